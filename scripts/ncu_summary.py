"""Print key metrics of an ncu report (details page) and the hottest SASS."""
import csv
import subprocess
import sys

rep = sys.argv[1]
keys = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Executed Ipc Active',
        'Issue Slots Busy', 'No Eligible', 'Warp Cycles Per Issued Instruction', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Avg. Active Threads Per Warp', 'L1/TEX Hit Rate',
        'L2 Hit Rate', 'Dynamic Shared Memory Per Block', 'Static Shared Memory Per Block']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
seen = set()
for r in csv.reader(out.splitlines()):
    if len(r) > 14 and r[12] in keys and r[12] not in seen:
        seen.add(r[12])
        print(f"  {r[12]:40s} {r[14]:>12s} {r[13]}")
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr = rows[0]
for m in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum', 'gpu__time_duration.sum'):
    if m in hdr:
        print(f"  {m:40s} {rows[2][hdr.index(m)]:>12s} {rows[1][hdr.index(m)]}")
if len(sys.argv) > 2:
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True,
                         text=True).stdout.splitlines()
    data = list(csv.reader(src))
    h = data[1]
    ie, sc, st = h.index('Instructions Executed'), h.index('Source'), h.index('Warp Stall Sampling (All Samples)')
    body = [r for r in data[2:] if len(r) > ie]
    tot = sum(float(r[ie] or 0) for r in body)
    stot = sum(float(r[st] or 0) for r in body)
    for r in sorted(body, key=lambda r: -float(r[st] or 0))[:int(sys.argv[2])]:
        print(f"  {r[0][-5:]} inst {100*float(r[ie] or 0)/tot:5.2f}% stall {100*float(r[st] or 0)/stot:5.2f}%  {r[sc][:70]}")
