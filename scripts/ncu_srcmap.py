"""Per-source-line instruction share of an ncu report, grouped by hot SASS region."""
import csv
import subprocess
import sys

txt = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(txt))
cur_file = cur_line = None
out = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split('/')[-1]
        continue
    if not r or r[0] == "Line No" or len(r) < 8:
        continue
    if r[0]:
        cur_line = (cur_file, r[0], r[1].strip()[:70])
        continue
    if r[2].startswith('0x'):
        out[int(r[2], 16) & 0xfffff] = (cur_line, float(r[7] or 0), float(r[4] or 0))
tot = sum(v[1] for v in out.values())
stot = sum(v[2] for v in out.values())
agg = {}
for a, (k, ie, st) in out.items():
    x = agg.setdefault(k, [0, 0])
    x[0] += ie
    x[1] += st
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, (ie, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"inst {100 * ie / tot:5.2f}%  stall {100 * st / stot:5.2f}%  {k[0]}:{k[1]}  {k[2]}")
