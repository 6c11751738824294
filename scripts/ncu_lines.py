"""Per-CUDA-line instruction / stall attribution from an ncu report (cuda,sass view)."""
import csv
import subprocess
import sys

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
fname, cur, hdr = None, None, None
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[2] == '-' and r[0] != '-':  # cuda line summary row
        ie = hdr.index('Instructions Executed')
        st = hdr.index('Warp Stall Sampling (All Samples)')
        try:
            agg.append((float(r[ie] or 0), float(r[st] or 0), fname, r[0], r[1][:80]))
        except ValueError:
            pass
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for a in sorted(agg, key=lambda a: -a[0])[:n]:
    print(f"inst {100*a[0]/ti:5.1f}%  stall {100*a[1]/ts:5.1f}%  {a[2]}:{a[3]:>4s}  {a[4]}")
