"""Hot contiguous SASS regions of an ncu report (instructions executed)."""
import csv
import subprocess
import sys

src = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src))
h = rows[1]
data = [r for r in rows[2:] if len(r) > 5]
ie, sc, st = h.index("Instructions Executed"), h.index("Source"), h.index('Warp Stall Sampling (All Samples)')
tot = sum(float(r[ie] or 0) for r in data)
stot = sum(float(r[st] or 0) for r in data)
reg, cur = [], None
for r in data:
    v = float(r[ie] or 0) / tot * 100
    if v < 0.02:
        if cur:
            reg.append(cur)
            cur = None
        continue
    if cur is None:
        cur = [r[0][-5:], r[0][-5:], 0, 0, 0, r[sc][:50]]
    cur[1] = r[0][-5:]
    cur[2] += v
    cur[3] += 1
    cur[4] += float(r[st] or 0) / stot * 100
if cur:
    reg.append(cur)
for c in sorted(reg, key=lambda c: -c[2])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{c[0]}-{c[1]} inst {c[2]:6.2f}% stall {c[4]:6.2f}% n={c[3]:4d} {c[5]}")
