"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]
ki, vi, gi = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Grid Size')
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e18
tot, cnt = {}, {}
for n, r in enumerate(rows[hi + 1:]):
    name = r[ki].split('(')[0].split('::')[-1]
    v = float(r[vi])
    tot[name] = tot.get(name, 0) + v
    cnt[name] = cnt.get(name, 0) + 1
    if v > thr:
        print(f"#{n:4d} {name:22s} {v/1e3:10.1f} us grid {r[gi]}")
allt = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:22s} n={cnt[k]:5d} {v/1e6:9.3f} ms  {100*v/allt:5.1f}%")
