"""Executed-instruction mix by SASS opcode (optionally restricted to source lines of one file)."""
import collections
import csv
import subprocess
import sys

txt = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout.splitlines()
only = sys.argv[2] if len(sys.argv) > 2 else None
cur_file = None
mix = collections.Counter()
seen = set()
for r in csv.reader(txt):
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split('/')[-1]
        continue
    if not r or r[0] == "Line No" or len(r) < 8 or r[0] or not r[2].startswith('0x'):
        continue
    if r[2] in seen:
        continue
    seen.add(r[2])
    if only and cur_file != only:
        continue
    op = r[3].split()
    op = [o for o in op if not o.startswith('@')]
    mix[op[0].split('.')[0] if op else '?'] += float(r[7] or 0)
tot = sum(mix.values())
for k, v in mix.most_common(30):
    print(f"{k:12s} {100 * v / tot:6.2f}%")
