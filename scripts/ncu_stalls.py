"""Warp stall reasons and pipe utilisation from an ncu report (raw page)."""
import csv
import subprocess
import sys

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, vals = rows[0], rows[2]
items = []
for h, v in zip(hdr, vals):
    if 'warps_issue_stalled' in h and 'pcsamp' in h and 'not_issued' not in h:
        try:
            items.append((float(v.replace(',', '')), h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
        except ValueError:
            pass
tot = sum(v for v, _ in items) or 1
print('  stalls: ' + ', '.join(f"{h} {100*v/tot:.0f}%" for v, h in sorted(items, reverse=True)[:8]))
for key in ['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
            'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']:
    for h, v in zip(hdr, vals):
        if h == key:
            print(f"  {key} {v}")
