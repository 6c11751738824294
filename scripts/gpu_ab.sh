#!/bin/bash
# A/B of the device-arena policies on QFT-34, then the QFT-30 launch list
for a in heap bump heap bump; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-link --no-cpu-baseline --arena $a 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; ph=r['phases']
print(d['config']['arena'], 'ms %.1f'%d['ms_per_step'], ' '.join('%s %.1fms'%(k,v['ms']) for k,v in ph.items()), d['store']['compactions'])"
done
Q=30 THR=100000 bash scripts/gpu_launches.sh | tail -16
