#!/bin/bash
# A/B of code-domain stages reading zero-free chunks from the payload (PermSrc).
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
line() {
  timeout 600 python bench.py $1 --steps 3 --warmup 3 --no-e2e --no-link --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; ph=r['phases']
print('$2', d['config']['workload'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%r['frac'], ' '.join('%s %.0fms'%(k,v['ms']) for k,v in ph.items()))"
}
for rep in 1 2; do
  line "" permsrc
  BMQ_DBG_NO_PERMSRC=1 line "" base
done
line "--qubits 30" permsrc
BMQ_DBG_NO_PERMSRC=1 line "--qubits 30" base
line "--workload ghz --qubits 30" permsrc
BMQ_DBG_NO_PERMSRC=1 line "--workload ghz --qubits 30" base
