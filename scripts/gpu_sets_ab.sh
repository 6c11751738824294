#!/bin/bash
# two buffer sets (overlapped batches) vs one: parity suite, then bench lines
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
line() {
  timeout 900 python bench.py $1 --steps 3 --warmup 2 --no-e2e --no-link --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; ph=r['phases']
print('$2', d['config']['workload'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%r['frac'], ' '.join('%s %.0fms'%(k,v['ms']) for k,v in ph.items()))"
}
for wl in "--workload qaoa3reg --qubits 30 --error-bound 1e-4" "--workload random --qubits 30 --layers 20" "--workload qaoa3reg --qubits 32 --error-bound 1e-3" "" "--workload qaoa3reg --qubits 32 --error-bound 1e-3 --device-plan --inner-size 16"; do
  line "$wl" two
  BMQ_DBG_ONE_SET=1 line "$wl" one
done
