#!/bin/bash
# iteration: parity suites, then dense bench lines with and without the streaming pass
timeout 1200 python -m pytest tests/test_codec_gpu.py tests/test_engine_gpu.py tests/test_headline_layout_gpu.py tests/test_gates_gpu.py -q -x 2>&1 | tail -4
line() {
  timeout 600 python bench.py $1 --steps 3 --warmup 3 --no-e2e --no-link --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; ph=r['phases']
print('$2', d['config']['workload'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%r['frac'], ' '.join('%s %.0fms %.2f'%(k,v['ms'],v['frac']) for k,v in ph.items()), 'fid', d['fidelity'])"
}
for wl in "--workload qaoa3reg --qubits 30 --error-bound 1e-4" "--workload random --qubits 30 --layers 20" ""; do
  BMQ_FUSED_DECODE=1 line "$wl" fused
  line "$wl" stream
  BMQ_DBG_NO_STREAM=1 line "$wl" tiled
done
