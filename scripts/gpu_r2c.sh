#!/bin/bash
# re-entry check: full GPU parity suite, smoke, default bench line, dense bench lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/tests.txt; cat gpurun_out/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
for wl in "--workload qaoa3reg --qubits 30 --error-bound 1e-4" "--workload qaoa3reg --qubits 30 --error-bound 1e-3" "--workload random --qubits 30 --layers 20"; do
  timeout 600 python bench.py $wl --steps 3 --warmup 3 --no-e2e --no-link --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; ph=r['phases']
print(d['config']['workload'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%r['frac'], ' '.join('%s %.0fms %.2f'%(k,v['ms'],v['frac']) for k,v in ph.items()), 'fid', d['fidelity'])"
done
