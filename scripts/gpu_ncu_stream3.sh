#!/bin/bash
mkdir -p gpurun_out
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound 1e-4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q28d.csv $BQ > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_q28d.csv 1e18 > gpurun_out/launches_q28d.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream_pass|k_gate_pass_fast" -s 40 -c 8 -o gpurun_out/q28u -f $BQ > gpurun_out/ncu_q28u.log 2>&1
BQ="python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qft30.csv $BQ > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_qft30.csv 1e18 > gpurun_out/launches_qft30.txt 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-link --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; ph=r['phases']
print(d['config']['workload'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%r['frac'], ' '.join('%s %.0fms'%(k,v['ms']) for k,v in ph.items()))"
