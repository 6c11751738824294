#!/bin/bash
mkdir -p gpurun_out
for br in 1e-4 1e-3; do
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound $br --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q28_$br.csv $BQ > /dev/null 2>&1
echo "== $br"; python scripts/launches.py gpurun_out/launches_q28_$br.csv 1e18 | head -6
done
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound 1e-4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream_pass|k_gate_pass_fast" -s 40 -c 6 -o gpurun_out/q28t -f $BQ > gpurun_out/ncu_q28t.log 2>&1
tail -1 gpurun_out/ncu_q28t.log
