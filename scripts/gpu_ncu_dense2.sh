#!/bin/bash
# ncu --set full of one mid-run dense stage of QAOA-3reg-28 @1e-4: quantising gate pass, doubles decode, emit
mkdir -p gpurun_out
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound 1e-4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q28.csv $BQ > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_q28.csv 1e18 > gpurun_out/launches_q28.txt; cat gpurun_out/launches_q28.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gate_pass_fast|k_dec_chunk|k_cmp_emit" -s 120 -c 6 -o gpurun_out/q28 -f $BQ > gpurun_out/ncu_q28.log 2>&1
tail -3 gpurun_out/ncu_q28.log
ls -la gpurun_out
