#!/bin/bash
mkdir -p gpurun_out
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound 1e-4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q28c.csv $BQ > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_q28c.csv 1e18 > gpurun_out/launches_q28c.txt; cat gpurun_out/launches_q28c.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream_pass" -s 40 -c 2 -o gpurun_out/q28s -f $BQ > gpurun_out/ncu_q28s.log 2>&1
tail -2 gpurun_out/ncu_q28s.log
