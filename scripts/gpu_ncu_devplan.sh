#!/bin/bash
# launch list + ncu of the tiled passes of a device-aware-plan dense run (QAOA-3reg-28 @1e-4)
mkdir -p gpurun_out
BQ="python bench.py --workload random --qubits 28 --layers 20 --device-plan --inner-size 16 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r28dp.csv $BQ > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_r28dp.csv 1e18 > gpurun_out/launches_r28dp.txt; cat gpurun_out/launches_r28dp.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gate_pass_fast" -s 4 -c 2 -o gpurun_out/r28dp -f $BQ > /dev/null 2>&1
ls -la gpurun_out/r28dp.ncu-rep
