#!/bin/bash
# per-kernel launch list + ncu of the dense QAOA-28 stage kernels (one capture set)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_codec_gpu.py -q -x 2>&1 | tail -2
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound 1e-4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q28b.csv $BQ > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_q28b.csv 1e18 > gpurun_out/launches_q28b.txt; cat gpurun_out/launches_q28b.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gate_pass_fast|k_dec_chunk|k_cmp_emit" -s 120 -c 6 -o gpurun_out/q28b -f $BQ > gpurun_out/ncu_q28b.log 2>&1
tail -2 gpurun_out/ncu_q28b.log
