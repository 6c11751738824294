#!/bin/bash
# One GPU session: parity tests, bench, launch list and ncu capture.
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
if [ "$1" == "prof" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --qubits 26 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gate_pass_fast|k_cmp_emit|k_cmp_stats|k_dec_chunk|k_dec_index|k_cmp_plan" -s 40 -c 8 -o gpurun_out/prof python bench.py --qubits 26 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1
fi
