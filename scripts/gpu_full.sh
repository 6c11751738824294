#!/bin/bash
# Full measurement session: tests, bench (with CPU baseline + e2e), reference arm,
# launch list of the bench command, ncu --set full of the top kernels.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
B="python bench.py --qubits 28 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q28.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gate_pass_fast|k_cmp_emit|k_dec_chunk" -s 60 -c 6 -o gpurun_out/prof_full $B > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
