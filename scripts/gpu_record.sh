#!/bin/bash
# Measurement session for profiles/: tests, smoke, default bench (with CPU
# baseline + e2e), reference arm, other workloads, QFT-30 launch list, and
# ncu --set full captures of the top kernels.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash scripts/gpu_workloads.sh > /dev/null 2>&1
Q=30 THR=1e18 bash scripts/gpu_launches.sh > /dev/null 2>&1
W=qaoa3reg Q=28 A="--error-bound 1e-4" bash scripts/gpu_launches_w.sh > /dev/null 2>&1
B="python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s 18 -c 1 -o gpurun_out/rec_chain $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s 16 -c 1 -o gpurun_out/rec_chain0 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_perm_pass -s 0 -c 1 -o gpurun_out/rec_perm $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dec_chunk -s 17 -c 1 -o gpurun_out/rec_dec $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cmp_emit -s 18 -c 1 -o gpurun_out/rec_emit $B > /dev/null 2>&1
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound 1e-4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s 60 -c 1 -o gpurun_out/rec_qaoa_pass $BQ > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cmp_emit -s 40 -c 1 -o gpurun_out/rec_qaoa_emit $BQ > /dev/null 2>&1
ls -la gpurun_out
