#!/bin/bash
# Stage profile of QFT-34 + ncu of perm and emit (QFT-30).
mkdir -p gpurun_out
timeout 300 python scripts/stage_profile.py qft 34 20 2 > gpurun_out/stages_qft34.txt 2>&1
B="python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_perm_pass -s 0 -c 1 -o gpurun_out/prof_perm $B > gpurun_out/ncu_perm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cmp_emit -s 18 -c 1 -o gpurun_out/prof_emit $B > gpurun_out/ncu_emit.log 2>&1
ls -la gpurun_out/*.ncu-rep
