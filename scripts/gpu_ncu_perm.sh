#!/bin/bash
# ncu --set full of the QFT-30 code-domain permutation passes (k_perm_pass launches 0 and 1).
mkdir -p gpurun_out
B="python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_perm_pass -s 0 -c 2 -o gpurun_out/prof_perm $B > gpurun_out/ncu_perm.log 2>&1
ls -la gpurun_out/*.ncu-rep
