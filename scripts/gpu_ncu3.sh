#!/bin/bash
# ncu --set full of the three kernels of a code-domain stage (QFT-30 swap stage).
mkdir -p gpurun_out
B="python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_perm_pass -s 0 -c 1 -o gpurun_out/prof_code $B > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dec_chunk -s 17 -c 1 -o gpurun_out/prof_decc $B > gpurun_out/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cmp_emit -s 18 -c 1 -o gpurun_out/prof_emitc $B > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out/*.ncu-rep
