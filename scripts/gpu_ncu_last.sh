#!/bin/bash
# ncu --set full of the quantising last pass of the QFT-30 chain stage (k_gate_pass_fast launch 18).
mkdir -p gpurun_out
B="python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s ${S:-18} -c 1 -o gpurun_out/prof_last $B > gpurun_out/ncu_last.log 2>&1
ls -la gpurun_out/*.ncu-rep
