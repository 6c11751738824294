#!/bin/bash
# ncu --set full of the chain-stage gate passes (QFT-30: passes 17 and 19 of k_gate_pass_fast).
mkdir -p gpurun_out
B="python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s 16 -c 1 -o gpurun_out/prof_chainA $B > gpurun_out/ncu4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s 18 -c 1 -o gpurun_out/prof_chainC $B > gpurun_out/ncu5.log 2>&1
ls -la gpurun_out/*.ncu-rep
