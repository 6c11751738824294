#!/bin/bash
B="python bench.py --qubits 26 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s 14 -c 1 -o gpurun_out/prof_chain $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s 17 -c 1 -o gpurun_out/prof_epi $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cmp_emit -s 15 -c 1 -o gpurun_out/prof_emit $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dec_chunk -s 15 -c 1 -o gpurun_out/prof_dec $B > /dev/null 2>&1
ls -la gpurun_out
