#!/bin/bash
# ncu --set full of one kernel launch: K=<name regex> S=<skip> Q=<qubits> OUT=<name>
mkdir -p gpurun_out
B="python bench.py --qubits ${Q:-30} --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${S:-0} -c 1 -o gpurun_out/prof_$OUT $B > gpurun_out/ncu_$OUT.log 2>&1
ls -la gpurun_out/prof_$OUT.ncu-rep
