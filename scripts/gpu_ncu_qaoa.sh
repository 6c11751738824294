#!/bin/bash
# ncu --set full of a QAOA-3reg-28 gate pass (k_gate_pass_fast launch ${S:-60}).
mkdir -p gpurun_out
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound 1e-4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s ${S:-60} -c 1 -o gpurun_out/prof_qaoa $BQ > gpurun_out/ncu_qaoa.log 2>&1
ls -la gpurun_out/*.ncu-rep
