#!/bin/bash
# Bench lines of the other BASELINE.json workload shapes on one GPU.
mkdir -p gpurun_out
run() { timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e "$@" 2>> gpurun_out/workloads.err | tail -1 >> gpurun_out/workloads.jsonl; }
: > gpurun_out/workloads.jsonl
run --workload ghz --qubits 30 --block-bits 20
run --workload qaoa3reg --qubits 30 --block-bits 20 --error-bound 1e-4
run --workload qaoa3reg --qubits 32 --block-bits 20 --error-bound 1e-3
run --workload random --qubits 30 --block-bits 20 --layers 20
run --workload qft --qubits 34 --block-bits 20 --inner-size 6
cat gpurun_out/workloads.jsonl | cut -c1-400
tail -5 gpurun_out/workloads.err
