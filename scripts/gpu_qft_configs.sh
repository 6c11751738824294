#!/bin/bash
# QFT-34 at the other (block bits, inner) configurations of BASELINE C3.
mkdir -p gpurun_out
: > gpurun_out/qft_configs.jsonl
for cfg in "14 2" "14 6" "17 4" "20 4" "24 6"; do
  set -- $cfg
  timeout 600 python bench.py --workload qft --qubits 34 --block-bits $1 --inner-size $2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>> gpurun_out/qft_configs.err | tail -1 >> gpurun_out/qft_configs.jsonl
done
cat gpurun_out/qft_configs.jsonl | cut -c1-300
