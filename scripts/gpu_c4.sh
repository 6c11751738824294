#!/bin/bash
# C4 at full size: QAOA MaxCut p=4 on a 34-node random 3-regular graph, 1e-4, 1 B200
free -g | head -2; nproc
timeout 1500 python bench.py --workload qaoa3reg --qubits 34 --error-bound 1e-4 --layers 4 --steps 1 --warmup ${W:-1} \
  --no-e2e --no-link > gpurun_out/c4_qaoa34.json 2> gpurun_out/c4_qaoa34.err
tail -3 gpurun_out/c4_qaoa34.err; cat gpurun_out/c4_qaoa34.json
