#!/bin/bash
# C5 shape on one B200: random circuit (sqrt-X/Y/W + CZ grid) depth 40, 1e-3,
# device arena fixed below the compressed state so most payloads live in the
# pinned host level (prefetched / written back on the copy streams)
free -g | head -2
timeout 2400 python bench.py --workload random --qubits ${N:-34} --layers 40 --error-bound 1e-3 --steps 1 --warmup ${W:-1} \
  --no-e2e --device-pool-gib ${DEV:-24} --host-pool-gib ${HOST:-120} > gpurun_out/c5_random${N:-34}.json 2> gpurun_out/c5_random${N:-34}.err
tail -3 gpurun_out/c5_random${N:-34}.err; cat gpurun_out/c5_random${N:-34}.json
