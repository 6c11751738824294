#!/bin/bash
# Stage fusion A/B: union size (BMQ_FUSE_INNER) and round trip in the pass vs k_round.
mkdir -p gpurun_out; B=gpurun_out; T=${T:-fuse2}
timeout 600 python -m pytest tests/test_fusion_gpu.py -m gpu -q -x 2>&1 | tail -3 > $B/${T}_tests.txt; tail -1 $B/${T}_tests.txt
run() { echo "$1" >> $B/${T}.jsonl; shift; timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-link "$@" 2>> $B/${T}.err | tail -1 >> $B/${T}.jsonl; }
: > $B/${T}.jsonl
for W in "--workload qaoa3reg --qubits 30 --error-bound 1e-4" "--workload qaoa3reg --qubits 32 --error-bound 1e-3" "--workload random --qubits 30 --layers 20"; do
  for K in 4 6 8; do
    BMQ_FUSE_INNER=$K run "K=$K pass" $W --fuse-stages
    BMQ_DBG_FUSE_KROUND=1 BMQ_FUSE_INNER=$K run "K=$K kround" $W --fuse-stages
  done
done
python - <<'PY'
import json, os
tag = None
for line in open(f"gpurun_out/{os.environ.get('T','fuse2')}.jsonl"):
    if not line.startswith("{"): tag = line.strip(); continue
    d = json.loads(line)
    print(tag, d["config"]["workload"], d["config"].get("stage_fusion"), "ms %.1f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"], "peak", d["max_footprint_bytes"])
PY
