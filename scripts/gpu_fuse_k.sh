#!/bin/bash
# Union cap sweep (BMQ_FUSE_INNER) on the dense lines.
mkdir -p gpurun_out; B=gpurun_out; T=${T:-fk}
run() { echo "$1" >> $B/${T}.jsonl; shift; timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-link "$@" 2>> $B/${T}.err | tail -1 >> $B/${T}.jsonl; }
: > $B/${T}.jsonl
for K in 7 9 10; do
  BMQ_FUSE_INNER=$K run "K=$K" --workload qaoa3reg --qubits 32 --error-bound 1e-3
  BMQ_FUSE_INNER=$K run "K=$K" --workload random --qubits 30 --layers 20
done
python - <<'PY'
import json, os
tag = None
for line in open(f"gpurun_out/{os.environ.get('T','fk')}.jsonl"):
    if not line.startswith("{"): tag = line.strip(); continue
    d = json.loads(line)
    print(tag, d["config"]["workload"], d["config"].get("stage_fusion"), "ms %.1f" % d["ms_per_step"])
PY
