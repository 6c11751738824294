#!/bin/bash
# A/B of the quantising streaming pass occupancy: fused + unfused dense lines and the headline.
mkdir -p gpurun_out; B=gpurun_out; T=${T:-d4}
run() { timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-link "$@" 2>> $B/${T}.err | tail -1 >> $B/${T}.jsonl; }
: > $B/${T}.jsonl
run --workload qaoa3reg --qubits 30 --error-bound 1e-4
run --workload qaoa3reg --qubits 32 --error-bound 1e-3
run --workload qaoa3reg --qubits 30 --error-bound 1e-4 --no-fuse-stages
run --workload random --qubits 30 --layers 20 --no-fuse-stages
run --steps 3 --warmup 3
python - <<'PY'
import json, os
for line in open(f"gpurun_out/{os.environ.get('T','d4')}.jsonl"):
    if not line.startswith("{"): print("!!", line[:300]); continue
    d = json.loads(line)
    print(d["config"]["workload"], d["config"].get("stage_fusion"), "ms %.1f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"])
PY
