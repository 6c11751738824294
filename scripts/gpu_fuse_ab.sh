#!/bin/bash
# Stage fusion: GPU suite, then the dense lines with and without fusion.
mkdir -p gpurun_out; B=gpurun_out; T=${T:-fuse}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > $B/${T}_tests.txt; tail -3 $B/${T}_tests.txt
run() { timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-link "$@" 2>> $B/${T}.err | tail -1 >> $B/${T}.jsonl; }
: > $B/${T}.jsonl
for W in "--workload qaoa3reg --qubits 30 --error-bound 1e-4" "--workload qaoa3reg --qubits 32 --error-bound 1e-3" "--workload random --qubits 30 --layers 20" "--qubits 30"; do
  run $W; run $W --fuse-stages
done
python - <<'PY'
import json, os
for line in open(f"gpurun_out/{os.environ.get('T','fuse')}.jsonl"):
    if not line.startswith("{"): print("!!", line[:300]); continue
    d = json.loads(line)
    print(d["config"]["workload"], d["config"].get("stage_fusion"), "ms %.1f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"], "ratio %.3f" % d["compression_ratio"], "peak", d["max_footprint_bytes"], "fid", d.get("fidelity"))
PY
