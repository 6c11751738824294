#!/bin/bash
# Fusion on by default: full GPU suite, smoke, headline, dense lines fused vs not, C4.
mkdir -p gpurun_out; B=gpurun_out; T=${T:-fuse3}
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -30 > $B/${T}_tests.txt; tail -3 $B/${T}_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $B/${T}_smoke.txt 2>&1; tail -1 $B/${T}_smoke.txt
run() { timeout 1500 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-link "$@" 2>> $B/${T}.err | tail -1 >> $B/${T}.jsonl; }
: > $B/${T}.jsonl
run --workload qaoa3reg --qubits 30 --error-bound 1e-4
run --workload qaoa3reg --qubits 32 --error-bound 1e-3
run --workload random --qubits 30 --layers 20
run --workload qaoa3reg --qubits 34 --error-bound 1e-3 --steps 1 --warmup 1
run --workload qaoa3reg --qubits 34 --error-bound 1e-4 --steps 1 --warmup 1
python - <<'PY'
import json, os
for line in open(f"gpurun_out/{os.environ.get('T','fuse3')}.jsonl"):
    if not line.startswith("{"): print("!!", line[:300]); continue
    d = json.loads(line)
    print(d["config"]["workload"], d["config"].get("stage_fusion"), "ms %.1f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"], "ratio %.3f" % d["compression_ratio"], "peak", d["max_footprint_bytes"], "fid", d.get("fidelity"))
PY
