#!/bin/bash
# A/B check after a kernel change: GPU suite, then the dense lines and the headline (T = tag).
mkdir -p gpurun_out; B=gpurun_out; T=${T:-ab}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $B/${T}_tests.txt; cat $B/${T}_tests.txt
run() { timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-link "$@" 2>> $B/${T}.err | tail -1 >> $B/${T}.jsonl; }
: > $B/${T}.jsonl
run --workload qaoa3reg --qubits 30 --error-bound 1e-4
run --workload qaoa3reg --qubits 32 --error-bound 1e-3
run --workload random --qubits 30 --layers 20
run --workload qaoa3reg --qubits 30 --error-bound 1e-4 --device-plan --inner-size 16
run --steps 3 --warmup 3
python - <<'PY'
import json, os
for line in open(f"gpurun_out/{os.environ.get('T','ab')}.jsonl"):
    if not line.startswith("{"): print("!!", line[:200]); continue
    d = json.loads(line)
    print(d["config"]["workload"], d["config"].get("plan"), "ms %.1f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"])
PY
