#!/bin/bash
# After the chain-stage exclusion: fusion + headline-layout suites, QFT inner 6, QAOA-30.
mkdir -p gpurun_out; B=gpurun_out; T=${T:-fchk}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $B/${T}_tests.txt; tail -1 $B/${T}_tests.txt
run() { timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-link "$@" 2>> $B/${T}.err | tail -1 >> $B/${T}.jsonl; }
: > $B/${T}.jsonl
run --inner-size 6
run --inner-size 4
run --workload qaoa3reg --qubits 30 --error-bound 1e-4
python - <<'PY'
import json, os
for line in open(f"gpurun_out/{os.environ.get('T','fchk')}.jsonl"):
    if not line.startswith("{"): print("!!", line[:300]); continue
    d = json.loads(line)
    print(d["config"]["workload"], d["config"].get("stage_fusion"), "ms %.1f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"])
PY
