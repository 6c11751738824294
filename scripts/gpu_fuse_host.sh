#!/bin/bash
# Stage fusion with a pinned host level: host-level parity tests, then a spilling dense line fused vs unfused.
mkdir -p gpurun_out; B=gpurun_out; T=${T:-fh}
timeout 900 python -m pytest tests -m gpu -q -x -k "host or spill or fusion or fused or disk or shard or checkpoint" 2>&1 | tail -3
run() { timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-link "$@" 2>> $B/${T}.err | tail -1 >> $B/${T}.jsonl; }
: > $B/${T}.jsonl
run --workload random --qubits 30 --layers 20 --device-pool-gib 2 --host-pool-gib 16 --arena heap
run --workload random --qubits 30 --layers 20 --device-pool-gib 2 --host-pool-gib 16 --arena heap --no-fuse-stages
python - <<'PY'
import json, os
for line in open(f"gpurun_out/{os.environ.get('T','fh')}.jsonl"):
    if not line.startswith("{"): print("!!", line[:300]); continue
    d = json.loads(line)
    print(d["config"]["workload"], d["config"].get("stage_fusion"), "ms %.1f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"], "peak", d["max_footprint_bytes"], "host", d["store"]["host_spill_bytes"], d["store"]["link_h2d_bytes"], d["store"]["link_d2h_bytes"])
PY
