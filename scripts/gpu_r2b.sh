#!/bin/bash
# Round-2 measurement set (r2b): headline + reference arm, dense workloads,
# device-aware plans, C4 at 34 q, sharded N=1 through the C ABI, launch lists
# and ncu captures of the top kernels.
mkdir -p gpurun_out
B=gpurun_out
timeout 1200 python bench.py > $B/r2b_bench_qft34.json 2> $B/r2b_bench_qft34.err; tail -c 600 $B/r2b_bench_qft34.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $B/r2b_bench_reference.json 2> $B/r2b_ref.err; tail -c 300 $B/r2b_bench_reference.json
run() { timeout 1200 python bench.py --steps 2 --warmup 1 --no-e2e "$@" 2>> $B/r2b_workloads.err | tail -1 >> $B/r2b_bench_workloads.jsonl; }
: > $B/r2b_bench_workloads.jsonl
run --workload ghz --qubits 30
run --workload qaoa3reg --qubits 30 --error-bound 1e-4
run --workload qaoa3reg --qubits 32 --error-bound 1e-3
run --workload random --qubits 30 --layers 20
run --inner-size 6
run --device-plan --inner-size 16
run --workload qaoa3reg --qubits 30 --error-bound 1e-4 --device-plan --inner-size 16
run --workload random --qubits 30 --layers 20 --device-plan --inner-size 16
timeout 1500 python bench.py --workload qaoa3reg --qubits 34 --error-bound 1e-4 --steps 1 --warmup 1 --no-e2e > $B/r2b_c4_qaoa34.json 2>> $B/r2b_workloads.err
timeout 1500 python bench.py --workload qaoa3reg --qubits 34 --error-bound 1e-4 --steps 1 --warmup 1 --no-e2e --device-plan --inner-size 16 > $B/r2b_c4_qaoa34_devplan.json 2>> $B/r2b_workloads.err
timeout 900 python bench.py --qubits 30 --sharded --steps 3 --warmup 2 --no-e2e > $B/r2b_sharded_qft30.json 2>> $B/r2b_workloads.err
timeout 900 python bench.py --qubits 30 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $B/r2b_direct_qft30.json 2>> $B/r2b_workloads.err
python - <<'PY'
import json
for f in ["gpurun_out/r2b_bench_workloads.jsonl", "gpurun_out/r2b_c4_qaoa34.json", "gpurun_out/r2b_c4_qaoa34_devplan.json", "gpurun_out/r2b_sharded_qft30.json", "gpurun_out/r2b_direct_qft30.json"]:
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"): continue
        d = json.loads(line); r = d.get("roofline") or {}
        print(d["config"]["workload"], d["config"].get("plan", d["config"].get("parallelism")), "stages", d["config"]["stages"], "ms %.1f" % d["ms_per_step"], "frac", round(r.get("frac", 0) or 0, 3), "fid", d.get("fidelity"))
PY
Q=30 THR=1e18 bash scripts/gpu_launches.sh > /dev/null 2>&1
W=qaoa3reg Q=28 A="--error-bound 1e-4" bash scripts/gpu_launches_w.sh > /dev/null 2>&1
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound 1e-4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream_pass|k_gate_pass_fast|k_dec_chunk|k_cmp_emit" -s 120 -c 8 -o $B/r2b_q28 -f $BQ > /dev/null 2>&1
BQ="python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s 18 -c 1 -o $B/r2b_qft30_chain -f $BQ > /dev/null 2>&1
ls -la $B | tail -30
