#!/bin/bash
# Round-2 closing measurement set (r2i, stage fusion on by default, round-trip variant at 2 CTAs/SM, chain stages unfused; final HEAD): parity suites, smoke, headline + reference arm,
# dense workloads with both plans, C4 and QAOA-34 @1e-3, three-level store line,
# launch lists and one ncu capture per hot kernel family.
mkdir -p gpurun_out
B=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $B/r2i_tests.txt; cat $B/r2i_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $B/r2i_smoke.txt 2>&1; tail -1 $B/r2i_smoke.txt
timeout 1200 python bench.py > $B/r2i_bench_qft34.json 2> $B/r2i_bench_qft34.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $B/r2i_bench_reference.json 2> $B/r2i_ref.err
run() { timeout 1500 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline "$@" 2>> $B/r2i_workloads.err | tail -1 >> $B/r2i_bench_workloads.jsonl; }
: > $B/r2i_bench_workloads.jsonl
run --workload ghz --qubits 30
run --workload qaoa3reg --qubits 30 --error-bound 1e-4
run --workload qaoa3reg --qubits 30 --error-bound 1e-4 --no-fuse-stages
run --workload qaoa3reg --qubits 30 --error-bound 1e-4 --device-plan --inner-size 16
run --workload qaoa3reg --qubits 32 --error-bound 1e-3
run --workload qaoa3reg --qubits 32 --error-bound 1e-3 --no-fuse-stages
run --workload qaoa3reg --qubits 32 --error-bound 1e-3 --device-plan --inner-size 16
run --workload random --qubits 30 --layers 20
run --workload random --qubits 30 --layers 20 --no-fuse-stages
run --workload random --qubits 30 --layers 20 --device-plan --inner-size 16
run --inner-size 6
run --device-plan --inner-size 16
run --workload random --qubits 28 --layers 20 --device-pool-gib 0.4 --host-pool-gib 0.4 --disk-pool-gib 4 --arena heap
run --workload qaoa3reg --qubits 34 --error-bound 1e-3 --steps 1 --warmup 1 --device-plan --inner-size 16
run --workload qaoa3reg --qubits 34 --error-bound 1e-4 --steps 1 --warmup 1 --device-plan --inner-size 16
run --workload qaoa3reg --qubits 34 --error-bound 1e-3 --steps 1 --warmup 1
run --workload qaoa3reg --qubits 34 --error-bound 1e-4 --steps 1 --warmup 1
python - <<'PY'
import json
for line in open("gpurun_out/r2i_bench_workloads.jsonl"):
    line = line.strip()
    if not line.startswith("{"): print("!!", line[:200]); continue
    d = json.loads(line); r = d.get("roofline") or {}
    print(d["config"]["workload"], d["config"].get("plan"), "stages", d["config"]["stages"], "ms %.1f" % d["ms_per_step"], "frac", round(r.get("frac", 0) or 0, 3), "ratio %.2f" % d["compression_ratio"], d["config"].get("stage_fusion"), "fid", d.get("fidelity"), d["store"].get("disk_spill_bytes"))
PY
Q=30 THR=1e18 bash scripts/gpu_launches.sh > /dev/null 2>&1
W=qaoa3reg Q=28 A="--error-bound 1e-4" bash scripts/gpu_launches_w.sh > /dev/null 2>&1
W=qaoa3reg Q=28 A="--error-bound 1e-4 --device-plan --inner-size 16" bash scripts/gpu_launches_w.sh > /dev/null 2>&1 ; mv $B/launches_qaoa3reg28.txt $B/launches_qaoa3reg28_dp.txt 2>/dev/null
W=qaoa3reg Q=28 A="--error-bound 1e-4" bash scripts/gpu_launches_w.sh > /dev/null 2>&1
BQ="python bench.py --workload qaoa3reg --qubits 28 --error-bound 1e-4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream_pass|k_gate_pass_fast|k_dec_chunk|k_cmp_emit" -s 120 -c 8 -o $B/r2i_q28 -f $BQ > /dev/null 2>&1

BQ30="python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gate_pass_fast|k_perm_pass|k_cmp_emit|k_dec_chunk" -s 60 -c 8 -o $B/r2i_qft30 -f $BQ30 > /dev/null 2>&1
ls $B | grep r2i
