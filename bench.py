#!/usr/bin/env python
"""Benchmark of the BMQSim hot path on B200 (BASELINE.json metric).

Workload (one "step" = one complete simulation): QFT on 34 qubits, block
b = 20 (2^20 amplitudes per block), inner_size = 2 (reference default),
point-wise bound 1e-3, 98 stages. Metric: amplitude-stages per second,
2^34 x stages / simulation time (higher is better), next to the absolute sim
time, compression ratio, peak footprint and fidelity (analytic: QFT|0> is the
uniform state).

  python bench.py [--gpus N --steps K --warmup W]      this implementation
  python bench.py --impl reference                      the reference CPU path
                                                        (oracle/_ref) on the host

value      device time (CUDA events on the engine stream) of init + stages;
           inputs (plan, codec tables, device buffers) resident beforehand.
e2e        the same metric through the public C ABI from host data each step:
           bmq_simulator_create (gates H2D, partition, allocation) -> run ->
           bmq_simulator_get_payloads (every final payload D2H) -> destroy.
roofline   the dominant device phase: algorithmic bytes / its
           CUDA-event time, against MEASURED_PEAKS.json hbm_gbs.
The working set per batch (16 GiB of dense group buffers) is far larger than
L2 (126 MB), so no explicit flush is needed between steps.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(name="qft", n=34, b=20, inner=2, error_bound=1e-3, layers=1)


def metric_name(w):
    label = {"qft": "QFT", "ghz": "GHZ", "qaoa3reg": "QAOA-3reg", "random": "random", "qaoa": "QAOA-ring",
             "bv": "BV"}.get(w["name"], w["name"])
    extra = f", p={w['layers']}" if w["name"] in ("qaoa", "qaoa3reg") else (
        f", depth={w['layers']}" if w["name"] == "random" else "")
    return f"amp-stages/s ({label}-{w['n']}{extra}, b={w['b']}, inner={w['inner']}, b_r={w['error_bound']:g})"


def workload_tag(w):
    lay = f"_l{w['layers']}" if w["name"] in ("qaoa", "qaoa3reg", "random") else ""
    return f"{w['name']}{w['n']}{lay}_b{w['b']}_i{w['inner']}_br{w['error_bound']:g}"


def data_desc(w):
    what = {"qft": "QFT|0> circuit", "ghz": "GHZ circuit", "qaoa3reg": "QAOA MaxCut on a seeded random 3-regular graph",
            "random": "seeded sqrt-X/Y/W + CZ grid random circuit"}.get(w["name"], w["name"] + " circuit")
    return f"synthetic ({what} generated in-process; no datasets)"


def fidelity_of(cbq, sim, circ, cfg, w):
    """QFT|0> and GHZ have analytic ideal states; other circuits are compared
    with an uncompressed FP64 device run when its dense state fits (n <= 32)."""
    if w["name"] == "qft":
        return sim.fidelity_analytic("uniform")
    if w["name"] in ("ghz", "cat_state"):
        return sim.fidelity_analytic("ghz")
    if w["n"] > 32:
        return None
    import dataclasses
    with cbq.Simulator(circ, dataclasses.replace(cfg, compress=False)) as exact:
        exact.run()
        return sim.fidelity_with(exact)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        loaded = [s for s in self.samples if s[7].replace(".", "").isdigit() and float(s[7]) > 0] or self.samples
        sm = [float(s[0]) for s in loaded if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    # the driver reads one JSON line from rank 0: keep NCCL's banner off stdout
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return world, rank, local, dist
    return 1, 0, 0, None


def barrier_sync(dist):
    import torch
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(dist, value):
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def qft_stage_sample(ref, w):
    """Stratified sample of the QFT|0> run for the reference CPU pipeline.

    Before stage s the QFT|0> state is exactly |+> on the qubits whose H gate
    precedes the stage and |0> on the rest (make_qft, benchmarks.hpp:97-114:
    every CP's control j < i is still |0> when it is applied), so per stage the
    number of groups holding a nonzero block is 2^(#H'd outer qubits) and the
    rest are ALL_ZERO groups, which the reference processes too (it has no
    zero skipping: engine.hpp:109-120). The sample takes, per stage, one
    nonzero group (outer value 0, its blocks built from that state) and, when
    the stage has any, one ALL_ZERO group; each group runs the reference
    pipeline with the stage's real gates. Returns (plan, samples, counts)."""
    import numpy as np
    n, b = w["n"], w["b"]
    gl = ref.generate_benchmark("qft", n)
    plan = ref.partition(n, gl, b, w["inner"])
    h_at = {g[1]: i for i, g in enumerate(gl) if g[0] == 0}  # GateKind::H
    cache = {}

    def payload(hset, nonzero):
        key = (frozenset(q for q in hset if q < b), nonzero)
        if key not in cache:
            blk = np.zeros(2 << b)
            if nonzero:
                lmask = sum(1 << q for q in range(b) if q not in hset)
                loc = np.arange(1 << b, dtype=np.int64)
                blk[: 1 << b][(loc & lmask) == 0] = 2.0 ** (-len(hset) / 2)
            cache[key] = ref.compress_block(blk, w["error_bound"])
        return cache[key]

    samples, counts = [], []
    for s, (gb, ge, inner) in enumerate(plan):
        hset = {q for q, i in h_at.items() if i < gb}
        outer = [q for q in range(b, n) if q not in inner]
        groups = ref.enumerate_groups(n, b, (gb, ge, inner))
        nz = 1 << sum(1 for q in outer if q in hset)
        zero = groups.shape[0] - nz
        gmask = sum(1 << (q - b) for q in range(b, n) if q not in hset)
        ids = groups[0]
        samples.append((s, ids, [payload(hset, (int(g) & gmask) == 0) for g in ids]))
        counts.append(nz)
        if zero:
            j = next(k for k, q in enumerate(outer) if q not in hset)  # an outer |0> qubit set to 1
            samples.append((s, groups[1 << j], [payload(hset, False)] * groups.shape[1]))
            counts.append(zero)
    return gl, plan, samples, counts


def reference_qft_rate(ref, w, gl, plan, samples, counts, cores):
    """One pass of the stratified sample on `cores` threads; the full-run time
    is the measured per-group times weighted by each stage's group counts,
    divided over the threads (perfect scaling assumed: favourable to the CPU)."""
    gms, wall = ref.stage_groups(w["n"], gl, plan, w["b"], w["error_bound"], cores, samples)
    full_s = float(sum(c * t for c, t in zip(counts, gms))) / 1e3 / cores
    return (1 << w["n"]) * len(plan) / full_s, full_s, wall


def run_reference(args):
    """--impl reference: the reference CPU pipeline (oracle/_ref, unmodified
    headers) on a stratified sample of the same workload, all host threads."""
    world, rank, local, dist = dist_setup()
    if rank != 0:
        return 0
    from oracle import oracle
    ref = oracle.ref()
    w = WORKLOAD
    cores = os.cpu_count() or 1
    gl, plan, samples, counts = qft_stage_sample(ref, w)
    rates, walls, fulls = [], [], []
    for step in range(args.warmup + args.steps):
        rate, full_s, wall = reference_qft_rate(ref, w, gl, plan, samples, counts, cores)
        if step >= args.warmup:
            rates.append(rate)
            walls.append(wall)
            fulls.append(full_s)
    value = statistics.median(rates)
    sample = (f"{len(samples)} groups per step (x{1 << w['inner']} blocks of 2^{w['b']} amps): one nonzero and one "
              f"ALL_ZERO group of each of the {len(plan)} stages of {workload_tag(w)}, with QFT|0>'s exact input "
              f"state, through the reference per-group pipeline (engine.hpp:203-225) on {cores} threads; full-run "
              f"time = per-group times x the stage's group counts / threads (extrapolated)")
    line = {
        "impl": "reference", "metric": metric_name(w), "value": value,
        "unit": "amp-stages/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(walls), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (QFT|0> circuit; stratified per-stage sample)",
        "config": {"workload": workload_tag(w), "stages": len(plan), "sample_groups": len(samples)},
        "extrapolated_full_run_s": statistics.median(fulls),
        "cpu_baseline": {"value": value, "unit": "amp-stages/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "amp-stages/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline(full_runs=True):
    """The reference CPU path on this host: the stratified QFT-34 sample
    (extrapolated, labelled) plus complete Simulator::run calls of smaller
    QFT configurations (measured, engine.hpp:97-134)."""
    from oracle import oracle
    ref = oracle.ref()
    w = WORKLOAD
    cores = os.cpu_count() or 1
    gl, plan, samples, counts = qft_stage_sample(ref, w)
    rate, full_s, wall = reference_qft_rate(ref, w, gl, plan, samples, counts, cores)
    out = {"value": rate, "unit": "amp-stages/s", "cores": cores, "kind": "reference",
           "sample": f"{len(samples)} groups (one nonzero + one ALL_ZERO group per stage of {workload_tag(w)}) "
                     f"through the unmodified reference pipeline in {wall / 1e3:.1f} s on {cores} threads; "
                     f"full run extrapolated from per-stage group counts",
           "extrapolated_full_run_s": full_s}
    if full_runs:
        runs = []
        for n, b in ((20, 14), (24, 20)):
            g = ref.generate_benchmark("qft", n)
            res = ref.simulate(n, g, b, w["inner"], w["error_bound"], workers=cores, want_payloads=False)
            r = res.report
            runs.append({"workload": f"qft{n}_b{b}_i{w['inner']}", "wall_s": r["wall_ms"] / 1e3,
                         "stages": r["stage_count"],
                         "amp_stages_per_s": (1 << n) * r["stage_count"] / (r["wall_ms"] / 1e3),
                         "measured": "complete Simulator::run (init + stages + final state_norm)"})
        out["full_runs"] = runs
    return out


def measure_e2e(cbq, circ, cfg, amp_stages, args, dist, world):
    """The same simulation end to end through the C ABI, host buffers in and
    out: gate list from pinned host memory -> bmq_simulator_create (H2D,
    partition, allocation) -> run -> bmq_simulator_get_payloads into a pinned
    host buffer (every final payload D2H) -> destroy."""
    import ctypes as C
    import numpy as np
    import torch
    from paper_2410_14088_b200 import _lib
    lib = _lib.lib
    gates = circ.c_array()
    gate_bytes = C.sizeof(gates)
    pinned_in = torch.empty(gate_bytes, dtype=torch.uint8, pin_memory=True)
    C.memmove(pinned_in.data_ptr(), C.addressof(gates), gate_bytes)
    gates_ptr = C.c_void_p(pinned_in.data_ptr())
    ccfg = cfg.to_c()
    pinned_out, sizes = None, None
    times = []
    h2d = d2h = 0
    for step in range(max(1, min(args.steps, 3)) + 1):
        barrier_sync(dist)
        t0 = time.perf_counter()
        h = C.c_void_p()
        cbq._check(lib.bmq_simulator_create(circ.num_qubits, gates_ptr, len(gates), C.byref(ccfg), C.byref(h)))
        rep = _lib.bmq_report()
        cbq._check(lib.bmq_simulator_run(h, C.byref(rep), None, 0))
        total = C.c_uint64()
        if sizes is None:
            nblk = 1 << (circ.num_qubits - cfg.block_bits)
            sizes = np.zeros(nblk, dtype=np.uint64)
        cbq._check(lib.bmq_simulator_get_payloads(h, None, 0, sizes.ctypes.data, C.byref(total)))
        if pinned_out is None or pinned_out.numel() < total.value:
            pinned_out = torch.empty(max(1, total.value), dtype=torch.uint8, pin_memory=True)
        cbq._check(lib.bmq_simulator_get_payloads(h, C.c_void_p(pinned_out.data_ptr()), total.value,
                                                  sizes.ctypes.data, C.byref(total)))
        lib.bmq_simulator_destroy(h)
        dt = time.perf_counter() - t0
        if step > 0:  # first call is the warm-up (module load, table cache, pinned buffer)
            times.append(dt)
        h2d = gate_bytes
        d2h = int(total.value) + 8 * len(sizes)
    t_e2e = max_over_ranks(dist, statistics.median(times))
    return {"value": world * amp_stages / t_e2e, "unit": "amp-stages/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "seconds": t_e2e}


def measure_link():
    """Pinned host <-> device copy bandwidth (GB/s) of this GPU: 1 GiB each way,
    CUDA events on the copy stream, best of 3 (north_star's BW_link)."""
    import torch
    n = 1 << 30
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {}
    for name, dst, src in (("h2d", dev, host), ("d2h", host, dev)):
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            e1.synchronize()
            best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
        out[name + "_gbs"] = best
    del host, dev
    torch.cuda.empty_cache()
    return out


def roofline(d, t_dev, link):
    """t_roof = max(B_HBM / BW_HBM, B_link / BW_link) with B_HBM the
    model bytes (reference-exact payload bytes of every block of every group
    holding a nonzero block, read + written, plus 32 B per amplitude of those
    groups) and B_link the host-tier payload bytes; frac = t_roof / t_sim.
    Beside it, each device phase's own bytes over its CUDA-event time and the
    dominant kernel's ncu DRAM traffic (profiles/traffic.json)."""
    peak, peak_kind = load_peaks()
    t = t_dev / 1e3
    b_hbm = d["model_bytes"]
    b_link = d["link_h2d_bytes"] + d["link_d2h_bytes"]
    bw_link = min(link["h2d_gbs"], link["d2h_gbs"]) if link else None
    t_hbm = b_hbm / (peak * 1e9)
    # the link is full duplex: prefetches (H2D) and write-backs (D2H) overlap
    t_link = max(d["link_h2d_bytes"] / (link["h2d_gbs"] * 1e9), d["link_d2h_bytes"] / (link["d2h_gbs"] * 1e9)) \
        if (link and b_link) else 0.0
    bound = "hbm" if t_hbm >= t_link else "link"
    phases = {"decompress": (d["decompress_ms"], d["decompress_bytes"]),
              "gate": (d["gate_ms"], d["gate_bytes"]),
              "compress": (d["compress_ms"], d["compress_bytes"])}
    dom = max(phases, key=lambda k: phases[k][0])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(workload_tag(WORKLOAD), {}).get(dom)
        except Exception:
            traffic = None
    achieved = (b_hbm if bound == "hbm" else b_link) / t / 1e9
    ref_bw = peak if bound == "hbm" else (b_link / t_link / 1e9 if t_link else bw_link)  # duplex link rate
    return {"bound": bound, "kernel": "stage loop (SURVEY 8(d) model bytes / device-timed simulation)",
            "achieved": achieved, "peak": ref_bw, "unit": "GB/s", "frac": max(t_hbm, t_link) / t,
            "peak_source": peak_kind if bound == "hbm" else "measured pinned copy (bench.py measure_link)",
            "traffic": traffic, "model_bytes": b_hbm, "model_groups": d["model_groups"],
            "link": dict(link or {}, bytes=b_link, h2d_bytes=d["link_h2d_bytes"], d2h_bytes=d["link_d2h_bytes"],
                         copy_ms=d["link_ms"]),
            "phases": {k: {"ms": v[0], "bytes": v[1], "gbs": v[1] / (v[0] / 1e3) / 1e9 if v[0] > 0 else None,
                           "frac": v[1] / (v[0] / 1e3) / 1e9 / peak if v[0] > 0 else None}
                       for k, v in phases.items()},
            "dominant_phase": dom}


def main_sharded_capi(args, world, rank, local, dist, circ, cfg):
    """N GPUs, one simulation through the C ABI's sharded stage loop
    (bmq_simulator_run_sharded: host C++ driver over an NCCL communicator that
    libbmq creates from a unique id broadcast by rank 0)."""
    import torch
    from paper_2410_14088_b200 import cbq
    w = WORKLOAD
    uid = [cbq.Collective.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    col = cbq.Collective.nccl(uid[0], rank, world, local)
    sim = cbq.Simulator(circ, cfg)
    stages = len(sim.plan().stages)
    amp_stages = (1 << w["n"]) * stages
    for _ in range(args.warmup):
        sim.run_sharded(col)
    reps, dev_ms = [], []
    barrier_sync(dist)
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            barrier_sync(dist)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            reps.append(sim.run_sharded(col))
            torch.cuda.synchronize()
            ev1.record()
            ev1.synchronize()
            dev_ms.append(ev0.elapsed_time(ev1))
        barrier_sync(dist)
    t_dev = max_over_ranks(dist, statistics.median(dev_ms))
    rep = reps[-1]
    fidelity = None
    if w["name"] == "qft":  # |<u|psi>| from the all-reduced block sums of every rank's share
        import ctypes
        import numpy as np
        s3 = (ctypes.c_double * 3)()
        cbq._check(cbq.lib.bmq_simulator_partial_sums(sim._h, s3))
        sums = torch.tensor(list(s3), dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(sums)
        fidelity = float(np.hypot(float(sums[1]), float(sums[2])) * 2.0 ** (-0.5 * w["n"]))
    value = amp_stages / (t_dev / 1e3)
    e2e = None
    if not args.no_e2e:
        times, h2d, d2h = [], 0, 0
        gates_arr = circ.c_array()
        for step in range(max(1, min(args.steps, 3)) + 1):
            barrier_sync(dist)
            t0 = time.perf_counter()
            with cbq.Simulator(circ, cfg) as s2:
                s2.run_sharded(col)
                pays = s2.payloads()  # this rank's blocks (the others read as ALL_ZERO headers)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if step > 0:
                times.append(dt)
            h2d = len(bytes(gates_arr)) + 8
            d2h = sum(len(p) for p in pays)
        t_e2e = max_over_ranks(dist, statistics.median(times))
        e2e = {"value": amp_stages / t_e2e, "unit": "amp-stages/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "seconds": t_e2e}
    sim.close()
    col.close()
    line = {
        "metric": metric_name(w), "value": value, "unit": "amp-stages/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": data_desc(w),
        "config": {"workload": workload_tag(w), "stages": stages,
                   "parallelism": f"shard{world} (device qubits; C ABI driver, NCCL payload remaps)",
                   "zero_group_skip": True, "identity_skip": not args.no_identity_skip,
                   "stage_fusion": "off (sharded runs)",
                   "l2": "working set (16 GiB batches) >> 126 MB L2; no flush needed"},
        "sim_time_s": t_dev / 1e3, "compression_ratio": rep.compression_ratio,
        "max_footprint_bytes": rep.max_footprint_bytes, "fidelity": fidelity, "final_norm": rep.final_norm,
        "gpu_launches": int(rep.device["kernel_launches"]),
        "clocks": clocks.summary(), "e2e": e2e,
    }
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))
    return 0


def main_sharded(args, world, rank, local, dist):
    """N GPUs, one simulation: the stage loop sharded over device qubits with
    payload remaps over NCCL (paper_2410_14088_b200/shard.py). Total work is
    fixed (strong scaling); value = amp-stages of the one simulation / the
    max over ranks of the device-timed run."""
    import torch
    from paper_2410_14088_b200 import cbq
    from paper_2410_14088_b200.shard import EngineShard, ShardedSimulator, TorchCollective
    if dist is None:  # --sharded at N=1: a one-rank NCCL group
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
    w = WORKLOAD
    circ = cbq.generate_benchmark(w["name"], w["n"], cbq.BenchmarkParams(layers=w["layers"]))
    cfg = cbq.Config(block_bits=w["b"], inner_size=w["inner"], error_bound=w["error_bound"], device=local,
                     identity_skip=not args.no_identity_skip)
    if not args.py_shard:
        return main_sharded_capi(args, world, rank, local, dist, circ, cfg)
    col = TorchCollective(torch.device("cuda", local))
    be = EngineShard(circ, cfg, rank, world)
    ssim = ShardedSimulator(be, col)
    stages = len(ssim.stages)
    amp_stages = (1 << w["n"]) * stages
    for _ in range(args.warmup):
        ssim.run()
    reps, dev_ms = [], []
    barrier_sync(dist)
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            barrier_sync(dist)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            reps.append(ssim.run())
            torch.cuda.synchronize()
            ev1.record()
            ev1.synchronize()
            dev_ms.append(ev0.elapsed_time(ev1))
        barrier_sync(dist)
    t_dev = max_over_ranks(dist, statistics.median(dev_ms))
    rep = reps[-1]
    local_rep = be.report()
    fidelity = ssim.fidelity_uniform() if w["name"] == "qft" else None
    value = amp_stages / (t_dev / 1e3)
    be.close()
    e2e = None
    if not args.no_e2e:
        times, h2d, d2h = [], 0, 0
        gates_arr = circ.c_array()
        for step in range(max(1, min(args.steps, 3)) + 1):
            barrier_sync(dist)
            t0 = time.perf_counter()
            b2 = EngineShard(circ, cfg, rank, world)
            s2 = ShardedSimulator(b2, col)
            s2.run()
            pays = s2.gather_payloads(0)
            b2.close()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if step > 0:
                times.append(dt)
            h2d = len(bytes(gates_arr)) + 8
            d2h = sum(len(p) for p in pays) + 8 * len(pays) if pays else 0
        t_e2e = max_over_ranks(dist, statistics.median(times))
        e2e = {"value": amp_stages / t_e2e, "unit": "amp-stages/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "seconds": t_e2e}
    line = {
        "metric": metric_name(w), "value": value, "unit": "amp-stages/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": data_desc(w),
        "config": {"workload": workload_tag(w), "stages": stages,
                   "parallelism": f"shard{world} (device qubits, NCCL payload remaps)",
                   "zero_group_skip": True, "identity_skip": not args.no_identity_skip,
                   "l2": "working set (16 GiB batches) >> 126 MB L2; no flush needed"},
        "sim_time_s": t_dev / 1e3, "compression_ratio": rep.compression_ratio,
        "max_footprint_bytes": rep.max_footprint_bytes, "fidelity": fidelity, "final_norm": rep.final_norm,
        "gpu_launches": int(rep.device["kernel_launches"]),
        "groups_processed": rep.device["groups_processed"], "groups_skipped": rep.device["groups_skipped"],
        "remaps": ssim.remaps, "exchange_ms_rank0": ssim.exchange_ms, "account_ms_rank0": ssim.account_ms,
        "roofline": dict(roofline(local_rep.device, t_dev, None), scope="rank 0"),
        "clocks": clocks.summary(), "e2e": e2e,
    }
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))
    return 0


def e2e_once(args):
    """--e2e-once (internal): ONE create -> run -> get_payloads -> destroy through
    the C ABI in a fresh process, timed from before create (CUDA context,
    codec-table build and allocation included): a one-shot caller's cost."""
    import ctypes as C
    import numpy as np
    from paper_2410_14088_b200 import _lib, cbq
    w = WORKLOAD
    circ = cbq.generate_benchmark(w["name"], w["n"], cbq.BenchmarkParams(layers=w["layers"]))
    cfg = cbq.Config(block_bits=w["b"], inner_size=w["inner"], error_bound=w["error_bound"],
                     fuse_stages=args.fuse_stages)
    gates = circ.c_array()
    ccfg = cfg.to_c()
    lib = _lib.lib
    t0 = time.perf_counter()
    h = C.c_void_p()
    cbq._check(lib.bmq_simulator_create(circ.num_qubits, gates, len(gates), C.byref(ccfg), C.byref(h)))
    rep = _lib.bmq_report()
    cbq._check(lib.bmq_simulator_run(h, C.byref(rep), None, 0))
    sizes = np.zeros(1 << (circ.num_qubits - cfg.block_bits), dtype=np.uint64)
    total = C.c_uint64()
    cbq._check(lib.bmq_simulator_get_payloads(h, None, 0, sizes.ctypes.data, C.byref(total)))
    out = np.empty(max(1, total.value), dtype=np.uint8)
    cbq._check(lib.bmq_simulator_get_payloads(h, out.ctypes.data, total.value, sizes.ctypes.data, C.byref(total)))
    lib.bmq_simulator_destroy(h)
    print(json.dumps({"seconds": time.perf_counter() - t0, "payload_bytes": int(total.value)}))
    return 0


def cold_first_call(args):
    cmd = [sys.executable, os.path.abspath(__file__), "--e2e-once", "--workload", WORKLOAD["name"],
           "--qubits", str(WORKLOAD["n"]), "--block-bits", str(WORKLOAD["b"]), "--inner-size",
           str(WORKLOAD["inner"]), "--error-bound", repr(WORKLOAD["error_bound"]), "--layers",
           str(WORKLOAD["layers"])] + ([] if args.fuse_stages else ["--no-fuse-stages"])
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0")))
        return json.loads(r.stdout.strip().splitlines()[-1])["seconds"]
    except Exception:
        return None


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec the same
    command as N ranks (one per GPU) on this node."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="bmq", choices=["bmq", "reference"])
    ap.add_argument("--workload", default=WORKLOAD["name"], choices=["qft", "ghz", "qaoa3reg", "random", "qaoa", "bv"])
    ap.add_argument("--layers", type=int, default=None, help="QAOA layers p / random-circuit depth")
    ap.add_argument("--error-bound", type=float, default=None)
    ap.add_argument("--qubits", type=int, default=WORKLOAD["n"])
    ap.add_argument("--block-bits", type=int, default=WORKLOAD["b"])
    ap.add_argument("--inner-size", type=int, default=WORKLOAD["inner"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-identity-skip", action="store_true",
                    help="process every block of every nonzero group (no diagonal-stage block skipping)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent full simulations instead of one sharded simulation")
    ap.add_argument("--sharded", action="store_true", help="use the sharded driver even at N=1")
    ap.add_argument("--no-link", action="store_true", help="skip the pinned host-link bandwidth measurement")
    ap.add_argument("--device-pool-gib", type=float, default=0.0,
                    help="fixed device payload arena (GiB); 0 = automatic, growing")
    ap.add_argument("--arena", default="auto", choices=["auto", "heap", "bump"],
                    help="device arena placement policy (payload bytes are identical)")
    ap.add_argument("--host-pool-gib", type=float, default=0.0,
                    help="pinned host level of the store (GiB); 0 = none")
    ap.add_argument("--disk-pool-gib", type=float, default=0.0,
                    help="disk level beneath the host level (spill file, GiB); 0 = none")
    ap.add_argument("--device-plan", action="store_true",
                    help="plan with bmq_plan_device_aware (inner size chosen for the device, --inner-size caps it)")
    ap.add_argument("--no-fuse-stages", dest="fuse_stages", action="store_false",
                    help="turn off BMQ_FLAG_STAGE_FUSION (runs of consecutive FP stages decoded / emitted once; "
                         "same payloads)")
    ap.add_argument("--py-shard", action="store_true",
                    help="N>1: the Python sharded driver (shard.py over torch.distributed) instead of the C ABI one")
    ap.add_argument("--e2e-once", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        return relaunch_under_torchrun(args)
    if env_world is not None and int(env_world) != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={env_world}"}))
        return 2
    if args.impl == "reference":
        return run_reference(args)
    WORKLOAD.update(name=args.workload, n=args.qubits, b=args.block_bits, inner=args.inner_size)
    if args.layers is not None:
        WORKLOAD["layers"] = args.layers
    elif args.workload in ("qaoa", "qaoa3reg"):
        WORKLOAD["layers"] = 4
    elif args.workload == "random":
        WORKLOAD["layers"] = 40
    if args.error_bound is not None:
        WORKLOAD["error_bound"] = args.error_bound
    if args.e2e_once:
        return e2e_once(args)
    if args.workload != "qft":
        args.no_cpu_baseline = True  # the sampled CPU baseline is defined on the QFT plan
    world, rank, local, dist = dist_setup()
    import torch
    torch.cuda.set_device(local)
    if (world > 1 and not args.replicas) or args.sharded:
        return main_sharded(args, world, rank, local, dist)
    from paper_2410_14088_b200 import cbq
    w = WORKLOAD
    circ = cbq.generate_benchmark(w["name"], w["n"], cbq.BenchmarkParams(layers=w["layers"]))
    cfg = cbq.Config(block_bits=w["b"], inner_size=w["inner"], error_bound=w["error_bound"], device=local,
                     identity_skip=not args.no_identity_skip, device_pool_bytes=int(args.device_pool_gib * 2**30),
                     host_pool_bytes=int(args.host_pool_gib * 2**30), arena=args.arena,
                     disk_pool_bytes=int(args.disk_pool_gib * 2**30), device_plan=args.device_plan,
                     fuse_stages=args.fuse_stages)
    sim = cbq.Simulator(circ, cfg)
    plan = sim.plan().stages
    stages = len(plan)
    amp_stages = (1 << w["n"]) * stages
    reps = []
    for _ in range(args.warmup):
        sim.reset()
        sim.run()
    barrier_sync(dist)
    with ClockSampler(local) as clocks:
        barrier_sync(dist)
        for _ in range(args.steps):
            sim.reset()
            reps.append(sim.run())
        barrier_sync(dist)
    dev_ms = [r.device["device_ms"] for r in reps]
    wall_ms = [r.wall_ms for r in reps]
    t_dev = max_over_ranks(dist, statistics.median(dev_ms))
    rep = reps[-1]
    fidelity = fidelity_of(cbq, sim, circ, cfg, w)
    sim.close()
    value = world * amp_stages / (t_dev / 1e3)
    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(cbq, circ, cfg, amp_stages, args, dist, world)
        if rank == 0:
            cold = cold_first_call(args)
            e2e["cold_first_call_s"] = cold
            e2e["cold_first_call_note"] = ("one create->run->get_payloads->destroy in a fresh process, timed from "
                                           "before create: CUDA context, codec tables, allocation included")
    link = measure_link() if not args.no_link else None
    roof = roofline(rep.device, t_dev, link)
    line = {
        "metric": metric_name(w), "value": value, "unit": "amp-stages/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev,
        "higher_is_better": True, "scaling": "weak" if world > 1 else "strong", "vs_baseline": None,
        "dtype": "f64", "data": data_desc(w),
        "config": {"workload": workload_tag(w), "stages": stages,
                   "plan": ("device-aware (bmq_plan_device_aware): inner "
                            f"{max((len(s.inner) for s in plan), default=0)}" if args.device_plan
                            else f"partition_circuit inner_size={w['inner']}"),
                   "parallelism": f"replicas{world}" if world > 1 else "1gpu",
                   "zero_group_skip": True, "identity_skip": not args.no_identity_skip,
                   "device_pool": f"{args.device_pool_gib:g} GiB fixed" if args.device_pool_gib else "automatic",
                   "stage_fusion": (f"{rep.device['fused_stages']} stages in {rep.device['fused_sets']} fused runs"
                                    if args.fuse_stages else "off"),
                   "host_pool_gib": args.host_pool_gib, "arena": args.arena,
                   "l2": "working set (16 GiB batches) >> 126 MB L2; no flush needed"},
        "sim_time_s": t_dev / 1e3, "wall_ms_median": statistics.median(wall_ms),
        "compression_ratio": rep.compression_ratio, "max_footprint_bytes": rep.max_footprint_bytes,
        "fidelity": fidelity, "final_norm": rep.final_norm,
        "gpu_launches": int(rep.device["kernel_launches"]),
        "groups_processed": rep.device["groups_processed"], "groups_skipped": rep.device["groups_skipped"],
        "device_peak_bytes": int(rep.device["device_peak_bytes"]),
        "store": {k: rep.device[k] for k in ("arena_bytes", "compactions", "compact_bytes", "pool_growths",
                                             "host_spill_bytes", "host_peak_bytes", "link_h2d_bytes",
                                             "link_d2h_bytes", "link_ms", "disk_spill_bytes", "disk_read_bytes",
                                             "disk_peak_bytes", "disk_gds")},
        "gate_passes": {"total": int(rep.device["gate_passes"]), "streaming": int(rep.device["stream_passes"])},
        "roofline": roof, "clocks": clocks.summary(), "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline()
        except Exception as e:  # the oracle is optional at run time
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
