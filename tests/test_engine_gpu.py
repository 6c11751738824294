"""Device Simulator parity (cbq::Simulator, engine.hpp:58-250): final
payloads byte-identical to the reference run, reports (stages, peak
footprint replayed in put order, spills, compression ratio, calls) equal,
norm and fidelity within stated tolerances."""
import ctypes as C
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NORM_RTOL = 1e-10        # sums over up to 2^20 amplitudes in a different order
FIDELITY_ATOL = 1e-6     # north_star: within 1e-6 of the reference fidelity


def fnv(port, payloads):
    f = port.lib.cbqo_fnv1a64
    f.restype, f.argtypes = C.c_uint64, [C.c_char_p, C.c_uint64, C.c_uint64]
    h = 0xCBF29CE484222325
    for p in payloads:
        if p:
            h = f(p, len(p), h)
    return h


def golden_cases():
    with open(os.path.join(GOLDEN, "sim_golden.json")) as f:
        return json.load(f)["simulations"]


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: f"{c['name']}{c['n']}-b{c['b']}-i{c['inner']}-{c['error_bound']}")
def test_simulator_matches_reference_golden(gpu, port, case):
    c = gpu.generate_benchmark(case["name"], case["n"], gpu.BenchmarkParams(layers=case["layers"], seed=1))
    with gpu.Simulator(c, gpu.Config(block_bits=case["b"], inner_size=case["inner"],
                                     error_bound=case["error_bound"])) as sim:
        rep = sim.run()
        want = case["report"]
        assert rep.stage_count == want["stage_count"]
        assert rep.max_footprint_bytes == want["max_footprint_bytes"]
        assert rep.compression_ratio == want["compression_ratio"]
        assert rep.spilled_blocks == want["spilled_blocks"]
        assert rep.stage_compress_calls == want["stage_compress_calls"]
        assert rep.stage_decompress_calls == want["stage_decompress_calls"]
        assert rep.final_norm == pytest.approx(want["final_norm"], rel=NORM_RTOL)
        assert f"{fnv(port, sim.payloads()):016x}" == case["payload_fnv"]
        if want.get("has_fidelity"):
            ideal = gpu.dense_reference(c)
            f = sim.fidelity_dense(ideal)
            assert abs(f - want["fidelity"]) <= FIDELITY_ATOL
            if case["error_bound"] <= 1e-3:
                assert f >= 0.99


def random_circuit(gpu, rng, n, count):
    gl = []
    for _ in range(count):
        k = int(rng.integers(15))
        q0 = int(rng.integers(n))
        q1 = int((q0 + 1 + rng.integers(n - 1)) % n)
        gl.append((k, q0, q1 if k >= 12 else 0, float(rng.uniform(0, 6.28))))
    return gl, gpu.Circuit(n, [gpu.Gate(gpu.GateKind(k), a, b, ang) for k, a, b, ang in gl])


@pytest.mark.parametrize("seed", range(8))
def test_random_circuits_match_oracle(gpu, port, seed):
    rng = np.random.default_rng(100 + seed)
    n = 6 + seed % 9
    gl, c = random_circuit(gpu, rng, n, 50)
    b = 1 + int(rng.integers(n))
    inner = int(rng.integers(5))
    br = [1e-2, 1e-3, 1e-4, 0.5][seed % 4]
    res = port.simulate(n, gl, b, inner, br, want_state=True)
    with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=inner, error_bound=br)) as sim:
        rep = sim.run()
        assert sim.payloads() == res.payloads
        assert rep.max_footprint_bytes == res.report["max_footprint_bytes"]
        assert rep.final_norm == pytest.approx(res.report["final_norm"], rel=NORM_RTOL)
        st = sim.extract_state()
        assert np.array_equal(st.view(np.uint64), res.state.view(np.uint64))
        k = int(rng.integers(1 << n))
        assert sim.amplitude(k) == res.state[k]


def test_zero_group_skip_is_exact(gpu):
    c = gpu.generate_benchmark("qft", 16)
    outs = []
    for skip in (True, False):
        with gpu.Simulator(c, gpu.Config(block_bits=10, inner_size=2, zero_group_skip=skip)) as sim:
            rep = sim.run()
            outs.append((sim.payloads(), rep.max_footprint_bytes))
            if skip:
                assert rep.device["groups_skipped"] > 0
            else:
                assert rep.device["groups_skipped"] == 0
    assert outs[0] == outs[1]


@pytest.mark.parametrize("seed", [0, 1])
def test_cancellation_inside_stage_is_exact(gpu, port, seed):
    """A dense state whose stage undoes itself (RY layer, then H twice on every
    qubit, then RY back): later passes of the stage see groups the earlier
    passes zeroed although the decoded batch had none (zero-group summary)."""
    n, b = 17, 12
    rng = np.random.default_rng(900 + seed)
    ang = [float(a) for a in rng.uniform(0.2, 1.2, n)]
    gl = [(0, q, 0, 0.0) for q in range(n)]
    gl += [(9, q, 0, ang[q]) for q in range(n)]
    gl += [(0, q, 0, 0.0) for q in range(n)] * 2
    gl += [(9, q, 0, -ang[q]) for q in range(n)]
    gl += [(0, q, 0, 0.0) for q in range(n)]
    c = gpu.Circuit(n, [gpu.Gate(gpu.GateKind(k), a, bb, t) for k, a, bb, t in gl])
    want = port.simulate(n, gl, b, 2, 1e-3)
    with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=2, error_bound=1e-3)) as sim:
        rep = sim.run()
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]


@pytest.mark.parametrize("name,n,b,inner,layers", [("qft", 18, 12, 2, 1), ("qft", 17, 12, 4, 1),
                                                   ("qaoa", 16, 12, 2, 2), ("bv", 16, 13, 2, 1)])
def test_identity_skip_is_exact(gpu, port, name, n, b, inner, layers):
    c = gpu.generate_benchmark(name, n, gpu.BenchmarkParams(layers=layers))
    want = port.simulate(n, [g.as_tuple() for g in c.gates], b, inner, 1e-3)
    # (stage fusion off: a fused run processes every block of its union groups)
    with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=inner, identity_skip=True, fuse_stages=False)) as sim:
        rep = sim.run()
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=NORM_RTOL)
        if name == "qft":  # QFT stages are mostly controlled phases: many blocks skipped
            assert rep.device["blocks_processed"] < rep.stage_count * (1 << (n - b))


def test_arena_compaction_is_exact(gpu, port):
    c = gpu.generate_benchmark("qaoa", 16, gpu.BenchmarkParams(layers=2))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    biggest = max(len(p) for p in want.payloads)
    pool = 24 * (biggest + 16)  # the live state plus about two batches
    with gpu.Simulator(c, gpu.Config(block_bits=12, inner_size=2, device_pool_bytes=pool, arena="bump",
                                     work_bytes=4 * (16 << 12), fuse_stages=False)) as sim:
        rep = sim.run()
        assert rep.device["compactions"] > 0
        assert sim.payloads() == want.payloads


@pytest.mark.parametrize("arena", ["heap", "bump"])
def test_host_spill_is_exact(gpu, port, arena):
    """Two-level store (store.hpp:47-300): with a device arena far smaller than
    the live state, payloads land in the pinned host arena and are read back
    from there by the next stage; the result is unchanged byte for byte."""
    c = gpu.generate_benchmark("qaoa", 16, gpu.BenchmarkParams(layers=2))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    biggest = max(len(p) for p in want.payloads)
    pool = 6 * (biggest + 16)  # about one batch: most payloads must go to the host
    cfg = gpu.Config(block_bits=12, inner_size=2, device_pool_bytes=pool, work_bytes=4 * (16 << 12),
                     host_pool_bytes=64 << 20, arena=arena)
    with gpu.Simulator(c, cfg) as sim:
        rep = sim.run()
        assert rep.device["host_spill_batches"] > 0
        assert rep.device["host_spill_bytes"] > 0
        assert sim.payloads() == want.payloads
        for i in (0, 3, 15):
            assert sim.get_payload(i) == want.payloads[i]
        assert abs(sim.state_norm() - want.report["final_norm"]) <= NORM_RTOL * want.report["final_norm"]
    cfg = gpu.Config(block_bits=12, inner_size=2, device_pool_bytes=pool, work_bytes=4 * (16 << 12), arena=arena)
    with gpu.Simulator(c, cfg) as sim:
        with pytest.raises(gpu.StoreError):
            sim.run()


@pytest.mark.parametrize("arena", ["heap", "bump"])
def test_host_level_reclaims_rewritten_payloads(gpu, port, arena):
    """The host level reuses the extents of rewritten payloads: over the run
    far more payload bytes go to the host than the host arena holds, every
    stage's host-level payloads are prefetched on the copy stream (H2D) and
    written back on the other (D2H), and the result is byte-identical."""
    c = gpu.generate_benchmark("qaoa", 16, gpu.BenchmarkParams(layers=2))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    biggest = max(len(p) for p in want.payloads)
    state = sum(len(p) for p in want.payloads)
    host = 2 * state + 16 * (biggest + 16)
    cfg = gpu.Config(block_bits=12, inner_size=2, device_pool_bytes=6 * (biggest + 16), work_bytes=4 * (16 << 12),
                     host_pool_bytes=host, arena=arena)
    with gpu.Simulator(c, cfg) as sim:
        rep = sim.run()
        d = rep.device
        assert d["host_spill_bytes"] > host  # more than the arena holds: rewritten payloads were reclaimed
        assert d["link_h2d_bytes"] > 0 and d["link_d2h_bytes"] > 0
        assert d["host_peak_bytes"] <= host
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=NORM_RTOL)


def test_in_place_compaction_keeps_live_payloads(gpu, port):
    """A fixed device arena a little larger than the live state: compactions
    slide the live payloads down in place (directly or through the staging
    buffer) many times; every payload stays byte-identical."""
    c = gpu.generate_benchmark("qaoa", 16, gpu.BenchmarkParams(layers=3))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    state = sum((len(p) + 15) // 16 * 16 for p in want.payloads)
    biggest = max(len(p) for p in want.payloads)
    cfg = gpu.Config(block_bits=12, inner_size=2, device_pool_bytes=state + 5 * (biggest + 16),
                     work_bytes=4 * (16 << 12), arena="bump", fuse_stages=False)
    with gpu.Simulator(c, cfg) as sim:
        rep = sim.run()
        assert rep.device["compactions"] >= rep.stage_count
        assert rep.device["compact_bytes"] > 0
        assert sim.payloads() == want.payloads


def test_heap_arena_reuses_decoded_extents(gpu, port):
    """Heap-mode arena (one extent per payload, freed when its block is
    rewritten): a fixed arena only a few payloads larger than the live state
    runs every dense stage without compaction or host spill, byte-exact."""
    c = gpu.generate_benchmark("qaoa", 16, gpu.BenchmarkParams(layers=3))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    state = sum((len(p) + 15) // 16 * 16 for p in want.payloads)
    biggest = max(len(p) for p in want.payloads)
    cfg = gpu.Config(block_bits=12, inner_size=2, device_pool_bytes=state + 8 * (biggest + 16),
                     work_bytes=4 * (16 << 12), arena="heap")
    with gpu.Simulator(c, cfg) as sim:
        rep = sim.run()
        assert rep.device["host_spill_bytes"] == 0
        assert rep.device["compactions"] <= 1
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]


@pytest.mark.parametrize("arena", ["heap", "bump"])
@pytest.mark.parametrize("name,layers", [("qft", 1), ("qaoa3reg", 2), ("random", 12)])
def test_arena_policies_are_exact(gpu, port, arena, name, layers):
    """Both device-arena policies on automatic sizing give the oracle's bytes."""
    c = gpu.generate_benchmark(name, 16, gpu.BenchmarkParams(layers=layers, seed=3))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 10, 2, 1e-3)
    with gpu.Simulator(c, gpu.Config(block_bits=10, inner_size=2, arena=arena, work_bytes=8 * (16 << 10))) as sim:
        rep = sim.run()
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]


def test_small_batches_are_exact(gpu, port):
    c = gpu.generate_benchmark("qaoa", 14, gpu.BenchmarkParams(layers=2))
    want = port.simulate(14, [g.as_tuple() for g in c.gates], 9, 2, 1e-3)
    with gpu.Simulator(c, gpu.Config(block_bits=9, inner_size=2, work_bytes=3 * (16 << 9) * 4)) as sim:
        sim.run()
        assert sim.payloads() == want.payloads


def test_spill_accounting(gpu, port):
    c = gpu.generate_benchmark("qft", 16)
    gl = [g.as_tuple() for g in c.gates]
    want = port.simulate(16, gl, 8, 2, 1e-3, memory_budget=20000)
    with gpu.Simulator(c, gpu.Config(block_bits=8, inner_size=2, memory_budget=20000)) as sim:
        rep = sim.run()
        assert rep.spilled_blocks == want.report["spilled_blocks"] > 0
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert sim.payloads() == want.payloads


def test_uncompressed_mode(gpu, port):
    rng = np.random.default_rng(21)
    gl, c = random_circuit(gpu, rng, 10, 60)
    want = port.simulate(10, gl, 4, 2, 1e-3, compress=False, want_state=True)
    with gpu.Simulator(c, gpu.Config(block_bits=4, inner_size=2, compress=False)) as sim:
        rep = sim.run()
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert np.array_equal(sim.extract_state(), want.state)  # values equal (zero signs may differ)
        assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=NORM_RTOL)


def test_fidelity_paths_agree(gpu):
    c = gpu.generate_benchmark("qft", 14)
    with gpu.Simulator(c, gpu.Config(block_bits=8, inner_size=2)) as sim, \
            gpu.Simulator(c, gpu.Config(block_bits=8, inner_size=2, compress=False)) as exact:
        sim.run()
        exact.run()
        f_dense = sim.fidelity_dense(gpu.dense_reference(c))
        f_pair = sim.fidelity_with(exact)
        f_uni = sim.fidelity_analytic("uniform")
        assert f_dense >= 0.99
        assert f_pair == pytest.approx(f_dense, abs=1e-9)
        assert f_uni == pytest.approx(f_dense, abs=1e-9)
    g = gpu.generate_benchmark("ghz", 14)
    with gpu.Simulator(g, gpu.Config(block_bits=6, inner_size=2)) as sim:
        sim.run()
        assert sim.fidelity_analytic("ghz") == pytest.approx(sim.fidelity_dense(gpu.dense_reference(g)), abs=1e-12)


def test_payload_round_trip_and_errors(gpu, port):
    c = gpu.generate_benchmark("qaoa", 10, gpu.BenchmarkParams(layers=1))
    with gpu.Simulator(c, gpu.Config(block_bits=5, inner_size=2)) as sim:
        sim.init_state()
        with pytest.raises(gpu.EngineError, match="already initialized"):
            sim.init_state()
        x = np.linspace(-0.1, 0.1, 64)
        p = port.compress_block(x, 1e-3)
        sim.put_payload(3, p)
        assert sim.get_payload(3) == p
        assert sim.amplitude(3 * 32 + 5) == complex(port.decompress_block(p)[5], port.decompress_block(p)[37])
        with pytest.raises(gpu.CodecError, match="codes truncated"):
            sim.put_payload(4, p[:-1])
        assert sim.get_payload(4) == port.compress_block(np.zeros(64), 1e-3)
    big = gpu.generate_benchmark("ghz", 26)
    with gpu.Simulator(big, gpu.Config(block_bits=20, inner_size=2)) as sim:
        with pytest.raises(gpu.EngineError, match="dense verification refused: 26 qubits exceeds the cap of 24"):
            sim.extract_state()


def test_stage_by_stage_driver(gpu):
    c = gpu.generate_benchmark("qft", 12)
    with gpu.Simulator(c, gpu.Config(block_bits=6, inner_size=2)) as a, \
            gpu.Simulator(c, gpu.Config(block_bits=6, inner_size=2)) as b:
        a.run()
        nst = len(b.plan().stages)
        for s in range(nst):
            b.run_stages(s, s + 1)
        assert a.payloads() == b.payloads()
        with pytest.raises(gpu.EngineError, match="stages must run in order"):
            b.run_stages(0, 1)


@pytest.mark.slow
def test_ghz30_b20_block_sizes(gpu):
    """C2 shape: GHZ-30, b=20, inner=2 — only the two end blocks are nonzero."""
    c = gpu.generate_benchmark("ghz", 30)
    with gpu.Simulator(c, gpu.Config(block_bits=20, inner_size=2)) as sim:
        rep = sim.run()
        assert rep.stage_count == 9
        sizes = [len(sim.get_payload(i)) for i in (0, 1, 1023)]
        assert sizes[1] == 26
        assert sim.fidelity_analytic("ghz") >= 0.99
        assert abs(rep.final_norm - 1) < 2e-3


def monomial_circuit(gpu, rng, n, count):
    """A dense complex state (H, T, RX layers) followed by `count` random
    unit-entry monomial gates (X, Y, Z, S, Sdg, CX, CZ) and a closing RY
    layer, so the plan holds code-domain stages between FP64 stages."""
    gl = []
    for q in range(n):
        gl += [(0, q, 0, 0.0), (6, q, 0, 0.0), (8, q, 0, 0.1 + 0.05 * q)]
    mono = [1, 2, 3, 4, 5, 12, 13]
    for _ in range(count):
        k = int(rng.choice(mono))
        q0 = int(rng.integers(n))
        q1 = int((q0 + 1 + rng.integers(n - 1)) % n)
        gl.append((k, q0, q1 if k >= 12 else 0, 0.0))
    gl += [(9, q, 0, 0.3) for q in range(0, n, 3)]
    return gl, gpu.Circuit(n, [gpu.Gate(gpu.GateKind(k), a, b, ang) for k, a, b, ang in gl])


@pytest.mark.parametrize("seed,n,b,inner,br", [(0, 16, 12, 2, 1e-3), (1, 17, 12, 3, 1e-4), (2, 16, 13, 1, 1e-2),
                                               (3, 18, 12, 2, 1e-3)])
def test_code_domain_stages_are_exact(gpu, port, seed, n, b, inner, br):
    """Stages of X/Y/Z/S/Sdg/CX/CZ run on quantiser codes (BMQ_FLAG_CODE_DOMAIN):
    payloads byte-identical to the oracle, with the path on and off."""
    rng = np.random.default_rng(500 + seed)
    gl, c = monomial_circuit(gpu, rng, n, 120)
    want = port.simulate(n, gl, b, inner, br)
    for on in (True, False):
        with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=inner, error_bound=br, code_domain=on)) as sim:
            rep = sim.run()
            assert (rep.device["code_domain_batches"] > 0) == on
            assert sim.payloads() == want.payloads
            assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
            assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=NORM_RTOL)


@pytest.mark.parametrize("seed,kinds", [(0, (1, 3, 12, 13)), (1, (1, 3, 12, 13, 4)), (2, (12,)), (3, (2, 12, 13))])
def test_code_domain_real_states_are_exact(gpu, port, seed, kinds):
    """A real state (H, RY) under X/Z/CX/CZ keeps its imaginary halves zero:
    the code-domain passes leave them untouched. With S or Y in the stage the
    halves mix and are processed; payloads byte-identical to the oracle."""
    rng = np.random.default_rng(700 + seed)
    n, b = 17, 12
    gl = [(0, q, 0, 0.0) for q in range(n)] + [(9, q, 0, 0.2 + 0.1 * q) for q in range(n)]
    for _ in range(60):
        k = int(rng.choice(kinds))
        q0 = int(rng.integers(n))
        q1 = int((q0 + 1 + rng.integers(n - 1)) % n)
        gl.append((k, q0, q1 if k >= 12 else 0, 0.0))
    gl += [(9, q, 0, 0.3) for q in range(0, n, 4)]
    c = gpu.Circuit(n, [gpu.Gate(gpu.GateKind(k), a, bb, ang) for k, a, bb, ang in gl])
    want = port.simulate(n, gl, b, 2, 1e-3)
    with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=2, error_bound=1e-3)) as sim:
        rep = sim.run()
        assert rep.device["code_domain_batches"] > 0
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]


def test_code_domain_qft_swaps(gpu, port):
    """QFT's closing bit-reversal (CX triples) runs in the code domain."""
    c = gpu.generate_benchmark("qft", 18)
    want = port.simulate(18, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    with gpu.Simulator(c, gpu.Config(block_bits=12, inner_size=2, identity_skip=True)) as sim:
        rep = sim.run()
        assert rep.device["code_domain_batches"] > 0
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        # final sums (one-bit-code chunks are counted, not decoded)
        assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=NORM_RTOL)
        amps = sim.extract_state()
        assert sim.fidelity_analytic("uniform") == pytest.approx(abs(amps.sum()) / np.sqrt(len(amps)), rel=1e-9)


@pytest.mark.parametrize("arena", ["heap", "bump"])
def test_pool_growth_is_exact(gpu, port, arena):
    """Arenas that start small double after compactions (BMQ_FLAG_POOL_GROW);
    payloads stay byte-identical to the oracle."""
    c = gpu.generate_benchmark("qaoa", 16, gpu.BenchmarkParams(layers=2))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    biggest = max(len(p) for p in want.payloads)
    pool = 8 * (biggest + 16)
    with gpu.Simulator(c, gpu.Config(block_bits=12, inner_size=2, device_pool_bytes=pool, pool_grow=True,
                                     work_bytes=4 * (16 << 12), arena=arena)) as sim:
        rep = sim.run()
        assert rep.device["pool_growths"] > 0
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]


def lazy_cx_circuit(gpu, rng, n, count):
    """Dense start, then random CX (controls inside and outside the tile),
    CP runs sharing a control (phase chains), H / RX / RZ / CZ: exercises the
    lazy-CX index map, its materialisation before chains, and the gather on
    store."""
    gl = [(0, q, 0, 0.0) for q in range(n)] + [(10, q, 0, 0.3 + 0.1 * q) for q in range(n)]
    for _ in range(count):
        r = rng.random()
        if r < 0.45:
            a, b = rng.choice(n, 2, replace=False)
            gl.append((12, int(a), int(b), 0.0))
        elif r < 0.6:  # a phase chain: CP(j, c) for descending j
            c = int(rng.integers(3, n))
            for j in sorted(rng.choice(c, size=min(c, 4), replace=False), reverse=True):
                gl.append((14, int(j), c, float(np.pi / 2 ** (c - j))))
        elif r < 0.75:
            gl.append((0, int(rng.integers(n)), 0, 0.0))
        elif r < 0.9:
            gl.append((8 + int(rng.integers(3)), int(rng.integers(n)), 0, float(rng.uniform(0, 6.28))))
        else:
            a, b = rng.choice(n, 2, replace=False)
            gl.append((13, int(a), int(b), 0.0))
    return gl, gpu.Circuit(n, [gpu.Gate(gpu.GateKind(k), a, b, ang) for k, a, b, ang in gl])


@pytest.mark.parametrize("seed,n,b,inner", [(0, 16, 12, 2), (1, 17, 13, 3), (2, 16, 12, 4), (3, 18, 14, 2)])
def test_lazy_cx_passes_are_exact(gpu, port, seed, n, b, inner):
    rng = np.random.default_rng(900 + seed)
    gl, c = lazy_cx_circuit(gpu, rng, n, 160)
    want = port.simulate(n, gl, b, inner, 1e-3)
    with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=inner, error_bound=1e-3)) as sim:
        rep = sim.run()
        assert rep.device["lazy_cx"] > 0 and rep.device["perm_materialisations"] > 0
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=NORM_RTOL)


@pytest.mark.parametrize("n,b,inner", [(18, 12, 2), (19, 13, 3)])
def test_qft_sparse_stages_are_exact(gpu, port, n, b, inner):
    """QFT|0>: the phase chains act only on exact zeros (skipped walks) and
    early H sweeps mostly on zero pairs; payloads stay byte-exact."""
    c = gpu.generate_benchmark("qft", n)
    want = port.simulate(n, [g.as_tuple() for g in c.gates], b, inner, 1e-3)
    with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=inner, identity_skip=True)) as sim:
        sim.run()
        assert sim.payloads() == want.payloads


def test_support_tracking_matches_full_sweeps(gpu):
    """Tile support tracking (ops visit only positions that can be nonzero)
    against full sweeps (BMQ_DBG_FULL_SUPPORT=1 in a child process): same bytes."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); from paper_2410_14088_b200 import cbq; import hashlib\n"
            "for name, n, b in (('qft', 18, 12), ('ghz', 18, 12), ('bv', 17, 12)):\n"
            "    c = cbq.generate_benchmark(name, n)\n"
            "    with cbq.Simulator(c, cbq.Config(block_bits=b, inner_size=2)) as s:\n"
            "        s.run(); print(hashlib.sha256(b''.join(s.payloads())).hexdigest())\n") % os.path.dirname(os.path.dirname(GOLDEN))
    outs = []
    for env in ({}, {"BMQ_DBG_FULL_SUPPORT": "1"}):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env={**os.environ, **env})
        assert r.returncode == 0, r.stderr
        outs.append(r.stdout)
    assert outs[0] == outs[1] and outs[0].count("\n") == 3


@pytest.mark.parametrize("name,n,b,cut", [("qft", 18, 12, 7), ("qaoa", 16, 12, 5)])
def test_checkpoint_resume_is_exact(gpu, tmp_path, name, n, b, cut):
    """save() after `cut` stages, load() into a fresh simulator, run the rest:
    payloads, max_footprint and norm equal the uninterrupted run."""
    c = gpu.generate_benchmark(name, n, gpu.BenchmarkParams(layers=2)) if name == "qaoa" \
        else gpu.generate_benchmark(name, n)
    cfg = gpu.Config(block_bits=b, inner_size=2, error_bound=1e-3)
    with gpu.Simulator(c, cfg) as full:
        rep_full = full.run()
        want = full.payloads()
        nstages = len(full.plan().stages)
    path = str(tmp_path / "state.bmqckpt")
    with gpu.Simulator(c, cfg) as a:
        a.run_stages(0, cut)
        a.save(path)
    with gpu.Simulator(c, cfg) as b2:
        assert b2.load(path) == cut
        b2.run_stages(cut, nstages)
        rep = b2.report()
        assert b2.payloads() == want
        assert rep.max_footprint_bytes == rep_full.max_footprint_bytes
        assert rep.stage_compress_calls == rep_full.stage_compress_calls
        assert rep.final_norm == pytest.approx(rep_full.final_norm, rel=1e-12)
    # a simulator of another bound, or a damaged file, is refused
    with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=2, error_bound=1e-4)) as other:
        with pytest.raises(Exception, match="checkpoint"):
            other.load(path)
    with open(path, "rb") as f:
        data = f.read()
    bad = str(tmp_path / "short.bmqckpt")
    with open(bad, "wb") as f:
        f.write(data[: len(data) // 2])
    with gpu.Simulator(c, cfg) as other:
        with pytest.raises(Exception, match="checkpoint"):
            other.load(bad)


@pytest.mark.parametrize("name,n,layers,b,br", [("qft", 18, 1, 12, 1e-3), ("qaoa3reg", 18, 2, 12, 1e-4),
                                                ("random", 17, 8, 12, 1e-3)])
def test_device_plan_matches_reference_at_chosen_inner(gpu, port, name, n, layers, b, br):
    """Config.device_plan (BMQ_FLAG_DEVICE_PLAN): the engine
    plans with plan_device_aware (cap inner_size) and the result is the
    reference's run at the inner size it chose, byte for byte."""
    c = gpu.generate_benchmark(name, n, gpu.BenchmarkParams(layers=layers, seed=1))
    plan, ch = gpu.plan_device_aware(c, b, max_inner=n - b)
    want = port.simulate(n, [g.as_tuple() for g in c.gates], b, ch.inner_size, br)
    with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=n - b, error_bound=br, device_plan=True)) as sim:
        rep = sim.run()
        assert rep.stage_count == len(plan.stages) == want.report["stage_count"]
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]


@pytest.mark.parametrize("arena", ["heap", "bump"])
def test_disk_level_is_exact(gpu, port, arena):
    """Third level (the reference's spill file, store.hpp:234-283):
    device arena and host level both far smaller than the live state, so most
    payloads go to the spill file (pread / pwrite through a pinned bounce;
    cuFile with BMQ_GDS=1) and every stage reads them back; payloads,
    peak footprint, norm and the per-payload reads are unchanged."""
    c = gpu.generate_benchmark("qaoa", 16, gpu.BenchmarkParams(layers=2))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    biggest = max(len(p) for p in want.payloads)
    pool = 6 * (biggest + 16)
    cfg = gpu.Config(block_bits=12, inner_size=2, device_pool_bytes=pool, work_bytes=4 * (16 << 12),
                     host_pool_bytes=3 * (biggest + 16), disk_pool_bytes=64 << 20, arena=arena)
    with gpu.Simulator(c, cfg) as sim:
        rep = sim.run()
        d = rep.device
        assert d["disk_spill_bytes"] > 0 and d["disk_read_bytes"] > 0
        assert d["disk_peak_bytes"] <= 64 << 20
        assert sim.payloads() == want.payloads
        for i in (0, 3, 15):
            assert sim.get_payload(i) == want.payloads[i]
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert abs(sim.state_norm() - want.report["final_norm"]) <= NORM_RTOL * want.report["final_norm"]
        psi = sim.extract_state()  # decode path outside the stage loop
        assert abs(np.linalg.norm(psi) - want.report["final_norm"]) <= 1e-9
    with pytest.raises(gpu.InvalidArgument, match="host level"):
        gpu.Simulator(c, gpu.Config(block_bits=12, disk_pool_bytes=1 << 20))


def test_disk_level_posix_path(gpu, port, tmp_path):
    """Same run with GPUDirect Storage explicitly off (BMQ_NO_GDS): pread /
    pwrite through the pinned bounce buffer, spill file in a given directory."""
    import subprocess
    import sys
    code = f"""
import sys; sys.path.insert(0, {repr(os.path.dirname(GOLDEN) + '/../..')})
sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(GOLDEN)))})
from paper_2410_14088_b200 import cbq
from oracle import oracle
port = oracle.port()
c = cbq.generate_benchmark("qaoa", 16, cbq.BenchmarkParams(layers=2))
want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
big = max(len(p) for p in want.payloads)
cfg = cbq.Config(block_bits=12, inner_size=2, device_pool_bytes=6 * (big + 16), work_bytes=4 * (16 << 12),
                 host_pool_bytes=3 * (big + 16), disk_pool_bytes=64 << 20, disk_dir={repr(str(tmp_path))})
with cbq.Simulator(c, cfg) as sim:
    rep = sim.run()
    assert rep.device["disk_gds"] == 0 and rep.device["disk_spill_bytes"] > 0
    assert sim.payloads() == want.payloads
print("ok")
"""
    env = dict(os.environ, BMQ_NO_GDS="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_three_levels_with_device_plan_queries_and_checkpoint(gpu, port, tmp_path):
    """The optional pieces together: a device-aware plan (equal to the
    reference at the chosen inner size) on a state spilled across all three
    store levels; sampling / top-k / amplitude queries and a checkpoint read
    the disk-resident payloads; the resumed run equals the uninterrupted one."""
    c = gpu.generate_benchmark("qaoa3reg", 16, gpu.BenchmarkParams(layers=2, seed=1))
    plan, ch = gpu.plan_device_aware(c, 12, max_inner=3)
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, ch.inner_size, 1e-3, want_state=True)
    biggest = max(len(p) for p in want.payloads)
    cfg = gpu.Config(block_bits=12, inner_size=3, error_bound=1e-3, device_plan=True, work_bytes=8 * (16 << 12),
                     device_pool_bytes=5 * (biggest + 16), host_pool_bytes=3 * (biggest + 16),
                     disk_pool_bytes=16 << 20, disk_dir=str(tmp_path))
    with gpu.Simulator(c, cfg) as sim:
        rep = sim.run()
        assert rep.device["disk_spill_bytes"] > 0
        assert sim.payloads() == want.payloads
        psi = sim.extract_state()
        idx, amp = sim.top_k(5)
        key = psi.real * psi.real + psi.imag * psi.imag
        nz = np.flatnonzero(key)
        assert np.array_equal(idx.astype(np.int64), nz[np.lexsort((nz, -key[nz]))][:5])
        assert sim.amplitude(int(idx[0])) == psi[int(idx[0])]
        s = sim.sample(2000, seed=5)
        assert np.all(key[s.astype(np.int64)] > 0)
        ck = str(tmp_path / "state.bmqckpt")
        sim.save(ck)
    with gpu.Simulator(c, cfg) as sim2:
        assert sim2.load(ck) == rep.stage_count
        assert sim2.payloads() == want.payloads
