"""Stage fusion (BMQ_FLAG_STAGE_FUSION): consecutive FP stages of the
reference's plan decoded once and emitted once, with the quantiser round
trip (decompress_block(compress_block(.)), codec.hpp:227-344) applied in
place between them. The final payloads, the peak footprint replayed in each
stage's put order (store.hpp:64-83), the call counts and the norm must equal
the C oracle's run of the same plan (engine.hpp:97-134); batches holding
fewer union groups (small work buffers) and stages the engine keeps unfused
(code-domain, block-wise diagonal) are covered too."""
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # name, n, layers, b, inner, error bound
    ("qaoa3reg", 16, 2, 12, 2, 1e-4),
    ("qaoa3reg", 18, 1, 12, 3, 1e-3),
    ("random", 16, 8, 12, 2, 1e-3),
    ("random", 18, 6, 13, 2, 1e-2),
    ("qft", 16, 1, 12, 2, 1e-3),
    ("ghz", 16, 1, 12, 2, 1e-3),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}{c[1]}-b{c[3]}-i{c[4]}-{c[5]}")
@pytest.mark.parametrize("work_blocks", [0, 8], ids=["auto", "8blocks"])
def test_fused_run_matches_oracle(gpu, port, case, work_blocks):
    name, n, layers, b, inner, br = case
    c = gpu.generate_benchmark(name, n, gpu.BenchmarkParams(layers=layers, seed=1))
    want = port.simulate(n, [g.as_tuple() for g in c.gates], b, inner, br)
    cfg = gpu.Config(block_bits=b, inner_size=inner, error_bound=br, fuse_stages=True,
                     work_bytes=work_blocks * (16 << b))
    with gpu.Simulator(c, cfg) as sim:
        rep = sim.run()
        assert sim.payloads() == want.payloads
        assert rep.stage_count == want.report["stage_count"]
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert rep.spilled_blocks == want.report["spilled_blocks"]
        assert rep.stage_compress_calls == want.report["stage_compress_calls"]
        assert rep.stage_decompress_calls == want.report["stage_decompress_calls"]
        assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=1e-10)
        if name in ("qaoa3reg", "random") and (work_blocks == 0 or inner == 2):  # else no two stages fit 8 blocks
            assert rep.device["fused_stages"] >= 2 and rep.device["fused_sets"] >= 1


@pytest.mark.parametrize("name", ["qaoa3reg", "random"])
def test_fused_equals_unfused_with_budget(gpu, name):
    """A memory budget (spills counted by the store model) and both arena
    policies: the fused run's payloads and accounting equal the unfused run's."""
    c = gpu.generate_benchmark(name, 18, gpu.BenchmarkParams(layers=3, seed=2))
    out = []
    for fuse, arena in ((False, "auto"), (True, "heap"), (True, "bump")):
        cfg = gpu.Config(block_bits=12, inner_size=2, error_bound=1e-3, fuse_stages=fuse, arena=arena,
                         memory_budget=200_000)
        with gpu.Simulator(c, cfg) as sim:
            rep = sim.run()
            out.append((sim.payloads(), rep.max_footprint_bytes, rep.spilled_blocks, rep.device["fused_stages"]))
    assert out[0][3] == 0 and out[1][3] > 0 and out[2][3] > 0
    for got in out[1:]:
        assert got[:3] == out[0][:3]


@pytest.mark.parametrize("cut", [1, 3, 5])
def test_fused_resume_from_checkpoint(gpu, port, tmp_path, cut):
    """A checkpoint taken after `cut` stages (possibly inside what would be a
    fused run) and resumed with run(): the remaining stages run unfused up to
    the next fused run's first stage, then fused; the final payloads and the
    peak equal the oracle's uninterrupted run."""
    c = gpu.generate_benchmark("qaoa3reg", 16, gpu.BenchmarkParams(layers=2, seed=1))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-4)
    cfg = gpu.Config(block_bits=12, inner_size=2, error_bound=1e-4)
    path = str(tmp_path / "state.bmqckpt")
    with gpu.Simulator(c, cfg) as a:
        a.run_stages(0, cut)
        a.save(path)
    with gpu.Simulator(c, cfg) as b:
        assert b.load(path) == cut
        rep = b.run()
        assert b.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=1e-10)
