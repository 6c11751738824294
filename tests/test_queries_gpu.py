"""Sampling and top-k amplitude queries on the compressed state (SURVEY §8
f3; the reference offers only the dense, 24-qubit-capped extract_state,
engine.hpp:138-147). Checked against the decompressed dense state of the
same simulator."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run(gpu, name, n, b, layers=1, br=1e-3, inner=2):
    c = gpu.generate_benchmark(name, n, gpu.BenchmarkParams(layers=layers, seed=1))
    sim = gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=inner, error_bound=br))
    sim.run()
    return sim


def test_sampling_matches_state_distribution(gpu):
    with run(gpu, "qaoa3reg", 16, 12, layers=2, br=1e-4) as sim:
        psi = sim.extract_state()
        p = psi.real * psi.real + psi.imag * psi.imag
        p /= p.sum()
        shots = 200_000
        s = sim.sample(shots, seed=7)
        assert s.shape == (shots,) and s.dtype == np.uint64
        assert np.all(p[s.astype(np.int64)] > 0)
        # coarse bins (top 6 index bits): total variation within sampling noise
        got = np.bincount((s >> 10).astype(np.int64), minlength=64) / shots
        want = np.add.reduceat(p, np.arange(0, 1 << 16, 1 << 10))
        assert 0.5 * np.abs(got - want).sum() < 0.01
        assert np.array_equal(sim.sample(1000, seed=7), s[:1000])  # deterministic per seed
        assert not np.array_equal(sim.sample(1000, seed=8), s[:1000])


def test_sampling_sparse_state(gpu):
    with run(gpu, "ghz", 20, 12) as sim:
        s = sim.sample(20_000, seed=3)
        assert set(np.unique(s).tolist()) == {0, (1 << 20) - 1}
        assert abs(np.mean(s == 0) - 0.5) < 0.02


@pytest.mark.parametrize("k", [1, 10, 1000, 70_000])
def test_top_k_matches_dense(gpu, k):
    with run(gpu, "qaoa3reg", 16, 12, layers=2, br=1e-4) as sim:
        psi = sim.extract_state()
        key = psi.real * psi.real + psi.imag * psi.imag
        nz = np.flatnonzero(key)
        order = nz[np.lexsort((nz, -key[nz]))]  # largest first, ties to the lower index
        idx, amp = sim.top_k(k)
        m = min(k, nz.size)
        assert idx.size == m
        assert np.array_equal(idx.astype(np.int64), order[:m])
        assert np.array_equal(amp, psi[order[:m]])


def test_top_k_sparse_and_ties(gpu):
    with run(gpu, "ghz", 20, 12) as sim:
        assert sim.top_k(0)[0].size == 0
        idx, amp = sim.top_k(3)
        assert idx.tolist() == [0, (1 << 20) - 1]  # equal magnitudes: lower index first
        assert np.allclose(np.abs(amp), 2 ** -0.5, rtol=2e-3)
    with run(gpu, "qft", 14, 12) as sim:  # QFT|0>: uniform magnitudes, ties everywhere
        idx, _ = sim.top_k(100)
        psi = sim.extract_state()
        key = psi.real * psi.real + psi.imag * psi.imag
        nz = np.flatnonzero(key)
        assert np.array_equal(idx.astype(np.int64), nz[np.lexsort((nz, -key[nz]))][:100])
