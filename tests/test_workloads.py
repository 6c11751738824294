"""BASELINE.json workloads built from the reference gate set (SURVEY.md
section 8d): QAOA MaxCut on a random 3-regular graph (C4) and the
sqrt-X/Y/W + CZ grid random circuit (C5). Host checks of their structure and
determinism, a QASM round trip through the reference parser, and (GPU) the
device simulation byte-exact against the oracle at small sizes."""
import collections
import math

import numpy as np
import pytest


def edges_of(gates):
    """(i, j) of every CX-RZ-CX triple of the first QAOA layer."""
    out = []
    for k in range(0, len(gates) - 2):
        a, b, c = gates[k], gates[k + 1], gates[k + 2]
        if a.kind == c.kind == 12 and b.kind == 10 and (a.q0, a.q1) == (c.q0, c.q1) and b.q0 == a.q1:
            out.append((a.q0, a.q1))
    return out


@pytest.mark.parametrize("n", [4, 16, 34])
def test_qaoa3reg_structure(cbq, n):
    layers = 4
    c = cbq.generate_benchmark("qaoa3reg", n, cbq.BenchmarkParams(layers=layers, seed=1))
    ne = 3 * n // 2
    assert len(c.gates) == layers * (3 * ne + n)  # 748 for n = 34
    per_layer = 3 * ne + n
    first = c.gates[:per_layer]
    e = edges_of(first)[:ne]
    assert len(set(e)) == ne and all(i < j for i, j in e)
    deg = collections.Counter(q for ij in e for q in ij)
    assert all(deg[q] == 3 for q in range(n))
    # angles per layer drawn like make_qaoa (benchmarks.hpp:123-126): the ring
    # QAOA with the same seed has the same gamma / beta sequence
    ring = cbq.generate_benchmark("qaoa", n, cbq.BenchmarkParams(layers=layers, seed=1))
    ring_g = [g.angle for g in ring.gates if g.kind == 10][::n]
    ring_b = [g.angle for g in ring.gates if g.kind == 8][::n]
    mine_g = [g.angle for g in c.gates if g.kind == 10][::ne]
    mine_b = [g.angle for g in c.gates if g.kind == 8][::n]
    assert mine_g == ring_g and mine_b == ring_b
    again = cbq.generate_benchmark("qaoa3reg", n, cbq.BenchmarkParams(layers=layers, seed=1))
    assert again == c
    other = cbq.generate_benchmark("qaoa3reg", n, cbq.BenchmarkParams(layers=layers, seed=2))
    assert other != c


def test_qaoa3reg_errors(cbq):
    with pytest.raises(cbq.InvalidArgument, match="even node count"):
        cbq.generate_benchmark("qaoa3reg", 7)
    with pytest.raises(cbq.InvalidArgument, match="at least one layer"):
        cbq.generate_benchmark("qaoa3reg", 8, cbq.BenchmarkParams(layers=0))


@pytest.mark.parametrize("n,rows,cols", [(16, 4, 4), (36, 6, 6), (12, 3, 4)])
def test_random_circuit_structure(cbq, n, rows, cols):
    cycles = 9
    c = cbq.generate_benchmark("random", n, cbq.BenchmarkParams(layers=cycles, seed=1))
    kinds = collections.Counter(g.kind for g in c.gates)
    assert set(kinds) <= {8, 9, 10, 13}  # RX, RY, RZ, CZ only
    # walk the cycles: n single-qubit "slots" (1 or 3 gates) then a CZ layer
    pos, prev = 0, [None] * n
    for cy in range(cycles):
        for q in range(n):
            g = c.gates[pos]
            assert g.q0 == q
            if g.kind == 10:  # sqrt(W) = RZ(-pi/4) RX(pi/2) RZ(pi/4)
                assert g.angle == -math.pi / 4 and c.gates[pos + 1].kind == 8 and c.gates[pos + 2].angle == math.pi / 4
                kind, pos = "w", pos + 3
            else:
                assert g.angle == math.pi / 2
                kind, pos = ("x" if g.kind == 8 else "y"), pos + 1
            assert kind != prev[q]
            prev[q] = kind
        pat = cy % 4
        while pos < len(c.gates) and c.gates[pos].kind == 13:
            a, b = c.gates[pos].q0, c.gates[pos].q1
            ra, ca = divmod(a, cols)
            if pat < 2:
                assert b == a + 1 and ca % 2 == pat
            else:
                assert b == a + cols and ra % 2 == pat - 2
            pos += 1
    assert pos == len(c.gates)


def test_workloads_round_trip_through_reference_qasm(cbq, ref):
    """The workloads are plain reference circuits: their QASM text parses in
    the unmodified reference parser (qasm.hpp) to the same gate list."""
    from oracle import oracle
    for name, n, layers in (("qaoa3reg", 10, 2), ("random", 12, 5)):
        c = cbq.generate_benchmark(name, n, cbq.BenchmarkParams(layers=layers))
        text = cbq.emit_qasm(c)
        nq, gl, _ = oracle.ref_parse_qasm(text)
        assert nq == n
        assert [tuple(g) for g in gl] == [g.as_tuple() for g in c.gates]
        assert cbq.parse_qasm(text) == c


@pytest.mark.gpu
@pytest.mark.parametrize("name,n,b,inner,layers,br", [("qaoa3reg", 16, 12, 2, 2, 1e-4), ("qaoa3reg", 14, 10, 3, 4, 1e-3),
                                                      ("random", 16, 12, 2, 6, 1e-3), ("random", 15, 11, 4, 8, 1e-3)])
def test_workloads_match_oracle(gpu, port, name, n, b, inner, layers, br):
    c = gpu.generate_benchmark(name, n, gpu.BenchmarkParams(layers=layers))
    gl = [g.as_tuple() for g in c.gates]
    want = port.simulate(n, gl, b, inner, br)
    with gpu.Simulator(c, gpu.Config(block_bits=b, inner_size=inner, error_bound=br, identity_skip=True)) as sim:
        rep = sim.run()
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=1e-10)
        f = sim.fidelity_dense(gpu.dense_reference(c))
        assert f >= 0.99
