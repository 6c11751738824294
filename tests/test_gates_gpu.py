"""Device gate engine parity: bmq_apply_gate / bmq_apply_stage /
bmq_dense_reference must be bit-identical to apply_unitary2/4, apply_stage
and dense_reference (kernel.hpp:24-122, engine.hpp:254-296)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.complex128).view(np.uint64)


def test_gate_golden(gpu):
    z = np.load(os.path.join(GOLDEN, "gate_golden.npz"))
    for i, g in enumerate(z["gates"]):
        gate = gpu.Gate(gpu.GateKind(int(g[0])), int(g[1]), int(g[2]), float(g[3]))
        a = z[f"in_{i}"].copy()
        if gpu.is_two_qubit(gate.kind):
            out = gpu.apply_unitary4(a, gate.q0, gate.q1, gpu.unitary4(gate))
        else:
            out = gpu.apply_unitary2(a, gate.q0, gpu.unitary2(gate))
        assert np.array_equal(bits(out), bits(z[f"out_{i}"])), i


@pytest.mark.parametrize("nbits", [1, 2, 5, 8, 12, 13, 17, 20])
def test_random_gates_match_oracle(gpu, port, nbits):
    rng = np.random.default_rng(nbits)
    for _ in range(12):
        a = rng.standard_normal(1 << nbits) + 1j * rng.standard_normal(1 << nbits)
        kind = gpu.GateKind(int(rng.integers(15)))
        if gpu.is_two_qubit(kind) and nbits < 2:
            continue
        q0 = int(rng.integers(nbits))
        q1 = int((q0 + 1 + rng.integers(max(1, nbits - 1))) % nbits) if nbits > 1 else 0
        g = gpu.Gate(kind, q0, q1, float(rng.uniform(-7, 7)))
        if gpu.is_two_qubit(kind):
            got = gpu.apply_unitary4(a.copy(), q0, q1, gpu.unitary4(g))
            want = port.apply_gate(a, port.unitary(g.as_tuple()), q0, q1)
        else:
            got = gpu.apply_unitary2(a.copy(), q0, gpu.unitary2(g))
            want = port.apply_gate(a, port.unitary(g.as_tuple()), q0)
        assert np.array_equal(bits(got), bits(want)), (kind, q0, q1)


def test_general_matrices(gpu, port):
    rng = np.random.default_rng(2)
    a = rng.standard_normal(1 << 10) + 1j * rng.standard_normal(1 << 10)
    u4 = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
    u4[1, 2] = 0
    u4[3, 0] = 1
    u4[0, 1] = -1j
    assert np.array_equal(bits(gpu.apply_unitary4(a.copy(), 7, 2, u4)), bits(port.apply_gate(a, u4, 7, 2)))
    u2 = np.array([[0.3, 1j], [-1, 0.5 - 0.25j]])
    assert np.array_equal(bits(gpu.apply_unitary2(a.copy(), 9, u2)), bits(port.apply_gate(a, u2, 9)))


def test_gate_bit_errors(gpu):
    with pytest.raises(gpu.InvalidArgument, match="gate bit out of range for buffer"):
        gpu.apply_unitary2(np.zeros(2, complex), 1, np.eye(2))
    with pytest.raises(gpu.InvalidArgument, match="gate bits invalid for buffer"):
        gpu.apply_unitary4(np.zeros(4, complex), 1, 1, np.eye(4))


def random_gates(rng, n, count):
    out = []
    for _ in range(count):
        k = int(rng.integers(15))
        q0 = int(rng.integers(n))
        q1 = int((q0 + 1 + rng.integers(n - 1)) % n)
        out.append((k, q0, q1 if k >= 12 else 0, float(rng.uniform(0, 6.28))))
    return out


def test_apply_stage_matches_oracle(gpu, port):
    rng = np.random.default_rng(4)
    for t in range(25):
        n = 4 + t % 12
        gl = random_gates(rng, n, 40)
        b = 2 + int(rng.integers(n - 1))
        c = gpu.Circuit(n, [gpu.Gate(gpu.GateKind(k), a, bb, ang) for k, a, bb, ang in gl])
        plan = gpu.partition_circuit(c, b, 1 + int(rng.integers(4)))
        L = gpu.make_layout(n, b)
        for st in plan.stages:
            buf_len = 1 << (b + len(st.inner))
            amps = rng.standard_normal(buf_len) + 1j * rng.standard_normal(buf_len)
            gb = gpu.GroupBuffer(gpu.SVGroup(0, []), amps.copy())
            gpu.apply_stage(gb, st, c, L)
            want = port.apply_stage(amps, n, gl, (st.gate_begin, st.gate_end, st.inner), b)
            assert np.array_equal(bits(gb.amps), bits(want))


def test_dense_reference_matches_oracle(gpu, port):
    rng = np.random.default_rng(8)
    for n in (1, 3, 7, 12, 16):
        gl = random_gates(rng, n, 60) if n > 1 else [(0, 0, 0, 0.0), (10, 0, 0, 0.3)]
        c = gpu.Circuit(n, [gpu.Gate(gpu.GateKind(k), a, bb, ang) for k, a, bb, ang in gl])
        # exact values; an exact zero may carry either sign (the codec maps both to the same bytes)
        assert np.array_equal(gpu.dense_reference(c), port.dense_reference(n, gl))
    for name in ("qft", "qaoa", "bv", "ghz"):
        c = gpu.generate_benchmark(name, 14, gpu.BenchmarkParams(layers=2))
        want = port.dense_reference(14, [g.as_tuple() for g in c.gates])
        assert np.array_equal(gpu.dense_reference(c), want)


def test_qft_is_dft(gpu):
    n = 5
    c = gpu.generate_benchmark("qft", n)
    N = 1 << n
    cols = []
    for k in range(N):
        gb = gpu.GroupBuffer(gpu.SVGroup(0, [0]), np.eye(N, dtype=complex)[k])
        gpu.apply_stage(gb, gpu.Stage(0, len(c.gates), []), c, gpu.make_layout(n, n))
        cols.append(gb.amps)
    dft = np.exp(2j * np.pi * np.outer(range(N), range(N)) / N) / np.sqrt(N)
    assert np.abs(np.array(cols).T - dft).max() <= 1e-12
