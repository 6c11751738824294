"""Pin the CPU oracle (oracle/cbq_oracle.c) before trusting it.

* SPEC known answers and the reference's own test
  expectations (proj/tests/*.cc) checked on the C restatement;
* golden fixtures generated from the unmodified reference
  (tests/golden/make_golden.py) replayed on the restatement;
* differential port-vs-reference runs when oracle/_ref is present.
"""
import ctypes as C
import json
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fnv(port, payloads):
    f = port.lib.cbqo_fnv1a64
    f.restype, f.argtypes = C.c_uint64, [C.c_char_p, C.c_uint64, C.c_uint64]
    h = 0xCBF29CE484222325
    for p in payloads:
        if p:
            h = f(p, len(p), h)
    return h


# ------------------------------------------------------------- known answers

def test_error_bound_known_answers(port):
    assert port.log2_abs(1.0) == 1.0
    assert port.log2_abs(3.0) == 2.0
    assert port.log2_abs(1e-3) == 0.0014419741739063218
    assert port.log2_abs(1e-4) == 0.00014426229109453829
    for bad in (0.0, -1.0, math.inf, math.nan):
        with pytest.raises(Exception, match="positive and finite"):
            port.log2_abs(bad)


def test_all_zero_block_is_header_only(port):
    p = port.compress_block(np.zeros(1 << 15), 1e-3)
    assert len(p) == 26 and p[25] == 1
    assert np.array_equal(port.decompress_block(p), np.zeros(1 << 15))


def test_one_is_exact_and_4_at_3(port):
    assert port.decompress_block(port.compress_block(np.array([1.0]), 1e-3))[0] == 1.0
    p = port.compress_block(np.array([4.0]), 3.0)
    assert len(p) == 31
    assert int.from_bytes(p[16:24], "little", signed=True) == 1 and p[24] == 1
    assert port.decompress_block(p)[0] == 4.0


def test_prescan_2pow20_zero_bits(port):
    enc = port.prescan_encode(np.zeros((1 << 20) // 64, dtype=np.uint64), 1 << 20)
    assert len(enc) == 64 and enc == bytes(64)


@pytest.mark.parametrize("b_r", [1e-2, 1e-3, 1e-4])
def test_pointwise_bound_million_scalars(port, b_r):
    rng = np.random.default_rng(5)
    n = 10**6
    x = np.sign(rng.standard_normal(n)) * 10.0 ** rng.uniform(-30, 0, n)
    x[rng.random(n) < 0.05] = 0.0
    y = port.decompress_block(port.compress_block(x, b_r))
    nz = x != 0
    rel = np.abs(y[nz] - x[nz]) / np.abs(x[nz])
    assert rel.max() <= math.sqrt(1 + b_r) - 1 + 1e-15
    assert np.array_equal(np.signbit(y[nz]), np.signbit(x[nz]))
    assert np.all(y[~nz] == 0.0)


def test_reference_test_expectations(port):
    # circuit_test.cc:184-197 (QFT-3 gate count), :248-258 (QAOA count)
    assert len(port.generate_benchmark("qft", 3)) == 9
    assert len(port.generate_benchmark("qaoa", 5, layers=2)) == 2 * (3 * 5 + 5)
    assert port.generate_benchmark("qaoa", 5, layers=2, seed=3) == port.generate_benchmark("qaoa", 5, layers=2, seed=3)
    # partition_test.cc:138-145 (group ids)
    assert port.enumerate_groups(6, 2, (0, 0, [3, 5])).tolist() == [[0, 2, 8, 10], [1, 3, 9, 11], [4, 6, 12, 14],
                                                                    [5, 7, 13, 15]]
    # partition_test.cc:175-182 (buffer bits)
    st = (0, 0, [3, 5])
    assert [port.buffer_bit_of_qubit(6, 2, st, q) for q in (0, 1, 3, 5)] == [0, 1, 2, 3]
    with pytest.raises(Exception, match="outer index"):
        port.buffer_bit_of_qubit(6, 2, st, 4)
    # partition_test.cc:60-71 expects 3 stages; Alg. 1 and the implementation give 2
    g = [("h", 2, 0), ("h", 3, 0), ("h", 4, 0), ("h", 5, 0)]
    assert port.partition(6, g, 2, 2) == [(0, 2, [2, 3]), (2, 4, [4, 5])]


def test_qft_equals_dft(port):
    # circuit_test.cc:199-218 — QFT == DFT matrix to 1e-12 (columns via apply_stage)
    n = 3
    g = port.generate_benchmark("qft", n)
    N = 1 << n
    cols = []
    for k in range(N):
        e = np.zeros(N, complex)
        e[k] = 1
        cols.append(port.apply_stage(e, n, g, (0, len(g), []), n))
    U = np.array(cols).T
    dft = np.exp(2j * np.pi * np.outer(range(N), range(N)) / N) / np.sqrt(N)
    assert np.abs(U - dft).max() <= 1e-12


def test_staged_equals_dense(port):
    # partition_test.cc:187-225 — staged uncompressed run == dense reference
    rng = np.random.default_rng(3)
    for t in range(20):
        n = 3 + t % 6
        gates = []
        for _ in range(30):
            k = int(rng.integers(15))
            q0 = int(rng.integers(n))
            q1 = int((q0 + 1 + rng.integers(n - 1)) % n)
            gates.append((k, q0, q1, float(rng.uniform(0, 6.28))))
        b = 1 + int(rng.integers(n))
        res = port.simulate(n, gates, b, int(rng.integers(4)), 1e-3, compress=False, want_payloads=False,
                            want_state=True)
        dense = port.dense_reference(n, gates)
        assert np.abs(res.state - dense).max() <= 1e-12


# ------------------------------------------------------------------ golden

def test_codec_golden(port):
    z = np.load(os.path.join(GOLDEN, "codec_golden.npz"))
    for i, name in enumerate(z["names"]):
        x, want, br = z[f"in_{i}"], z[f"out_{i}"].tobytes(), float(z["bounds"][i])
        assert port.compress_block(x, br) == want, name


def test_gate_golden(port):
    z = np.load(os.path.join(GOLDEN, "gate_golden.npz"))
    for i, g in enumerate(z["gates"]):
        kind, q0, q1, ang = int(g[0]), int(g[1]), int(g[2]), float(g[3])
        u = port.unitary((kind, q0, q1, ang))
        got = port.apply_gate(z[f"in_{i}"], u, q0, q1) if kind >= 12 else port.apply_gate(z[f"in_{i}"], u, q0)
        assert np.array_equal(got.view(np.uint64), z[f"out_{i}"].view(np.uint64)), i


def _sim_cases():
    with open(os.path.join(GOLDEN, "sim_golden.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _sim_cases()["simulations"], ids=lambda c: f"{c['name']}{c['n']}-b{c['b']}-i{c['inner']}-{c['error_bound']}")
def test_simulator_golden(port, case):
    gl = port.generate_benchmark(case["name"], case["n"], layers=case["layers"], seed=1)
    res = port.simulate(case["n"], gl, case["b"], case["inner"], case["error_bound"])
    want = case["report"]
    for k in ("qubits", "gate_count", "stage_count", "max_footprint_bytes", "spilled_blocks",
              "stage_compress_calls", "stage_decompress_calls"):
        assert res.report[k] == want[k], k
    assert res.report["compression_ratio"] == want["compression_ratio"]
    assert res.report["final_norm"] == want["final_norm"]
    assert f"{fnv(port, res.payloads):016x}" == case["payload_fnv"]


def test_plans_golden(port):
    d = _sim_cases()
    for p in d["plans"]:
        gl = port.generate_benchmark(p["name"], p["n"])
        assert len(gl) == p["gates"]
        assert len(port.partition(p["n"], gl, p["b"], p["inner"])) == p["stages"], p
    gr = d["groups"]
    assert port.enumerate_groups(gr["n"], gr["b"], tuple(gr["stage"])).tolist() == gr["ids"]


def test_spill_equivalence(port):
    # a small budget spills but the state is bit-identical
    gl = port.generate_benchmark("qft", 16)
    a = port.simulate(16, gl, 8, 2, 1e-3)
    b = port.simulate(16, gl, 8, 2, 1e-3, memory_budget=20000)
    assert b.report["spilled_blocks"] > 0
    assert a.payloads == b.payloads


# ----------------------------------------------------- differential vs _ref

def test_port_matches_reference_codec(port, ref):
    rng = np.random.default_rng(11)
    for n in (1, 7, 64, 4095, 4096, 4097, 12288, 1 << 15):
        x = rng.standard_normal(n) * 10.0 ** rng.uniform(-300, 10, n)
        x[rng.random(n) < 0.3] = 0.0
        for br in (1e-1, 1e-3, 1e-4, 7.0):
            p = ref.compress_block(x, br)
            assert port.compress_block(x, br) == p
            assert np.array_equal(port.decompress_block(p).view(np.uint64), ref.decompress_block(p).view(np.uint64))


def test_port_matches_reference_errors(port, ref):
    good = ref.compress_block(np.linspace(-1, 1, 9000), 1e-3)
    cases = [good[:10], good[:27], good[:-1], good + b"\0", good[:26] + b"\xff" + good[27:]]
    for bad in cases:
        with pytest.raises(Exception) as e1:
            ref.decompress_block(bad)
        with pytest.raises(Exception) as e2:
            port.decompress_block(bad)
        assert str(e1.value) == str(e2.value)


def test_port_matches_reference_simulation(port, ref):
    rng = np.random.default_rng(7)
    for t in range(12):
        n = 4 + t % 7
        gates = []
        for _ in range(25):
            k = int(rng.integers(15))
            q0 = int(rng.integers(n))
            q1 = int((q0 + 1 + rng.integers(n - 1)) % n)
            gates.append((k, q0, q1, float(rng.uniform(0, 6.28))))
        b = 1 + int(rng.integers(n))
        inner = int(rng.integers(4))
        br = [1e-2, 1e-3, 1e-4][t % 3]
        a = port.simulate(n, gates, b, inner, br)
        r = ref.simulate(n, gates, b, inner, br, workers=1)
        assert a.payloads == r.payloads
        for k in ("max_footprint_bytes", "final_norm", "stage_count"):
            assert a.report[k] == r.report[k]
