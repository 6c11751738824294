"""Regenerate tests/golden/* from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists and
`make -C oracle` built oracle/_ref/libcbqref.so):

    python tests/golden/make_golden.py

Outputs (committed):
  codec_golden.npz   input scalars, relative bounds and the reference payload
                     bytes of compress_block (codec.hpp:227-295)
  gate_golden.npz    random states, gates and apply_unitary2/4 results
                     (kernel.hpp:24-64)
  sim_golden.json    Simulator::run reports (workers = 1) + FNV-1a-64 of the
                     final payloads in id order, plans, group ids
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

SIM_CASES = [
    # name, n, b, inner, b_r, layers
    ("qft", 20, 14, 2, 1e-3, 1),
    ("qft", 20, 10, 5, 1e-3, 1),
    ("ghz", 20, 14, 2, 1e-3, 1),
    ("bv", 20, 14, 2, 1e-3, 1),
    ("qaoa", 20, 14, 2, 1e-3, 2),
    ("qaoa", 20, 14, 2, 1e-4, 4),
    ("qaoa", 18, 10, 3, 1e-3, 4),
    ("qft", 12, 3, 2, 1e-3, 1),
    ("qft", 9, 9, 2, 1e-2, 1),
    ("ghz", 16, 1, 2, 1e-3, 1),
    ("qaoa", 10, 2, 0, 3.0, 1),
]

PLAN_CASES = [("qft", 34, b, i) for b, i in [(14, 2), (14, 6), (17, 4), (20, 2), (20, 4), (20, 6), (24, 6)]]


def fnv_payloads(payloads):
    h = 0xCBF29CE484222325
    port = O.port()
    for p in payloads:
        h = port.lib.cbqo_fnv1a64(p, len(p), h) if p else h
    return h


def main():
    r = O.ref()
    port = O.port()
    port.lib.cbqo_fnv1a64.restype = __import__("ctypes").c_uint64
    port.lib.cbqo_fnv1a64.argtypes = [__import__("ctypes").c_char_p, __import__("ctypes").c_uint64,
                                      __import__("ctypes").c_uint64]
    rng = np.random.default_rng(20241014)
    # ---------------------------------------------------------------- codec
    inputs, bounds, payloads, names = [], [], [], []

    def add(name, x, br):
        x = np.ascontiguousarray(x, dtype=np.float64)
        inputs.append(x)
        bounds.append(br)
        payloads.append(np.frombuffer(r.compress_block(x, br), dtype=np.uint8))
        names.append(name)

    n = 1 << 15
    logu = np.sign(rng.standard_normal(n)) * 10.0 ** rng.uniform(-30, 0, n)
    logu[rng.random(n) < 0.1] = 0.0
    logu[rng.random(n) < 0.01] = -0.0
    for br in (1e-2, 1e-3, 1e-4):
        add(f"loguniform_1e{int(np.log10(br))}", logu, br)
    add("all_zero_b14", np.zeros(n), 1e-3)
    add("one_scalar_4_at_3", np.array([4.0]), 3.0)
    for b in (10, 14):
        e0 = np.zeros(2 << b)
        e0[0] = 1.0
        add(f"e0_b{b}", e0, 1e-3)
    add("uniform_real_b14", np.concatenate([np.full(1 << 14, 2.0 ** -10), np.zeros(1 << 14)]), 1e-3)
    g = rng.standard_normal(n) / 128.0
    add("gaussian_b14", g, 1e-3)
    add("gaussian_partial_5000", g[:5000], 1e-3)
    mixed = g.copy()
    mixed[: 3 * 4096] = 0.0
    mixed[4096 * 4: 4096 * 5] = -np.abs(mixed[4096 * 4: 4096 * 5])
    add("chunk_tags_all0_all1", mixed, 1e-3)
    add("subnormals", np.array([5e-324, -1e-310, 2.5e-308, 1.0, -3e-320, 0.0]), 1e-3)
    add("large_values", np.array([1e300, -1e-300, 1e10, 7.0]), 1e-2)
    np.savez_compressed(os.path.join(HERE, "codec_golden.npz"), names=np.array(names),
                        bounds=np.array(bounds),
                        **{f"in_{i}": x for i, x in enumerate(inputs)},
                        **{f"out_{i}": p for i, p in enumerate(payloads)})
    # ---------------------------------------------------------------- gates
    states, gspec, outs = [], [], []
    for t in range(40):
        nb = 2 + t % 7
        a = rng.uniform(-1, 1, 1 << nb) + 1j * rng.uniform(-1, 1, 1 << nb)
        kind = int(rng.integers(15))
        q0 = int(rng.integers(nb))
        q1 = int((q0 + 1 + rng.integers(nb - 1)) % nb)
        ang = float(rng.uniform(0, 2 * np.pi))
        gt = (kind, q0, q1 if kind >= 12 else 0, ang)
        u = r.unitary(gt)
        o = r.apply_gate(a, u, q0, q1) if kind >= 12 else r.apply_gate(a, u, q0)
        states.append(a)
        gspec.append(gt)
        outs.append(o)
    np.savez_compressed(os.path.join(HERE, "gate_golden.npz"), gates=np.array(gspec, dtype=np.float64),
                        **{f"in_{i}": x for i, x in enumerate(states)},
                        **{f"out_{i}": x for i, x in enumerate(outs)})
    # ------------------------------------------------------------ simulator
    sims = []
    for name, nq, b, inner, br, layers in SIM_CASES:
        gl = r.generate_benchmark(name, nq, layers=layers, seed=1)
        res = r.simulate(nq, gl, b, inner, br, workers=1, want_payloads=True, with_fidelity=nq <= 20)
        rep = {k: v for k, v in res.report.items() if k not in ("wall_ms", "stage_ms", "pad")}
        sims.append({"name": name, "n": nq, "b": b, "inner": inner, "error_bound": br, "layers": layers,
                     "report": rep, "payload_fnv": f"{fnv_payloads(res.payloads):016x}",
                     "payload_sizes_head": [len(p) for p in res.payloads[:16]]})
        print(name, nq, b, inner, br, rep["max_footprint_bytes"], rep.get("fidelity"))
    plans = []
    for name, nq, b, inner in PLAN_CASES:
        gl = r.generate_benchmark(name, nq)
        plans.append({"name": name, "n": nq, "b": b, "inner": inner, "gates": len(gl),
                      "stages": len(r.partition(nq, gl, b, inner))})
    groups = {"n": 6, "b": 2, "stage": [0, 0, [3, 5]],
              "ids": r.enumerate_groups(6, 2, (0, 0, [3, 5])).tolist()}
    with open(os.path.join(HERE, "sim_golden.json"), "w") as f:
        json.dump({"simulations": sims, "plans": plans, "groups": groups}, f, indent=1)


if __name__ == "__main__":
    main()
