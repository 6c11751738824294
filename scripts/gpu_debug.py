"""Quick GPU parity probe (development aid)."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, '.')
from paper_2410_14088_b200 import cbq
from oracle import oracle as O
r = O.ref()
ok = True
def check(name, cond):
    global ok
    print(("PASS " if cond else "FAIL ") + name, flush=True)
    ok &= bool(cond)
rng = np.random.default_rng(1)
# codec
for n in [0, 4, 100, 4096, 8192, 32768, 5000, 2**21]:
    x = rng.standard_normal(n) * 10.0**rng.uniform(-30, 0, n)
    x[rng.random(n) < 0.2] = 0
    if n > 10: x[10:4106] = 0  # an all-zero chunk-ish region
    for br in [1e-2, 1e-3, 1e-4, 3.0]:
        try:
            a = cbq.compress_block(x, br); b = r.compress_block(x, br)
            eq = a == b
            if not eq:
                i = next((k for k in range(min(len(a), len(b))) if a[k] != b[k]), None)
                print(f"  n={n} br={br} len {len(a)} vs {len(b)} first diff at {i}")
            check(f"compress n={n} br={br}", eq)
            da = cbq.decompress_block(b); db = r.decompress_block(b)
            check(f"decompress n={n} br={br}", np.array_equal(da.view(np.uint64), db.view(np.uint64)))
        except Exception as e:
            traceback.print_exc(); check(f"codec n={n} br={br}", False)
# gates
for trial in range(20):
    nb = 2 + trial % 12
    a = rng.standard_normal(1 << nb) + 1j * rng.standard_normal(1 << nb)
    for g in [cbq.gates.h(rng.integers(nb)), cbq.gates.rx(rng.integers(nb), 0.3), cbq.gates.rz(rng.integers(nb), 1.3)]:
        u = cbq.unitary2(g)
        x = cbq.apply_unitary2(a.copy(), g.q0, u)
        y = r.apply_gate(a, u, g.q0)
        check(f"gate1 nb={nb}", np.array_equal(x.view(np.uint64), y.view(np.uint64)))
    q0, q1 = rng.choice(nb, 2, replace=False)
    for g in [cbq.gates.cx(q0, q1), cbq.gates.cp(q0, q1, 0.77), cbq.gates.cz(q0,q1)]:
        u = cbq.unitary4(g)
        x = cbq.apply_unitary4(a.copy(), int(q0), int(q1), u)
        y = r.apply_gate(a, u, int(q0), int(q1))
        check(f"gate2 nb={nb}", np.array_equal(x.view(np.uint64), y.view(np.uint64)))
# simulator
for name, n, b, inner, br, layers in [("qft",10,4,2,1e-3,1),("qaoa",10,3,3,1e-4,2),("ghz",12,3,2,1e-3,1),("bv",11,3,2,1e-3,1),
                                      ("qft",20,14,2,1e-3,1), ("qaoa",16,12,2,1e-4,2), ("qft", 16, 11, 4, 1e-3, 1)]:
    c = cbq.generate_benchmark(name, n, cbq.BenchmarkParams(layers=layers))
    t = time.time()
    try:
        sim = cbq.Simulator(c, cbq.Config(block_bits=b, inner_size=inner, error_bound=br))
        rep = sim.run(); pays = sim.payloads(); t1 = time.time()
        R = r.simulate(n, [g.as_tuple() for g in c.gates], b, inner, br, workers=8, want_payloads=True)
        t2 = time.time()
        same = pays == R.payloads
        if not same:
            bad = [i for i in range(len(pays)) if pays[i] != R.payloads[i]]
            print("  payload mismatch ids", bad[:10], len(bad))
        check(f"sim {name}-{n} b={b} i={inner} payloads", same)
        check(f"sim {name}-{n} peak {rep.max_footprint_bytes} vs {R.report['max_footprint_bytes']}", rep.max_footprint_bytes == R.report['max_footprint_bytes'])
        check(f"sim {name}-{n} norm {rep.final_norm} vs {R.report['final_norm']}", abs(rep.final_norm - R.report['final_norm']) < 1e-12)
        print(f"  gpu {t1-t:.3f}s ref {t2-t1:.3f}s dev {rep.device}")
    except Exception:
        traceback.print_exc(); check(f"sim {name}", False)
print("ALL OK" if ok else "SOME FAILED")
