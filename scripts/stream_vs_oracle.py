"""Bisect the streaming pass: small circuits of one gate family each, run
through the simulator and compared with the C oracle (payload bytes)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle
from paper_2410_14088_b200 import cbq

port = oracle.port()
G = cbq.GateKind
n, b = 14, 12
rng = np.random.default_rng(1)
def run(name, gl, inner=2, br=1e-3):
    c = cbq.Circuit(n, [cbq.Gate(G(k), a, q, x) for k, a, q, x in gl])
    want = port.simulate(n, [g.as_tuple() for g in c.gates], b, inner, br)
    with cbq.Simulator(c, cbq.Config(block_bits=b, inner_size=inner, error_bound=br)) as sim:
        sim.run()
        got = sim.payloads()
    ok = got == want.payloads
    print(f"{name:40s} {'ok' if ok else 'DIFF'}", flush=True)
    return ok
H = [(0, q, 0, 0.0) for q in range(n)]
run("H all", H)
for q in (0, 3, 5, 6, 9, 12, 13):
    run(f"H all + RX q{q}", H + [(8, q, 0, 0.3)])
    run(f"H all + RZ q{q}", H + [(10, q, 0, 0.3)])
    run(f"H all + CX 1->{q}", H + [(12, 1 if q != 1 else 2, q, 0.0)])
    run(f"H all + CX {q}->4", H + [(12, q, 4 if q != 4 else 3, 0.0)])
    run(f"H all + CP {q},7", H + [(14, q, 7 if q != 7 else 8, 0.7)])
    run(f"H all + RY q{q} + CZ", H + [(9, q, 0, 0.4), (13, q, (q + 3) % n, 0.0)])
for s in range(4):
    gl = list(H)
    for _ in range(12):
        k = int(rng.choice([8, 9, 10, 12, 13, 14, 0]))
        a, q = rng.choice(n, 2, replace=False)
        gl.append((k, int(a), int(q), float(rng.uniform(0, 6))))
    run(f"random mix {s}", gl)
