"""Per-stage wall time of one simulation (development aid): which stages dominate."""
import sys, collections
sys.path.insert(0, '.')
from paper_2410_14088_b200 import cbq
name = sys.argv[1] if len(sys.argv) > 1 else "qft"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 34
b = int(sys.argv[3]) if len(sys.argv) > 3 else 20
inner = int(sys.argv[4]) if len(sys.argv) > 4 else 2
br = float(sys.argv[5]) if len(sys.argv) > 5 else 1e-3
c = cbq.generate_benchmark(name, n, cbq.BenchmarkParams(layers=4))
cfg = cbq.Config(block_bits=b, inner_size=inner, error_bound=br, identity_skip=True)
sim = cbq.Simulator(c, cfg)
rep = sim.run(); sim.reset(); rep = sim.run()
plan = sim.plan()
print("total device ms", rep.device["device_ms"], rep.device)
rows = []
for i, (st, ms) in enumerate(zip(plan.stages, rep.stage_ms)):
    kinds = collections.Counter(cbq.gate_name(c.gates[g].kind) for g in range(st.gate_begin, st.gate_end))
    rows.append((ms, i, st.inner, dict(kinds)))
for ms, i, inn, k in sorted(rows, reverse=True)[:40]:
    print(f"stage {i:3d} {ms:9.2f} ms inner={inn} {k}")
print("sum stage ms", sum(r[0] for r in rows))
