"""Find the first stage whose payloads differ between two engine settings (debug aid)."""
import os, subprocess, sys, json
sys.path.insert(0, '.')
from paper_2410_14088_b200 import cbq
n, b, inner = 20, 14, 2
c = cbq.generate_benchmark("qft", n)
plan = cbq.partition_circuit(c, b, inner)
if len(sys.argv) > 1:
    sim = cbq.Simulator(c, cbq.Config(block_bits=b, inner_size=inner))
    out = []
    for s in range(len(plan.stages)):
        sim.run_stages(s, s + 1)
        out.append(hash(tuple(sim.payloads())))
    print(json.dumps(out))
    sys.exit(0)
a = json.loads(subprocess.run([sys.executable, __file__, "x"], capture_output=True, text=True).stdout)
env = dict(os.environ, BMQ_DBG_FULL_SUPPORT="1")
bb = json.loads(subprocess.run([sys.executable, __file__, "x"], capture_output=True, text=True, env=env).stdout)
for s, (x, y) in enumerate(zip(a, bb)):
    if x != y:
        st = plan.stages[s]
        print("first differing stage", s, st.inner, [(cbq.gate_name(c.gates[g].kind), c.gates[g].q0, c.gates[g].q1) for g in range(st.gate_begin, st.gate_end)])
        break
else:
    print("no difference")
