import sys, subprocess, os
import numpy as np
sys.path.insert(0, '.')
from paper_2410_14088_b200 import cbq
G = cbq.GateKind
n, b = 14, 12
gl = [(0, q, 0, 0.0) for q in range(n)]
c = cbq.Circuit(n, [cbq.Gate(G(k), a, q, x) for k, a, q, x in gl])
with cbq.Simulator(c, cbq.Config(block_bits=b, inner_size=2, error_bound=1e-3)) as sim:
    rep = sim.run()
    st = sim.extract_state()
    pays = sim.payloads()
np.save(f"gpurun_out/st_{os.environ.get('BMQ_DBG_NO_STREAM','s')}.npy", st)
print("passes", rep.device.get('gate_passes'), "sizes", [len(p) for p in pays], "norm", rep.final_norm)
print("first", st[:4], "nonzero", np.count_nonzero(st), "max", np.abs(st).max(), "min", np.abs(st).min())
