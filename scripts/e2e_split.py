"""Split the e2e step (create -> run -> get_payloads -> destroy) of bench.py's
headline workload into its parts (host wall clock, after one warm-up)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14088_b200 import _lib, cbq  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 34
lib = _lib.lib
circ = cbq.generate_benchmark("qft", n)
cfg = cbq.Config(block_bits=20, inner_size=2, error_bound=1e-3, identity_skip=True)
gates = circ.c_array()
ccfg = cfg.to_c()
nblk = 1 << (n - 20)
sizes = np.zeros(nblk, dtype=np.uint64)
out = None
for step in range(4):
    t = [time.perf_counter()]
    h = C.c_void_p()
    cbq._check(lib.bmq_simulator_create(n, C.byref(gates), len(gates), C.byref(ccfg), C.byref(h)))
    t.append(time.perf_counter())
    rep = _lib.bmq_report()
    cbq._check(lib.bmq_simulator_run(h, C.byref(rep), None, 0))
    t.append(time.perf_counter())
    total = C.c_uint64()
    cbq._check(lib.bmq_simulator_get_payloads(h, None, 0, sizes.ctypes.data, C.byref(total)))
    if out is None:
        out = torch.empty(total.value, dtype=torch.uint8, pin_memory=True)
    t.append(time.perf_counter())
    cbq._check(lib.bmq_simulator_get_payloads(h, C.c_void_p(out.data_ptr()), total.value, sizes.ctypes.data,
                                              C.byref(total)))
    t.append(time.perf_counter())
    lib.bmq_simulator_destroy(h)
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"step {step}: create {d[0]:.1f} run {d[1]:.1f} sizes {d[2]:.1f} payloads {d[3]:.1f} destroy {d[4]:.1f} "
          f"total {sum(d):.1f} ms (device sim {rep.device_ms if hasattr(rep, 'device_ms') else float('nan'):.1f})",
          flush=True)
