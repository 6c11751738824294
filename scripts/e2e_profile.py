"""Time the parts of one end-to-end simulation through the C ABI (development aid)."""
import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2410_14088_b200 import cbq, _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 34
circ = cbq.generate_benchmark("qft", n)
cfg = cbq.Config(block_bits=20, inner_size=2, error_bound=1e-3, identity_skip=True)
pinned = None
for it in range(3):
    t0 = time.perf_counter(); s = cbq.Simulator(circ, cfg); t1 = time.perf_counter()
    rep = s.run(); t2 = time.perf_counter()
    nblk = s.layout().num_blocks()
    sizes = np.zeros(nblk, dtype=np.uint64); total = C.c_uint64()
    _lib.lib.bmq_simulator_get_payloads(s._h, None, 0, sizes.ctypes.data, C.byref(total))
    if pinned is None or pinned.numel() < total.value:
        pinned = torch.empty(total.value, dtype=torch.uint8, pin_memory=True)
    t3 = time.perf_counter()
    _lib.lib.bmq_simulator_get_payloads(s._h, C.c_void_p(pinned.data_ptr()), total.value, sizes.ctypes.data, C.byref(total))
    t4 = time.perf_counter()
    pays = s.payloads(); t5 = time.perf_counter()
    s.close(); t6 = time.perf_counter()
    print(f"create {t1-t0:.3f} run {t2-t1:.3f} (device {rep.device['device_ms']/1e3:.3f}, wall {rep.wall_ms/1e3:.3f}) "
          f"sizes {t3-t2:.3f} get_payloads(pinned) {t4-t3:.3f} payloads(list) {t5-t4:.3f} close {t6-t5:.3f} total_bytes {total.value}")
