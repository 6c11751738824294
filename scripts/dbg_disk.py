import sys, time
sys.path.insert(0, '.')
from paper_2410_14088_b200 import cbq
from oracle import oracle
port = oracle.port()
c = cbq.generate_benchmark("qaoa", 16, cbq.BenchmarkParams(layers=2))
want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
big = max(len(p) for p in want.payloads)
cfg = cbq.Config(block_bits=12, inner_size=2, device_pool_bytes=6 * (big + 16), work_bytes=4 * (16 << 12),
                 host_pool_bytes=3 * (big + 16), disk_pool_bytes=64 << 20, arena=sys.argv[1])
t = time.time()
with cbq.Simulator(c, cfg) as sim:
    print("created", time.time() - t, flush=True)
    rep = sim.run()
    print("ran", time.time() - t, rep.device["disk_spill_bytes"], rep.device["disk_read_bytes"], rep.device["disk_gds"], flush=True)
    print("payloads equal", sim.payloads() == want.payloads, flush=True)
