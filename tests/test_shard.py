"""Sharded stage loop: device-qubit planning, the exchange
protocol and the accounting replay, on CPU (gloo, world_size 2, and threads)
with the oracle as each rank's backend; and on the GPU with device engines.
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch

from paper_2410_14088_b200 import cbq
from paper_2410_14088_b200.shard import (LocalCollective, LocalHub, ShardedSimulator, TorchCollective, owners,
                                         remap_lists, shard_plan)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _remaps(bits):
    return sum(1 for s in range(1, len(bits)) if not np.array_equal(bits[s - 1], bits[s]))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_plan_keeps_device_qubits_outer(world):
    c = cbq.generate_benchmark("qft", 34)
    plan = cbq.partition_circuit(c, 20, 2)
    bits = shard_plan(34, 20, plan.stages, world)
    assert bits.shape == (len(plan.stages), world.bit_length() - 1)
    for st, row in zip(plan.stages, bits):
        assert len(set(row.tolist())) == len(row)
        assert all(20 <= q < 34 and q not in st.inner for q in row.tolist())
    # a slot only changes when its qubit becomes inner in that stage
    for s in range(1, len(bits)):
        for j in range(bits.shape[1]):
            if bits[s, j] != bits[s - 1, j]:
                assert bits[s - 1, j] in plan.stages[s].inner
    assert bits.tolist() == shard_plan(34, 20, plan.stages, world).tolist()  # deterministic
    assert _remaps(bits) <= 16


def test_plan_refuses_too_few_outer_bits():
    c = cbq.generate_benchmark("qft", 12)
    plan = cbq.partition_circuit(c, 9, 2)  # c = 3, inner 2 -> 1 outer bit
    shard_plan(12, 9, plan.stages, 2)
    with pytest.raises(cbq.InvalidArgument, match="too few"):
        shard_plan(12, 9, plan.stages, 4)
    with pytest.raises(cbq.InvalidArgument, match="power of two"):
        shard_plan(12, 9, plan.stages, 3)


def test_remap_lists_partition_the_moving_ids():
    nid, b = 64, 4
    prev = owners(nid, [4, 5], b)
    nxt = owners(nid, [4, 7], b)
    moved = 0
    for r in range(4):
        sends, recvs = remap_lists(prev, nxt, r, 4)
        for p in range(4):
            assert all(prev[i] == r and nxt[i] == p for i in sends[p].tolist())
            assert all(prev[i] == p and nxt[i] == r for i in recvs[p].tolist())
            got = remap_lists(prev, nxt, p, 4)[1][r]
            assert sends[p].tolist() == got.tolist()
        moved += sum(len(x) for x in sends)
    assert moved == int((prev != nxt).sum()) == nid // 2


CASES = [("qft", 12, 6, 2, 1e-3, {}), ("qaoa", 12, 5, 2, 1e-3, {"layers": 2}), ("ghz", 12, 5, 2, 1e-3, {})]


def _oracle_run(port, rank, world, col, name, n, b, inner, br, kw):
    from shard_oracle import OracleShard
    gates = port.generate_benchmark(name, n, **kw)
    be = OracleShard(port, n, gates, b, inner, br, rank, world)
    sim = ShardedSimulator(be, col)
    rep = sim.run()
    return sim, rep, sim.gather_payloads(0)


def _gloo_worker(rank, world, port_no, case, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import torch.distributed as dist
    from oracle import oracle
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sim, rep, payloads = _oracle_run(oracle.port(), rank, world, TorchCollective("cpu"), *case)
        out_q.put((rank, rep.max_footprint_bytes, rep.final_norm, sim.remaps, sim.moved_bytes,
                   [bytes(p) for p in payloads] if payloads else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES[:2], ids=[c[0] for c in CASES[:2]])
def test_gloo_world2_matches_single_process(port, case):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pn = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, pn, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    name, n, b, inner, br, kw = case
    gates = port.generate_benchmark(name, n, **kw)
    want = port.simulate(n, gates, b, inner, br)
    assert res[0][5] == want.payloads
    for r in (0, 1):
        assert res[r][1] == want.report["max_footprint_bytes"]
        assert res[r][2] == pytest.approx(want.report["final_norm"], rel=1e-12)
    assert res[0][3] == res[1][3]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_threads_match_single_process(port, case, world):
    hub = LocalHub(world)
    out = [None] * world
    errs = []

    def work(r):
        try:
            out[r] = _oracle_run(port, r, world, LocalCollective(hub, r), *case)
        except BaseException as e:  # pragma: no cover - surfaced below
            errs.append(e)
            hub.bar.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    assert not errs, errs
    name, n, b, inner, br, kw = case
    gates = port.generate_benchmark(name, n, **kw)
    want = port.simulate(n, gates, b, inner, br)
    assert out[0][2] == want.payloads
    for r in range(world):
        assert out[r][1].max_footprint_bytes == want.report["max_footprint_bytes"]
        assert out[r][1].spilled_blocks == want.report["spilled_blocks"]


# ---------------------------------------------------------------- GPU


def _engine_threads(circuit, cfg, world):
    from paper_2410_14088_b200.shard import EngineShard
    hub = LocalHub(world)
    out = [None] * world
    errs = []

    def work(r):
        try:
            be = EngineShard(circuit, cfg, r, world)
            try:
                sim = ShardedSimulator(be, LocalCollective(hub, r, "cuda:0"))
                rep = sim.run()
                out[r] = (sim, rep, sim.gather_payloads(0), sim.fidelity_uniform())
            finally:
                be.close()
        except BaseException as e:  # pragma: no cover
            errs.append(e)
            hub.bar.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    assert not errs, errs
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name,n,b,kw", [("qft", 16, 8, {}), ("qaoa", 16, 8, {"layers": 2})])
def test_engine_shards_match_single_gpu(gpu, port, name, n, b, kw, world):
    c = gpu.generate_benchmark(name, n, gpu.BenchmarkParams(**kw))
    want = port.simulate(n, [g.as_tuple() for g in c.gates], b, 2, 1e-3)
    cfg = gpu.Config(block_bits=b, inner_size=2, work_bytes=8 * (16 << b))
    out = _engine_threads(c, cfg, world)
    sim, rep, payloads, _ = out[0]
    assert payloads == want.payloads
    assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
    assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=1e-10)
    assert sim.remaps > 0


@pytest.mark.gpu
def test_engine_shards_spill_to_host(gpu, port):
    c = gpu.generate_benchmark("qaoa", 16, gpu.BenchmarkParams(layers=2))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 10, 2, 1e-3)
    biggest = max(len(p) for p in want.payloads)
    cfg = gpu.Config(block_bits=10, inner_size=2, work_bytes=4 * (16 << 10), device_pool_bytes=6 * (biggest + 16),
                     host_pool_bytes=64 << 20)
    out = _engine_threads(c, cfg, 2)
    assert out[0][2] == want.payloads
    assert out[0][1].device["host_spill_bytes"] > 0


@pytest.mark.gpu
def test_nccl_world1_path(gpu, port):
    """The NCCL collective path of the driver (world 1: the device-tensor
    plumbing the multi-GPU bench uses)."""
    import torch.distributed as dist
    from paper_2410_14088_b200.shard import EngineShard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        c = gpu.generate_benchmark("qft", 14)
        want = port.simulate(14, [g.as_tuple() for g in c.gates], 7, 2, 1e-3)
        be = EngineShard(c, gpu.Config(block_bits=7, inner_size=2), 0, 1)
        try:
            sim = ShardedSimulator(be, TorchCollective())
            rep = sim.run()
            assert sim.gather_payloads(0) == want.payloads
            assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
            assert sim.fidelity_uniform() == pytest.approx(0.9989, abs=2e-3)
        finally:
            be.close()
    finally:
        dist.destroy_process_group()


def _merged(per_rank):
    """Each id's payload from the rank that holds it (the others read ALL_ZERO)."""
    out = []
    for ps in zip(*per_rank):
        held = [p for p in ps if len(p) > 26 or (len(p) == 26 and p[25] != 1)]
        out.append(held[0] if held else ps[0])
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name,n,layers,b,br", [("qft", 18, 1, 12, 1e-3), ("qaoa3reg", 18, 2, 12, 1e-4)])
def test_c_abi_sharded_run_matches_single(gpu, port, world, name, n, layers, b, br):
    """bmq_simulator_run_sharded (host C++ driver) with the
    in-process collective: `world` engines on one GPU driven by threads;
    payloads (each from its owner), peak footprint and norm equal the
    single-GPU run's, which equals the oracle's."""
    import threading
    c = gpu.generate_benchmark(name, n, gpu.BenchmarkParams(layers=layers, seed=1))
    cfg = gpu.Config(block_bits=b, inner_size=2, error_bound=br)
    want = port.simulate(n, [g.as_tuple() for g in c.gates], b, 2, br)
    cols = gpu.Collective.local(world)
    sims = [gpu.Simulator(c, cfg) for _ in range(world)]
    reps, errs = [None] * world, []

    def go(r):
        try:
            reps[r] = sims[r].run_sharded(cols[r])
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=go, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert _merged([s.payloads() for s in sims]) == want.payloads
    for rep in reps:
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
        assert rep.final_norm == pytest.approx(want.report["final_norm"], rel=1e-10)
    for s in sims:
        s.close()
    for col in cols:
        col.close()


@pytest.mark.gpu
def test_c_abi_sharded_run_nccl_world1(gpu, port):
    """The NCCL collective (libnccl.so.2 at run time) for one rank."""
    c = gpu.generate_benchmark("qft", 16)
    cfg = gpu.Config(block_bits=12, inner_size=2, error_bound=1e-3)
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    col = gpu.Collective.nccl(gpu.Collective.nccl_unique_id(), 0, 1, 0)
    with gpu.Simulator(c, cfg) as sim:
        rep = sim.run_sharded(col)
        assert sim.payloads() == want.payloads
        assert rep.max_footprint_bytes == want.report["max_footprint_bytes"]
    col.close()


@pytest.mark.gpu
def test_c_abi_sharded_run_with_host_level(gpu, port):
    """Sharded ranks whose device arenas overflow into their pinned host
    levels: remaps export payloads from either level; the result is the
    single-GPU run's."""
    import threading
    c = gpu.generate_benchmark("qaoa3reg", 16, gpu.BenchmarkParams(layers=2, seed=1))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, 1e-3)
    biggest = max(len(p) for p in want.payloads)
    cfg = gpu.Config(block_bits=12, inner_size=2, error_bound=1e-3, work_bytes=4 * (16 << 12),
                     device_pool_bytes=3 * (biggest + 16), host_pool_bytes=32 << 20)
    cols = gpu.Collective.local(2)
    sims = [gpu.Simulator(c, cfg) for _ in range(2)]
    reps, errs = [None, None], []

    def go(r):
        try:
            reps[r] = sims[r].run_sharded(cols[r])
        except Exception as e:
            errs.append(e)

    th = [threading.Thread(target=go, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert sum(r.device["host_spill_bytes"] for r in reps) > 0
    assert _merged([s.payloads() for s in sims]) == want.payloads
    assert reps[0].max_footprint_bytes == want.report["max_footprint_bytes"]
    for s in sims:
        s.close()
    for col in cols:
        col.close()
