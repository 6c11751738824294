"""shard.py — the stage loop of cbq::Simulator::run (engine.hpp:97-134) over
several GPUs, one process (or thread) per GPU.

The reference is single-node: within a stage every SV group is independent
(engine.hpp:114-115) and only the grouping changes between stages. A sharded
run picks log2(world) *device qubits* among each stage's outer qubits
(`bmq_shard_plan`, furthest-next-use); a group then lives wholly on the rank
named by its device-qubit values, and a stage needs no communication at all.
Only when the next stage needs a device qubit as an inner qubit do the device
qubits change, and the compressed payloads whose owner changes move:

    meta  (size + block sums, 32 B per moving id)   all_to_all_v
    bytes (payloads, 16-byte aligned slots)          all_to_all_v

The receiving side knows which ids it gets (ownership is a pure function of
the plan), so only sizes travel before the bytes. Per stage, one sum
all-reduce of the per-id sizes (2^c u64) lets every rank replay the
reference BlockStore accounting (store.hpp:64-83) in the reference's put
order, so max_footprint_bytes / spilled_blocks equal the single-GPU run.
Norm and fidelity are sums of per-block partial sums, all-reduced.

Transport is `torch.distributed` (NCCL over NVLink on GPUs, gloo on CPU) or,
for several shards in one process, `LocalCollective` (threads). Payload
buffers stay on the device for NCCL: the engine packs into / unpacks from
the tensors' device memory directly.
"""
from __future__ import annotations

import ctypes as C
import threading
import time

import numpy as np
import torch

from . import cbq
from ._lib import lib, bmq_report, bmq_stage

# ------------------------------------------------------------------ planning


def shard_plan(num_qubits: int, block_bits: int, stages, world: int) -> np.ndarray:
    """Device qubits per stage: array (num_stages, log2 world); entry [s, j]
    is the qubit whose value is bit j of the rank that owns a group of s."""
    m = int(world).bit_length() - 1
    arr = (bmq_stage * max(1, len(stages)))()
    for i, st in enumerate(stages):
        arr[i] = st.to_c() if hasattr(st, "to_c") else st
    out = np.zeros(max(1, len(stages) * m), dtype=np.uint32)
    cbq._check(lib.bmq_shard_plan(num_qubits, block_bits, arr, len(stages), world,
                                  out.ctypes.data_as(C.POINTER(C.c_uint32))))
    return out[: len(stages) * m].reshape(len(stages), m)


def owners(num_blocks: int, device_qubits, block_bits: int) -> np.ndarray:
    """Owning rank of every block id under one stage's device qubits."""
    ids = np.arange(num_blocks, dtype=np.uint64)
    r = np.zeros(num_blocks, dtype=np.uint64)
    for j, q in enumerate(device_qubits):
        r |= ((ids >> np.uint64(int(q) - block_bits)) & np.uint64(1)) << np.uint64(j)
    return r.astype(np.int64)


def remap_lists(own_prev: np.ndarray, own_next: np.ndarray, rank: int, world: int):
    """Ids this rank sends to / receives from each peer (ascending id order)."""
    ids = np.arange(len(own_prev), dtype=np.uint64)
    leaving = own_prev == rank
    arriving = own_next == rank
    sends = [ids[leaving & (own_next == p)] if p != rank else ids[:0] for p in range(world)]
    recvs = [ids[arriving & (own_prev == p)] if p != rank else ids[:0] for p in range(world)]
    return sends, recvs


def _aligned(sizes: np.ndarray) -> np.ndarray:
    return (sizes.astype(np.int64) + 15) // 16 * 16


# --------------------------------------------------------------- transports


class TorchCollective:
    """torch.distributed process group (nccl: CUDA tensors; gloo: CPU)."""

    def __init__(self, device: torch.device | str | None = None, group=None):
        import torch.distributed as dist
        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if device is None:
            device = (torch.device("cuda", torch.cuda.current_device())
                      if dist.get_backend(group) == "nccl" else torch.device("cpu"))
        self.device = torch.device(device)

    def all_to_all_v(self, send: torch.Tensor, send_counts, recv_counts) -> torch.Tensor:
        out = torch.empty(int(sum(recv_counts)), dtype=send.dtype, device=self.device)
        if self.world == 1:
            out.copy_(send[: out.numel()])
            return out
        self._dist.all_to_all_single(out, send, [int(c) for c in recv_counts], [int(c) for c in send_counts],
                                     group=self.group)
        return out

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            self._dist.all_reduce(t, group=self.group)
        return t

    def barrier(self):
        if self.world > 1:
            self._dist.barrier(group=self.group)

    def synchronize(self):
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)


class LocalHub:
    """Shared state of the LocalCollectives of one process (one per thread)."""

    def __init__(self, world: int):
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)


class LocalCollective:
    """Same interface as TorchCollective for `world` shards driven by threads
    of one process (e.g. several engines sharing one GPU)."""

    def __init__(self, hub: LocalHub, rank: int, device: torch.device | str = "cpu"):
        self.hub, self.rank, self.world = hub, rank, hub.world
        self.device = torch.device(device)

    def _exchange(self, item):
        self.hub.slots[self.rank] = item
        self.hub.bar.wait()
        got = list(self.hub.slots)
        self.hub.bar.wait()
        return got

    def all_to_all_v(self, send: torch.Tensor, send_counts, recv_counts) -> torch.Tensor:
        self.synchronize()
        got = self._exchange((send, [int(c) for c in send_counts]))
        parts = []
        for q, (buf, counts) in enumerate(got):
            start = sum(counts[: self.rank])
            parts.append(buf[start: start + counts[self.rank]].to(self.device))
        out = torch.cat(parts) if parts else torch.empty(0, dtype=send.dtype, device=self.device)
        assert out.numel() == sum(int(c) for c in recv_counts)
        self.synchronize()
        self.hub.bar.wait()  # every peer has copied its part out of our send buffer
        return out

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        got = self._exchange(t.clone())
        total = got[0].to(t.device).clone()
        for x in got[1:]:
            total += x.to(t.device)
        t.copy_(total)
        return t

    def barrier(self):
        self.hub.bar.wait()

    def synchronize(self):
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)


# ------------------------------------------------------------------ backends


class EngineShard:
    """One rank's share of the state in a device engine (libbmq)."""

    def __init__(self, circuit: cbq.Circuit, config: cbq.Config, rank: int, world: int):
        self.sim = cbq.Simulator(circuit, config)
        self.rank, self.world = rank, world
        self.layout = self.sim.layout()
        self.stages = self.sim.plan().stages
        self.block_bits = config.block_bits
        self.error_bound = config.error_bound
        if world > 1:
            cbq._check(lib.bmq_simulator_shard(self.sim._h, rank, world))

    def close(self):
        self.sim.close()

    @property
    def _h(self):
        return self.sim._h

    def init(self):
        self.sim.init_state()

    def reset(self):
        self.sim.reset()

    def run_stage(self, s: int):
        cbq._check(lib.bmq_simulator_run_stages(self._h, s, s + 1))

    @staticmethod
    def _ids(ids: np.ndarray):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        return ids, ids.ctypes.data_as(C.POINTER(C.c_uint64))

    def meta(self, ids: np.ndarray) -> np.ndarray:
        ids, p = self._ids(ids)
        meta = np.zeros((len(ids), 4), dtype=np.uint64)
        cbq._check(lib.bmq_simulator_export(self._h, p, len(ids), meta.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            None, 0))
        return meta

    def pack(self, ids: np.ndarray, out: torch.Tensor) -> None:
        ids, p = self._ids(ids)
        meta = np.zeros((len(ids), 4), dtype=np.uint64)
        cbq._check(lib.bmq_simulator_export(self._h, p, len(ids), meta.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            C.c_void_p(out.data_ptr() if out.numel() else None), out.numel()))

    def unpack(self, ids: np.ndarray, meta: np.ndarray, buf: torch.Tensor) -> None:
        ids, p = self._ids(ids)
        meta = np.ascontiguousarray(meta, dtype=np.uint64)
        cbq._check(lib.bmq_simulator_import(self._h, p, len(ids), meta.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            C.c_void_p(buf.data_ptr() if buf.numel() else None)))

    def drop(self, ids: np.ndarray) -> None:
        ids, p = self._ids(ids)
        cbq._check(lib.bmq_simulator_drop(self._h, p, len(ids)))

    def stage_sizes(self, s: int) -> np.ndarray:
        out = np.zeros(self.layout.num_blocks(), dtype=np.uint64)
        cbq._check(lib.bmq_simulator_stage_sizes(self._h, s, out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    def account_stage(self, s: int, sizes: np.ndarray) -> None:
        sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
        cbq._check(lib.bmq_simulator_account_stage(self._h, s, sizes.ctypes.data_as(C.POINTER(C.c_uint64))))

    def partial_sums(self) -> np.ndarray:
        out = np.zeros(3)
        cbq._check(lib.bmq_simulator_partial_sums(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def report(self) -> cbq.SimulationReport:
        r = bmq_report()
        cbq._check(lib.bmq_simulator_report(self._h, C.byref(r)))
        return cbq.report_from_c(r, [])


# ------------------------------------------------------------------- driver

_SUMMED = ("groups_processed", "groups_skipped", "blocks_processed", "payload_bytes_read", "payload_bytes_written",
           "dense_bytes", "kernel_launches", "gate_passes", "batches", "decompress_bytes", "gate_bytes",
           "compress_bytes", "fused_batches", "compactions", "host_spill_bytes", "host_spill_batches",
           "code_domain_batches", "pool_growths", "lazy_cx", "perm_materialisations", "model_bytes", "model_groups",
           "link_h2d_bytes", "link_d2h_bytes", "link_ms", "compact_bytes", "host_peak_bytes", "arena_bytes")


class ShardedSimulator:
    """cbq::Simulator::run over `collective.world` ranks; every rank calls
    run() (SPMD). `backend` holds this rank's blocks (EngineShard on a GPU)."""

    def __init__(self, backend, collective):
        self.backend, self.col = backend, collective
        self.rank, self.world = collective.rank, collective.world
        if backend.world != self.world or backend.rank != self.rank:
            raise cbq.InvalidArgument("backend and collective disagree on rank / world")
        L = backend.layout
        self.layout = L
        self.stages = backend.stages
        self.bits = shard_plan(L.n, L.b, self.stages, self.world)
        if hasattr(backend, "set_bits"):  # backends that do not plan themselves
            backend.set_bits(self.bits)
        self._own = {}
        self._ran = False
        self.remaps = 0
        self.moved_bytes = 0  # payload bytes this rank sent
        self.exchange_ms = 0.0
        self.account_ms = 0.0

    def owners_of(self, s: int) -> np.ndarray:
        if s not in self._own:
            self._own[s] = owners(self.layout.num_blocks(), self.bits[s], self.layout.b)
        return self._own[s]

    def _i64(self, a: np.ndarray) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(self.col.device)

    def _exchange(self, sends, recvs):
        """Move the listed payloads: meta first, then the packed bytes."""
        be, col = self.backend, self.col
        send_ids = np.concatenate(sends)
        recv_ids = np.concatenate(recvs)
        meta = be.meta(send_ids)
        rmeta_t = col.all_to_all_v(self._i64(meta.reshape(-1)), [4 * len(x) for x in sends],
                                   [4 * len(x) for x in recvs])
        rmeta = rmeta_t.cpu().numpy().view(np.uint64).reshape(-1, 4)
        sbytes = _aligned(meta[:, 0])
        rbytes = _aligned(rmeta[:, 0])
        scounts, rcounts, a, b = [], [], 0, 0
        for p in range(self.world):
            scounts.append(int(sbytes[a: a + len(sends[p])].sum()))
            rcounts.append(int(rbytes[b: b + len(recvs[p])].sum()))
            a += len(sends[p])
            b += len(recvs[p])
        sbuf = torch.empty(sum(scounts), dtype=torch.uint8, device=col.device)
        be.pack(send_ids, sbuf)
        rbuf = col.all_to_all_v(sbuf, scounts, rcounts)
        col.synchronize()
        be.unpack(recv_ids, rmeta, rbuf)
        be.drop(send_ids)
        self.moved_bytes += sum(scounts)

    def _remap(self, s: int):
        prev, nxt = self.owners_of(s - 1), self.owners_of(s)
        if np.array_equal(self.bits[s - 1], self.bits[s]):
            return
        t0 = time.perf_counter()
        sends, recvs = remap_lists(prev, nxt, self.rank, self.world)
        self._exchange(sends, recvs)
        self.remaps += 1
        self.exchange_ms += (time.perf_counter() - t0) * 1e3

    def run(self) -> cbq.SimulationReport:
        be, col = self.backend, self.col
        t0 = time.perf_counter()
        if self._ran:
            be.reset()
        self._ran = True
        self.remaps, self.moved_bytes, self.exchange_ms, self.account_ms = 0, 0, 0.0, 0.0
        be.init()
        stage_ms = []
        for s in range(len(self.stages)):
            ts = time.perf_counter()
            if s and self.world > 1:
                self._remap(s)
            be.run_stage(s)
            if self.world > 1:
                ta = time.perf_counter()
                sizes = self._i64(be.stage_sizes(s))
                col.all_reduce_sum(sizes)
                be.account_stage(s, sizes.cpu().numpy().view(np.uint64))
                self.account_ms += (time.perf_counter() - ta) * 1e3
            stage_ms.append((time.perf_counter() - ts) * 1e3)
        rep = self._global_report(stage_ms)
        rep.wall_ms = (time.perf_counter() - t0) * 1e3
        return rep

    def _global_report(self, stage_ms) -> cbq.SimulationReport:
        be, col = self.backend, self.col
        rep = be.report()
        sums = torch.tensor(be.partial_sums(), dtype=torch.float64, device=col.device)
        col.all_reduce_sum(sums)
        self.global_sums = sums.cpu().numpy()
        rep.final_norm = float(np.sqrt(self.global_sums[0]))
        counts = torch.tensor([rep.device[k] for k in _SUMMED], dtype=torch.int64, device=col.device)
        col.all_reduce_sum(counts)
        for k, v in zip(_SUMMED, counts.cpu().tolist()):
            rep.device[k] = v
        rep.stage_ms = stage_ms
        rep.device["remaps"] = self.remaps
        rep.device["exchange_ms"] = self.exchange_ms
        rep.device["account_ms"] = self.account_ms
        return rep

    def norm(self) -> float:
        sums = torch.tensor(self.backend.partial_sums(), dtype=torch.float64, device=self.col.device)
        self.col.all_reduce_sum(sums)
        return float(np.sqrt(sums[0].item()))

    def fidelity_uniform(self) -> float:
        """|<u|psi>| with u = 2^(-n/2) (1, ..., 1): the QFT-of-|0> ideal."""
        sums = torch.tensor(self.backend.partial_sums(), dtype=torch.float64, device=self.col.device)
        self.col.all_reduce_sum(sums)
        re, im = float(sums[1]), float(sums[2])
        return float(np.hypot(re, im) * 2.0 ** (-0.5 * self.layout.n))

    def gather_payloads(self, root: int = 0):
        """Every payload in id order on `root` (None elsewhere)."""
        be, col = self.backend, self.col
        last = self.owners_of(len(self.stages) - 1) if len(self.stages) else np.zeros(self.layout.num_blocks(),
                                                                                           np.int64)
        ids = np.arange(self.layout.num_blocks(), dtype=np.uint64)
        mine = ids[last == self.rank]
        empty = ids[:0]
        sends = [mine if p == root else empty for p in range(self.world)]
        recvs = [ids[last == q] if self.rank == root else empty for q in range(self.world)]
        meta = be.meta(mine)
        rmeta = col.all_to_all_v(self._i64(meta.reshape(-1)), [4 * len(x) for x in sends],
                                 [4 * len(x) for x in recvs]).cpu().numpy().view(np.uint64).reshape(-1, 4)
        sb = int(_aligned(meta[:, 0]).sum())
        sbuf = torch.empty(sb, dtype=torch.uint8, device=col.device)
        be.pack(mine, sbuf)
        rcounts = []
        a = 0
        rb = _aligned(rmeta[:, 0])
        for q in range(self.world):
            rcounts.append(int(rb[a: a + len(recvs[q])].sum()))
            a += len(recvs[q])
        rbuf = col.all_to_all_v(sbuf, [sb if p == root else 0 for p in range(self.world)], rcounts)
        if self.rank != root:
            return None
        raw = rbuf.cpu().numpy().tobytes()
        out = [b""] * self.layout.num_blocks()
        zero = zero_payload(self.layout.b, be.error_bound)
        pos = 0
        order = np.concatenate(recvs)
        for i, id_ in enumerate(order.tolist()):
            size = int(rmeta[i, 0])
            out[id_] = raw[pos: pos + size] if size else zero
            pos += int(rb[i])
        return out


def zero_payload(block_bits: int, error_bound: float) -> bytes:
    """The canonical ALL_ZERO payload of a block (codec.hpp:263-271)."""
    hdr = bytearray(26)
    hdr[0:8] = (2 << block_bits).to_bytes(8, "little")
    hdr[8:16] = np.float64(error_bound).tobytes()
    hdr[25] = 1
    return bytes(hdr)
