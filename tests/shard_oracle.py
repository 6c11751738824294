"""CPU stand-in for one rank's EngineShard, built on the oracle (test
infrastructure only). It runs the reference's per-group pipeline
(engine.hpp:203-225: decompress -> assemble -> apply_stage -> split ->
compress) with the oracle's C restatement, so the shard driver's planning,
exchange protocol and accounting can be checked on CPU over gloo, world 2.
"""
from __future__ import annotations

import numpy as np
import torch

from paper_2410_14088_b200 import cbq
from paper_2410_14088_b200.shard import owners


class StoreReplay:
    """BlockStore accounting (store.hpp:64-117,188-232), sequential order."""

    def __init__(self, nid, budget=2**64 - 1):
        self.size = [0] * nid
        self.flag = [4] * nid  # bit0 spilled, bit1 shared, bit2 absent
        self.budget = budget
        self.resident = self.spilled_live = self.peak = self.spilled_blocks = 0
        self.shared_refs = self.shared_size = 0
        self.shared_spilled = False

    def _detach(self, i):
        f = self.flag[i]
        if f & 4:
            return
        if f & 2:
            self.shared_refs -= 1
            if self.shared_refs == 0:
                if self.shared_spilled:
                    self.spilled_live -= self.shared_size
                else:
                    self.resident -= self.shared_size
        elif f & 1:
            self.spilled_live -= self.size[i]
        else:
            self.resident -= self.size[i]
        self.flag[i] = 4

    def _place(self, size):
        if size <= self.budget and self.resident <= self.budget - size:
            self.resident += size
            return False
        self.spilled_live += size
        self.spilled_blocks += 1
        return True

    def put(self, i, size):
        self._detach(i)
        self.flag[i] = 1 if self._place(size) else 0
        self.size[i] = size
        self.peak = max(self.peak, self.resident + self.spilled_live)

    def put_shared(self, first, last, size):
        for i in range(first, last):
            self._detach(i)
        self.shared_spilled = self._place(size)
        self.shared_size = size
        self.shared_refs = last - first
        for i in range(first, last):
            self.flag[i] = 2
            self.size[i] = size
        self.peak = max(self.peak, self.resident + self.spilled_live)


def _is_zero(p: bytes) -> bool:
    return len(p) == 26 and p[25] & 1


class OracleShard:
    def __init__(self, port, n, gates, block_bits, inner_size, error_bound, rank, world):
        self.port, self.n, self.gates = port, n, gates
        self.block_bits, self.error_bound = block_bits, error_bound
        self.rank, self.world = rank, world
        self.layout = cbq.make_layout(n, block_bits)
        self.plan = port.partition(n, gates, block_bits, inner_size)
        self.stages = [cbq.Stage(b, e, list(inner)) for b, e, inner in self.plan]
        self.payload: dict[int, bytes] = {}
        self.sums: dict[int, tuple] = {}
        self.store = StoreReplay(self.layout.num_blocks())
        self.groups_processed = 0
        self._bits = None

    def set_bits(self, bits):
        self._bits = bits

    def _sums(self, x):
        h = len(x) // 2
        return (float(np.dot(x, x)), float(x[:h].sum()), float(x[h:].sum()))

    def init(self):
        nid = self.layout.num_blocks()
        e0 = np.zeros(2 << self.block_bits)
        e0[0] = 1.0
        p = self.port.compress_block(e0, self.error_bound)
        self.store.put(0, len(p))
        if nid > 1:
            self.store.put_shared(1, nid, 26)
        if self.rank == 0:
            self.payload[0] = p
            self.sums[0] = self._sums(self.port.decompress_block(p))

    def run_stage(self, s):
        b = self.block_bits
        st = self.plan[s]
        own = owners(self.layout.num_blocks(), self._bits[s], b)
        for ids in self.port.enumerate_groups(self.n, b, st):
            ids = [int(i) for i in ids]
            if own[ids[0]] != self.rank:
                continue
            if all(i not in self.payload for i in ids):
                continue
            self.groups_processed += 1
            buf = np.zeros(len(ids) << b, dtype=np.complex128)
            for v, i in enumerate(ids):
                if i in self.payload:
                    x = self.port.decompress_block(self.payload[i])
                    buf[v << b: (v + 1) << b] = x[: 1 << b] + 1j * x[1 << b:]
            buf = self.port.apply_stage(buf, self.n, self.gates, st, b)
            for v, i in enumerate(ids):
                blk = buf[v << b: (v + 1) << b]
                p = self.port.compress_block(np.concatenate([blk.real, blk.imag]), self.error_bound)
                if _is_zero(p):
                    self.payload.pop(i, None)
                    self.sums.pop(i, None)
                else:
                    self.payload[i] = p
                    self.sums[i] = self._sums(self.port.decompress_block(p))

    def meta(self, ids):
        m = np.zeros((len(ids), 4), dtype=np.uint64)
        for k, i in enumerate(np.asarray(ids).tolist()):
            if i in self.payload:
                m[k, 0] = len(self.payload[i])
                m[k, 1:] = np.array(self.sums[i], dtype=np.float64).view(np.uint64)
        return m

    def pack(self, ids, out: torch.Tensor):
        pos = 0
        view = out.numpy()
        for i in np.asarray(ids).tolist():
            p = self.payload.get(i, b"")
            view[pos: pos + len(p)] = np.frombuffer(p, dtype=np.uint8)
            pos += (len(p) + 15) // 16 * 16
        assert pos == out.numel()

    def unpack(self, ids, meta, buf: torch.Tensor):
        raw = buf.cpu().numpy().tobytes()
        pos = 0
        for k, i in enumerate(np.asarray(ids).tolist()):
            size = int(meta[k, 0])
            if size:
                self.payload[i] = raw[pos: pos + size]
                self.sums[i] = tuple(np.asarray(meta[k, 1:], dtype=np.uint64).view(np.float64).tolist())
            else:
                self.payload.pop(i, None)
                self.sums.pop(i, None)
            pos += (size + 15) // 16 * 16

    def drop(self, ids):
        for i in np.asarray(ids).tolist():
            self.payload.pop(i, None)
            self.sums.pop(i, None)

    def stage_sizes(self, s):
        own = owners(self.layout.num_blocks(), self._bits[s], self.block_bits)
        out = np.zeros(self.layout.num_blocks(), dtype=np.uint64)
        for i in range(len(out)):
            if own[i] == self.rank:
                out[i] = len(self.payload[i]) if i in self.payload else 26
        return out

    def account_stage(self, s, sizes):
        for ids in self.port.enumerate_groups(self.n, self.block_bits, self.plan[s]):
            for i in ids.tolist():
                self.store.put(i, int(sizes[i]))

    def partial_sums(self):
        out = np.zeros(3)
        for v in self.sums.values():
            out += np.array(v)
        return out

    def report(self):
        L = self.layout
        dev = {k: 0 for k in cbq.DEVICE_REPORT_KEYS}
        dev["groups_processed"] = self.groups_processed
        std = float(2 ** (L.n + 4))
        return cbq.SimulationReport(L.n, len(self.gates), len(self.plan), self.store.peak, std,
                                    std / self.store.peak if self.store.peak else 0.0, self.store.spilled_blocks,
                                    0.0, [], None, 0.0, 0, 0, dev)
