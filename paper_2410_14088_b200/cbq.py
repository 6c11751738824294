"""Python mirror of the reference's ``namespace cbq`` surface over libbmq.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/cbq); the work happens in libbmq (host C++ for
descriptors, sm_100a CUDA for the codec / gates / simulator):

=========================  ==================================================
reference (file:line)       here
=========================  ==================================================
GateKind, Gate, Circuit     ``GateKind``, ``Gate``, ``Circuit`` (circuit.hpp:20-130)
unitary2 / unitary4         ``unitary2`` / ``unitary4`` (circuit.hpp:133-198)
generate_benchmark          ``generate_benchmark`` (benchmarks.hpp:148-166)
Layout / make_layout        ``Layout`` / ``make_layout`` (partition.hpp:14-31)
Stage, PartitionPlan        ``Stage``, ``PartitionPlan`` (partition.hpp:36-46)
partition_circuit           ``partition_circuit`` (partition.hpp:59-101)
SVGroup, enumerate_groups   ``SVGroup``, ``enumerate_groups`` (partition.hpp:50-153)
buffer_bit_of_qubit         ``buffer_bit_of_qubit`` (partition.hpp:158-169)
ErrorBound                  ``ErrorBound`` (codec.hpp:19-29)
compress_block              ``compress_block`` / ``compress_blocks`` (codec.hpp:227)
decompress_block            ``decompress_block`` / ``decompress_blocks`` (codec.hpp:299)
apply_unitary2/4            ``apply_unitary2`` / ``apply_unitary4`` (kernel.hpp:24-64)
apply_stage                 ``apply_stage`` (kernel.hpp:111-122)
Config, SimulationReport    ``Config``, ``SimulationReport`` (engine.hpp:23-53)
Simulator                   ``Simulator`` (engine.hpp:58-250)
dense_reference, fidelity   ``dense_reference``, ``fidelity`` (engine.hpp:254-308)
CodecError / StoreError /   same names; std::invalid_argument -> ``InvalidArgument``
EngineError / QasmError     (a ValueError), std::logic_error -> ``LogicError``
=========================  ==================================================
"""
from __future__ import annotations

import ctypes as C
import os
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import lib, bmq_gate, bmq_stage, bmq_config, bmq_report


# ---------------------------------------------------------------- errors

class BmqError(RuntimeError):
    code = -1


class InvalidArgument(BmqError, ValueError):
    code = _lib.BMQ_ERR_INVALID_ARGUMENT


class LogicError(BmqError):
    code = _lib.BMQ_ERR_LOGIC


class CodecError(BmqError):
    code = _lib.BMQ_ERR_CODEC


class StoreError(BmqError):
    code = _lib.BMQ_ERR_STORE


class EngineError(BmqError):
    code = _lib.BMQ_ERR_ENGINE


class QasmError(BmqError):
    """cbq::QasmError (qasm.hpp:17-31): message 'line L, col C: ...'."""
    code = _lib.BMQ_ERR_QASM

    def __init__(self, msg):
        super().__init__(msg)
        import re
        m = re.match(r"line (\d+), col (\d+): ", msg)
        self.line = int(m.group(1)) if m else 0
        self.col = int(m.group(2)) if m else 0


class CudaError(BmqError):
    code = _lib.BMQ_ERR_CUDA


class NoDeviceError(BmqError):
    code = _lib.BMQ_ERR_NO_DEVICE


class OutOfMemory(BmqError, MemoryError):
    code = _lib.BMQ_ERR_OUT_OF_MEMORY


class BufferTooSmall(BmqError):
    code = _lib.BMQ_ERR_BUFFER_TOO_SMALL


_ERRORS = {c.code: c for c in (InvalidArgument, LogicError, CodecError, StoreError, EngineError, QasmError,
                               CudaError, NoDeviceError, OutOfMemory, BufferTooSmall)}


def _check(rc):
    if rc:
        msg = lib.bmq_last_error().decode()
        raise _ERRORS.get(rc, BmqError)(msg)


def device_count() -> int:
    n = C.c_int()
    _check(lib.bmq_device_count(C.byref(n)))
    return n.value


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------- circuit

class GateKind(enum.IntEnum):
    H = 0
    X = 1
    Y = 2
    Z = 3
    S = 4
    Sdg = 5
    T = 6
    Tdg = 7
    RX = 8
    RY = 9
    RZ = 10
    P = 11
    CX = 12
    CZ = 13
    CP = 14


_TWO = {GateKind.CX, GateKind.CZ, GateKind.CP}
_PARAM = {GateKind.RX, GateKind.RY, GateKind.RZ, GateKind.P, GateKind.CP}
_NAMES = ["h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "p", "cx", "cz", "cp"]


def is_two_qubit(kind) -> bool:
    return GateKind(kind) in _TWO


def is_parameterized(kind) -> bool:
    return GateKind(kind) in _PARAM


def gate_name(kind) -> str:
    return _NAMES[int(kind)]


@dataclass(frozen=True)
class Gate:
    """cbq::Gate (circuit.hpp:65-72); q0 is the high sub-index bit of 2q gates."""
    kind: GateKind
    q0: int = 0
    q1: int = 0
    angle: float = 0.0

    def to_c(self) -> bmq_gate:
        return bmq_gate(int(self.kind), self.q0, self.q1 if is_two_qubit(self.kind) else 0, 0, float(self.angle))

    def as_tuple(self):
        return (int(self.kind), self.q0, self.q1 if is_two_qubit(self.kind) else 0, float(self.angle))


class gates:  # cbq::gates (circuit.hpp:74-92)
    h = staticmethod(lambda q: Gate(GateKind.H, q))
    x = staticmethod(lambda q: Gate(GateKind.X, q))
    y = staticmethod(lambda q: Gate(GateKind.Y, q))
    z = staticmethod(lambda q: Gate(GateKind.Z, q))
    s = staticmethod(lambda q: Gate(GateKind.S, q))
    sdg = staticmethod(lambda q: Gate(GateKind.Sdg, q))
    t = staticmethod(lambda q: Gate(GateKind.T, q))
    tdg = staticmethod(lambda q: Gate(GateKind.Tdg, q))
    rx = staticmethod(lambda q, a: Gate(GateKind.RX, q, 0, a))
    ry = staticmethod(lambda q, a: Gate(GateKind.RY, q, 0, a))
    rz = staticmethod(lambda q, a: Gate(GateKind.RZ, q, 0, a))
    p = staticmethod(lambda q, a: Gate(GateKind.P, q, 0, a))
    cx = staticmethod(lambda c, t: Gate(GateKind.CX, c, t))
    cz = staticmethod(lambda a, b: Gate(GateKind.CZ, a, b))
    cp = staticmethod(lambda a, b, ang: Gate(GateKind.CP, a, b, ang))


def _gate_array(gs):
    arr = (bmq_gate * max(1, len(gs)))()
    for i, g in enumerate(gs):
        arr[i] = g.to_c()
    return arr


def _gate_from_c(g: bmq_gate) -> Gate:
    k = GateKind(g.kind)
    return Gate(k, g.q0, g.q1 if k in _TWO else 0, g.angle)


class Circuit:
    """cbq::Circuit (circuit.hpp:97-130): validated ordered gate list."""

    def __init__(self, num_qubits: int = 1, gate_list=None):
        if not (1 <= num_qubits <= 62):
            raise InvalidArgument(f"qubit count must be in [1, 62], got {num_qubits}")
        self.num_qubits = num_qubits
        self.gates: list[Gate] = []
        for g in gate_list or []:
            self.add(g)

    def add(self, g: Gate) -> None:
        _check(lib.bmq_circuit_validate(self.num_qubits, C.byref(g.to_c()), 1))
        self.gates.append(g)

    def c_array(self):
        return _gate_array(self.gates)

    def __eq__(self, other):
        return isinstance(other, Circuit) and self.num_qubits == other.num_qubits and self.gates == other.gates

    def __len__(self):
        return len(self.gates)


Mat2 = np.ndarray
Mat4 = np.ndarray


def _unitary(g: Gate) -> np.ndarray:
    out = np.zeros(32)
    _check(lib.bmq_gate_unitary(C.byref(g.to_c()), _ptr(out)))
    m = 4 if is_two_qubit(g.kind) else 2
    return (out[0::2] + 1j * out[1::2])[: m * m].reshape(m, m)


def unitary2(g: Gate) -> np.ndarray:
    if is_two_qubit(g.kind):
        raise LogicError("unitary2 called on a two-qubit gate")
    return _unitary(g)


def unitary4(g: Gate) -> np.ndarray:
    if not is_two_qubit(g.kind):
        raise LogicError("unitary4 called on a single-qubit gate")
    return _unitary(g)


class Benchmark(enum.Enum):
    Ghz = "ghz"
    CatState = "cat_state"
    Bv = "bv"
    Qft = "qft"
    Qaoa = "qaoa"


def benchmark_from_name(name: str) -> Benchmark:
    try:
        return Benchmark(name)
    except ValueError:
        raise InvalidArgument(f"unknown benchmark '{name}'") from None


@dataclass
class BenchmarkParams:
    layers: int = 1
    secret: str | None = None
    seed: int = 1


def generate_benchmark(bench, n: int, params: BenchmarkParams | None = None) -> Circuit:
    """generate_benchmark (benchmarks.hpp:148-166)."""
    p = params or BenchmarkParams()
    name = bench.value if isinstance(bench, Benchmark) else str(bench)
    count = C.c_uint64()
    rc = lib.bmq_generate_benchmark(name.encode(), n, p.layers, p.seed, (p.secret or "").encode(), None, 0,
                                    C.byref(count))
    if rc and rc != _lib.BMQ_ERR_BUFFER_TOO_SMALL:
        _check(rc)
    arr = (bmq_gate * max(1, count.value))()
    _check(lib.bmq_generate_benchmark(name.encode(), n, p.layers, p.seed, (p.secret or "").encode(), arr,
                                      count.value, C.byref(count)))
    c = Circuit(n)
    c.gates = [_gate_from_c(arr[i]) for i in range(count.value)]
    return c


def parse_qasm(text: str, warnings: list | None = None) -> Circuit:
    """parse_qasm (qasm.hpp:387-389): OPENQASM 2.0 subset, parsed by libbmq's host C++."""
    data = text.encode()
    nq, count, nw = C.c_uint32(), C.c_uint64(), C.c_uint64()
    wbuf = C.create_string_buffer(4096)
    rc = lib.bmq_parse_qasm(data, C.byref(nq), None, 0, C.byref(count), wbuf, 4096, C.byref(nw))
    if rc and rc != _lib.BMQ_ERR_BUFFER_TOO_SMALL:
        _check(rc)
    arr = (bmq_gate * max(1, count.value))()
    _check(lib.bmq_parse_qasm(data, C.byref(nq), arr, count.value, C.byref(count), wbuf, 4096, C.byref(nw)))
    if warnings is not None and nw.value:
        warnings.extend(wbuf.value.decode().split("\n"))
    c = Circuit(nq.value)
    c.gates = [_gate_from_c(arr[i]) for i in range(count.value)]
    return c


def emit_qasm(circuit: Circuit) -> str:
    """emit_qasm (qasm.hpp:392-411)."""
    size = C.c_uint64()
    rc = lib.bmq_emit_qasm(circuit.num_qubits, circuit.c_array(), len(circuit.gates), None, 0, C.byref(size))
    if rc and rc != _lib.BMQ_ERR_BUFFER_TOO_SMALL:
        _check(rc)
    buf = C.create_string_buffer(size.value + 1)
    _check(lib.bmq_emit_qasm(circuit.num_qubits, circuit.c_array(), len(circuit.gates), buf, size.value + 1,
                             C.byref(size)))
    return buf.value.decode()


# ------------------------------------------------------------- partition

@dataclass(frozen=True)
class Layout:
    n: int = 1
    b: int = 1
    c: int = 0

    def num_blocks(self) -> int:
        return 1 << self.c

    def block_size(self) -> int:
        return 1 << self.b


def make_layout(n: int, b: int) -> Layout:
    if not (1 <= n <= 62):
        raise InvalidArgument("layout qubit count must be in [1, 62]")
    if not (1 <= b <= n):
        raise InvalidArgument("local index bits must be in [1, n]")
    return Layout(n, b, n - b)


@dataclass
class Stage:
    gate_begin: int = 0
    gate_end: int = 0
    inner: list = field(default_factory=list)

    def to_c(self) -> bmq_stage:
        st = bmq_stage()
        st.gate_begin, st.gate_end, st.inner_count = self.gate_begin, self.gate_end, len(self.inner)
        for i, q in enumerate(self.inner):
            st.inner[i] = q
        return st

    @staticmethod
    def from_c(s: bmq_stage) -> "Stage":
        return Stage(s.gate_begin, s.gate_end, list(s.inner[: s.inner_count]))


@dataclass
class PartitionPlan:
    layout: Layout
    inner_size: int
    stages: list


def partition_circuit(circuit: Circuit, block_bits: int, inner_size: int) -> PartitionPlan:
    """partition_circuit (partition.hpp:59-101), computed by libbmq's host C++."""
    layout = make_layout(circuit.num_qubits, block_bits)
    cap = max(1, len(circuit.gates))
    out = (bmq_stage * cap)()
    ns = C.c_uint64()
    _check(lib.bmq_partition(circuit.num_qubits, circuit.c_array(), len(circuit.gates), block_bits, inner_size,
                             out, cap, C.byref(ns)))
    return PartitionPlan(layout, inner_size, [Stage.from_c(out[i]) for i in range(ns.value)])


@dataclass
class PlanChoice:
    """What plan_device_aware chose and the modelled time of every candidate."""
    inner_size: int
    stages: int
    passes: int
    remaps: int
    model_s: float
    candidates: dict  # inner size -> modelled seconds


def plan_device_aware(circuit: Circuit, block_bits: int, *, work_bytes: int = 16 << 30, hbm_gbs: float = 6500.0,
                      link_gbs: float = 700.0, ratio: float = 4.0, stage_overhead_s: float = 100e-6,
                      world: int = 1, max_inner: int = 0):
    """Device-aware staging (bmq_plan_device_aware): the
    partition_circuit plan (partition.hpp:59-101) at the inner size this
    engine's cost model prefers for the device; returns (PartitionPlan,
    PlanChoice). Replaying it in the reference needs inner_size =
    choice.inner_size."""
    layout = make_layout(circuit.num_qubits, block_bits)
    m = _lib.bmq_plan_model()
    lib.bmq_plan_model_default(C.byref(m))
    m.work_bytes, m.hbm_gbs, m.link_gbs, m.ratio = work_bytes, hbm_gbs, link_gbs, ratio
    m.stage_overhead_s, m.world, m.max_inner = stage_overhead_s, world, max_inner
    cap = max(1, len(circuit.gates))
    out = (bmq_stage * cap)()
    ns = C.c_uint64()
    ch = _lib.bmq_plan_choice()
    _check(lib.bmq_plan_device_aware(circuit.num_qubits, circuit.c_array(), len(circuit.gates), block_bits,
                                     C.byref(m), out, cap, C.byref(ns), C.byref(ch)))
    choice = PlanChoice(ch.inner_size, ch.stages, ch.passes, ch.remaps, ch.model_s_best,
                        {ch.inner[i]: ch.model_s[i] for i in range(ch.candidates)})
    return PartitionPlan(layout, ch.inner_size, [Stage.from_c(out[i]) for i in range(ns.value)]), choice


@dataclass
class SVGroup:
    outer_value: int = 0
    block_ids: list = field(default_factory=list)


def enumerate_groups(stage: Stage, layout: Layout) -> list:
    """enumerate_groups (partition.hpp:120-153)."""
    st = stage.to_c()
    cap = 1 << layout.c
    ids = np.zeros(max(1, cap), dtype=np.uint64)
    cnt = C.c_uint64()
    _check(lib.bmq_enumerate_groups(layout.n, layout.b, C.byref(st), _ptr(ids), cap, C.byref(cnt)))
    per = 1 << len(stage.inner)
    rows = ids[: cnt.value].reshape(-1, per)
    return [SVGroup(o, [int(x) for x in row]) for o, row in enumerate(rows)]


def buffer_bit_of_qubit(stage: Stage, layout: Layout, q: int) -> int:
    st = stage.to_c()
    out = C.c_uint32()
    _check(lib.bmq_buffer_bit_of_qubit(layout.n, layout.b, C.byref(st), q, C.byref(out)))
    return out.value


# ----------------------------------------------------------------- codec

kPayloadHeaderBytes = 26
kFlagAllZero = 0x1


class ErrorBound:
    """ErrorBound (codec.hpp:19-29)."""

    def __init__(self, b_r: float):
        out = C.c_double()
        _check(lib.bmq_error_bound(float(b_r), C.byref(out)))
        self.relative = float(b_r)
        self.log2_abs = out.value


def relative_to_absolute_bound(b_r: float) -> float:
    return ErrorBound(b_r).log2_abs


@dataclass
class PayloadHeader:
    scalar_count: int = 0
    relative_bound: float = 0.0
    code_min: int = 0
    code_width: int = 0
    flags: int = 0

    def all_zero(self) -> bool:
        return bool(self.flags & kFlagAllZero)


def parse_header(payload: bytes) -> PayloadHeader:
    """parse_header (codec.hpp:213-222)."""
    if len(payload) < kPayloadHeaderBytes:
        raise CodecError("header truncated")
    count, bound, cmin = np.frombuffer(payload[:24], dtype="<u8").tolist()
    return PayloadHeader(count, float(np.array([bound], dtype=np.uint64).view(np.float64)[0]),
                         int(np.array([cmin], dtype=np.uint64).view(np.int64)[0]), payload[24], payload[25])


def compress_blocks(scalars: np.ndarray, bound) -> list:
    """Compress each row of a 2-D float64 array (one block per row) on the GPU."""
    b_r = bound.relative if isinstance(bound, ErrorBound) else float(bound)
    a = np.ascontiguousarray(scalars, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    nblk, n = a.shape
    cap = int(lib.bmq_compress_bound(n)) * max(1, nblk)
    out = np.empty(max(1, cap), dtype=np.uint8)
    sizes = np.zeros(max(1, nblk), dtype=np.uint64)
    _check(lib.bmq_compress_blocks(_ptr(a), nblk, n, b_r, _ptr(out), cap, _ptr(sizes)))
    res, off = [], 0
    for s in sizes[:nblk].tolist():
        res.append(out[off: off + s].tobytes())
        off += s
    return res


def compress_block(scalars, bound) -> bytes:
    """compress_block (codec.hpp:227-295): byte-identical payload."""
    return compress_blocks(np.asarray(scalars, dtype=np.float64).reshape(1, -1), bound)[0]


def decompress_blocks(payloads: list) -> list:
    blob = b"".join(payloads)
    nblk = len(payloads)
    sizes = np.array([len(p) for p in payloads], dtype=np.uint64)
    offs = np.zeros(nblk, dtype=np.uint64)
    if nblk > 1:
        offs[1:] = np.cumsum(sizes)[:-1]
    data = np.frombuffer(blob + b"\0", dtype=np.uint8)
    counts = np.zeros(max(1, nblk), dtype=np.uint64)
    out = np.zeros(1, dtype=np.float64)
    rc = lib.bmq_decompress_blocks(_ptr(data), _ptr(offs), _ptr(sizes), nblk, _ptr(out), 0, _ptr(counts))
    if rc == _lib.BMQ_ERR_BUFFER_TOO_SMALL:
        out = np.zeros(max(1, int(counts[:nblk].sum())), dtype=np.float64)
        rc = lib.bmq_decompress_blocks(_ptr(data), _ptr(offs), _ptr(sizes), nblk, _ptr(out), out.size, _ptr(counts))
    _check(rc)
    res, pos = [], 0
    for c in counts[:nblk].tolist():
        res.append(out[pos: pos + c].copy())
        pos += c
    return res


def decompress_block(payload: bytes) -> np.ndarray:
    """decompress_block (codec.hpp:299-344): bit-identical values."""
    return decompress_blocks([bytes(payload)])[0]


# ---------------------------------------------------------------- kernel

SVBlock = np.ndarray


@dataclass
class GroupBuffer:
    group: SVGroup
    amps: np.ndarray


def _apply(amps, u, two, hi, lo):
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    um = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(-1))
    ud = np.empty(2 * um.size)
    ud[0::2], ud[1::2] = um.real, um.imag
    _check(lib.bmq_apply_gate(_ptr(a), a.size, _ptr(ud), int(two), hi, lo))
    return a


def apply_unitary2(amps: np.ndarray, bit: int, u) -> np.ndarray:
    """apply_unitary2 (kernel.hpp:24-38); returns the updated buffer (in place when contiguous complex128)."""
    out = _apply(amps, u, False, bit, 0)
    if out is not amps and isinstance(amps, np.ndarray) and amps.dtype == np.complex128:
        amps[...] = out
    return out


def apply_unitary4(amps: np.ndarray, hi_bit: int, lo_bit: int, u) -> np.ndarray:
    """apply_unitary4 (kernel.hpp:42-64)."""
    out = _apply(amps, u, True, hi_bit, lo_bit)
    if out is not amps and isinstance(amps, np.ndarray) and amps.dtype == np.complex128:
        amps[...] = out
    return out


def assemble_group_buffer(group: SVGroup, blocks: list) -> GroupBuffer:
    """assemble_group_buffer (kernel.hpp:66-84)."""
    if not blocks or (len(blocks) & (len(blocks) - 1)):
        raise InvalidArgument("group block count must be a nonzero power of two")
    if len(blocks) != len(group.block_ids):
        raise InvalidArgument("block list does not match the group")
    if any(len(b) != len(blocks[0]) for b in blocks):
        raise InvalidArgument("group blocks must have equal length")
    return GroupBuffer(group, np.concatenate([np.asarray(b, dtype=np.complex128) for b in blocks]))


def split_buffer(buf: GroupBuffer, block_bits: int) -> list:
    """split_buffer (kernel.hpp:87-98)."""
    bs = 1 << block_bits
    if buf.amps.size % bs:
        raise InvalidArgument("buffer length not divisible by the block size")
    return [buf.amps[o: o + bs].copy() for o in range(0, buf.amps.size, bs)]


def apply_stage(buf: GroupBuffer, stage: Stage, circuit: Circuit, layout: Layout) -> None:
    """apply_stage (kernel.hpp:111-122) on the GPU, in place on buf.amps."""
    a = np.ascontiguousarray(buf.amps, dtype=np.complex128)
    st = stage.to_c()
    _check(lib.bmq_apply_stage(_ptr(a), a.size, circuit.num_qubits, circuit.c_array(), len(circuit.gates),
                               C.byref(st), layout.b))
    buf.amps = a


# ---------------------------------------------------------------- engine

kUnlimitedBudget = 2**64 - 1


@dataclass
class Config:
    """cbq::Config (engine.hpp:23-37) plus device knobs."""
    block_bits: int = 1
    inner_size: int = 2
    error_bound: float = 1e-3
    memory_budget: int = kUnlimitedBudget
    workers: int = 1
    compress: bool = True
    verify_cap_qubits: int = 24
    device: int = 0
    device_pool_bytes: int = 0
    work_bytes: int = 0
    zero_group_skip: bool = True
    identity_skip: bool = False
    code_domain: bool = True
    pool_grow: bool = False
    arena: str = "auto"  # device arena placement: "auto", "heap" (extent per payload) or "bump" (cursor + compaction)
    host_pool_bytes: int = 0
    device_plan: bool = False  # plan with plan_device_aware (inner_size = cap) instead of partition_circuit
    fuse_stages: bool = True  # BMQ_FLAG_STAGE_FUSION: consecutive FP stages decoded / emitted once
    disk_pool_bytes: int = 0   # third level: spill file beneath the host level (needs host_pool_bytes)
    disk_dir: str = ""         # directory of the spill file ("" = /tmp)

    def to_c(self) -> bmq_config:
        c = bmq_config()
        lib.bmq_config_default(C.byref(c))
        c.block_bits, c.inner_size, c.error_bound = self.block_bits, self.inner_size, self.error_bound
        c.memory_budget, c.workers, c.compress = self.memory_budget, self.workers, int(self.compress)
        c.verify_cap_qubits, c.device = self.verify_cap_qubits, self.device
        c.device_pool_bytes, c.work_bytes = self.device_pool_bytes, self.work_bytes
        c.host_pool_bytes = self.host_pool_bytes
        c.disk_pool_bytes = self.disk_pool_bytes
        self._disk_dir_c = self.disk_dir.encode() if self.disk_dir else None  # kept alive with the config
        c.disk_dir = self._disk_dir_c
        c.flags = (_lib.BMQ_FLAG_ZERO_GROUP_SKIP if self.zero_group_skip else 0) | \
                  (_lib.BMQ_FLAG_IDENTITY_SKIP if self.identity_skip else 0) | \
                  (_lib.BMQ_FLAG_CODE_DOMAIN if self.code_domain else 0) | \
                  (_lib.BMQ_FLAG_POOL_GROW if self.pool_grow else 0) | \
                  (_lib.BMQ_FLAG_DEVICE_PLAN if self.device_plan else 0) | \
                  (_lib.BMQ_FLAG_STAGE_FUSION if self.fuse_stages else 0) | \
                  {"auto": 0, "heap": _lib.BMQ_FLAG_HEAP_ARENA, "bump": _lib.BMQ_FLAG_BUMP_ARENA}[self.arena]
        return c


class Collective:
    """One rank's collective of a sharded run (bmq_collective): NCCL (one
    process per GPU) or in-process (one thread per rank, any devices)."""

    def __init__(self, handle):
        self._h = handle

    @staticmethod
    def local(world: int) -> list:
        hs = (C.c_void_p * world)()
        _check(lib.bmq_collective_local_create(world, hs))
        return [Collective(C.c_void_p(h)) for h in hs]

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib.bmq_nccl_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl(uid: bytes, rank: int, world: int, device: int = 0) -> "Collective":
        h = C.c_void_p()
        _check(lib.bmq_collective_nccl_create((C.c_uint8 * 128).from_buffer_copy(uid), rank, world, device,
                                              C.byref(h)))
        return Collective(h)

    def close(self):
        if self._h:
            lib.bmq_collective_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class SimulationReport:
    """cbq::SimulationReport (engine.hpp:39-53) plus device counters."""
    qubits: int = 0
    gate_count: int = 0
    stage_count: int = 0
    max_footprint_bytes: int = 0
    standard_bytes: float = 0.0
    compression_ratio: float = 0.0
    spilled_blocks: int = 0
    wall_ms: float = 0.0
    stage_ms: list = field(default_factory=list)
    fidelity: float | None = None
    final_norm: float = 0.0
    stage_compress_calls: int = 0
    stage_decompress_calls: int = 0
    device: dict = field(default_factory=dict)


DEVICE_REPORT_KEYS = ("device_ms", "groups_processed", "groups_skipped", "blocks_processed",
                      "payload_bytes_read", "payload_bytes_written", "dense_bytes", "kernel_launches",
                      "device_peak_bytes", "gate_passes", "decompress_ms", "gate_ms", "compress_ms", "batches",
                      "decompress_bytes", "gate_bytes", "compress_bytes", "fused_batches", "compactions",
                      "host_spill_bytes", "host_spill_batches", "code_domain_batches", "pool_growths",
                      "lazy_cx", "perm_materialisations",
                      "model_bytes", "model_groups", "link_h2d_bytes", "link_d2h_bytes", "link_ms",
                      "compact_bytes", "host_peak_bytes", "arena_bytes", "fused_decode_batches", "stream_passes",
                      "disk_spill_bytes", "disk_read_bytes", "disk_peak_bytes", "disk_gds",
                      "fused_stages", "fused_sets")


def report_from_c(r: bmq_report, stage_ms: list) -> SimulationReport:
    dev = {k: getattr(r, k) for k in DEVICE_REPORT_KEYS}
    return SimulationReport(r.qubits, r.gate_count, r.stage_count, r.max_footprint_bytes, r.standard_bytes,
                            r.compression_ratio, r.spilled_blocks, r.wall_ms, stage_ms,
                            r.fidelity if r.has_fidelity else None, r.final_norm, r.stage_compress_calls,
                            r.stage_decompress_calls, dev)


class Simulator:
    """cbq::Simulator (engine.hpp:58-250) running on one B200."""

    def __init__(self, circuit: Circuit, config: Config):
        self.circuit = circuit
        self.config = config
        self._h = C.c_void_p()
        self._cfg = config.to_c()
        _check(lib.bmq_simulator_create(circuit.num_qubits, circuit.c_array(), len(circuit.gates),
                                        C.byref(self._cfg), C.byref(self._h)))
        self._layout = make_layout(circuit.num_qubits, config.block_bits)

    def close(self):
        if self._h:
            lib.bmq_simulator_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def layout(self) -> Layout:
        return self._layout

    def plan(self) -> PartitionPlan:
        cnt = C.c_uint64()
        cap = max(1, len(self.circuit.gates))
        out = (bmq_stage * cap)()
        _check(lib.bmq_simulator_plan(self._h, out, cap, C.byref(cnt)))
        return PartitionPlan(self._layout, self.config.inner_size, [Stage.from_c(out[i]) for i in range(cnt.value)])

    def init_state(self) -> None:
        _check(lib.bmq_simulator_init_state(self._h))

    def run(self) -> SimulationReport:
        r = bmq_report()
        nst = max(1, len(self.circuit.gates))
        stage_ms = np.zeros(nst)
        _check(lib.bmq_simulator_run(self._h, C.byref(r), _ptr(stage_ms), nst))
        return report_from_c(r, stage_ms[: r.stage_count].tolist())

    def run_sharded(self, col: "Collective") -> SimulationReport:
        """Simulator::run as one rank of a sharded run (bmq_simulator_run_sharded,
        SURVEY §8e): every rank calls it with its own simulator of the same
        circuit and config; the report's norm and counters are global."""
        r = bmq_report()
        nst = max(1, len(self.circuit.gates))
        stage_ms = np.zeros(nst)
        _check(lib.bmq_simulator_run_sharded(self._h, col._h, C.byref(r), _ptr(stage_ms), nst))
        return report_from_c(r, stage_ms[: r.stage_count].tolist())

    def reset(self) -> None:
        """Drop the state; the next run() starts from |0...0> again."""
        _check(lib.bmq_simulator_reset(self._h))

    def run_stages(self, first: int, last: int) -> None:
        _check(lib.bmq_simulator_run_stages(self._h, first, last))

    def report(self) -> SimulationReport:
        """Report of the stages run so far (final_norm taken now; wall/device time 0)."""
        r = bmq_report()
        _check(lib.bmq_simulator_report(self._h, C.byref(r)))
        r.final_norm = self.state_norm()
        return report_from_c(r, [])

    def save(self, path: str) -> None:
        """Checkpoint: payloads, block sums, store accounting and the stage cursor."""
        _check(lib.bmq_simulator_save(self._h, os.fsencode(path)))

    def load(self, path: str) -> int:
        """Resume from save(); returns the next stage to run."""
        nxt = C.c_uint64()
        _check(lib.bmq_simulator_load(self._h, os.fsencode(path), C.byref(nxt)))
        return nxt.value

    def state_norm(self) -> float:
        out = C.c_double()
        _check(lib.bmq_simulator_state_norm(self._h, C.byref(out)))
        return out.value

    def extract_state(self) -> np.ndarray:
        n = self.circuit.num_qubits
        if n > self.config.verify_cap_qubits:
            raise EngineError(f"dense verification refused: {n} qubits exceeds the cap of "
                              f"{self.config.verify_cap_qubits}")
        out = np.zeros(1 << n, dtype=np.complex128)
        _check(lib.bmq_simulator_extract_state(self._h, _ptr(out), out.size))
        return out

    def amplitude(self, index: int) -> complex:
        re, im = C.c_double(), C.c_double()
        _check(lib.bmq_simulator_amplitude(self._h, index, C.byref(re), C.byref(im)))
        return complex(re.value, im.value)

    def sample(self, shots: int, seed: int = 1) -> np.ndarray:
        """Basis-state indices drawn from |a_i|^2 of the stored state
        (bmq_simulator_sample), deterministic for a seed."""
        out = np.empty(max(1, shots), dtype=np.uint64)
        _check(lib.bmq_simulator_sample(self._h, shots, seed, _ptr(out)))
        return out[:shots]

    def top_k(self, k: int):
        """(indices, amplitudes) of the k largest |a|^2, largest first, ties to
        the lower index (bmq_simulator_top_k)."""
        idx = np.empty(max(1, k), dtype=np.uint64)
        re = np.empty(max(1, k))
        im = np.empty(max(1, k))
        n = C.c_uint64()
        _check(lib.bmq_simulator_top_k(self._h, k, _ptr(idx), _ptr(re), _ptr(im), C.byref(n)))
        m = n.value
        return idx[:m], re[:m] + 1j * im[:m]

    def get_payload(self, block_id: int) -> bytes:
        size = C.c_uint64()
        _check(lib.bmq_simulator_get_payload(self._h, block_id, None, 0, C.byref(size)))
        buf = np.empty(max(1, size.value), dtype=np.uint8)
        _check(lib.bmq_simulator_get_payload(self._h, block_id, _ptr(buf), size.value, C.byref(size)))
        return buf[: size.value].tobytes()

    def payloads(self) -> list:
        """Every block's payload in id order (store().get for all ids)."""
        nblk = self._layout.num_blocks()
        sizes = np.zeros(nblk, dtype=np.uint64)
        total = C.c_uint64()
        _check(lib.bmq_simulator_get_payloads(self._h, None, 0, _ptr(sizes), C.byref(total)))
        buf = np.empty(max(1, total.value), dtype=np.uint8)
        _check(lib.bmq_simulator_get_payloads(self._h, _ptr(buf), total.value, _ptr(sizes), C.byref(total)))
        raw = buf[: total.value].tobytes()
        out, off = [], 0
        for s in sizes.tolist():
            out.append(raw[off: off + s])
            off += s
        return out

    def put_payload(self, block_id: int, payload: bytes) -> None:
        data = np.frombuffer(bytes(payload) + b"\0", dtype=np.uint8)
        _check(lib.bmq_simulator_put_payload(self._h, block_id, _ptr(data), len(payload)))

    def fidelity_dense(self, ideal: np.ndarray) -> float:
        a = np.ascontiguousarray(ideal, dtype=np.complex128)
        out = C.c_double()
        _check(lib.bmq_simulator_fidelity_dense(self._h, _ptr(a), a.size, C.byref(out)))
        return out.value

    def fidelity_with(self, other: "Simulator") -> float:
        out = C.c_double()
        _check(lib.bmq_simulator_fidelity(self._h, other._h, C.byref(out)))
        return out.value

    def fidelity_analytic(self, kind: str) -> float:
        out = C.c_double()
        _check(lib.bmq_simulator_fidelity_analytic(self._h, {"uniform": 0, "ghz": 1}[kind], C.byref(out)))
        return out.value


def dense_reference(circuit: Circuit, verify_cap_qubits: int = 24) -> np.ndarray:
    """dense_reference (engine.hpp:254-296) on the GPU."""
    n = circuit.num_qubits
    if n > verify_cap_qubits:
        raise EngineError(f"dense reference refused: {n} qubits exceeds the cap of {verify_cap_qubits}")
    out = np.zeros(1 << n, dtype=np.complex128)
    _check(lib.bmq_dense_reference(n, circuit.c_array(), len(circuit.gates), _ptr(out), verify_cap_qubits))
    return out


def fidelity(a: np.ndarray, b: np.ndarray) -> float:
    """fidelity (engine.hpp:299-308): |<a|b>|, unnormalised."""
    if len(a) != len(b):
        raise InvalidArgument("fidelity requires equal-length states")
    return float(abs(np.vdot(a, b)))
