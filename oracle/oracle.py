"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes front-end over the two CPU checkers built by oracle/Makefile:

* ``port()`` — the plain-C restatement ``oracle/_build/libcbq_oracle.so``
  (oracle/cbq_oracle.c), always buildable;
* ``ref()``  — the unmodified reference headers compiled where they lie,
  ``oracle/_ref/libcbqref.so`` (oracle/ref_shim.cpp), present in this container
  and shipped prebuilt to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package never
does (it fails loudly without its CUDA extension instead).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libcbq_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcbqref.so")

GATE_KINDS = ["h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "p", "cx", "cz", "cp"]
TWO_QUBIT = {12, 13, 14}


class Gate(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("q0", C.c_uint32), ("q1", C.c_uint32), ("pad", C.c_uint32),
                ("angle", C.c_double)]


class Stage(C.Structure):
    _fields_ = [("gate_begin", C.c_uint64), ("gate_end", C.c_uint64), ("inner_count", C.c_uint32),
                ("pad", C.c_uint32), ("inner", C.c_uint32 * 64)]


class Report(C.Structure):
    _fields_ = [("qubits", C.c_uint64), ("gate_count", C.c_uint64), ("stage_count", C.c_uint64),
                ("max_footprint_bytes", C.c_uint64), ("standard_bytes", C.c_double),
                ("compression_ratio", C.c_double), ("spilled_blocks", C.c_uint64),
                ("wall_ms", C.c_double), ("has_fidelity", C.c_int32), ("pad", C.c_int32),
                ("fidelity", C.c_double), ("final_norm", C.c_double),
                ("stage_compress_calls", C.c_uint64), ("stage_decompress_calls", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "pad"}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def fnv1a64(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    arr = np.frombuffer(data, dtype=np.uint8)
    for b in arr.tolist():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def gates_array(gates):
    """gates: list of (kind, q0, q1, angle) with kind a name or an int."""
    arr = (Gate * max(1, len(gates)))()
    for i, g in enumerate(gates):
        k = g[0] if isinstance(g[0], int) else GATE_KINDS.index(g[0])
        arr[i] = Gate(k, g[1], g[2] if k in TWO_QUBIT else 0, 0, g[3] if len(g) > 3 else 0.0)
    return arr


def gates_to_list(arr, count):
    return [(arr[i].kind, arr[i].q0, arr[i].q1, arr[i].angle) for i in range(count)]


def stage_struct(begin, end, inner):
    st = Stage()
    st.gate_begin, st.gate_end, st.inner_count = begin, end, len(inner)
    for i, q in enumerate(inner):
        st.inner[i] = q
    return st


@dataclass
class SimResult:
    report: dict
    payloads: list
    state: np.ndarray | None


class _Lib:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.path = path
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self._f("last_error")().decode())

    def log2_abs(self, b_r):
        out = C.c_double()
        self._check(self._f("log2_abs")(C.c_double(b_r), C.byref(out)))
        return out.value

    def compress_block(self, scalars, b_r) -> bytes:
        s = np.ascontiguousarray(scalars, dtype=np.float64)
        cap = 64 + 2 * (len(s) // 8 + 1024) + 8 * len(s)
        out = (C.c_uint8 * cap)()
        size = C.c_uint64()
        self._check(self._f("compress_block")(s.ctypes.data_as(C.c_void_p), C.c_uint64(len(s)),
                                              C.c_double(b_r), out, C.c_uint64(cap), C.byref(size)))
        return bytes(out[: size.value])

    def decompress_block(self, payload: bytes) -> np.ndarray:
        p = (C.c_uint8 * max(1, len(payload))).from_buffer_copy(payload or b"\0")
        cnt = C.c_uint64()
        out = np.zeros(16, dtype=np.float64)
        rc = self._f("decompress_block")(p, C.c_uint64(len(payload)), out.ctypes.data_as(C.c_void_p),
                                         C.c_uint64(0), C.byref(cnt))
        if rc == 10:
            out = np.zeros(max(1, cnt.value), dtype=np.float64)
            rc = self._f("decompress_block")(p, C.c_uint64(len(payload)), out.ctypes.data_as(C.c_void_p),
                                             C.c_uint64(cnt.value), C.byref(cnt))
        elif rc == 0:
            return out[: cnt.value].copy()
        self._check(rc)
        return out[: cnt.value].copy()

    def prescan_encode(self, words, bit_count) -> bytes:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        if len(w) == 0:
            w = np.zeros(1, dtype=np.uint64)
        cap = 1024 + bit_count // 4
        out = (C.c_uint8 * cap)()
        size = C.c_uint64()
        self._check(self._f("prescan_encode")(w.ctypes.data_as(C.c_void_p), C.c_uint64(bit_count), out,
                                              C.c_uint64(cap), C.byref(size)))
        return bytes(out[: size.value])

    def unitary(self, gate):
        g = gates_array([gate])
        out = np.zeros(32, dtype=np.float64)
        self._check(self._f("unitary")(C.byref(g[0]), out.ctypes.data_as(C.c_void_p)))
        m = 4 if g[0].kind in TWO_QUBIT else 2
        return (out[0::2] + 1j * out[1::2])[: m * m].reshape(m, m)

    def generate_benchmark(self, name, n, layers=1, seed=1, secret=None):
        cap = 8 * n * n + 16 * n * layers + 64
        arr = (Gate * cap)()
        cnt = C.c_uint64()
        self._check(self._f("generate_benchmark")(name.encode(), C.c_uint32(n), C.c_uint32(layers),
                                                  C.c_uint64(seed), (secret or "").encode(), arr,
                                                  C.c_uint64(cap), C.byref(cnt)))
        return gates_to_list(arr, cnt.value)

    def partition(self, n, gates, block_bits, inner_size):
        arr = gates_array(gates)
        cap = max(1, len(gates))
        out = (Stage * cap)()
        ns = C.c_uint64()
        self._check(self._f("partition")(C.c_uint32(n), arr, C.c_uint64(len(gates)), C.c_uint32(block_bits),
                                         C.c_uint32(inner_size), out, C.c_uint64(cap), C.byref(ns)))
        return [(out[i].gate_begin, out[i].gate_end, list(out[i].inner[: out[i].inner_count]))
                for i in range(ns.value)]

    def enumerate_groups(self, n, block_bits, stage):
        st = stage_struct(*stage)
        cap = 1 << (n - block_bits)
        ids = np.zeros(cap, dtype=np.uint64)
        cnt = C.c_uint64()
        self._check(self._f("enumerate_groups")(C.c_uint32(n), C.c_uint32(block_bits), C.byref(st),
                                                ids.ctypes.data_as(C.c_void_p), C.c_uint64(cap),
                                                C.byref(cnt)))
        per = 1 << len(stage[2])
        return ids[: cnt.value].reshape(-1, per)

    def buffer_bit_of_qubit(self, n, block_bits, stage, q):
        st = stage_struct(*stage)
        out = C.c_uint32()
        self._check(self._f("buffer_bit_of_qubit")(C.c_uint32(n), C.c_uint32(block_bits), C.byref(st),
                                                   C.c_uint32(q), C.byref(out)))
        return out.value

    def apply_gate(self, amps, u, hi_bit, lo_bit=0):
        a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
        um = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(-1))
        ud = np.empty(2 * len(um))
        ud[0::2], ud[1::2] = um.real, um.imag
        self._check(self._f("apply_gate")(a.ctypes.data_as(C.c_void_p), C.c_uint64(len(a)),
                                          ud.ctypes.data_as(C.c_void_p), C.c_int(len(um) == 16),
                                          C.c_uint32(hi_bit), C.c_uint32(lo_bit)))
        return a

    def apply_stage(self, amps, n, gates, stage, block_bits):
        a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
        arr = gates_array(gates)
        st = stage_struct(*stage)
        self._check(self._f("apply_stage")(a.ctypes.data_as(C.c_void_p), C.c_uint64(len(a)), C.c_uint32(n),
                                           arr, C.c_uint64(len(gates)), C.byref(st),
                                           C.c_uint32(block_bits)))
        return a

    def dense_reference(self, n, gates):
        out = np.zeros(1 << n, dtype=np.complex128)
        arr = gates_array(gates)
        self._check(self._f("dense_reference")(C.c_uint32(n), arr, C.c_uint64(len(gates)),
                                               out.ctypes.data_as(C.c_void_p)))
        return out

    def fidelity(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.complex128)
        b = np.ascontiguousarray(b, dtype=np.complex128)
        out = C.c_double()
        self._check(self._f("fidelity")(a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                        C.c_uint64(len(a)), C.byref(out)))
        return out.value


class Port(_Lib):
    prefix = "cbqo_"

    def simulate(self, n, gates, block_bits, inner_size=2, error_bound=1e-3, memory_budget=2**64 - 1,
                 compress=True, want_payloads=True, want_state=False):
        arr = gates_array(gates)
        rep = Report()
        nblk = 1 << (n - block_bits)
        sizes = np.zeros(nblk, dtype=np.uint64)
        state = np.zeros(1 << n, dtype=np.complex128) if want_state else None
        self._check(self._f("simulate")(C.c_uint32(n), arr, C.c_uint64(len(gates)), C.c_uint32(block_bits),
                                        C.c_uint32(inner_size), C.c_double(error_bound),
                                        C.c_uint64(memory_budget), C.c_int(int(compress)), C.byref(rep),
                                        None, C.c_uint64(0), sizes.ctypes.data_as(C.c_void_p),
                                        state.ctypes.data_as(C.c_void_p) if want_state else None))
        payloads = []
        if want_payloads:
            total = int(sizes.sum())
            buf = (C.c_uint8 * max(1, total))()
            self._check(self._f("simulate")(C.c_uint32(n), arr, C.c_uint64(len(gates)), C.c_uint32(block_bits),
                                            C.c_uint32(inner_size), C.c_double(error_bound),
                                            C.c_uint64(memory_budget), C.c_int(int(compress)), C.byref(rep),
                                            buf, C.c_uint64(total), sizes.ctypes.data_as(C.c_void_p), None))
            raw = bytes(buf[:total])
            off = 0
            for s in sizes.tolist():
                payloads.append(raw[off: off + s])
                off += s
        return SimResult(rep.as_dict(), payloads, state)


class Ref(_Lib):
    prefix = "cbqref_"

    def simulate(self, n, gates, block_bits, inner_size=2, error_bound=1e-3, memory_budget=2**64 - 1,
                 compress=True, workers=1, want_payloads=True, want_state=False, with_fidelity=False,
                 spill_dir=None):
        arr = gates_array(gates)
        rep = Report()
        nblk = 1 << (n - block_bits)
        sizes = np.zeros(nblk, dtype=np.uint64)
        state = np.zeros(1 << n, dtype=np.complex128) if want_state else None

        def call(buf, cap, st):
            nst = 4096
            stage_ms = np.zeros(nst)
            self._check(self._f("simulate")(
                C.c_uint32(n), arr, C.c_uint64(len(gates)), C.c_uint32(block_bits), C.c_uint32(inner_size),
                C.c_double(error_bound), C.c_uint64(memory_budget), C.c_uint32(workers), C.c_int(int(compress)),
                (spill_dir or "").encode(), C.byref(rep), stage_ms.ctypes.data_as(C.c_void_p), C.c_uint64(nst),
                buf, C.c_uint64(cap), sizes.ctypes.data_as(C.c_void_p),
                st.ctypes.data_as(C.c_void_p) if st is not None else None, C.c_int(int(with_fidelity))))
            return stage_ms

        stage_ms = call(None, 0, state)
        payloads = []
        if want_payloads:
            total = int(sizes.sum())
            buf = (C.c_uint8 * max(1, total))()
            call(buf, total, None)
            raw = bytes(buf[:total])
            off = 0
            for s in sizes.tolist():
                payloads.append(raw[off: off + s])
                off += s
        d = rep.as_dict()
        d["stage_ms"] = stage_ms[: d["stage_count"]].tolist()
        return SimResult(d, payloads, state)

    def group_pipeline(self, n, gates, stage, block_bits, error_bound, workers, group_ids, payloads):
        """Time the reference per-group pipeline (engine.hpp:203-225) on given groups."""
        arr = gates_array(gates)
        st = stage_struct(*stage)
        ids = np.ascontiguousarray(group_ids, dtype=np.uint64).reshape(-1)
        sizes = np.array([len(p) for p in payloads], dtype=np.uint64)
        offs = np.zeros_like(sizes)
        if len(sizes) > 1:
            offs[1:] = np.cumsum(sizes)[:-1]
        blob = b"".join(payloads)
        buf = (C.c_uint8 * max(1, len(blob))).from_buffer_copy(blob or b"\0")
        wall = C.c_double()
        outb = C.c_uint64()
        per = 1 << len(stage[2])
        self._check(self._f("group_pipeline")(
            C.c_uint32(n), arr, C.c_uint64(len(gates)), C.byref(st), C.c_uint32(block_bits),
            C.c_double(error_bound), C.c_uint32(workers), ids.ctypes.data_as(C.c_void_p),
            C.c_uint64(len(ids) // per), buf, offs.ctypes.data_as(C.c_void_p), sizes.ctypes.data_as(C.c_void_p),
            C.byref(wall), C.byref(outb)))
        return wall.value, outb.value

    def stage_groups(self, n, gates, stages, block_bits, error_bound, workers, samples):
        """Time the reference per-group pipeline on groups of several stages at
        once. samples: list of (stage index, block ids of one group, payloads).
        Returns (per-group thread ms, wall ms of the parallel region)."""
        arr = gates_array(gates)
        st = (Stage * len(stages))(*[stage_struct(*x) for x in stages])
        gstage = np.array([s for s, _, _ in samples], dtype=np.uint64)
        ids = np.concatenate([np.asarray(i, dtype=np.uint64).reshape(-1) for _, i, _ in samples])
        first = np.zeros(len(samples), dtype=np.uint64)
        first[1:] = np.cumsum([len(i) for _, i, _ in samples])[:-1]
        pays = [p for _, _, ps in samples for p in ps]
        sizes = np.array([len(p) for p in pays], dtype=np.uint64)
        offs = np.zeros_like(sizes)
        offs[1:] = np.cumsum(sizes)[:-1]
        blob = b"".join(pays)
        buf = (C.c_uint8 * max(1, len(blob))).from_buffer_copy(blob or b"\0")
        gms = np.zeros(len(samples))
        wall = C.c_double()
        vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self._f("stage_groups")(
            C.c_uint32(n), arr, C.c_uint64(len(gates)), st, C.c_uint64(len(stages)), C.c_uint32(block_bits),
            C.c_double(error_bound), C.c_uint32(workers), vp(gstage), vp(first), C.c_uint64(len(samples)),
            vp(ids), buf, vp(offs), vp(sizes), vp(gms), C.byref(wall)))
        return gms, wall.value


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build()
        _port = Port(PORT_SO)
    return _port


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref(REF_SO)
    return _ref


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref_parse_qasm(text: str):
    """Reference parse_qasm through oracle/_ref: (num_qubits, gates, n_warnings) or raises OracleError."""
    r = ref()
    cap = 1 << 16
    arr = (Gate * cap)()
    nq, cnt, nw = C.c_uint32(), C.c_uint64(), C.c_uint64()
    r._check(r._f("parse_qasm")(text.encode(), C.byref(nq), arr, C.c_uint64(cap), C.byref(cnt), C.byref(nw)))
    return nq.value, gates_to_list(arr, cnt.value), nw.value


def ref_emit_qasm(n: int, gates) -> str:
    r = ref()
    arr = gates_array(gates)
    cap = 64 * (len(gates) + 8)
    buf = C.create_string_buffer(cap)
    size = C.c_uint64()
    r._check(r._f("emit_qasm")(C.c_uint32(n), arr, C.c_uint64(len(gates)), buf, C.c_uint64(cap), C.byref(size)))
    return buf.value.decode()
