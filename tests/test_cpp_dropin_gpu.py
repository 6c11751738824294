"""The C++ drop-in surface (include/bmq/cbq.hpp) on the device: a program
written against the reference's `namespace cbq` API (tests/cpp/dropin_gpu.cpp)
is compiled with g++ against the header and libbmq.so, runs Simulator::run,
the QASM loader/emitter and the kernel.hpp group-buffer functions on the B200,
and its outputs are compared with the oracle / the unmodified reference."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from test_engine_gpu import FIDELITY_ATOL, NORM_RTOL

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def fnv_bytes(payloads):
    h = 0xCBF29CE484222325
    for p in payloads:
        for c in p:
            h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.fixture(scope="module")
def dropin(tmp_path_factory, gpu):
    from paper_2410_14088_b200 import _lib
    libdir = os.path.dirname(_lib.LIB_PATH)
    d = tmp_path_factory.mktemp("dropin")
    exe = d / "dropin_gpu"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"{ROOT}/tests/cpp/dropin_gpu.cpp",
                    f"-L{libdir}", "-lbmq", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    qaoa16 = gpu.emit_qasm(gpu.generate_benchmark("qaoa3reg", 16, gpu.BenchmarkParams(layers=1, seed=1)))
    qaoa10 = gpu.emit_qasm(gpu.generate_benchmark("qaoa3reg", 10, gpu.BenchmarkParams(layers=1, seed=1)))
    blob = d / "apply_stage.bin"
    r = subprocess.run([str(exe), str(blob), qaoa16, qaoa10], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return r.stdout.splitlines(), blob


def parse_case(lines, tag):
    line = next(x for x in lines if x.startswith(tag + " "))
    f = line.split()[1:]
    return dict(zip(f[0::2], f[1::2]))


@pytest.mark.parametrize("tag,name,layers,br", [("qft16", "qft", 1, 1e-3), ("qaoa3reg16", "qaoa3reg", 1, 1e-4)])
def test_cpp_simulator_run_matches_oracle(dropin, gpu, port, tag, name, layers, br):
    lines, _ = dropin
    got = parse_case(lines, tag)
    c = gpu.generate_benchmark(name, 16, gpu.BenchmarkParams(layers=layers, seed=1))
    want = port.simulate(16, [g.as_tuple() for g in c.gates], 12, 2, br, want_state=True)
    assert int(got["stages"]) == want.report["stage_count"]
    assert int(got["peak"]) == want.report["max_footprint_bytes"] == int(got["fp_peak"])
    assert int(got["fnv"], 16) == fnv_bytes(want.payloads)
    assert float(got["norm"]) == pytest.approx(want.report["final_norm"], rel=NORM_RTOL)
    ideal = gpu.dense_reference(c)
    exact = abs(np.vdot(ideal, want.state))
    assert abs(float(got["fidelity"]) - exact) <= FIDELITY_ATOL


def test_cpp_qasm_surface(dropin, ref):
    lines, _ = dropin
    assert "qasm_roundtrip 1" in lines
    assert "qasm_warnings 1" in lines
    err = next(x for x in lines if x.startswith("qasm_error "))
    # QasmError(line, col) carries the unmodified reference parser's position and text
    from oracle import oracle
    with pytest.raises(oracle.OracleError) as e:
        oracle.ref_parse_qasm("OPENQASM 2.0;\nqreg q[2];\nh q[5];\n")
    assert err == f"qasm_error 3 5 {e.value}"


def test_cpp_apply_stage_matches_reference(dropin, gpu, ref):
    lines, blob = dropin
    assert "apply_stage_written 4" in lines  # a CX-RZ-CX stage needs both outer qubits inner: 4 blocks
    raw = open(blob, "rb").read()
    s, n_in, n_blocks, per = np.frombuffer(raw[:32], dtype=np.uint64)
    amps = np.frombuffer(raw[32: 32 + 16 * int(n_in)], dtype=np.complex128).copy()
    out = np.frombuffer(raw[32 + 16 * int(n_in):], dtype=np.complex128)
    c = gpu.generate_benchmark("qaoa3reg", 10, gpu.BenchmarkParams(layers=1, seed=1))
    gl = [g.as_tuple() for g in c.gates]
    plan = ref.partition(10, gl, 4, 1)
    want = ref.apply_stage(amps, 10, gl, plan[int(s)], 4)
    assert out.view(np.uint64).tolist() == np.asarray(want).view(np.uint64).tolist()


def test_cpp_kernel_errors(dropin):
    lines, _ = dropin
    assert "invalid_argument gate bit out of range for buffer" in lines
    assert "invalid_argument gate bits invalid for buffer" in lines
    assert "invalid_argument group block count must be a nonzero power of two" in lines
