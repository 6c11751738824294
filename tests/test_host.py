"""Host-side checks of libbmq (no GPU needed): the C ABI loads and exports
every symbol include/bmq.h declares, and the host descriptor logic
(benchmarks, unitaries, partition, groups, buffer bits, validation) matches
the pinned oracle exactly."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "bmq.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(bmq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(cbq):
    from paper_2410_14088_b200 import _lib
    declared = declared_symbols()
    assert len(declared) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (bmq_\w+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), "ctypes table and header disagree"


def test_library_is_sm100a(cbq):
    from paper_2410_14088_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_bounds(cbq):
    assert b"sm_100a" in cbq.lib.bmq_version()
    assert cbq.ErrorBound(1e-3).log2_abs == 0.0014419741739063218
    assert cbq.ErrorBound(1.0).log2_abs == 1.0
    with pytest.raises(cbq.InvalidArgument, match="positive and finite"):
        cbq.ErrorBound(0.0)


@pytest.mark.parametrize("name", ["ghz", "cat_state", "bv", "qft", "qaoa"])
def test_benchmarks_match_oracle(cbq, port, name):
    for n in (2, 5, 13, 34):
        c = cbq.generate_benchmark(name, n, cbq.BenchmarkParams(layers=3, seed=9))
        assert [g.as_tuple() for g in c.gates] == [tuple(x) for x in port.generate_benchmark(name, n, 3, 9)]


def test_benchmark_errors(cbq):
    with pytest.raises(cbq.InvalidArgument, match="unknown benchmark"):
        cbq.generate_benchmark("nope", 4)
    with pytest.raises(cbq.InvalidArgument, match="at least 2 qubits"):
        cbq.generate_benchmark("qft", 1)
    with pytest.raises(cbq.InvalidArgument, match="only '0' and '1'"):
        cbq.generate_benchmark("bv", 4, cbq.BenchmarkParams(secret="012"))


def test_unitaries_bit_identical(cbq, port):
    rng = np.random.default_rng(0)
    for kind in cbq.GateKind:
        for _ in range(5):
            ang = float(rng.uniform(-7, 7))
            g = cbq.Gate(kind, 0, 1 if cbq.is_two_qubit(kind) else 0, ang if cbq.is_parameterized(kind) else 0.0)
            a = cbq._unitary(g)
            b = port.unitary(g.as_tuple())
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), kind
    with pytest.raises(cbq.LogicError):
        cbq.unitary2(cbq.gates.cx(0, 1))


def random_circuit(rng, n, count):
    gl = []
    for _ in range(count):
        k = int(rng.integers(15))
        q0 = int(rng.integers(n))
        q1 = int((q0 + 1 + rng.integers(n - 1)) % n)
        gl.append((k, q0, q1 if k >= 12 else 0, float(rng.uniform(0, 6.28)) if k in (8, 9, 10, 11, 14) else 0.0))
    return gl


def to_circuit(cbq, n, gl):
    return cbq.Circuit(n, [cbq.Gate(cbq.GateKind(k), a, b, ang) for k, a, b, ang in gl])


def test_partition_and_groups_match_oracle(cbq, port):
    rng = np.random.default_rng(11)
    for t in range(60):
        n = 3 + t % 12
        gl = random_circuit(rng, n, 1 + int(rng.integers(80)))
        b = 1 + int(rng.integers(n))
        inner = int(rng.integers(5))
        c = to_circuit(cbq, n, gl)
        plan = cbq.partition_circuit(c, b, inner)
        assert [(s.gate_begin, s.gate_end, s.inner) for s in plan.stages] == port.partition(n, gl, b, inner)
        L = cbq.make_layout(n, b)
        for s in plan.stages:
            ids = [g.block_ids for g in cbq.enumerate_groups(s, L)]
            assert ids == port.enumerate_groups(n, b, (s.gate_begin, s.gate_end, s.inner)).tolist()
            for q in range(n):
                st = (s.gate_begin, s.gate_end, s.inner)
                try:
                    want = port.buffer_bit_of_qubit(n, b, st, q)
                except Exception:
                    with pytest.raises(cbq.LogicError, match="outer index"):
                        cbq.buffer_bit_of_qubit(s, L, q)
                else:
                    assert cbq.buffer_bit_of_qubit(s, L, q) == want


def test_qft34_plans(cbq):
    c = cbq.generate_benchmark("qft", 34)
    assert len(c.gates) == 646
    want = {(14, 2): 200, (14, 6): 43, (17, 4): 54, (20, 2): 98, (20, 4): 37, (20, 6): 21, (24, 6): 10}
    for (b, i), stages in want.items():
        assert len(cbq.partition_circuit(c, b, i).stages) == stages


def test_validation_messages(cbq):
    with pytest.raises(cbq.InvalidArgument, match=r"qubit count must be in \[1, 62\], got 0"):
        cbq.Circuit(0)
    c = cbq.Circuit(3)
    with pytest.raises(cbq.InvalidArgument, match="gate operand 3 out of range for 3 qubits"):
        c.add(cbq.gates.h(3))
    with pytest.raises(cbq.InvalidArgument, match="operands must be distinct"):
        c.add(cbq.gates.cx(1, 1))
    with pytest.raises(cbq.InvalidArgument, match=r"local index bits must be in \[1, n\]"):
        cbq.make_layout(4, 5)
    with pytest.raises(cbq.InvalidArgument, match="outside the global index range"):
        cbq.enumerate_groups(cbq.Stage(0, 0, [1]), cbq.make_layout(6, 2))


def test_cpp_dropin_header(cbq, tmp_path):
    """include/bmq/cbq.hpp compiles like the reference headers and agrees with them."""
    from paper_2410_14088_b200 import _lib
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = tmp_path / "dropin"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", f"{ROOT}/tests/cpp/dropin_host.cpp",
                    f"-L{libdir}", "-lbmq", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines()
    assert "qft34_gates 646" in out
    assert "stages 14 2 200" in out and "stages 20 2 98" in out and "stages 20 6 21" in out
    assert "group0 0 2 8 10" in out
    assert "h00 0.70710678118654746" in out
    assert "invalid_argument two-qubit gate operands must be distinct" in out
    assert "logic_error qubit 4 is an outer index for this stage" in out


def test_no_cpu_fallback_without_device(cbq):
    if cbq.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(cbq.NoDeviceError):
        cbq.compress_block(np.ones(8), 1e-3)
    with pytest.raises(cbq.NoDeviceError):
        cbq.Simulator(cbq.generate_benchmark("ghz", 4), cbq.Config(block_bits=2))


def test_host_level_extent_heap(tmp_path):
    """ExtentHeap (csrc/store.hpp), the pinned host level's allocator: random
    alloc / free sequences against a brute-force model (no overlap, best fit,
    coalesced free list, double frees rejected without damage, full
    coalescing at the end). Built with g++ from the product source."""
    exe = tmp_path / "eht"
    csrc = os.path.join(ROOT, "paper_2410_14088_b200", "csrc")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"-I{csrc}",
                    os.path.join(ROOT, "tests", "cpp", "extent_heap_test.cpp"), os.path.join(csrc, "store_host.cpp"),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "extent_heap ok" in out.stdout


@pytest.mark.parametrize("name,n,layers,b", [("qft", 34, 1, 20), ("qaoa3reg", 34, 4, 20), ("random", 30, 20, 14),
                                             ("ghz", 30, 1, 20)])
def test_device_aware_plan(cbq, name, n, layers, b):
    """plan_device_aware returns partition_circuit's plan at
    the inner size whose modelled time is least, never beyond the work
    budget (2^(b+k) complex doubles) or the outer bits the shards need."""
    c = cbq.generate_benchmark(name, n, cbq.BenchmarkParams(layers=layers, seed=1))
    for world, work in ((1, 16 << 30), (8, 16 << 30), (1, 16 << (b + 3))):
        plan, ch = cbq.plan_device_aware(c, b, world=world, work_bytes=work)
        k = ch.inner_size
        assert plan.stages == cbq.partition_circuit(c, b, k).stages
        assert ch.stages == len(plan.stages) and ch.model_s == min(ch.candidates.values())
        assert ch.model_s == ch.candidates[k]
        assert (16 << (b + k)) <= work or k == 2
        assert k <= (n - b) - (world.bit_length() - 1)
        assert all(len(s.inner) <= k for s in plan.stages)
        assert world > 1 or ch.remaps == 0
    default = cbq.partition_circuit(c, b, 2)
    plan, ch = cbq.plan_device_aware(c, b)
    assert len(plan.stages) <= len(default.stages)


def test_device_aware_plan_errors(cbq):
    c = cbq.generate_benchmark("qft", 12)
    with pytest.raises(cbq.InvalidArgument, match="power of two"):
        cbq.plan_device_aware(c, 6, world=3)
    with pytest.raises(cbq.InvalidArgument, match="positive"):
        cbq.plan_device_aware(c, 6, hbm_gbs=0.0)
    plan, ch = cbq.plan_device_aware(c, 6, max_inner=3)
    assert ch.inner_size <= 3
