"""QASM loader of the drop-in surface (qasm.hpp) against the reference
parser compiled from /root/reference (oracle/_ref): same circuits, same
warnings, same "line L, col C" error messages, exact emit round trip."""
import pytest

PROGRAMS = [
    'OPENQASM 2.0;\ninclude "qelib1.inc";\nqreg q[3];\nh q[0];\ncx q[0],q[1];\n',
    "qreg r[4];\nu1(pi/4) r[1];\ncu1(-pi/2 + 0.25*pi) r[1],r[3];\nCX r[0],r[2];\nswap r[3],r[0];\n",
    "qreg q[2]; creg c[2]; rz(2*(pi - 1e-3)) q[1]; barrier q; measure q[0] -> c[0]; measure q[1] -> c[1];",
    "// only a comment\nqreg q[1];\nrx(-(1.5e-2)) q[0]; ry(+3) q[0]; p(1/3) q[0]; t q[0]; tdg q[0]; s q[0]; sdg q[0];",
    "qreg q[62]; y q[61]; z q[0]; cz q[5],q[60]; cp(.5) q[1],q[2];",
    "qreg q[2]; rx(1e) q[0]; ry(2.5E-1) q[1];",  # std::stod accepts the "1e" prefix, like the reference
]

BAD = [
    "qreg q[3]; h q[3];", "h q[0];", "qreg q[2]; foo q[0];", "qreg q[2]; rx q[0];", "qreg q[2];\n cx q[0],q[0];",
    "qreg q[2]; rx(1/0) q[0];", "qreg q[2]; h q[0] $", "qreg q[2]; qreg r[2];", "qreg q[63];", "qreg q[2]; h(1) q[0];",
    "qreg q[2]; cx q[0];", "qreg q[2]; h r[0];", 'include "x.inc', "qreg q[1.5];", "qreg q[2]; h q[0]", "", "OPENQASM;",
]


@pytest.mark.parametrize("text", PROGRAMS)
def test_parse_matches_reference(cbq, ref, text):
    from oracle import oracle
    warnings = []
    c = cbq.parse_qasm(text, warnings)
    n, gl, nw = oracle.ref_parse_qasm(text)
    assert c.num_qubits == n
    assert [g.as_tuple() for g in c.gates] == [tuple(g) for g in gl]
    assert len(warnings) == nw


@pytest.mark.parametrize("text", BAD)
def test_errors_match_reference(cbq, ref, text):
    from oracle import oracle
    with pytest.raises(oracle.OracleError) as want:
        oracle.ref_parse_qasm(text)
    with pytest.raises(cbq.QasmError) as got:
        cbq.parse_qasm(text)
    assert str(got.value) == str(want.value)
    assert got.value.line >= 1 and got.value.col >= 1


@pytest.mark.parametrize("name", ["ghz", "bv", "qft", "qaoa"])
def test_emit_round_trip(cbq, ref, name):
    from oracle import oracle
    c = cbq.generate_benchmark(name, 9, cbq.BenchmarkParams(layers=2, seed=5))
    text = cbq.emit_qasm(c)
    assert text == oracle.ref_emit_qasm(9, [g.as_tuple() for g in c.gates])
    assert cbq.parse_qasm(text) == c
