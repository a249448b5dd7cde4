"""The `kernel` JSON protocol (reference cli.py:251-287) on the device path."""
from __future__ import annotations

import io
import json

import numpy as np
import pytest

from conftest import pairs_to_complex
from paper_2405_01250_b200 import cli


def call(monkeypatch, capsys, op, request):
    monkeypatch.setattr("sys.stdin", io.StringIO(json.dumps(request)))
    rc = cli.main(["kernel", op])
    out = capsys.readouterr()
    return rc, (json.loads(out.out) if out.out.strip() else None), out.err


def test_flat_qasm_matches_reference_lowering(kats):
    sim = kats["kernel_protocol"]["ghz4_simulate"]
    c = cli.parse_flat_qasm("OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[4];\ncreg c[4];\nh q[0];\n"
                            "cx q[0],q[1];\ncx q[1],q[2];\ncx q[2],q[3];\nmeasure q -> c;\n")
    assert c.n_qubits == sim["n_qubits"]
    assert [[o.name, list(o.qubits), list(o.params)] for o in c.ops] == sim["ops"]
    c2 = cli.parse_flat_qasm("qreg r[3]; u3(pi/2, -pi/4, 0.5*2) r[2]; rz(-0.25) r[0]; // note\nbarrier r;")
    assert c2.ops[0].params == (np.pi / 2, -np.pi / 4, 1.0) and c2.ops[1].params == (-0.25,)


def test_exit_codes_without_device(monkeypatch, capsys):
    rc, _, err = call(monkeypatch, capsys, "simulate", {"qasm": "qreg q[2]; frob q[0];"})
    assert rc == cli.EXIT_UNSUPPORTED and "unsupported" in err
    rc, _, err = call(monkeypatch, capsys, "simulate", {"qasm": "qreg q[2]; h q[0]"[:-3] + " q0;"})
    assert rc == cli.EXIT_PARSE
    rc, _, err = call(monkeypatch, capsys, "simulate", {"qasm": "qreg q[2]; gate foo a { h a; }"})
    assert rc == cli.EXIT_UNSUPPORTED
    rc, _, err = call(monkeypatch, capsys, "spmv", {"a": {"n": 2, "diags": {}}, "x": [[1, 0]]})
    assert rc == cli.EXIT_ERROR


@pytest.mark.gpu
def test_kernel_protocol_goldens(monkeypatch, capsys, kats):
    proto = kats["kernel_protocol"]
    rc, out, _ = call(monkeypatch, capsys, "from-dense", {"dense": proto["corner"]["dense"]})
    assert rc == 0 and out == proto["corner"]["wire"]
    rc, out, _ = call(monkeypatch, capsys, "to-dense", {"a": proto["corner"]["wire"]})
    assert rc == 0 and out["dense"] == proto["corner"]["round_trip"]
    mc = proto["matmul_case"]
    rc, out, _ = call(monkeypatch, capsys, "matmul", {"a": mc["a"], "b": mc["b"]})
    assert rc == 0 and out == mc["c"]
    rc, out, _ = call(monkeypatch, capsys, "spmv", {"a": mc["a"], "x": mc["x"]})
    assert rc == 0 and out["y"] == mc["y"]
    sim = proto["ghz4_simulate"]
    rc, out, _ = call(monkeypatch, capsys, "simulate",
                      {"qasm": "OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[4];\ncreg c[4];\nh q[0];\n"
                               "cx q[0],q[1];\ncx q[1],q[2];\ncx q[2],q[3];\nmeasure q -> c;\n",
                       "seed": 7, "shots": 1024, "emit_state": True})
    assert rc == 0 and out["counts"] == sim["result"]["counts"]
    assert np.array_equal(pairs_to_complex(out["state"]), pairs_to_complex(sim["result"]["state"]))
    rc, _, err = call(monkeypatch, capsys, "matmul", {"a": {"n": 2, "diags": {}}, "b": {"n": 3, "diags": {}}})
    assert rc == cli.EXIT_ERROR and "not multiplyable" in err
