"""`kernel` JSON-over-stdio protocol on the device path.

    python -m paper_2405_01250_b200.cli kernel {from-dense,to-dense,matmul,spmv,simulate} < request.json

Same requests, replies and exit codes as the reference's `diaqsim kernel`
(cli.py:251-287, docs/cli.md:95-114; exit codes cli.py:42-46, 351-369), so
the TypeScript client (frontend/src/core.ts:41-60) can point DIAQSIM_BIN at
this entry point.  `simulate` accepts the reference's `qasm` field for the
flat OpenQASM 2.0 subset (one qreg, catalog gates, measure/barrier; QASM
macros and includes beyond qelib1.inc are out of scope -> exit 3), or an
`ops` list ([[name, [qubits], [params]], ...]) plus `n_qubits`.
"""
from __future__ import annotations

import argparse
import ast
import json
import math
import operator
import re
import sys

import numpy as np

from . import __version__
from .errors import DiaqError, ParseError, ResourceError, UnsupportedFeatureError, UnsupportedGateError
from .gates import GATE_DEFS, Circuit, GateOp
from .matrix import from_dense, from_json_dict, matmul, spmv, to_dense, to_json_dict
from .sim import run as sim_run

EXIT_OK, EXIT_ERROR, EXIT_PARSE, EXIT_UNSUPPORTED, EXIT_RESOURCE = 0, 1, 2, 3, 4


def _complex_pairs(values) -> list[list[float]]:
    return [[float(v.real), float(v.imag)] for v in values]


def _pairs_to_complex(pairs) -> np.ndarray:
    arr = np.asarray(pairs, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[1] != 2:
        raise ValueError("expected a list of [re, im] pairs")
    return arr[:, 0] + 1j * arr[:, 1]


_OPS = {ast.Add: operator.add, ast.Sub: operator.sub, ast.Mult: operator.mul, ast.Div: operator.truediv,
        ast.Pow: operator.pow, ast.USub: operator.neg, ast.UAdd: operator.pos}


def _param(text: str, line: int) -> float:
    def ev(node):
        if isinstance(node, ast.Expression):
            return ev(node.body)
        if isinstance(node, ast.Constant) and isinstance(node.value, (int, float)):
            return float(node.value)
        if isinstance(node, ast.Name) and node.id == "pi":
            return math.pi
        if isinstance(node, ast.BinOp) and type(node.op) in _OPS:
            return _OPS[type(node.op)](ev(node.left), ev(node.right))
        if isinstance(node, ast.UnaryOp) and type(node.op) in _OPS:
            return _OPS[type(node.op)](ev(node.operand))
        raise ParseError(f"unsupported parameter expression '{text}'", line, 1)
    try:
        return ev(ast.parse(text.strip(), mode="eval"))
    except SyntaxError as exc:
        raise ParseError(f"bad parameter '{text}'", line, 1) from exc


_GATE_LINE = re.compile(r"^([a-z_][a-z0-9_]*)\s*(?:\((.*)\))?\s+(.+)$")
_QARG = re.compile(r"^([a-zA-Z_]\w*)\[(\d+)\]$")


def parse_flat_qasm(text: str, name: str = "qasm") -> Circuit:
    """Flat OpenQASM 2.0 subset: header, one qreg, catalog gates, measure, barrier."""
    n = None
    qreg = None
    ops = []
    body = re.sub(r"//[^\n]*", "", text)
    for line_no, stmt in enumerate((s.strip() for s in body.split(";")), start=1):
        if not stmt or stmt.startswith("OPENQASM") or stmt.startswith("include") or stmt.startswith("creg"):
            continue
        if stmt.startswith("qreg"):
            m = re.match(r"^qreg\s+([a-zA-Z_]\w*)\[(\d+)\]$", stmt)
            if not m:
                raise ParseError(f"bad qreg '{stmt}'", line_no, 1)
            if qreg is not None:
                raise UnsupportedFeatureError("more than one qreg", line_no, 1)
            qreg, n = m.group(1), int(m.group(2))
            continue
        if stmt.startswith("measure") or stmt.startswith("barrier"):
            # structural ops are kept like the reference lowering does (no Placement)
            kind, rest = stmt.split(None, 1)
            target = rest.split("->")[0].strip()
            qubits = []
            for a in target.split(","):
                a = a.strip()
                if a == qreg:
                    qubits.extend(range(n))
                    continue
                qa = _QARG.match(a)
                if not qa or qa.group(1) != qreg:
                    raise ParseError(f"bad qubit argument '{a}'", line_no, 1)
                qubits.append(int(qa.group(2)))
            ops.append(GateOp(kind, tuple(qubits)))
            continue
        if stmt.startswith("gate") or stmt.startswith("if") or stmt.startswith("opaque"):
            raise UnsupportedFeatureError(f"'{stmt.split()[0]}' is outside the flat subset", line_no, 1)
        m = _GATE_LINE.match(stmt)
        if not m:
            raise ParseError(f"cannot parse '{stmt}'", line_no, 1)
        gname, params, args = m.group(1), m.group(2), m.group(3)
        if gname not in GATE_DEFS:
            raise UnsupportedGateError(f"unknown gate '{gname}'")
        qubits = []
        for a in args.split(","):
            qa = _QARG.match(a.strip())
            if not qa or qa.group(1) != qreg:
                raise ParseError(f"bad qubit argument '{a.strip()}'", line_no, 1)
            qubits.append(int(qa.group(2)))
        ps = tuple(_param(p, line_no) for p in params.split(",")) if params else ()
        ops.append(GateOp(gname, tuple(qubits), ps))
    if n is None:
        raise ParseError("no qreg declared", 1, 1)
    return Circuit(n, ops, name=name)


def cmd_kernel(args) -> int:
    request = json.loads(sys.stdin.read())
    op = args.op
    if op == "from-dense":
        m = np.array([[complex(p[0], p[1]) for p in row] for row in request["dense"]], dtype=np.complex128)
        out = to_json_dict(from_dense(m, eps=float(request.get("eps", 0.0))))
    elif op == "to-dense":
        m = to_dense(from_json_dict(request["a"]))
        out = {"dense": [_complex_pairs(row) for row in m]}
    elif op == "matmul":
        out = to_json_dict(matmul(from_json_dict(request["a"]), from_json_dict(request["b"])))
    elif op == "spmv":
        out = {"y": _complex_pairs(spmv(from_json_dict(request["a"]), _pairs_to_complex(request["x"])))}
    else:
        if "ops" in request:
            circuit = Circuit(int(request["n_qubits"]), [GateOp(o[0], tuple(o[1]), tuple(o[2]))
                                                         for o in request["ops"]])
        else:
            circuit = parse_flat_qasm(request["qasm"], name=request.get("name", "qasm"))
        result = sim_run(circuit, backend=request.get("backend", "diaq"), shots=int(request.get("shots", 1024)),
                         seed=int(request.get("seed", 0)), emit_state=bool(request.get("emit_state", False)),
                         span_limit=request.get("span_limit"))
        out = {"counts": dict(sorted(result.counts.items())), "n_qubits": result.n_qubits,
               "backend": result.backend}
        if result.state is not None:
            out["state"] = _complex_pairs(result.state)
    json.dump(out, sys.stdout)
    sys.stdout.write("\n")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="diaqsim-b200", description="DiaQ kernels on the B200 path")
    parser.add_argument("--version", action="version", version=f"diaqsim-b200 {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)
    p_k = sub.add_parser("kernel", help="matrix kernels over JSON stdin/stdout")
    p_k.add_argument("op", choices=("from-dense", "to-dense", "matmul", "spmv", "simulate"))
    p_k.set_defaults(fn=cmd_kernel)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except ParseError as exc:
        print(f"parse error: {exc}", file=sys.stderr)
        return EXIT_PARSE
    except (UnsupportedFeatureError, UnsupportedGateError) as exc:
        print(f"unsupported: {exc}", file=sys.stderr)
        return EXIT_UNSUPPORTED
    except ResourceError as exc:
        print(f"resource guard: {exc}", file=sys.stderr)
        return EXIT_RESOURCE
    except DiaqError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_ERROR
    except (OSError, ValueError, KeyError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_ERROR


if __name__ == "__main__":
    sys.exit(main())
