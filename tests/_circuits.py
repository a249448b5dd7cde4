"""Seeded circuit generators shared by the GPU parity tests and the CPU
codegen test of the specialised fused passes."""
import numpy as np

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import workloads as W


def _perm_gate(q):
    """0/1 matrix moving old index c to new index q[c]."""
    m = np.zeros((len(q), len(q)), dtype=complex)
    for c, r in enumerate(q):
        m[r, c] = 1.0
    return m


def fuzz_circuit(seed, n=None):
    """Seeded random circuit over every gate kind the fused scheduler routes
    differently; returns (n, placements, rng) -- also used by the CPU
    codegen test of the specialised passes (test_jit_cpu.py).  `n` forces
    the state size (default: drawn from 11..18)."""
    rng = np.random.default_rng(1000 + seed)
    drawn = int(rng.integers(11, 19))
    n = drawn if n is None else int(n)
    names1 = ["h", "x", "y", "z", "s", "t", "rx", "ry", "rz", "u3", "sdg"]
    pls = []
    for _ in range(int(rng.integers(40, 90))):
        kind = rng.integers(8)
        q = [int(v) for v in rng.choice(n, size=3, replace=False)]
        if kind <= 2:
            nm = names1[int(rng.integers(len(names1)))]
            par = {"rx": (0.7,), "ry": (1.1,), "rz": (2.3,), "u3": (0.1, 0.2, 0.3)}.get(nm, ())
            ops = [(nm, (q[0],), par)]
        elif kind == 3:
            ops = [("cx", (q[0], q[1]), ()), ("cx", (q[1], q[2]), ()), ("swap", (q[0], q[2]), ())]
        elif kind == 4:
            ops = [("cz", (q[0], q[1]), ()), ("ccx", (q[0], q[1], q[2]), ())]
        else:
            ops = []
            if kind == 5:
                g, qs = W.haar(rng, 4), [q[0], q[1]]
            elif kind == 6:
                g = np.eye(8, dtype=complex)
                g[4:, 4:] = W.haar(rng, 4)
                qs = q
            else:
                g, qs = _perm_gate([2, 0, 3, 1]), [q[0], q[1]]
            lo, hi = min(qs), max(qs)
            pls.append(D.Placement(2**lo, None, 2 ** (n - 1 - hi), lo, hi, "u", gate=(g, [v - lo for v in qs])))
        if ops:
            pls += D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    return n, pls, rng
