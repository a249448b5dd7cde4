"""Wider fuzz of the fused passes (both numerics, interpreter and specialised kernels): the contracted schedule (lookahead, phase slots,
register exchanges, unit forms) against the bitwise gate-by-gate state:
  python tools/fuzz_contracted.py [first_seed] [last_seed]"""
import sys

sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import numpy as np

import paper_2405_01250_b200 as D
from _circuits import fuzz_circuit
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W
from paper_2405_01250_b200.shard import run_emulated

lo = int(sys.argv[1]) if len(sys.argv) > 1 else 6
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 40
C = L.CMUL_CONTRACT
worst = 0.0


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for seed in range(lo, hi):
    n, pls, rng = fuzz_circuit(seed)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=None, tile_bits=0).amps
    for jit in (0, 2):
        L.tune("fused_jit", jit)
        for tb in (11, 12):
            got = D.run_gates(x0, pls, cmul_mode=C, tile_bits=tb).amps
            e = rel(got, want)
            worst = max(worst, e)
            assert e < 1e-12, ("fuzz", seed, n, jit, tb, e)
            # the bitwise modes through the same kernels: equal to gate by gate
            assert np.array_equal(D.run_gates(x0, pls, cmul_mode=None, tile_bits=tb).amps, want), ("bitwise", seed, n, jit, tb)
    L.tune("fused_jit", 1)
print("fuzz circuits ok, worst rel L2", worst)

# QFT-like circuits: H, controlled phases (diagonal two-selector gates), swaps
for n in (13, 16, 19):
    ops = []
    for q in range(n):
        ops.append(("h", (q,), ()))
        for k in range(q + 1, min(n, q + 5)):
            ops.append(("cz", (k, q), ()))
            ops.append(("rz", (k,), (0.3 * (k - q),)))
    for q in range(n // 2):
        ops.append(("swap", (q, n - 1 - q), ()))
    for q in range(n):
        ops.append((("rx", "ry", "t", "s", "x", "y")[q % 6], (q,), (0.4 + q,) if q % 6 < 2 else ()))
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    want = D.run_gates(D.init_state(n), pls, cmul_mode=None, tile_bits=0).amps
    got = D.run_gates(D.init_state(n), pls, cmul_mode=C).amps
    e = rel(got, want)
    worst = max(worst, e)
    assert e < 1e-12, ("qft-like", n, e)
print("qft-like ok, worst", worst)

# layered circuits, sharded emulation (the local schedule per shard)
for n, layers, seed, p in ((18, 10, 3, 2), (20, 8, 4, 4), (21, 12, 5, 2), (22, 6, 6, 8)):
    ops = W.random_layered_ops(n, layers, seed=seed)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    want = D.run_gates(D.init_state(n), pls, cmul_mode=None).amps
    got = D.run_gates(D.init_state(n), pls, cmul_mode=C).amps
    e = rel(got, want)
    shards, _ = run_emulated(n, p, pls, cmul_mode=C)
    es = rel(np.concatenate([s.cpu().numpy() for s in shards]), want)
    worst = max(worst, e, es)
    assert e < 1e-12 and es < 1e-12, ("layered", n, layers, e, es)
print("layered + sharded ok, worst", worst)
