"""Fuzz circuits at a production-like size (default n=24: dynamic unit
order, pair stores and plain pairs all active) through the specialised
kernels and the interpreter, both numerics, against gate by gate:
  python tools/fuzz_large.py [n] [first_seed] [last_seed]"""
import sys

sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import numpy as np

import paper_2405_01250_b200 as D
from _circuits import fuzz_circuit
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 10
worst = 0.0
for seed in range(lo, hi):
    _, pls, rng = fuzz_circuit(seed, n=n)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=None, tile_bits=0).amps
    for jit in (2, 0):
        L.tune("fused_jit", jit)
        got = D.run_gates(x0, pls, cmul_mode=None, tile_bits=11).amps
        assert np.array_equal(got, want), ("bitwise", seed, jit)
        got = D.run_gates(x0, pls, cmul_mode=L.CMUL_CONTRACT, tile_bits=11).amps
        e = float(np.linalg.norm(got - want) / np.linalg.norm(want))
        worst = max(worst, e)
        assert e < 1e-12, ("contracted", seed, jit, e)
    L.tune("fused_jit", 1)
    print("seed", seed, "ok", flush=True)
print("n =", n, "seeds", lo, "..", hi - 1, "ok; worst contracted rel L2", worst)
