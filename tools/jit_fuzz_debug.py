"""Specialised vs AOT fused passes on the seeded fuzz circuits (tests/_circuits.py):
report every (seed, tile, switch) whose states differ."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import paper_2405_01250_b200 as D
from _circuits import fuzz_circuit
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    n, pls, rng = fuzz_circuit(seed)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=1, tile_bits=0).amps
    for ps in (1, 0):
        L.tune("fused_pair_store", ps)
        for sw in ({}, {"fused_gperm_rows": 1}, {"fused_seq": 0}, {"fused_perm": 0}):
            for k, v in sw.items():
                L.tune(k, v)
            for tb in (11, 12):
                L.tune("fused_jit", 2)
                got = D.run_gates(x0, pls, cmul_mode=1, tile_bits=tb).amps
                bad = np.flatnonzero(got != want)
                if len(bad):
                    print("MISMATCH seed", seed, "n", n, "tb", tb, "pair_store", ps, sw, "bad", len(bad), "first", bad[:4], flush=True)
            for k in sw:
                L.tune(k, {"fused_gperm_rows": 0}.get(k, 1))
print("done")
