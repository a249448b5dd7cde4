"""One fuzz circuit through the fused passes with the given knobs (debugging):
  python tools/jit_one.py SEED TILE [key=value ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import paper_2405_01250_b200 as D
from _circuits import fuzz_circuit
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

seed, tb = int(sys.argv[1]), int(sys.argv[2])
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    L.tune(k, int(v))
n, pls, rng = fuzz_circuit(seed)
x0 = D.StateVector(n, W.random_state(rng, 2**n))
want = D.run_gates(x0, pls, cmul_mode=1, tile_bits=0).amps
got = D.run_gates(x0, pls, cmul_mode=1, tile_bits=tb)
torch.cuda.synchronize()
g = got.amps
print("seed", seed, "n", n, "tb", tb, sys.argv[3:], "bad", int(np.count_nonzero(g != want)), flush=True)
