"""Profile driver: the metric's Haar4 layer at n=28 (14 Haar-random two-qubit
gates on a seeded random matching, as bench.py's secondary) through the
fused passes; argv[1] = cmul mode (default: reference rounding)."""
import sys

sys.path.insert(0, '/root/repo')
import numpy as np
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

mode = int(sys.argv[1]) if len(sys.argv) > 1 else None
L.tune("fused_jit", 2)
rng = np.random.default_rng(0)
perm = rng.permutation(28)
pls = []
for i in range(14):
    qa, qb = int(perm[2 * i]), int(perm[2 * i + 1])
    lo, hi = min(qa, qb), max(qa, qb)
    pls.append(D.Placement(2**lo, None, 2 ** (27 - hi), lo, hi, "haar", gate=(W.haar(rng, 4), [qa - lo, qb - lo])))
st = D.init_state(28)
for _ in range(2):
    D.run_gates(st, pls, cmul_mode=mode, inplace=True)
torch.cuda.synchronize()
print("ok", st.norm())
