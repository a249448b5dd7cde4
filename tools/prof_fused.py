"""Small driver for profiling the fused tile pass (one layer at n=24)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import workloads as W

from paper_2405_01250_b200 import _lib as L

# usage: prof_fused.py [n] [key=value ...]  (diaq_tune settings, e.g. fused_jit=2)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
cmul = None
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    if k == "cmul":  # 2: contracted arithmetic
        cmul = int(v)
        continue
    L.tune(k, int(v))
ops = W.random_layered_ops(n, 1, seed=0)
pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
st = D.init_state(n)
for _ in range(2):
    st = D.run_gates(st, pls, cmul_mode=cmul, inplace=True)
torch.cuda.synchronize()
print("ok", st.norm())
