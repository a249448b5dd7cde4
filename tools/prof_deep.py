"""Driver for profiling the deep (multi-layer) passes of the lookahead
schedule: a layered circuit under the contracted arithmetic, run twice.
  python tools/prof_deep.py [n] [layers] [key=value ...]  (diaq_tune settings)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 6
L.tune("fused_jit", 2)
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    L.tune(k, int(v))
ops = W.random_layered_ops(n, layers, seed=0)
pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
st = D.init_state(n, max_qubits=n)
timer = L.Timer(len(pls) + 1)
for _ in range(2):
    st = D.run_gates(st, pls, cmul_mode=L.CMUL_CONTRACT, inplace=True, timer=timer)
torch.cuda.synchronize()
print("ok", st.norm(), [round(float(v), 3) for v in timer.elapsed_ms() if v > 0])
