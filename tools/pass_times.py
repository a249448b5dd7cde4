#!/usr/bin/env python3
"""Per-pass structure of a random layered circuit's fused program (one run,
specialised passes compiled first), for pairing with an ncu launch list:
  DIAQ_JIT_TRACE=1 ncu --metrics gpu__time_duration.sum -k regex:diaq_jit_pass --csv \\
      python tools/pass_times.py N LAYERS [key=value ...]
The trace lines (stderr) and the ncu rows come in launch order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

n, layers = int(sys.argv[1]), int(sys.argv[2])
L.tune("fused_jit", 2)
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    L.tune(k, int(v))
ops = W.random_layered_ops(n, layers, seed=0)
pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
st = D.init_state(n, max_qubits=max(30, n))
D.run_gates(st, pls, inplace=True)
torch.cuda.synchronize()
print("norm", st.norm(), file=sys.stderr)
