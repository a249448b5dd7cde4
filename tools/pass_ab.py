#!/usr/bin/env python3
"""Per-pass device times of a random layered circuit's fused program with the
specialised passes compiled first (CUDA events at pass boundaries, median of
reps), e.g. for A/B-ing pass-body variants (env DIAQ_JIT_OLD_BODY=1):
  python tools/pass_ab.py N LAYERS [REPS] [key=value ...]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

n, layers = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
L.tune("fused_jit", 2)
for kv in sys.argv[4:]:
    k, v = kv.split("=")
    if k == "tile":
        D.sim.FUSE_TILE_BITS = int(v)
    else:
        L.tune(k, int(v))
ops = W.random_layered_ops(n, layers, seed=0)
pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
st = D.init_state(n, max_qubits=max(30, n))
D.run_gates(st, pls, inplace=True)
torch.cuda.synchronize()
per = []
tot = []
for _ in range(reps):
    tm = L.Timer(len(pls) + 1)
    D.run_gates(st, pls, timer=tm, inplace=True)
    ms = tm.elapsed_ms()
    per.append([float(m) for m in ms if m > 0])
    tot.append(float(sum(ms)))
npass = len(per[0])
med = [statistics.median(r[i] for r in per) for i in range(npass)]
print(json.dumps({"n": n, "layers": layers, "args": sys.argv[4:], "env": {k: v for k, v in os.environ.items() if k.startswith("DIAQ_JIT")},
                  "ms_total": round(statistics.median(tot), 4), "passes": npass,
                  "ms_per_pass": [round(m, 4) for m in med[:16]], "norm": st.norm()}), flush=True)
