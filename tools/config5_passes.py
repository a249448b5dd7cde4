"""Per-pass device times of config 5 at n=30 (20 layers) under a numerics
mode, with DIAQ_JIT_TRACE=1 giving each launch's structure on stderr:
  DIAQ_JIT_TRACE=1 python tools/config5_passes.py [cmul_mode] [n] [layers]"""
import sys

sys.path.insert(0, '/root/repo')
import numpy as np
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

import os
for kv in filter(None, os.environ.get("DIAQ_TUNE", "").split(",")):  # e.g. DIAQ_TUNE=fused_estore=0
    k, v = kv.split("=")
    L.tune(k, int(v))
mode = int(sys.argv[1]) if len(sys.argv) > 1 else L.CMUL_CONTRACT
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
layers = int(sys.argv[3]) if len(sys.argv) > 3 else 20
ops = W.random_layered_ops(n, layers, seed=0)
pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
st = D.init_state(n, max_qubits=n)
D.run_gates(st, pls, cmul_mode=mode, inplace=True)
L.call("diaq_jit_wait", -1.0)
tot = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    D.run_gates(st, pls, cmul_mode=mode, inplace=True)
    e1.record()
    torch.cuda.synchronize()
    tot.append(e0.elapsed_time(e1))
print(f"median of 3 whole-program runs: {sorted(tot)[1]:.2f} ms  ({', '.join(f'{t:.1f}' for t in tot)})")
timer = L.Timer(len(pls) + 1)
print("--- timed run", file=sys.stderr, flush=True)
D.run_gates(st, pls, cmul_mode=mode, inplace=True, timer=timer)
ms = timer.elapsed_ms()
per = [float(v) for v in ms if v > 0]
print(f"passes {len(per)} total {sum(per):.2f} ms")
floor = 32 * 2**n / 6.5517e12 * 1e3
for i, v in enumerate(per):
    print(f"{i:3d} {v:8.3f} ms  frac {floor / v:.3f}")
