#!/usr/bin/env python3
"""Memory-pattern probe for the fused passes: one pass of K RX gates whose
target state bits are given (same FP64 work, different tile bits), device
time per pass (median of reps):
  python tools/tile_pattern.py N REPS bits1 [bits2 ...]   (bits: comma lists)"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L

n, reps = int(sys.argv[1]), int(sys.argv[2])
L.tune("fused_jit", 2)
for spec in sys.argv[3:]:
    if "=" in spec:
        k, v = spec.split("=")
        L.tune(k, int(v))
        continue
    bits = [int(b) for b in spec.split(",")]
    ops = [D.GateOp("rx", (n - 1 - b,), (0.3 + 0.1 * i,)) for i, b in enumerate(bits)]
    pls = D.compile_circuit(D.Circuit(n, ops), span_limit=n)
    st = D.init_state(n, max_qubits=max(30, n))
    D.run_gates(st, pls, inplace=True)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        D.run_gates(st, pls, inplace=True)
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    print(json.dumps({"bits": bits, "ms": round(statistics.median(times), 4)}), flush=True)
    del st
