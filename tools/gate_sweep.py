#!/usr/bin/env python3
"""Time the fused multi-gate passes vs gate-by-gate at n=28 (and n=20) per tile size."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W
from paper_2405_01250_b200.sim import _GateProgram


def main():
    # usage: gate_sweep.py [key=value ...] -- diaq_tune settings; GATE_SWEEP_TILES="0,11" picks tile sizes
    for kv in sys.argv[1:]:
        k, v = kv.split("=")
        L.tune(k, int(v))
    tiles = [int(t) for t in os.environ.get("GATE_SWEEP_TILES", "0,8,9,10,11,12").split(",")]
    sizes = ((28, 1), (20, 40)) if not os.environ.get("GATE_SWEEP_N28_ONLY") else ((28, 1),)
    for n, layers in sizes:
        ops = W.random_layered_ops(n, layers, seed=0)
        pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
        prog = _GateProgram([p.compact() for p in pls])
        x = torch.zeros(2**n, dtype=torch.complex128, device="cuda")
        x[0] = 1
        s = torch.cuda.current_stream().cuda_stream
        ref = None
        for tb in tiles:
            npass = ctypes.c_int(0)

            def go():
                if tb == 0:
                    L.call("diaq_run_gates", n, prog.n, prog.arr, x.data_ptr(), 1, None, s)
                else:
                    L.call("diaq_run_gates_fused", n, prog.n, prog.arr, x.data_ptr(), 1, tb, None,
                           ctypes.addressof(npass), s)
            x.zero_(); x[0] = 1
            go()
            torch.cuda.synchronize()
            if ref is None:
                ref = x.clone()
            same = bool(torch.equal(ref, x))
            for _ in range(2):
                go()
            torch.cuda.synchronize()
            reps = 5 if n >= 26 else 20
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
            evs[0].record()
            for r in range(reps):
                go()
                evs[r + 1].record()
            torch.cuda.synchronize()
            per = sorted(evs[r].elapsed_time(evs[r + 1]) for r in range(reps))
            ms = per[len(per) // 2]  # median
            print(json.dumps({"tune": sys.argv[1:], "n": n, "gates": prog.n, "tile_bits": tb, "passes": npass.value if tb else prog.n,
                              "ms": round(ms, 3), "gates_per_s": round(prog.n / ms * 1e3, 1),
                              "ms_per_pass": round(ms / max(1, npass.value if tb else prog.n), 4),
                              "first_run_bitwise_same_as_unfused": same}), flush=True)


if __name__ == "__main__":
    main()
