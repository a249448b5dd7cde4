#!/usr/bin/env python3
"""Specialised (NVRTC) fused passes vs the AOT interpreter: bitwise check
and timing on the random layered circuits (n=28 one layer, n=20 40 layers).
  python tools/jit_check.py [n layers tile_bits] ...
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W
from paper_2405_01250_b200.sim import _GateProgram


def jit_stats():
    st = (ctypes.c_int64 * 6)()
    L.call("diaq_jit_stats", ctypes.addressof(st))
    return dict(zip(["compiled", "failed", "launches", "modules", "pending", "compile_ms"], list(st)))


def run_case(n, layers, tb):
    ops = W.random_layered_ops(n, layers, seed=0)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    prog = _GateProgram([p.compact() for p in pls])
    x = torch.zeros(2**n, dtype=torch.complex128, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    npass = ctypes.c_int(0)

    def go():
        L.call("diaq_run_gates_fused", n, prog.n, prog.arr, x.data_ptr(), 1, tb, None, ctypes.addressof(npass), s)

    def timed(reps):
        for _ in range(2):
            go()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        evs[0].record()
        for r in range(reps):
            go()
            evs[r + 1].record()
        torch.cuda.synchronize()
        per = sorted(evs[r].elapsed_time(evs[r + 1]) for r in range(reps))
        return per[len(per) // 2]

    out = {"n": n, "layers": layers, "tile_bits": tb, "gates": prog.n}
    res = {}
    for mode in (0, 2):
        L.tune("fused_jit", mode)
        x.zero_(); x[0] = 1
        t0 = time.perf_counter()
        go()
        torch.cuda.synchronize()
        out[f"first_call_s_jit{mode}"] = round(time.perf_counter() - t0, 3)
        res[mode] = x.clone()
        reps = 5 if n >= 26 else 20
        ms = timed(reps)
        out[f"ms_jit{mode}"] = round(ms, 3)
        out[f"gates_per_s_jit{mode}"] = round(prog.n / ms * 1e3, 1)
    out["passes"] = npass.value
    out["bitwise_equal"] = bool(torch.equal(res[0], res[2]))
    out["jit"] = jit_stats()
    L.tune("fused_jit", 1)
    print(json.dumps(out), flush=True)


def main():
    # JIT_TUNE="k=v,k=v": extra diaq_tune settings for both arms
    for kv in filter(None, os.environ.get("JIT_TUNE", "").split(",")):
        k, v = kv.split("=")
        L.tune(k, int(v))
    args = sys.argv[1:] or ["28", "1", "0", "20", "40", "0"]
    for i in range(0, len(args), 3):
        run_case(int(args[i]), int(args[i + 1]), int(args[i + 2]))
    err = L.load().diaq_jit_last_error()
    if err:
        print("jit last error:", err.decode()[:2000])


if __name__ == "__main__":
    main()
