#!/usr/bin/env python3
"""Sweep launch-geometry knobs of the spmv and gate kernels at n=28 (GPU).

Results never depend on the knobs (checked bitwise here); only time does.
"""
import ctypes
import itertools
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    N = 2**n
    c4 = W.config4(22, seed=0, with_x=False)
    span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    a = D.kron_identity(2 ** (n - 22), span, c4["right"])
    nbytes = 16 * sum(N - abs(d) for d in a.diag_indices()) + 32 * N
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.randn(N, dtype=torch.complex128, device="cuda", generator=g)
    y = torch.empty_like(x)
    st = a._struct()
    s = torch.cuda.current_stream().cuda_stream
    fn = lambda: L.call("diaq_spmv", ctypes.byref(st), x.data_ptr(), y.data_ptr(), s)
    ref = None
    res = []
    for asy, tma, stages, banded, strips, raster, chunk, xpol, ctas in (
            (0, 0, 2, 1, 1, 0, 1, 0, 0), (1, 0, 2, 1, 1, 0, 1, 0, 0), (1, 0, 2, 1, 1, 0, 1, 0, 12),
            (1, 0, 2, 1, 0, 0, 1, 0, 0)):
        L.tune("spmv_async", asy)
        L.tune("spmv_tma", tma)
        L.tune("spmv_tma_stages", stages)
        L.tune("spmv_banded", banded)
        L.tune("spmv_strips", strips)
        L.tune("spmv_raster", raster)
        L.tune("spmv_chunk", chunk)
        L.tune("spmv_xpol", xpol)
        L.tune("spmv_ctas_per_sm", ctas)
        ms = timeit(fn)
        if ref is None:
            ref = y.clone()
        same = bool(torch.equal(ref, y))
        rec = {"async": asy, "tma": tma, "stages": stages, "banded": banded, "strips": strips, "raster": raster, "chunk": chunk, "xpol": xpol, "ctas_per_sm": ctas, "ms": round(ms, 4),
               "GBs": round(nbytes / ms / 1e6, 1), "bitwise_same": same}
        print(json.dumps(rec), flush=True)
        res.append(rec)
    # gate kernel
    del a, span
    state = D.StateVector(n, x)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in W.random_layered_ops(n, 1, 0)]), span_limit=n)
    for ctas in (2, 4, 8, 16, 32):
        L.tune("gate_ctas_per_sm", ctas)
        ms = timeit(lambda: D.run_gates(state, pls, inplace=True), reps=3, warm=1) / len(pls)
        print(json.dumps({"gate_ctas_per_sm": ctas, "ms_per_gate": round(ms, 4),
                          "GBs": round(32 * N / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
