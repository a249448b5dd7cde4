"""Host cost per call of the config-1 spmv (n=14) and its pieces (us/call,
back-to-back calls, wall clock): python tools/host_cost_spmv.py"""
import ctypes
import sys
import time

sys.path.insert(0, '/root/repo')
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

c1 = W.config1(0)
a1 = D.kron_identity(c1["left"], D.from_dense(c1["u"], 0.0), c1["right"])
x1 = torch.from_numpy(c1["x"]).cuda()
n = a1.n_dim


def t(f, k=4000):
    for _ in range(100):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        f()
    dt = (time.perf_counter() - t0) / k * 1e6
    torch.cuda.synchronize()
    return round(dt, 2)


st = a1._struct()
ref = ctypes.byref(st)
y = L.empty_c128(n)
s = L.stream_handle()
lib = L.load()
out = {
    "stream_handle": t(L.stream_handle),
    "empty_like": t(lambda: torch.empty_like(x1)),
    "ctypes_call_only(diaq_spmv, prealloc y)": t(lambda: lib.diaq_spmv(ref, x1.data_ptr(), y.data_ptr(), s)),
    "D.spmv (fast path)": t(lambda: D.spmv(a1, x1)),
    "torch x1*2 (reference launch)": t(lambda: x1 * 2),
}
for k, v in out.items():
    print(f"{k:45s} {v:8.2f} us")
