"""Finer host-cost breakdown of the config-1 spmv call (us per call, 20000
back-to-back calls): python tools/host_cost_spmv2.py"""
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
lib = L.load()
st = a1._struct()
ref = ctypes.byref(st)
y = torch.empty_like(x1)
xp, yp, s = x1.data_ptr(), y.data_ptr(), L.stream_handle()


def t(f, k=20000):
    for _ in range(500):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        f()
    dt = (time.perf_counter() - t0) / k * 1e6
    torch.cuda.synchronize()
    return dt


rows = [
    ("D.spmv(a, x) full", lambda: D.spmv(a1, x1)),
    ("ctypes diaq_spmv, prealloc y, ints", lambda: lib.diaq_spmv(ref, xp, yp, s)),
    ("ctypes diaq_version() (no-op)", lambda: lib.diaq_version()),
    ("ctypes diaq_launch_count() (no-op)", lambda: lib.diaq_launch_count()),
    ("torch.empty_like(x)", lambda: torch.empty_like(x1)),
    ("L.stream_handle()", L.stream_handle),
    ("x.data_ptr()", x1.data_ptr),
    ("torch x*2 (torch's own launch)", lambda: x1 * 2),
]
for name, f in rows:
    print(f"{name:40s} {t(f):8.2f} us", flush=True)
