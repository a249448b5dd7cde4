"""spmv DRAM traffic vs offset structure (run under ncu for dram byte counts)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L

n = 28
N = 2**n
x = torch.randn(N, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
cases = {"diag0": [0], "near3": [-8, 0, 8], "far3": [-(2**21), 0, 2**21],
         "cfg4": [-(2**21) - 8, -(2**21), -(2**21) + 8, -8, 0, 8, 2**21 - 8, 2**21, 2**21 + 8]}
for name, offs in cases.items():
    a = D.DiaqMatrix._empty_device(N, np.array(offs))
    a.device_arena()[2].fill_(0.5)
    st = a._struct()
    L.call("diaq_spmv", ctypes.byref(st), x.data_ptr(), y.data_ptr(), s)
    torch.cuda.synchronize()
    alg = 16 * sum(N - abs(d) for d in offs) + 32 * N
    print(name, "alg_read_GB", round((alg - 16 * N) / 1e9, 3))
    del a, st
