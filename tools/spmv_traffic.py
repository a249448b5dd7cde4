"""Run the config-4 spmv once per raster/x-policy variant (for ncu dram byte counts)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

n = 28
c4 = W.config4(22, seed=0, with_x=False)
span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
a = D.kron_identity(2 ** (n - 22), span, c4["right"])
x = torch.randn(2**n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
st = a._struct()
s = torch.cuda.current_stream().cuda_stream
for banded, raster, chunk, xpol in ((1, 0, 1, 0), (0, 0, 1, 0), (1, 0, 1, 0)):
    L.tune("spmv_banded", banded)
    L.tune("spmv_raster", raster)
    L.tune("spmv_chunk", chunk)
    L.tune("spmv_xpol", xpol)
    L.call("diaq_spmv", ctypes.byref(st), x.data_ptr(), y.data_ptr(), s)
torch.cuda.synchronize()
print("ok")
