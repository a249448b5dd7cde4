import time, ctypes, sys
sys.path.insert(0, '/root/repo')
import torch
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L, workloads as W
from paper_2405_01250_b200.matrix import _as_device_vector
c1 = W.config1(0)
a1 = D.kron_identity(c1["left"], D.from_dense(c1["u"], 0.0), c1["right"])
x1 = torch.from_numpy(c1["x"]).cuda()
n = a1.n_dim
def t(f, k=2000):
    for _ in range(50): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): f()
    dt = (time.perf_counter() - t0) / k * 1e6
    torch.cuda.synchronize()
    return round(dt, 2)
st = a1._struct(); y = L.empty_c128(n); s = L.stream_handle()
print("stream_handle", t(L.stream_handle))
print("raw stream", t(lambda: torch._C._cuda_getCurrentRawStream(0)))
print("empty_c128", t(lambda: L.empty_c128(n)))
print("device()", t(L.device))
print("as_device_vector", t(lambda: _as_device_vector(x1, n)))
print("_struct", t(a1._struct))
print("call spmv", t(lambda: L.call("diaq_spmv", ctypes.byref(st), x1.data_ptr(), y.data_ptr(), s)))
print("D.spmv", t(lambda: D.spmv(a1, x1)))
