"""Where the launch-bound configs spend their time (GPU box):
  * config-1 spmv: host us/call vs device us/call (events over 200 calls);
  * run() sampling at n=20 (1024 shots): splitmix uniforms, the native
    sampler call (wall and device), counting/formatting.
python tools/host_breakdown.py"""
import ctypes
import statistics
import sys
import time

sys.path.insert(0, '/root/repo')
import numpy as np
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import sim
from paper_2405_01250_b200 import workloads as W

c1 = W.config1(0)
a1 = D.kron_identity(c1["left"], D.from_dense(c1["u"], 0.0), c1["right"])
x1 = torch.from_numpy(c1["x"]).cuda()
s = torch.cuda.current_stream()
for reps in (50, 200, 1000):
    for _ in range(20):
        D.spmv(a1, x1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(reps):
        D.spmv(a1, x1)
    e1.record(s)
    th = (time.perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    print(f"spmv x{reps}: host {th:.2f} us/call, device {e0.elapsed_time(e1) / reps * 1e3:.2f} us/call")
# graph of 50 spmvs: pure device cost per call
y = torch.empty_like(x1)
st = a1._struct()
ref = ctypes.byref(st)
lib = L.load()
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
with torch.cuda.stream(cs):
    lib.diaq_spmv(ref, x1.data_ptr(), y.data_ptr(), L.stream_handle())
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(50):
            lib.diaq_spmv(ref, x1.data_ptr(), y.data_ptr(), ctypes.c_void_p(cs.cuda_stream))
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10):
    g.replay()
e1.record(s)
torch.cuda.synchronize()
print(f"spmv in a CUDA graph: device {e0.elapsed_time(e1) / 500 * 1e3:.2f} us/call")

n = 20
ops = W.random_layered_ops(n, 40, seed=0)
pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
state = D.run_gates(D.init_state(n), pls)
torch.cuda.synchronize()
for _ in range(3):
    sim.measure_all_sample(state, 1024, 0)
T = {"uniforms": [], "native_wall": [], "native_dev": [], "count": [], "total": []}
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u = sim.splitmix64_uniforms(0, 1024)
    t1 = time.perf_counter()
    xd = state.device_amps
    hits = np.empty(1024, dtype=np.int64)
    nrm = ctypes.c_double(0.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    L.call("diaq_sample_hits", int(xd.numel()), xd.data_ptr(), u.ctypes.data, 1024, hits.ctypes.data,
           ctypes.addressof(nrm), L.stream_handle())
    e1.record(s)
    t2 = time.perf_counter()
    outcomes, freq = np.unique(hits, return_counts=True)
    d = {format(int(i), f"0{n}b"): int(c) for i, c in zip(outcomes, freq)}
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    T["uniforms"].append((t1 - t0) * 1e3)
    T["native_wall"].append((t2 - t1) * 1e3)
    T["native_dev"].append(e0.elapsed_time(e1))
    T["count"].append((t3 - t2) * 1e3)
    t0 = time.perf_counter()
    sim.measure_all_sample(state, 1024, 0)
    T["total"].append((time.perf_counter() - t0) * 1e3)
print("sampling n=20, ms (median of 10):", {k: round(statistics.median(v), 3) for k, v in T.items()})
