"""Host cost of the config-2 products: per matmul() call and per product of
a batched matmul_batch() sweep of the 64 seeded pairs (wall, us), with a
cProfile of one matmul() call's Python side:  python tools/host_cost_spgemm.py"""
import cProfile
import io
import pstats
import statistics
import sys
import time

sys.path.insert(0, '/root/repo')
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import workloads as W

pairs = []
for seed in range(64):
    p = W.config2(seed)
    span = D.build_span_unitary(D.from_dense(p["u4"], 0.0), p["u4_positions"], p["u4_span"])
    A = D.kron_identity(p["a_left"], span, p["a_right"])
    B = D.matmul(D.kron_identity(p["b1_left"], D.from_dense(p["u2"], 0.0), p["b1_right"]),
                 D.kron_identity(p["b0_left"], D.from_dense(W.rz(p["theta"]), 0.0), p["b0_right"]))
    pairs.append((A, B))
for A, B in pairs:  # warm: device tables of every operand
    D.matmul(A, B)
torch.cuda.synchronize()
per_call, batched = [], []
for _ in range(5):
    t0 = time.perf_counter()
    for A, B in pairs:
        D.matmul(A, B)
    torch.cuda.synchronize()
    per_call.append((time.perf_counter() - t0) / 64 * 1e6)
    t0 = time.perf_counter()
    D.matrix.matmul_batch(pairs)
    torch.cuda.synchronize()
    batched.append((time.perf_counter() - t0) / 64 * 1e6)
print(f"matmul() per call      {statistics.median(per_call):8.2f} us")
print(f"matmul_batch per prod  {statistics.median(batched):8.2f} us")
pr = cProfile.Profile()
pr.enable()
for A, B in pairs:
    D.matmul(A, B)
pr.disable()
buf = io.StringIO()
pstats.Stats(pr, stream=buf).sort_stats("tottime").print_stats(12)
print(buf.getvalue()[:3000])

# host-side vs device-side time of one batched sweep
for _ in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    Cs = D.matrix.matmul_batch(pairs)
    t_host = time.perf_counter() - t0
    e1.record()
    torch.cuda.synchronize()
    t_all = time.perf_counter() - t0
    print(f"batch: host enqueue {t_host * 1e6:8.1f} us, wall {t_all * 1e6:8.1f} us, device {e0.elapsed_time(e1) * 1e3:8.1f} us")
pr = cProfile.Profile()
pr.enable()
D.matrix.matmul_batch(pairs)
pr.disable()
buf = io.StringIO()
pstats.Stats(pr, stream=buf).sort_stats("tottime").print_stats(10)
print(buf.getvalue()[:2500])
