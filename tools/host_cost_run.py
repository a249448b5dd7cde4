"""Host cost of run() at config 3 (n=20, 40 layers, 1200 gates, 1024 shots):
wall per call, its phase timings, the device time of the gate loop, and a
cProfile of one call:  python tools/host_cost_run.py"""
import cProfile
import io
import pstats
import statistics
import sys
import time

sys.path.insert(0, '/root/repo')
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

ops = W.random_layered_ops(20, 40, seed=0)
circ = D.Circuit(20, [D.GateOp(*o) for o in ops])
for _ in range(3):
    D.run(circ, shots=1024, seed=0, span_limit=20)
L.call("diaq_jit_wait", -1.0)
walls, phases = [], []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = D.run(circ, shots=1024, seed=0, span_limit=20)
    walls.append((time.perf_counter() - t0) * 1e3)
    phases.append({k: v / 1e6 for k, v in r.timings_ns.items() if k != "per_gate"})
print(f"run() wall ms: median {statistics.median(walls):.3f}  min {min(walls):.3f}")
print("phases ms (last):", {k: round(v, 3) for k, v in phases[-1].items()})
pr = cProfile.Profile()
pr.enable()
D.run(circ, shots=1024, seed=0, span_limit=20)
pr.disable()
buf = io.StringIO()
pstats.Stats(pr, stream=buf).sort_stats("cumtime").print_stats(25)
print(buf.getvalue()[:5000])

# enqueue cost of the gate program alone vs its device time
import ctypes
from paper_2405_01250_b200.sim import _GateProgram
pls = D.compile_circuit(circ, span_limit=20)
prog = _GateProgram([p.compact() for p in pls])
st = D.init_state(20)
xd = st.device_amps
s = torch.cuda.current_stream()
np_ = ctypes.c_int(0)
for _ in range(3):
    L.call("diaq_run_gates_fused", 20, prog.n, prog.arr, xd.data_ptr(), 1, -1, None, ctypes.addressof(np_), L.stream_handle())
torch.cuda.synchronize()
enq, dev = [], []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    L.call("diaq_run_gates_fused", 20, prog.n, prog.arr, xd.data_ptr(), 1, -1, None, ctypes.addressof(np_), L.stream_handle())
    enq.append((time.perf_counter() - t0) * 1e3)
    e1.record(s)
    torch.cuda.synchronize()
    dev.append(e0.elapsed_time(e1))
print(f"gate program n=20: {np_.value} passes, enqueue {statistics.median(enq):.3f} ms, device {statistics.median(dev):.3f} ms")
