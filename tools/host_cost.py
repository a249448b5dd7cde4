import time, sys, ctypes
sys.path.insert(0,'.')
import torch
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import workloads as W, _lib as L
from paper_2405_01250_b200.sim import _GateProgram
ops = W.random_layered_ops(20, 40, seed=0)
pls = D.compile_circuit(D.Circuit(20, [D.GateOp(*o) for o in ops]), span_limit=20)
st = D.init_state(20)
for _ in range(3): D.run_gates(st, pls, inplace=True)
torch.cuda.synchronize()
prog = _GateProgram.for_placements(pls)
s = L.stream_handle()
x = st.device_amps
t = time.perf_counter()
for _ in range(10):
    L.call("diaq_run_gates_fused", 20, prog.n, prog.arr, x.data_ptr(), 1, 12, None, None, s)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host ms per native call", (t1 - t) / 10 * 1e3, "total ms per call incl drain", (t2 - t) / 10 * 1e3)
t = time.perf_counter()
for _ in range(10):
    D.run_gates(st, pls, inplace=True)
torch.cuda.synchronize()
print("run_gates wall ms", (time.perf_counter() - t) / 10 * 1e3)
