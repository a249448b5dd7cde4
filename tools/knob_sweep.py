"""Device time per HBM pass of the n=28 random layer under diaq_tune knob
settings, both numerics:
  python tools/knob_sweep.py KNOB v1 v2 ...        one knob, several values
  python tools/knob_sweep.py -s "a=1,b=0" "a=0"    several full settings
Median of 5 x 4 layers per setting."""
import ctypes
import statistics
import sys

sys.path.insert(0, '/root/repo')
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

if sys.argv[1] == "-s":
    settings = [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in a.split(",")) for a in sys.argv[2:]]
else:
    settings = [{sys.argv[1]: int(v)} for v in sys.argv[2:]]
knobs = sorted({k for st_ in settings for k in st_})
n = int(__import__("os").environ.get("KNOB_N", "28"))
ops = W.random_layered_ops(n, 1, seed=0)
pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
st = D.init_state(n)
s = torch.cuda.current_stream()
for mode, name in ((None, "reference"), (L.CMUL_CONTRACT, "contracted")):
    D.run_gates(st, pls, cmul_mode=mode, inplace=True)
    L.call("diaq_jit_wait", -1.0)
    for setting in settings:
        for k in knobs:
            L.tune(k, setting.get(k, 0))
        D.run_gates(st, pls, cmul_mode=mode, inplace=True)
        L.call("diaq_jit_wait", -1.0)
        ts = []
        for _ in range(5):
            l0 = L.launch_count()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(4):
                D.run_gates(st, pls, cmul_mode=mode, inplace=True)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / (L.launch_count() - l0))
        tag = ",".join(f"{k}={v}" for k, v in setting.items())
        print(f"{name:10s} {tag:30s}: {statistics.median(ts):.4f} ms/pass  (min {min(ts):.4f})", flush=True)
