"""Per-pass device times (CUDA events around each HBM pass) of the n=28
random layer under diaq_tune settings:  python tools/pass_split.py "a=1,b=0" ...
Prints, per setting and numerics, the median ms of every pass of the layer."""
import statistics
import sys

sys.path.insert(0, '/root/repo')
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

settings = [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in a.split(",")) for a in sys.argv[1:]] or [{}]
knobs = sorted({k for st_ in settings for k in st_})
n = 28
ops = W.random_layered_ops(n, 1, seed=0)
pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
st = D.init_state(n)
for mode, name in ((None, "reference"), (L.CMUL_CONTRACT, "contracted")):
    for setting in settings:
        for k in knobs:
            L.tune(k, setting.get(k, 0))
        D.run_gates(st, pls, cmul_mode=mode, inplace=True)
        L.call("diaq_jit_wait", -1.0)
        timer = L.Timer(len(pls) + 1)
        per = []
        for _ in range(7):
            D.run_gates(st, pls, cmul_mode=mode, inplace=True, timer=timer)
            ms = timer.elapsed_ms()
            per.append([float(v) for v in ms if v > 0])
        cols = list(zip(*per))
        tag = ",".join(f"{k}={v}" for k, v in setting.items())
        print(f"{name:10s} {tag:32s}: " + "  ".join(f"{statistics.median(c):.4f}" for c in cols), flush=True)
