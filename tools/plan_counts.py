"""HBM pass counts of the fused schedule per numerics mode (host only, no
device): python tools/plan_counts.py [n] [layers] [seed]
DIAQ_TUNE=fused_lookahead=0,... switches scheduler knobs."""
import ctypes
import os
import sys
import time

sys.path.insert(0, '/root/repo')
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W
from paper_2405_01250_b200.sim import _GateProgram


def plan(n, ops, mode, local_bits=None, tile_bits=0):
    lib = L.load()
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    prog = _GateProgram([p.compact() for p in pls])
    st = (ctypes.c_int * 5)()
    t0 = time.perf_counter()
    L.check(lib.diaq_fused_plan_mode(n, n if local_bits is None else local_bits, prog.n, prog.arr, tile_bits, mode, st),
            "diaq_fused_plan_mode")
    dt = time.perf_counter() - t0
    return dict(zip(["passes", "single", "phases", "folded", "smem_phases"], list(st))), dt


if __name__ == "__main__":
    for kv in filter(None, os.environ.get("DIAQ_TUNE", "").split(",")):
        k, v = kv.split("=")
        L.tune(k, int(v))
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    ops = W.random_layered_ops(n, layers, seed=seed)
    for name, mode in [("reference", L.CMUL_FMA), ("contracted", L.CMUL_CONTRACT)]:
        st, dt = plan(n, ops, mode)
        print(f"n={n} layers={layers} seed={seed} {name}: {st}  schedule {dt * 1e3:.1f} ms")
