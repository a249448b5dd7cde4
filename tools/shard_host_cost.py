"""Host vs device cost of the sharded run loop: config-5 shape at n=29 over
2 emulated shards (4 layers), wall clock, CUDA-event device time and a
cProfile of one run:  python tools/shard_host_cost.py [n] [world] [layers]"""
import cProfile
import io
import pstats
import sys
import time

sys.path.insert(0, '/root/repo')
import torch

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W
from paper_2405_01250_b200.shard import run_emulated

n = int(sys.argv[1]) if len(sys.argv) > 1 else 29
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
layers = int(sys.argv[3]) if len(sys.argv) > 3 else 4
ops = W.random_layered_ops(n, layers, seed=0)
pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
for remap in (False, True):
    run_emulated(n, world, pls, remap=remap)
    L.call("diaq_jit_wait", -1.0)
    torch.cuda.synchronize()
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        shards, st = run_emulated(n, world, pls, remap=remap)
        t_enq = time.perf_counter() - t0
        e1.record()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t0
        print(f"remap={remap}: wall {t_wall * 1e3:.1f} ms, host until return {t_enq * 1e3:.1f} ms, "
              f"device {e0.elapsed_time(e1):.1f} ms, stats {st}")
        del shards
pr = cProfile.Profile()
pr.enable()
shards, st = run_emulated(n, world, pls, remap=False)
torch.cuda.synchronize()
pr.disable()
buf = io.StringIO()
pstats.Stats(pr, stream=buf).sort_stats("cumtime").print_stats(25)
print(buf.getvalue()[:6000])
