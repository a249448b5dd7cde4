import sys, time, torch
sys.path.insert(0, '.')
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import workloads as W
for n in (20, 24, 28):
    ops = W.random_layered_ops(n, 1, seed=0)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    st = D.run_gates(D.init_state(n), pls, inplace=True)
    D.measure_all_sample(st, 16, 0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        D.measure_all_sample(st, 1024, 1)
    torch.cuda.synchronize()
    print(n, "sample 1024 shots ms", (time.perf_counter() - t) / 3 * 1e3)
