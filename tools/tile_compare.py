import sys, json, torch
sys.path.insert(0, '.')
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import workloads as W
for n, layers in ((28, 1), (30, 20), (20, 40)):
    ops = W.random_layered_ops(n, layers, seed=0)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    st = D.init_state(n, max_qubits=30)
    for tb in (11, 12, -1):
        D.run_gates(st, pls, inplace=True, tile_bits=tb)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        for i in range(3):
            D.run_gates(st, pls, inplace=True, tile_bits=tb)
            ev[i + 1].record()
        torch.cuda.synchronize()
        ms = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(3))[1]
        print(json.dumps({"n": n, "layers": layers, "tile": tb, "ms": round(ms, 3), "gates_per_s": round(len(pls) / ms * 1e3, 1)}))
    del st
