"""A layer of 14 Haar-random two-qubit gates on a random matching at n=28
(the metric's Haar4 gate kind): fused passes vs gate by gate, device time."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import workloads as W


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    rng = np.random.default_rng(0)
    perm = rng.permutation(n)
    pls = []
    for i in range(n // 2):
        a, b = int(perm[2 * i]), int(perm[2 * i + 1])
        lo, hi = min(a, b), max(a, b)
        pls.append(D.Placement(2**lo, None, 2 ** (n - 1 - hi), lo, hi, "haar",
                               gate=(W.haar(rng, 4), [a - lo, b - lo])))
    st = D.init_state(n)
    for tb in (0, 11, 12, -1):
        D.run_gates(st, pls, inplace=True, tile_bits=tb)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        for i in range(3):
            D.run_gates(st, pls, inplace=True, tile_bits=tb)
            ev[i + 1].record()
        torch.cuda.synchronize()
        ms = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(3))[1]
        print(json.dumps({"n": n, "gates": len(pls), "tile_bits": tb, "ms": round(ms, 3),
                          "gates_per_s": round(len(pls) / ms * 1e3, 1)}))


if __name__ == "__main__":
    main()
