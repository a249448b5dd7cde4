"""Device time of the row-sharded spmv kernel (diaq_spmv_sharded) against the
single-GPU banded cp.async kernel at config-4 size, one GPU: P = 1 (all x
local) and P = 2 emulated (this rank's half of the rows, x split in two
buffers on the same device -- the boundary-crossing reads hit the other
buffer exactly as they would hit a peer mapping)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W
from paper_2405_01250_b200.shard import ShardedDiaq


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        fn()
        ev[i + 1].record()
    torch.cuda.synchronize()
    e = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
    return e[len(e) // 2]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    c4 = W.config4(22, seed=0, with_x=False)
    span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    a = D.kron_identity(2 ** (n - 22), span, c4["right"])
    N = 2**n
    x = torch.randn(N, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    offs = a.diag_indices()
    alg = sum(N - abs(d) for d in offs) * 16 + 32 * N
    out = {"n": n}
    ms = timed(lambda: D.spmv(a, x, out=y))
    out["diaq_spmv"] = {"ms": round(ms, 3), "GB_s": round(alg / ms / 1e6, 1)}
    want = y.clone()
    for world in (1, 2):
        sd = ShardedDiaq.from_matrix(a, 0, world)
        parts = list(x.chunk(world))
        ys = torch.empty(sd.nrows, dtype=torch.complex128, device="cuda")
        ms = timed(lambda: sd.spmv(parts, ys))
        rows_alg = alg / world
        same = bool(torch.equal(ys, want[:sd.nrows]))
        out[f"sharded_P{world}_rank0"] = {"ms": round(ms, 3), "GB_s": round(rows_alg / ms / 1e6, 1), "bitwise": same}
        del sd, ys
    print(json.dumps(out))


if __name__ == "__main__":
    main()
