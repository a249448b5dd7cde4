"""Device time of the construction kernels at config-4 size (n=28):
kron_identity (write-only, 16 B per stored element) and
build_span_unitary / from_dense at their own sizes.  CUDA events on the
launching stream, median of 10 after 3 warm-ups."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    tm = L.Timer(reps + 1)
    torch.cuda.synchronize()
    tm.record(0)
    for i in range(reps):
        fn()
        tm.record(i + 1)
    torch.cuda.synchronize()
    e = sorted(tm.elapsed_ms().tolist())
    return e[len(e) // 2]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    c4 = W.config4(22, seed=0, with_x=False)
    u = D.from_dense(c4["u4"], 0.0)
    span = D.build_span_unitary(u, c4["positions"], c4["span"])
    out = {}
    a = D.kron_identity(2 ** (n - 22), span, c4["right"])
    stored = sum(2 ** n - abs(d) for d in a.diag_indices()) * 16
    del a
    for flat, ctas in ((0, 8), (1, 32)):
        L.tune("kron_flat", flat)
        L.tune("kron_ctas_per_sm", ctas)
        ms = timed(lambda: D.kron_identity(2 ** (n - 22), span, c4["right"]))
        out[f"kron_identity_flat{flat}_c{ctas}"] = {"n": n, "ms": round(ms, 3), "bytes": stored,
                                                    "GB_s": round(stored / ms / 1e6, 1)}
    L.tune("kron_flat", 1)
    L.tune("kron_ctas_per_sm", 8)
    ms = timed(lambda: D.build_span_unitary(u, c4["positions"], c4["span"]))
    out["build_span_unitary_19"] = {"ms": round(ms, 4)}
    buf = torch.empty(2 ** 31, dtype=torch.complex128, device="cuda")  # 34 GB
    ms = timed(lambda: buf.zero_())
    out["torch_zero_34GB"] = {"ms": round(ms, 3), "GB_s": round(buf.numel() * 16 / ms / 1e6, 1)}
    del buf
    print(json.dumps(out))


if __name__ == "__main__":
    main()
