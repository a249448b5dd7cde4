"""Run kron_identity at config-4 size a few times (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
if len(sys.argv) > 2:
    L.tune("kron_ctas_per_sm", int(sys.argv[2]))
c4 = W.config4(22, seed=0, with_x=False)
span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
for _ in range(3):
    a = D.kron_identity(2 ** (n - 22), span, c4["right"])
    del a
torch.cuda.synchronize()
