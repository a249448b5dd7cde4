"""Profile driver: the device sampler on a random n-qubit state (default 20)."""
import sys

sys.path.insert(0, '/root/repo')
import numpy as np

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
x = W.random_state(np.random.default_rng(0), 2**n)
st = D.StateVector(n, x)
for _ in range(3):
    D.measure_all_sample(st, 1024, 0)
print("ok")
