"""Measure pinned H2D / D2H / bidirectional copy bandwidth (the e2e ceiling)."""
import json
import time

import torch

N = 2**28  # complex128 elements = 4 GiB
xh = torch.empty(N, dtype=torch.complex128, pin_memory=True)
yh = torch.empty(N, dtype=torch.complex128, pin_memory=True)
xd = torch.empty(N, dtype=torch.complex128, device="cuda")
yd = torch.empty(N, dtype=torch.complex128, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
out = {}
for name, fn in (("h2d", lambda: xd.copy_(xh, non_blocking=True)),
                 ("d2h", lambda: yh.copy_(yd, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out[name + "_GBs"] = round(3 * 16 * N / (time.perf_counter() - t0) / 1e9, 1)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)
    torch.cuda.synchronize()
out["bidir_GBs_each"] = round(3 * 16 * N / (time.perf_counter() - t0) / 1e9, 1)
out["bidir_ms_4GiB_each_way"] = round((time.perf_counter() - t0) / 3 * 1e3, 1)
print(json.dumps(out))
