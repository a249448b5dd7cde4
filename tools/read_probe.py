"""Pure-read and multi-stream read bandwidth probes (context for the spmv roofline)."""
import json

import torch

out = {}
x = torch.ones(2**31, dtype=torch.float64, device="cuda")  # 16 GiB
for _ in range(2):
    x.sum()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    x.sum()
e1.record()
torch.cuda.synchronize()
out["torch_sum_read_GBs"] = round(5 * x.numel() * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
y = torch.empty_like(x)
e0.record()
for _ in range(5):
    y.copy_(x)
e1.record()
torch.cuda.synchronize()
out["torch_copy_GBs"] = round(5 * 2 * x.numel() * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
print(json.dumps(out))
