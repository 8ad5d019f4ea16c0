"""Measured HBM read bandwidth (torch.sum over 4 GiB fp32) next to the copy peak, for read-heavy kernels."""
import json
import torch

x = torch.ones(1 << 30, dtype=torch.float32, device="cuda")
for _ in range(3):
    x.sum()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(10):
    s.record()
    x.sum()
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
y = torch.empty_like(x)
bc = 1e9
for _ in range(10):
    s.record()
    y.copy_(x)
    e.record()
    torch.cuda.synchronize()
    bc = min(bc, s.elapsed_time(e))
print(json.dumps({"read_gbs": x.numel() * 4 / best / 1e6, "copy_gbs": 2 * x.numel() * 4 / bc / 1e6}))
