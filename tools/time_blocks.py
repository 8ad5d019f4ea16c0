"""Time 2-D block extraction / reassembly through tile_copy (Array-OL block tilers: an
[H, W] image cut into b x b blocks, each block a pattern, written as a dense [nblocks, b*b]
stream, and back): plan and GB/s."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import Tiler, _capi  # noqa: E402

H = W = 8192


def timed(task, T, ptrs):
    for _ in range(2):
        _capi.launch(task, 0, T, ptrs, (), 0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        _capi.launch(task, 0, T, ptrs, (), 0)
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / 5


x = torch.rand(H * W, device="cuda")
y = torch.empty(H * W, device="cuda")
for b in (4, 8, 16, 32):
    nb = (H // b, W // b)
    blk = Tiler((0, 0), ((b, 0), (0, b)), ((1, 0), (0, 1)), (b, b)).bind((H, W), nb)
    dense = Tiler((0,), ((W // b * b * b, b * b),), ((b, 1),), (b, b)).bind((H * W,), nb)
    for name, src, dst, a, c in (("extract", blk, dense, x, y), ("assemble", dense, blk, y, x)):
        task = _capi.make_task("tile_copy", "float32", [src, dst])
        T = nb[0] * nb[1]
        plan = _capi.plan_name(task, 0, T, [a.data_ptr(), c.data_ptr()])
        ms = timed(task, T, [a.data_ptr(), c.data_ptr()])
        print(f"{b:2d}x{b:<2d} {name:9s} plan={plan:24s} {ms:7.3f} ms  {2 * H * W * 4 / (ms * 1e-3) / 1e9:7.1f} GB/s",
              flush=True)
