"""Time a wrapping 9-element window sum over 2^26 elements (tile_sum.batched vs the table kernel)."""
import sys, torch
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
from paper_1105_4424_b200 import Tiler, _capi
N = 1 << 26
x = torch.rand(N, device="cuda"); y = torch.empty(N, device="cuda")
tx = Tiler((N - 4,), ((1,),), ((1,),), (9,)).bind((N,), (N,))
ts = Tiler((0,), ((1,),), ((0,),), (1,)).bind((N,), (N,))
task = _capi.make_task("tile_sum", "float32", [tx, ts])
ptrs = [x.data_ptr(), y.data_ptr()]
plan = _capi.plan_name(task, 0, N, ptrs)
for _ in range(3): _capi.launch(task, 0, N, ptrs, (), 0)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): _capi.launch(task, 0, N, ptrs, (), 0)
e.record(); e.synchronize()
ms = s.elapsed_time(e) / 10
print("wrap 9-sum 2^26", plan, round(ms, 3), "ms", round(2 * N * 4 / (ms * 1e-3) / 1e9), "GB/s")
