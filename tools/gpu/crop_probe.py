"""Time 2-D crops (tile_copy.rows_shift / tma_plane) for several extents and offsets."""
import sys, torch
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
from paper_1105_4424_b200 import Tiler, _capi
N = 16384
x = torch.rand(N * N, device="cuda"); y = torch.empty(N * N, device="cuda")
for (o0, o1), (R0, R1) in (((3, 5), (16376, 16376)), ((3, 5), (16381, 16379)), ((3, 5), (16381, 16376)),
                           ((3, 5), (16376, 16379)), ((0, 0), (16376, 16376)), ((3, 4), (16376, 16376))):
    src = Tiler((o0, o1), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((N, N), (R0, R1))
    dst = Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((N, N), (R0, R1))
    task = _capi.make_task("tile_copy", "float32", [src, dst])
    T = R0 * R1
    ptrs = [x.data_ptr(), y.data_ptr()]
    plan = _capi.plan_name(task, 0, T, ptrs)
    for _ in range(3): _capi.launch(task, 0, T, ptrs, (), 0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): _capi.launch(task, 0, T, ptrs, (), 0)
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 10
    print((o0, o1), (R0, R1), plan, round(ms, 3), "ms", round(2 * T * 4 / (ms * 1e-3) / 1e9), "GB/s", flush=True)
