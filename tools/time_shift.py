"""Time toroidal (wrapping) shifts through tile_copy: a 1-D circular shift of 2^28 elements and a 2-D torus shift of 16384^2."""
import sys, torch
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import Tiler, _capi
N = 1 << 28
x = torch.rand(N, device="cuda"); y = torch.empty(N, device="cuda")
for name, src in (("shift 1-D", Tiler((12345,), ((1,),), ((0,),), (1,)).bind((N,), (N,))),
                  ("shift rows 2-D", Tiler((3, 5), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((16384, 16384), (16384, 16384))),
                  ("crop 2-D (3, 5)", Tiler((3, 5), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((16384, 16384), (16376, 16376)))):
    dst = Tiler((0,), ((1,),), ((0,),), (1,)).bind((N,), (N,)) if src.rep == (N,) else Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((16384, 16384), src.rep)
    task = _capi.make_task("tile_copy", "float32", [src, dst])
    T = src.rep_total
    plan = _capi.plan_name(task, 0, T, [x.data_ptr(), y.data_ptr()])
    for _ in range(2): _capi.launch(task, 0, T, [x.data_ptr(), y.data_ptr()], (), 0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): _capi.launch(task, 0, T, [x.data_ptr(), y.data_ptr()], (), 0)
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 5
    print(name, plan, round(ms, 3), "ms", round(2 * T * 4 / (ms * 1e-3) / 1e9), "GB/s")
