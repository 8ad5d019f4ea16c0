import sys, torch
sys.path.insert(0, '.')
from paper_1105_4424_b200 import Tiler, _capi
N = 1 << 28
x = torch.rand(N, device="cuda"); y = torch.empty(N, device="cuda")
cases = {"1-D": (Tiler((12345,), ((1,),), ((0,),), (1,)).bind((N,), (N,)), Tiler((0,), ((1,),), ((0,),), (1,)).bind((N,), (N,))),
         "2-D": (Tiler((3, 5), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((16384, 16384), (16384, 16384)),
                 Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((16384, 16384), (16384, 16384)))}
for name, (src, dst) in cases.items():
    task = _capi.make_task("tile_copy", "float32", [src, dst])
    for mode in ("whole", "halves"):
        def run():
            if mode == "whole":
                _capi.launch(task, 0, N, [x.data_ptr(), y.data_ptr()], (), 0)
            else:
                _capi.launch(task, 0, N // 2, [x.data_ptr(), y.data_ptr()], (), 0)
                _capi.launch(task, N // 2, N - N // 2, [x.data_ptr(), y.data_ptr()], (), 0)
        plan = _capi.plan_name(task, 0, N if mode == "whole" else N // 2, [x.data_ptr(), y.data_ptr()])
        for _ in range(2): run()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5): run()
        e.record(); e.synchronize()
        ms = s.elapsed_time(e) / 5
        print(name, mode, plan, round(ms, 3), "ms", round(2 * N * 4 / (ms * 1e-3) / 1e9), "GB/s")
