"""Time tile_filter shapes outside the configs' specialised kernels (1-D FIR, decimating FIR,
2-D 3x3 downsample, a 16-tap line filter) on ~1e8-element arrays: plan and GB/s."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import Tiler, _capi, builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402


def run(name, x_arr, tx, y_arr, ty, rep, npx, npy):
    w = (np.arange(npx * npy, dtype=np.float32) + 1) / (npx * npy)
    fmt = lambda a: ",".join(map(str, a))  # noqa: E731
    model = builders.tile_task_model(
        "tile_filter", {"x": f"in float32 [{fmt(x_arr)}]", "w": f"in float32 [{w.size}]",
                        "y": f"out float32 [{fmt(y_arr)}]"}, {"x": tx, "y": ty}, rep)
    nx, ny = int(np.prod(x_arr)), int(np.prod(y_arr))
    x = torch.rand(nx, device="cuda")
    ex = Executor(model, build_schedule(model, 1), {"p_x": x, "p_w": torch.from_numpy(w).cuda()}, 1)
    t = ex.task(ex.schedule.steps[0].task_path)
    ptrs = [ex.storage.array(t.nodes[p]).data_ptr() for p in t.port_order]
    plan = _capi.plan_name(t.ctask, 0, int(np.prod(rep)), ptrs)
    for _ in range(2):
        ex.run()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        ex.run()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"{name:28s} plan={plan:28s} {ms:8.3f} ms  {(nx + ny) * 4 / (ms * 1e-3) / 1e9:8.1f} GB/s", flush=True)


N = 1 << 27
run("1-D FIR 8 taps", (N,), Tiler((0,), ((1,),), ((1,),), (8,)), (N,), Tiler((0,), ((1,),), ((0,),), (1,)), (N,), 8, 1)
run("1-D FIR 16 taps", (N,), Tiler((0,), ((1,),), ((1,),), (16,)), (N,), Tiler((0,), ((1,),), ((0,),), (1,)), (N,), 16, 1)
run("decimate 16 taps / 4", (N,), Tiler((0,), ((4,),), ((1,),), (16,)), (N // 4,),
    Tiler((0,), ((1,),), ((0,),), (1,)), (N // 4,), 16, 1)
H = W = 8192
run("2-D 2x2 downsample", (H, W), Tiler((0, 0), ((2, 0), (0, 2)), ((1, 0), (0, 1)), (2, 2)), (H // 2, W // 2),
    Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,)), (H // 2, W // 2), 4, 1)
run("line 16 taps along rows /8", (64, 2048, 2048), Tiler((0, 0, 0), ((1, 0, 0), (0, 1, 0), (0, 0, 8)), ((0,), (0,), (1,)), (16,)),
    (64, 2048, 256 * 2), Tiler((0, 0, 0), ((1, 0, 0), (0, 1, 0), (0, 0, 2)), ((0,), (0,), (1,)), (2,)), (64, 2048, 256), 16, 2)
run("2-D 3x3 stride 2 (torus)", (H, W), Tiler((H - 1, W - 1), ((2, 0), (0, 2)), ((1, 0), (0, 1)), (3, 3)),
    (H // 2, W // 2), Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,)), (H // 2, W // 2), 9, 1)
run("2-D 2x2 outputs per 4x4 window", (H, W), Tiler((0, 0), ((4, 0), (0, 4)), ((1, 0), (0, 1)), (4, 4)),
    (H // 2, W // 2), Tiler((0, 0), ((2, 0), (0, 2)), ((1, 0), (0, 1)), (2, 2)), (H // 4, W // 4), 16, 4)
run("1-D 8 taps /2, 2 outputs", (N,), Tiler((0,), ((2,),), ((1,),), (8,)), (N,), Tiler((0,), ((2,),), ((1,),), (2,)), (N // 2,), 8, 2)
run("1-D 13 taps /8, 3 outputs", (N,), Tiler((0,), ((8,),), ((1,),), (13,)), (N // 8 * 3,),
    Tiler((0,), ((3,),), ((1,),), (3,)), (N // 8,), 13, 3)
run("1-D 7 taps /3 (wrap)", (3 * (N // 3),), Tiler((5,), ((3,),), ((1,),), (7,)), (N // 3,),
    Tiler((0,), ((1,),), ((0,),), (1,)), (N // 3,), 7, 1)
run("rows 16 taps /8, 1 output", (64, 2048, 2048), Tiler((0, 0, 0), ((1, 0, 0), (0, 1, 0), (0, 0, 8)), ((0,), (0,), (1,)), (16,)),
    (64, 2048, 256), Tiler((0, 0, 0), ((1, 0, 0), (0, 1, 0), (0, 0, 1)), ((0,), (0,), (0,)), (1,)), (64, 2048, 256), 16, 1)
