"""Time toroidal K x K box stencils (K = 3, 5, 7) on a 16384^2 fp32 torus through the drop-in:
which plan each takes and its GB/s (x read once + y written once), CUDA events."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import Tiler, _capi, builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

n = 16384
for K in (3, 5, 7):
    h = K // 2
    tx = Tiler((n - h, n - h), ((1, 0), (0, 1)), ((1, 0), (0, 1)), (K, K))
    ty = Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,))
    w = (np.arange(K * K, dtype=np.float32) + 1) / (K * K)
    model = builders.tile_task_model(
        "stencil", {"x": f"in float32 [{n},{n}]", "w": f"in float32 [{K * K}]", "y": f"out float32 [{n},{n}]"},
        {"x": tx, "y": ty}, (n, n))
    x = torch.rand(n * n, device="cuda")
    ex = Executor(model, build_schedule(model, 1), {"p_x": x, "p_w": torch.from_numpy(w).cuda()}, 1)
    t = ex.task(ex.schedule.steps[0].task_path)
    ptrs = [ex.storage.array(t.nodes[p]).data_ptr() for p in t.port_order]
    plan = _capi.plan_name(t.ctask, 0, n * n, ptrs)
    for _ in range(3):
        ex.run()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        ex.run()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"K={K} plan={plan:28s} {ms:7.3f} ms  {2 * n * n * 4 / (ms * 1e-3) / 1e9:7.1f} GB/s")
    del ex, x
    torch.cuda.empty_cache()
