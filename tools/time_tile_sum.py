"""Time tile_sum (pattern reduction, pattern order) on row sums and column sums of a 16384^2
fp32 array through the drop-in: plan and GB/s (array read once + sums written), CUDA events."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import Tiler, _capi, builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

n = 16384
cases = {"row sums": Tiler((0, 0), ((1,), (0,)), ((0,), (1,)), (n,)),
         "column sums": Tiler((0, 0), ((0,), (1,)), ((1,), (0,)), (n,))}
x = torch.rand(n * n, device="cuda")
for name, tx in cases.items():
    ts = Tiler((0,), ((1,),), ((0,),), (1,))
    model = builders.tile_task_model("tile_sum", {"x": f"in float32 [{n},{n}]", "s": f"out float32 [{n}]"},
                                     {"x": tx, "s": ts}, (n,))
    ex = Executor(model, build_schedule(model, 1), {"p_x": x}, 1)
    t = ex.task(ex.schedule.steps[0].task_path)
    ptrs = [ex.storage.array(t.nodes[p]).data_ptr() for p in t.port_order]
    plan = _capi.plan_name(t.ctask, 0, n, ptrs)
    for _ in range(3):
        ex.run()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        ex.run()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"{name:12s} plan={plan:22s} {ms:8.3f} ms  {(n * n + n) * 4 / (ms * 1e-3) / 1e9:8.1f} GB/s")
