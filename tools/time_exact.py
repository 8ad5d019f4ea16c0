"""Time the exact-order MatMul (precision="exact": k ascending, no FMA, bit-identical to the
reference spmv order) at 2048^3 and 4096^3 through the drop-in."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import Tiler, _capi, builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

for n in (2048, 4096):
    ta = Tiler((0, 0), ((1, 0), (0, 0)), ((0,), (1,)), (n,))
    tb = Tiler((0, 0), ((0, 0), (0, 1)), ((1,), (0,)), (n,))
    tc = Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,))
    model = builders.tile_task_model("matmul", {"a": f"in float32 [{n},{n}]", "b": f"in float32 [{n},{n}]",
                                                "c": f"out float32 [{n},{n}]"}, {"a": ta, "b": tb, "c": tc}, (n, n))
    a = torch.randn(n * n, device="cuda")
    b = torch.randn(n * n, device="cuda")
    ex = Executor(model, build_schedule(model, 1), {"p_a": a, "p_b": b}, 1, precision="exact")
    t = ex.task(ex.schedule.steps[0].task_path)
    plan = _capi.plan_name(t.ctask, 0, n * n, [ex.storage.array(t.nodes[p]).data_ptr() for p in t.port_order])
    ex.run()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        ex.run()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / 3
    print(f"{n}^3 exact plan={plan:20s} {ms:9.3f} ms  {2 * n ** 3 / (ms * 1e-3) / 1e12:7.2f} TFLOP/s")
