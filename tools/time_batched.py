"""Time a batched MatMul task (repetition space [B, M, N]) through the drop-in: the per-slice
tcgen05 path vs the exact generic kernel, CUDA events, inputs resident in HBM."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import Tiler, _capi, builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

Bn, M, N, K = 16, 2048, 2048, 2048
ta = Tiler((0, 0, 0), ((1, 0, 0), (0, 1, 0), (0, 0, 0)), ((0,), (0,), (1,)), (K,))
tb = Tiler((0, 0, 0), ((1, 0, 0), (0, 0, 0), (0, 0, 1)), ((0,), (1,), (0,)), (K,))
tc = Tiler((0, 0, 0), ((1, 0, 0), (0, 1, 0), (0, 0, 1)), ((0,), (0,), (0,)), (1,))
model = builders.tile_task_model(
    "matmul", {"a": f"in float32 [{Bn},{M},{K}]", "b": f"in float32 [{Bn},{K},{N}]", "c": f"out float32 [{Bn},{M},{N}]"},
    {"a": ta, "b": tb, "c": tc}, (Bn, M, N))
a = torch.randn(Bn * M * K, device="cuda")
b = torch.randn(Bn * K * N, device="cuda")
for prec in ("default", "exact"):
    ex = Executor(model, build_schedule(model, 1), {"p_a": a, "p_b": b}, 1, precision=prec)
    t = ex.task(ex.schedule.steps[0].task_path)
    plan = _capi.plan_name(t.ctask, 0, Bn * M * N, [ex.storage.array(t.nodes[p]).data_ptr() for p in t.port_order])
    reps = 5 if prec == "default" else 1
    ex.run()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        ex.run()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"{prec:8s} plan={plan:30s} {ms:9.3f} ms  {2 * Bn * M * N * K / (ms * 1e-3) / 1e12:8.1f} TFLOP/s")
