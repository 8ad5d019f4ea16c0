"""Time the matmul task at 8192^3 in precision="3xtf32" (fp32-accurate) vs the TF32 default and
torch fp32 (cuBLAS, allow_tf32=False), CUDA events, inputs resident in HBM."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import aol_oracle as orc  # noqa: E402  (tiler dicts only)
from paper_1105_4424_b200 import Tiler, builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

M = N = K = 8192
g = orc.gemm_tilers(M, N, K)
model = builders.tile_task_model(
    "matmul", {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]", "c": f"out float32 [{M},{N}]"},
    {k: Tiler(v["origin"], v["paving"], v["fitting"], v["pattern"]) for k, v in g.items()}, (M, N))
a = torch.randn(M * K, device="cuda")
b = torch.randn(K * N, device="cuda")


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


for prec in ("default", "3xtf32"):
    ex = Executor(model, build_schedule(model, 1), {"p_a": a, "p_b": b}, 1, precision=prec)
    ms = timed(ex.run)
    print(f"{prec:8s} {ms:7.3f} ms  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s")
torch.backends.cuda.matmul.allow_tf32 = False
A, B = a.view(M, K), b.view(K, N)
ms = timed(lambda: A @ B)
print(f"cublas fp32 {ms:7.3f} ms  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s")
