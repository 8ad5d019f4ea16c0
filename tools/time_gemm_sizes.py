"""TF32 GEMM at 1024..8192 (square): the drop-in's kernel (Executor.run, inputs in HBM) against
cuBLAS TF32 (torch.matmul, allow_tf32) on the same operands, CUDA events, best of 20."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402


def best(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


torch.backends.cuda.matmul.allow_tf32 = True
for n in (1024, 2048, 3072, 4096, 6144, 8192):
    a = torch.randn(n * n, device="cuda")
    b = torch.randn(n * n, device="cuda")
    model = builders.matmul_model(n, n, n)
    ex = Executor(model, build_schedule(model, 1), {"p_a": a, "p_b": b}, 1)
    t_ours = best(ex.run)
    A, B = a.view(n, n), b.view(n, n)
    t_cub = best(lambda: A @ B)
    f = 2.0 * n ** 3
    print(f"{n:5d}^3  ours {f / t_ours / 1e9:7.1f} TFLOP/s  cuBLAS TF32 {f / t_cub / 1e9:7.1f}  ratio {t_cub / t_ours:.3f}",
          flush=True)
    del ex, a, b
    torch.cuda.empty_cache()
