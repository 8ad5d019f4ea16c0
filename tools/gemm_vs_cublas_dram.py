"""One launch each of the drop-in's TF32 GEMM (C2 8192^3) and cuBLAS TF32 (torch.matmul,
allow_tf32=True) on the same operands -- run under ncu to compare DRAM bytes and L2 hit rate:

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
      python tools/gemm_vs_cublas_dram.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

n = 8192
model = builders.matmul_model(n, n, n)
a = torch.randn(n * n, device="cuda")
b = torch.randn(n * n, device="cuda")
ex = Executor(model, build_schedule(model, 1), {"p_a": a, "p_b": b}, 1)
ex.run()
torch.backends.cuda.matmul.allow_tf32 = True
c = a.view(n, n) @ b.view(n, n)
torch.cuda.synchronize()
