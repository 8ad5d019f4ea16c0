"""matmul 8192^3 (C2) in every precision mode: time (CUDA events, inputs resident in HBM) and
normwise error against an fp64 product on 128 sampled rows of C.

  default  TF32 tcgen05 (the bench headline)
  3xtf32   fused fp32-faithful kernel: hi/lo split in shared memory, three tcgen05 products,
           K-chunked TMEM accumulation with round-to-nearest adds between chunks
  3xtf32 split (AOL_3XTF32_SPLIT=1): the round-1 form, operands split into HBM copies
  cuBLAS fp32 (allow_tf32=False): SIMT fp32, the library reference point
Prints one JSON line."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1105_4424_b200 import builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

M = N = K = int(os.environ.get("SIZE", "8192"))
model = builders.matmul_model(M, N, K)
a = torch.randn(M * K, device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
b = torch.randn(K * N, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
rows = torch.randperm(M, generator=torch.Generator().manual_seed(1))[:128].cuda()
ref = a.view(M, K)[rows].double() @ b.view(K, N).double()


def err(c):
    return float(torch.linalg.norm(c.view(M, N)[rows].double() - ref) / torch.linalg.norm(ref))


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


out = {"M": M, "N": N, "K": K}
VARIANTS = [("default", "default", {}), ("3xtf32", "3xtf32", {}),
            ("3xtf32_split", "3xtf32", {"AOL_3XTF32_SPLIT": "1"})]
for spec in os.environ.get("X3_SWEEP", "").split():          # e.g. "64:1 128:0"
    chunk, hi = spec.split(":")
    VARIANTS.append((f"3xtf32_chunk{chunk}_hi{hi}", "3xtf32", {"AOL_3XTF32_CHUNK": chunk, "AOL_3XTF32_HI": hi}))
for name, prec, env in VARIANTS:
    for k in ("AOL_3XTF32_SPLIT", "AOL_3XTF32_CHUNK", "AOL_3XTF32_HI"):
        os.environ.pop(k, None)
    os.environ.update(env)
    ex = Executor(model, build_schedule(model, 1), {"p_a": a, "p_b": b}, 1, precision=prec)
    ms = timed(ex.run)
    c = ex.outputs(on_device=True)["p_c"]
    out[name] = {"ms": ms, "TFLOPs": 2 * M * N * K / ms / 1e9, "normwise": err(c)}
    del ex, c
    torch.cuda.empty_cache()
torch.backends.cuda.matmul.allow_tf32 = False
A, B = a.view(M, K), b.view(K, N)
ms = timed(lambda: A @ B)
out["cublas_fp32"] = {"ms": ms, "TFLOPs": 2 * M * N * K / ms / 1e9, "normwise": err(A @ B)}
print(json.dumps(out))
