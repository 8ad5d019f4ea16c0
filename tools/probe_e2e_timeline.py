"""Timeline of one C2 e2e step through execute_schedule(pipeline=8) with pinned buffers (the 2-D
block path): wall time per call, then CUDA-event timestamps of every H2D, GEMM and D2H."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1105_4424_b200 import builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

M = N = K = 8192
model = builders.matmul_model(M, N, K)
sched = build_schedule(model, 1)
g = torch.Generator().manual_seed(7)
ha = torch.randn(M * K, generator=g).pin_memory()
hb = torch.randn(K * N, generator=g).pin_memory()
hc = torch.empty(M * N).pin_memory()


NUMPY = os.environ.get("PROBE_NUMPY") == "1"
na, nb = ha.numpy().copy(), hb.numpy().copy()


def call():
    if NUMPY:                                       # the reference's call: pageable in, fresh out
        ex = Executor(model, sched, {"p_a": na, "p_b": nb}, 1, pipeline=8)
        ex.run_streamed(None)
    else:
        ex = Executor(model, sched, {"p_a": ha, "p_b": hb}, 1, pipeline=8)
        ex.run_streamed({"p_c": hc})
    return ex


for _ in range(3):
    call()
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    call()
    print(f"call {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
os.environ["AOL_E2E_TIMELINE"] = "1"
ex = call()
for tag, ms in ex.timeline:
    print(f"{tag:10s} {ms:8.3f} ms")
