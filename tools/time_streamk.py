"""TF32 pair GEMM at C2's per-rank shards (M = 8192/ranks rows, N = K = 8192): split-K tail on
and off, alternated in one process (AOL_GEMM_STREAMK is read per launch), median of 3 each."""
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1105_4424_b200 import builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

K = N = 8192
a = torch.randn(8192 * K, device="cuda")
b = torch.randn(K * N, device="cuda")


def timed(ex, reps=30):
    for _ in range(3):
        ex.run()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        ex.run()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


for ranks in [int(x) for x in (sys.argv[1:] or ["1", "2", "4", "8", "16"])]:
    M = 8192 // ranks
    model = builders.matmul_model(M, N, K)
    ex = Executor(model, build_schedule(model, 1), {"p_a": a[:M * K], "p_b": b}, 1)
    res = {"0": [], "1": []}
    for _ in range(3):
        for mode in ("0", "1"):
            os.environ["AOL_GEMM_STREAMK"] = mode
            res[mode].append(timed(ex))
    off, on = statistics.median(res["0"]), statistics.median(res["1"])
    f = 2.0 * M * N * K / 1e9
    print(f"M={M:5d} ({ranks:2d} ranks): off {off:.4f} ms {f / off:6.1f} TF | split-K tail {on:.4f} ms "
          f"{f / on:6.1f} TF | {off / on:.3f}x", flush=True)
    del ex
