"""Break one matmul e2e step (execute_schedule with host buffers) into setup and streamed run."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402

w = bench.WORKLOADS["matmul"](torch, torch.device("cuda:0"), 0, 1)
w.e2e_setup()
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ex = Executor(w.model, w.schedule, w.hin, 1, pipeline=w.pipeline)
    t1 = time.perf_counter()
    ex.run_streamed(out=w.hout)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"setup {1e3 * (t1 - t0):.2f} ms  streamed {1e3 * (t2 - t1):.2f} ms")
