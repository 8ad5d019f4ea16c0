"""cProfile of the C1 path: execute_schedule on a 256^3 matmul, host numpy in/out."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

w = bench.C1Workload(torch, torch.device("cuda:0"), 0, 1)
for _ in range(20):
    w.step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    w.step()
print(f"{(time.perf_counter() - t0) / 200 * 1e6:.1f} us per execute_schedule")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    w.step()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
