"""Host memcpy rate pageable -> pinned (the staging ring's CPU side) for 16 MB pieces, by the
number of torch threads; and numpy's copyto for comparison."""
import os
import time

import numpy as np
import torch

src = np.random.default_rng(0).random(1 << 27, dtype=np.float32)          # 512 MB pageable
srct = torch.from_numpy(src).view(torch.uint8)
dst = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for th in (1, 2, 4, 8, 16, 32):
    torch.set_num_threads(th)
    t0 = time.perf_counter()
    for off in range(0, srct.numel(), dst.numel()):
        dst.copy_(srct[off:off + dst.numel()])
    dt = time.perf_counter() - t0
    print(f"torch copy_ threads={th:2d}: {srct.numel() / dt / 1e9:6.1f} GB/s", flush=True)
d = dst.numpy()
t0 = time.perf_counter()
for off in range(0, srct.numel(), dst.numel()):
    np.copyto(d, src.view(np.uint8)[off:off + dst.numel()])
dt = time.perf_counter() - t0
print(f"numpy copyto (1 thread): {srct.numel() / dt / 1e9:6.1f} GB/s")
