"""Break one CG solve (bench --workload cg) into setup / first run / cached runs."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402

w = bench.WORKLOADS[__import__("os").environ.get("DIAG_WL", "cg")](torch, torch.device("cuda:0"), 0, 1)
modes = sys.argv[1:] or ["graphs"]
for mode in modes:
    graphs = mode != "eager"
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ex = Executor(w.model, w.schedule, w.bind, 1, graphs=graphs)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    times = []
    for rep in range(int(__import__("os").environ.get("DIAG_REPS", "4")) if graphs else 1):
        it0 = ex.iterations
        ta = time.perf_counter()
        ex.run()
        torch.cuda.synchronize()
        times.append((time.perf_counter() - ta, ex.iterations - it0))
    print(f"{mode}: setup {1e3*(t1-t0):.2f} ms; runs " +
          ", ".join(f"{1e3*t:.2f} ms ({n} it, {1e6*t/n:.1f} us/it)" for t, n in times) +
          f"; persistent={getattr(ex, 'persistent_loops', 0)}")
