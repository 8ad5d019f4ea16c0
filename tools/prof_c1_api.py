"""cProfile of the C1 execute_schedule call (host numpy in/out and device-resident forms)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1105_4424_b200 import builders  # noqa: E402
from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

n = 256
model = builders.matmul_model(n, n, n)
sched = build_schedule(model, 1)
rng = np.random.default_rng(0)
bind = {"p_a": rng.standard_normal(n * n, dtype=np.float32), "p_b": rng.standard_normal(n * n, dtype=np.float32)}
dbind = {k: torch.from_numpy(v).cuda() for k, v in bind.items()}
for _ in range(20):
    execute_schedule(model, sched, bind, 1)
    execute_schedule(model, sched, dbind, 1, device_outputs=True)
torch.cuda.synchronize()
for name, fn in (("numpy", lambda: execute_schedule(model, sched, bind, 1)),
                 ("device", lambda: execute_schedule(model, sched, dbind, 1, device_outputs=True))):
    t0 = time.perf_counter()
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    print(name, f"{(time.perf_counter() - t0) / 200 * 1e6:.1f} us per call")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)
