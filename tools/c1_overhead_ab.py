"""Per-call time of execute_schedule on C1 (256^3 matmul) for the package at sys.argv[1]
(device-resident bindings + device outputs, and numpy in / numpy out), median of 5 x 200 calls."""
import statistics
import sys
import time

sys.path.insert(0, sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import aol_oracle as orc  # noqa: E402
from paper_1105_4424_b200 import Tiler, builders  # noqa: E402
from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

n = 256
g = orc.gemm_tilers(n, n, n)
model = builders.tile_task_model(
    "matmul", {"a": f"in float32 [{n},{n}]", "b": f"in float32 [{n},{n}]", "c": f"out float32 [{n},{n}]"},
    {k: Tiler(v["origin"], v["paving"], v["fitting"], v["pattern"]) for k, v in g.items()}, (n, n))
sched = build_schedule(model, 1)
rng = np.random.default_rng(0)
bind = {"p_a": rng.standard_normal(n * n, dtype=np.float32), "p_b": rng.standard_normal(n * n, dtype=np.float32)}
dbind = {k: torch.from_numpy(v).cuda() for k, v in bind.items()}
for name, fn in (("device", lambda: execute_schedule(model, sched, dbind, 1, device_outputs=True)),
                 ("numpy", lambda: execute_schedule(model, sched, bind, 1))):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    res = []
    for _ in range(5):
        t0 = time.perf_counter()
        for _ in range(200):
            fn()
        torch.cuda.synchronize()
        res.append((time.perf_counter() - t0) / 200 * 1e6)
    print(f"{sys.argv[1]}: {name} {statistics.median(res):.1f} us per call", flush=True)
