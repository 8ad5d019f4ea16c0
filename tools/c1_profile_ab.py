"""cProfile of the device-resident C1 call for the package at sys.argv[1] (cumulative)."""
import cProfile
import pstats
import sys

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
dbind = {k: torch.from_numpy(rng.standard_normal(n * n, dtype=np.float32)).cuda() for k in ("p_a", "p_b")}
for _ in range(50):
    execute_schedule(model, sched, dbind, 1, device_outputs=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    execute_schedule(model, sched, dbind, 1, device_outputs=True)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
