"""C1 (matmul 256^3) execute_schedule phases, host wall time per call: Executor construction
(DeviceStorage: arena, uploads, zero-fill; task validation), run(), outputs()."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1105_4424_b200 import builders  # noqa: E402
from paper_1105_4424_b200.executor import DeviceStorage, Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

n = 256
model = builders.matmul_model(n, n, n)
sched = build_schedule(model, 1)
rng = np.random.default_rng(0)
hb = {"p_a": rng.standard_normal(n * n, dtype=np.float32), "p_b": rng.standard_normal(n * n, dtype=np.float32)}
db = {k: torch.from_numpy(v).cuda() for k, v in hb.items()}
dev = torch.device("cuda", 0)
for name, bind, on_dev in (("device", db, True), ("numpy", hb, False)):
    t = {"storage": 0.0, "executor": 0.0, "run": 0.0, "outputs": 0.0}
    N = 300
    for i in range(N + 20):
        t0 = time.perf_counter()
        DeviceStorage(model, bind, dev)
        t1 = time.perf_counter()
        ex = Executor(model, sched, bind, 1)
        t2 = time.perf_counter()
        ex.run()
        t3 = time.perf_counter()
        ex.outputs(on_device=on_dev)
        t4 = time.perf_counter()
        if i >= 20:
            t["storage"] += t1 - t0
            t["executor"] += t2 - t1
            t["run"] += t3 - t2
            t["outputs"] += t4 - t3
    torch.cuda.synchronize()
    print(name, {k: round(v / N * 1e6, 1) for k, v in t.items()}, "us", flush=True)
