"""m = 8 row-stride sweep point inside the bench's SweepWorkload (main point resident, table
timing) against the same point built alone: is the bench-context slowdown the kernel's?"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
sw = bench.SweepWorkload(torch, dev, 0, 1)
pts = [(8, "rowstride", 10 ** 8), (8, "rowstride", 10 ** 7), (16, "rowstride", 10 ** 8), (8, "rowstride", 10 ** 8)]
sw.points = pts
for r in sw.measure_points():
    print("with main resident:", r["m"], r["paving"], r["T"], r["plan"], f"{r['ms']:.3f} ms floor_frac {r['floor_frac']:.3f} "
          f"copy {r.get('frac_of_copy', 0):.3f}", flush=True)
del sw.task
torch.cuda.empty_cache()
sw.points = pts
for r in sw.measure_points():
    print("main freed:        ", r["m"], r["paving"], r["T"], r["plan"], f"{r['ms']:.3f} ms floor_frac {r['floor_frac']:.3f} "
          f"copy {r.get('frac_of_copy', 0):.3f}", flush=True)
