"""CG (golden cg_k20) through execute_schedule with and without a caller stream, D = 1..6:
iterations and x must match bit for bit."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.model import model_from_dict  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

meta = json.loads((ROOT / "tests" / "golden" / "reference_golden.json").read_text())
data = np.load(ROOT / "tests" / "golden" / "reference_golden.npz")
model = model_from_dict(meta["cg_k20"]["model"])
bind = {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}
for D in range(1, 7):
    sched = build_schedule(model, D)
    for kw in ({}, {"graphs": False}):
        plain = execute_schedule(model, sched, bind, D, **kw)
        for rep in range(3):
            s = torch.cuda.Stream()
            r = execute_schedule(model, sched, bind, D, stream=s, **kw)
            torch.cuda.synchronize()
            same = np.array_equal(np.asarray(r.outputs["x"]), np.asarray(plain.outputs["x"]))
            if not same or r.iterations != plain.iterations:
                d = np.max(np.abs(np.asarray(r.outputs["x"]) - np.asarray(plain.outputs["x"])))
                print(f"D={D} {kw} rep={rep}: MISMATCH iters {r.iterations} vs {plain.iterations}, max|dx| {d:.3e}",
                      flush=True)
    print(f"D={D} done", flush=True)
