"""Repeated calls must not grow device or host memory: 3000 execute_schedule calls per form
(C1 through the prepared-executor cache with numpy / device / pinned-out forms, a streamed
stencil with pipeline=4, CG), device bytes allocated and process RSS sampled every 500 calls."""
import json
import resource
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1105_4424_b200 import builders  # noqa: E402
from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.model import model_from_dict  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

rng = np.random.default_rng(0)
n = 256
mm = builders.matmul_model(n, n, n)
mms = build_schedule(mm, 1)
hb = {"p_a": rng.standard_normal(n * n, dtype=np.float32), "p_b": rng.standard_normal(n * n, dtype=np.float32)}
db = {k: torch.from_numpy(v).cuda() for k, v in hb.items()}
pout = {"p_c": torch.empty(n * n).pin_memory()}
st = builders.stencil_model(512, 512)
sts = build_schedule(st, 2)
sb = {"p_x": rng.random(512 * 512).astype(np.float32), "p_w": np.ones(9, np.float32) / 9}
meta = json.loads((ROOT / "tests" / "golden" / "reference_golden.json").read_text())
data = np.load(ROOT / "tests" / "golden" / "reference_golden.npz")
cg = model_from_dict(meta["cg_k20"]["model"])
cgs = build_schedule(cg, 2)
cgb = {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}
forms = {
    "c1 numpy": lambda: execute_schedule(mm, mms, hb, 1),
    "c1 device": lambda: execute_schedule(mm, mms, db, 1, device_outputs=True),
    "c1 pinned out": lambda: execute_schedule(mm, mms, hb, 1, out=pout),
    "stencil pipeline=4": lambda: execute_schedule(st, sts, sb, 2, pipeline=4),
    "cg D=2": lambda: execute_schedule(cg, cgs, cgb, 2),
}
for name, fn in forms.items():
    samples = []
    for i in range(3000 if not name.startswith("cg") else 600):
        fn()
        if i % 500 == 0 or i == (2999 if not name.startswith("cg") else 599):
            torch.cuda.synchronize()
            samples.append((i, torch.cuda.memory_allocated() >> 20, resource.getrusage(resource.RUSAGE_SELF).ru_maxrss >> 10))
    print(name, "(call, device MiB allocated, max RSS MiB):", samples, flush=True)
