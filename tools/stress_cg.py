"""Random SPD sparse systems through the CG case study (cg.gmodel resized, refexec.py:552-596):
the device loop (persistent interpreter / CUDA graph) must give the same iteration count and
bit-identical x as host-driven iterations (graphs=False) at random n, nnz pattern and D.

    SEED=1 CASES=40 python tools/stress_cg.py"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.model import model_from_dict  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

meta = json.loads((ROOT / "tests" / "golden" / "reference_golden.json").read_text())
base = meta["cg_k20"]["model"]
rng = np.random.default_rng(int(os.environ.get("SEED", "1")))


def random_spd(n):
    """Symmetric, strictly diagonally dominant: random off-diagonal pairs (i, j), |v| < 1, and
    a diagonal larger than the row sums.  CSR rows sorted by column."""
    m = int(rng.integers(n, 8 * n))
    i = rng.integers(0, n, m)
    j = rng.integers(0, n, m)
    keep = i != j
    i, j = i[keep], j[keep]
    v = rng.uniform(-1, 1, i.size)
    rows = np.concatenate([i, j, np.arange(n)])
    cols = np.concatenate([j, i, np.arange(n)])
    vals = np.concatenate([v, v, np.zeros(n)])
    key = rows * n + cols
    order = np.argsort(key, kind="stable")
    key, rows, cols, vals = key[order], rows[order], cols[order], vals[order]
    uniq, start = np.unique(key, return_index=True)
    vals = np.add.reduceat(vals, start)
    rows, cols = uniq // n, uniq % n
    diag = rows == cols
    rowsum = np.bincount(rows[~diag], weights=np.abs(vals[~diag]), minlength=n)
    vals[diag] = rowsum[rows[diag]] + rng.uniform(0.5, 2.0, int(diag.sum()))
    rowptr = np.zeros(n + 1, np.int32)
    rowptr[1:] = np.cumsum(np.bincount(rows, minlength=n))
    return rowptr, cols.astype(np.int32), vals


for case in range(int(os.environ.get("CASES", "40"))):
    n = int(rng.integers(50, 60000))
    rowptr, colidx, values = random_spd(n)
    nnz = int(rowptr[-1])
    model = model_from_dict(bench._resize_model_dict(base, 400, 1920, n, nnz))
    D = int(rng.integers(1, 9))
    sched = build_schedule(model, D)
    bind = {"rowptr": rowptr, "colidx": colidx, "values": values, "b": rng.standard_normal(n)}
    eager = execute_schedule(model, sched, bind, D, graphs=False)
    dev = execute_schedule(model, sched, bind, D)
    ok = eager.iterations == dev.iterations and np.array_equal(eager.outputs["x"], dev.outputs["x"])
    if not ok:
        print(f"FAIL case {case}: n={n} nnz={nnz} D={D} iterations {eager.iterations} / {dev.iterations}", flush=True)
        sys.exit(1)
    print(f"case {case}: n={n} nnz={nnz} D={D} iterations={dev.iterations} relres={dev.final_relres:.2e} ok",
          flush=True)
print("all ok")
