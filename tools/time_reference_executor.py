"""Time the UNMODIFIED reference executor on C1 (build container only; the reference is not on
the GPU box, so bench.py cannot run it there -- it reads this file's committed output instead).

    python tools/time_reference_executor.py > profiles/r2_reference_executor_c1.json

C1 as the reference executes it: C = A B (256^3 fp32) is ONE spmv_csr
repetitive task over the Kronecker CSR matrix kron(A, I) (16.8 M nnz) applied to vec(B),
through gmodelc.refexec.execute_schedule (refexec.py:427-549) at D = 1 and D = 8 (simulated
devices, launches run one after another).  Reports end-to-end (the executor call, including its
_Storage copies) and op-only (refexec.spmv_range on the same plan) times, best of 3, and checks
the result against numpy's fp64 product."""
import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF_SRC = Path(os.environ.get("GMODELC_SRC", "/root/reference/pkg/src"))
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

import gmodelc                                        # noqa: E402
from gmodelc.partition import build_schedule          # noqa: E402
from gmodelc.refexec import execute_schedule          # noqa: E402

from make_golden import single_task_model             # noqa: E402


def kron_csr(A):
    n = A.shape[0]
    rows = np.repeat(np.arange(n * n), n)
    i, j = rows // n, rows % n
    k = np.tile(np.arange(n), n * n)
    colidx = (k * n + j).astype(np.int32)
    values = A[i, k].astype(np.float32)
    rowptr = (np.arange(n * n + 1) * n).astype(np.int32)
    return rowptr, colidx, values


def main():
    n = 256
    rng = np.random.default_rng(0)
    A = rng.standard_normal((n, n), dtype=np.float32)
    B = rng.standard_normal((n, n), dtype=np.float32)
    rowptr, colidx, values = kron_csr(A)
    N, nnz = n * n, int(rowptr[-1])
    model = single_task_model(
        "spmv_csr",
        [f"rowptr in int32 [{N + 1}]", f"colidx in int32 [{nnz}]", f"values in float32 [{nnz}]",
         f"x in float32 [{N}]", f"y out float32 [{N}]"],
        [f"rp in int32 [{N + 1}]", f"ci in int32 [{nnz}]", f"va in float32 [{nnz}]",
         f"vx in float32 [{N}]", f"o out float32 [{N}]"],
        ["rp -> t.rowptr", "ci -> t.colidx", "va -> t.values", "vx -> t.x", "t.y -> o"],
        ["allocate data rp onto dev.gmem", "allocate data ci onto dev.gmem", "allocate data va onto dev.gmem",
         "allocate data vx onto dev.gmem", "allocate data t.y onto dev.gmem", "allocate task t onto dev.cu"], N)
    bind = {"rp": rowptr, "ci": colidx, "va": values, "vx": B.ravel().copy()}
    ref64 = A.astype(np.float64) @ B.astype(np.float64)
    out = {"workload": "C1 matmul 256^3 fp32 as the reference executes it: one spmv_csr over kron(A, I) "
                       f"({nnz} nnz) applied to vec(B), gmodelc.refexec.execute_schedule",
           "host": {"cpu_count": os.cpu_count(), "machine": platform.machine(), "python": platform.python_version(),
                    "numpy": np.__version__, "where": "build container (the reference is absent on the GPU box)"},
           "runs": {}}
    for D in (1, 8):
        sched = build_schedule(model, D)
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            res = execute_schedule(model, sched, bind, D)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        C = res.outputs["o"].reshape(n, n)          # row i*n+j of kron(A, I) . vec(B) is C[i, j]
        err = float(np.linalg.norm(C - ref64) / np.linalg.norm(ref64))
        out["runs"][str(D)] = {"e2e_s": best, "TFLOP/s": 2.0 * n ** 3 / best / 1e12, "normwise_vs_fp64": err}
    # op-only: the executor's own spmv_range (refexec.py:111-121) on the ready arrays, plan cached
    from gmodelc import refexec
    plan = refexec.build_sweep_plan(rowptr, 0, N)
    best = None
    for _ in range(3):
        y = np.zeros(N, np.float32)
        t0 = time.perf_counter()
        refexec.spmv_range(rowptr, colidx, values, bind["vx"], 0, N, plan=plan, out=y)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    out["op_only"] = {"s": best, "TFLOP/s": 2.0 * n ** 3 / best / 1e12,
                      "what": "refexec.spmv_range over all rows with a cached sweep plan (D=1)"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
