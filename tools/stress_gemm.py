"""Random TF32 GEMM shapes / shard counts / operand majorness, repeated: every result inside the
stated TF32 bound and bit-identical when re-run (split-K counters, scratch reuse, mixed-width
off/on).  Prints one line per 20 cases; exits non-zero on the first failure."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_1105_4424_b200 import Tiler, builders  # noqa: E402
from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
n_cases = int(os.environ.get("CASES", "200"))
for case in range(n_cases):
    M = int(rng.integers(1, 9)) * int(rng.choice([64, 128, 256, 300]))
    N = int(rng.integers(1, 9)) * int(rng.choice([64, 128, 256, 264]))
    K = int(rng.choice([32, 64, 96, 512, 1024, 2048]))
    D = int(rng.integers(1, 8))
    a_mn, b_k = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
    if rng.random() < 0.2:
        os.environ["AOL_GEMM_SPLIT"] = str(int(rng.choice([2, 3, 4])))
    else:
        os.environ.pop("AOL_GEMM_SPLIT", None)
    os.environ["AOL_GEMM_NARROW"] = "1" if rng.random() < 0.2 else "0"
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    ta = Tiler((0, 0), ((0, 0), (1, 0)), ((1,), (0,)), (K,)) if a_mn else Tiler((0, 0), ((1, 0), (0, 0)), ((0,), (1,)), (K,))
    tb = Tiler((0, 0), ((0, 0), (0, 1)), ((1,), (0,)), (K,)) if not b_k else Tiler((0, 0), ((0, 1), (0, 0)), ((0,), (1,)), (K,))
    tc = Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,))
    a_arr = (K, M) if a_mn else (M, K)
    b_arr = (N, K) if b_k else (K, N)
    a_bind = np.ascontiguousarray(A.T if a_mn else A).ravel()
    b_bind = np.ascontiguousarray(B.T if b_k else B).ravel()
    model = builders.tile_task_model("matmul", {"a": f"in float32 [{a_arr[0]},{a_arr[1]}]",
                                                "b": f"in float32 [{b_arr[0]},{b_arr[1]}]",
                                                "c": f"out float32 [{M},{N}]"}, {"a": ta, "b": tb, "c": tc}, (M, N))
    sched = build_schedule(model, D)
    if os.environ.get("STRESS_VERBOSE"):
        print(f"case {case}: M={M} N={N} K={K} D={D} a_mn={a_mn} b_k={b_k} split={os.environ.get('AOL_GEMM_SPLIT')} "
              f"narrow={os.environ['AOL_GEMM_NARROW']}", flush=True)
    prec = str(rng.choice(["default", "default", "3xtf32", "exact"]))
    if prec == "exact" and M * N * K > 2 ** 27:
        prec = "default"
    c1 = execute_schedule(model, sched, {"p_a": a_bind, "p_b": b_bind}, D, precision=prec).outputs["p_c"].reshape(M, N)
    c2 = execute_schedule(model, sched, {"p_a": a_bind, "p_b": b_bind}, D, precision=prec).outputs["p_c"].reshape(M, N)
    a64, b64 = A.astype(np.float64), B.astype(np.float64)
    c64 = a64 @ b64
    same = np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    if prec == "default":
        bound = (2.0 ** -9 + K * 2.0 ** -23) * (np.abs(a64) @ np.abs(b64))
        ok = same and np.all(np.abs(c1 - c64) <= bound)
    elif prec == "3xtf32":
        ok = same and np.linalg.norm(c1 - c64) / np.linalg.norm(c64) <= 1e-6
    else:                                   # the reference's k-ascending order, bit for bit
        from oracle import aol_oracle as orc
        tl = {"a": dict(array=a_arr, rep=(M, N), pattern=(K,), origin=ta.origin, paving=ta.paving, fitting=ta.fitting),
              "b": dict(array=b_arr, rep=(M, N), pattern=(K,), origin=tb.origin, paving=tb.paving, fitting=tb.fitting),
              "c": dict(array=(M, N), rep=(M, N), pattern=(1,), origin=tc.origin, paving=tc.paving, fitting=tc.fitting)}
        ref = orc.run_tile_task("matmul", tl, {"a": a_bind, "b": b_bind}, {"c": (M * N, np.float32)}, M * N, D)["c"]
        ok = same and np.array_equal(c1.ravel().view(np.uint32), ref.view(np.uint32))
    if not ok:
        print(f"FAIL case {case}: M={M} N={N} K={K} D={D} a_mn={a_mn} b_k={b_k} prec={prec} "
              f"split={os.environ.get('AOL_GEMM_SPLIT')} narrow={os.environ['AOL_GEMM_NARROW']}", flush=True)
        sys.exit(1)
    if case % 20 == 19:
        print(f"{case + 1} cases ok", flush=True)
print("all ok")
