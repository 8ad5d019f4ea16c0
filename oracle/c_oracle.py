"""ctypes loader of oracle/_build/liboracle.so (the C restatement) — TEST INFRASTRUCTURE ONLY.

Used by tests/ (large-size cross-checks) and by bench.py's CPU baseline and
``--impl reference`` arm.  See oracle/aol_oracle.c for what it restates.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

I64x4 = C.c_int64 * 4


class OrcTiler(C.Structure):
    _fields_ = [("arr_rank", C.c_int32), ("rep_rank", C.c_int32), ("pat_rank", C.c_int32),
                ("reserved", C.c_int32), ("array", I64x4), ("rep", I64x4), ("pattern", I64x4),
                ("origin", I64x4), ("paving", I64x4 * 4), ("fitting", I64x4 * 4)]


def pack(d: dict) -> OrcTiler:
    t = OrcTiler()
    t.arr_rank, t.rep_rank, t.pat_rank = len(d["array"]), len(d["rep"]), len(d["pattern"])
    for i, v in enumerate(d["array"]):
        t.array[i] = v
        t.origin[i] = d["origin"][i]
        for j, pv in enumerate(d["paving"][i]):
            t.paving[i][j] = pv
        for k, fv in enumerate(d["fitting"][i]):
            t.fitting[i][k] = fv
    for j, v in enumerate(d["rep"]):
        t.rep[j] = v
    for k, v in enumerate(d["pattern"]):
        t.pattern[k] = v
    return t


_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        lib = C.CDLL(str(LIB))
        P = C.c_void_p
        lib.orc_threads.restype = C.c_int
        lib.orc_tiler_offsets.argtypes = [C.POINTER(OrcTiler), C.c_int64, C.c_int64, P]
        lib.orc_tile_copy.argtypes = [P, P, C.c_int, C.POINTER(OrcTiler), C.POINTER(OrcTiler), C.c_int64, C.c_int64]
        lib.orc_matmul_f32.argtypes = [P, P, P, C.POINTER(OrcTiler), C.POINTER(OrcTiler), C.POINTER(OrcTiler),
                                       C.c_int64, C.c_int64]
        lib.orc_gemm_rows_f32.argtypes = [P, P, P, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
        lib.orc_filter_f32.argtypes = [P, P, P, C.POINTER(OrcTiler), C.POINTER(OrcTiler), C.c_int64, C.c_int64]
        lib.orc_stencil3x3_rows_f32.argtypes = [P, P, P, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def threads() -> int:
    return int(load().orc_threads())


def tiler_offsets(t: dict, first: int, count: int) -> np.ndarray:
    P = int(np.prod(t["pattern"]))
    out = np.empty(count * P, dtype=np.int64)
    load().orc_tiler_offsets(C.byref(pack(t)), first, count, _p(out))
    return out.reshape(count, P)


def tile_copy(src: np.ndarray, dst: np.ndarray, ts: dict, td: dict, first: int, count: int) -> None:
    load().orc_tile_copy(_p(src), _p(dst), src.itemsize, C.byref(pack(ts)), C.byref(pack(td)), first, count)


def matmul(a, b, c, ta, tb, tc, first, count) -> None:
    load().orc_matmul_f32(_p(a), _p(b), _p(c), C.byref(pack(ta)), C.byref(pack(tb)), C.byref(pack(tc)),
                          first, count)


def gemm_rows(A: np.ndarray, B: np.ndarray, Cm: np.ndarray, N: int, K: int, lo: int, hi: int) -> None:
    load().orc_gemm_rows_f32(_p(A), _p(B), _p(Cm), N, K, lo, hi)


def tile_filter(x, w, y, tx, ty, first, count) -> None:
    load().orc_filter_f32(_p(x), _p(w), _p(y), C.byref(pack(tx)), C.byref(pack(ty)), first, count)


def stencil_rows(x, w, y, H: int, W: int, lo: int, hi: int) -> None:
    load().orc_stencil3x3_rows_f32(_p(x), _p(w), _p(y), H, W, lo, hi)
