"""ctypes binding of libaolb200.so (include/aol_b200.h).

The library is loaded eagerly on first use and the product path fails
loudly (``NativeLibraryError``) when it is missing or cannot find an
sm_100 device — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .tiler import MAX_RANK, BoundTiler

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libaolb200.so"
ABI_VERSION = 2
FLAG_DEVICE_SCALARS = 1
FLAG_STAGE_SMEM = 2
MAX_TILERS = 4

AOL_OK, AOL_EINVAL, AOL_ECUDA, AOL_EUNSUPPORTED, AOL_ENODEV = 0, -1, -2, -3, -4
DTYPE = {"float32": 0, "float64": 1, "int32": 2, "int64": 3}
OP = {"copy": 1, "sub": 2, "scale": 3, "axpy": 4, "spmv_csr": 5, "dot_partial": 6,
      "div": 7, "neg": 8, "rel_residual": 9, "partials_sum": 10, "scalar_seq": 11,
      "tile_copy": 16, "matmul": 17, "tile_filter": 18, "hfilter": 18, "vfilter": 18,
      "stencil": 18, "tile_sum": 19}
PRECISION = {"default": 0, "tf32": 1, "3xtf32": 2, "exact": 3}

EXPORTS = ("aol_abi_version", "aol_last_error", "aol_device_count", "aol_validate", "aol_launch",
           "aol_plan_name", "aol_tiler_offsets", "aol_launch_counter", "aol_launch_fused2", "aol_loop_begin",
           "aol_loop_end", "aol_loop_run", "aol_loop_destroy", "aol_loop_persistent", "aol_release_scratch",
           "aol_ipc_export", "aol_ipc_import", "aol_ipc_close", "aol_memcpy2d")


class NativeLibraryError(RuntimeError):
    pass


class AolError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"libaolb200 status {status}: {message}")
        self.status = status


I64x4 = C.c_int64 * MAX_RANK


class AolTiler(C.Structure):
    _fields_ = [("arr_rank", C.c_int32), ("rep_rank", C.c_int32), ("pat_rank", C.c_int32),
                ("reserved", C.c_int32), ("array", I64x4), ("rep", I64x4), ("pattern", I64x4),
                ("origin", I64x4), ("paving", I64x4 * MAX_RANK), ("fitting", I64x4 * MAX_RANK)]


class AolTask(C.Structure):
    _fields_ = [("op", C.c_int32), ("dtype", C.c_int32), ("index_dtype", C.c_int32),
                ("precision", C.c_int32), ("n_tilers", C.c_int32), ("n_scalars", C.c_int32),
                ("flags", C.c_int32), ("reserved", C.c_int32), ("tilers", AolTiler * MAX_TILERS)]


def pack_tiler(bt: BoundTiler) -> AolTiler:
    t = AolTiler()
    tl = bt.tiler
    t.arr_rank, t.rep_rank, t.pat_rank = len(bt.array), len(bt.rep), len(tl.pattern)
    for d, v in enumerate(bt.array):
        t.array[d] = v
        t.origin[d] = tl.origin[d]
        for j, pv in enumerate(tl.paving[d]):
            t.paving[d][j] = pv
        for k, fv in enumerate(tl.fitting[d]):
            t.fitting[d][k] = fv
    for j, v in enumerate(bt.rep):
        t.rep[j] = v
    for k, v in enumerate(tl.pattern):
        t.pattern[k] = v
    return t


def make_task(op: str, dtype: str, tilers: list[BoundTiler] = (), precision: str = "default",
              n_scalars: int = 0, index_dtype: str = "int32", flags: int = 0) -> AolTask:
    task = AolTask()
    task.flags = flags
    task.op = OP[op]
    task.dtype = DTYPE[dtype]
    task.index_dtype = DTYPE[index_dtype]
    task.precision = PRECISION[precision]
    task.n_tilers = len(tilers)
    task.n_scalars = n_scalars
    for i, bt in enumerate(tilers):
        task.tilers[i] = pack_tiler(bt)
    return task


_lib = None


def load(path: Path | str | None = None) -> C.CDLL:
    """Load (once) and type the library; raise NativeLibraryError if absent or mismatched."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path or os.environ.get("AOL_LIB", LIB_PATH))
    if not p.exists():
        raise NativeLibraryError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            f"(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name in EXPORTS:
        if not hasattr(lib, name):
            raise NativeLibraryError(f"{p} does not export {name}")
    lib.aol_abi_version.restype = C.c_int
    lib.aol_last_error.restype = C.c_char_p
    lib.aol_device_count.argtypes = [C.POINTER(C.c_int)]
    lib.aol_validate.argtypes = [C.POINTER(AolTask)]
    lib.aol_launch.argtypes = [C.POINTER(AolTask), C.c_int64, C.c_int64, C.POINTER(C.c_void_p),
                               C.POINTER(C.c_double), C.c_void_p]
    lib.aol_plan_name.argtypes = [C.POINTER(AolTask), C.c_int64, C.c_int64, C.POINTER(C.c_void_p),
                                  C.c_char_p, C.c_int]
    lib.aol_tiler_offsets.argtypes = [C.POINTER(AolTiler), C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
    lib.aol_launch_counter.restype = C.c_int64
    lib.aol_launch_fused2.argtypes = [C.POINTER(AolTask), C.POINTER(AolTask), C.c_int64, C.c_int64,
                                      C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p]
    lib.aol_loop_begin.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int64, C.POINTER(C.c_void_p)]
    lib.aol_loop_end.argtypes = [C.c_void_p]
    lib.aol_loop_run.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                 C.POINTER(C.c_int)]
    lib.aol_loop_destroy.argtypes = [C.c_void_p]
    lib.aol_ipc_export.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
    lib.aol_ipc_import.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]
    lib.aol_ipc_close.argtypes = [C.c_void_p]
    lib.aol_memcpy2d.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
    lib.aol_loop_persistent.argtypes = [C.POINTER(AolLoopOp), C.c_int, C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_double, C.c_int64, C.c_void_p,
                                        C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_int)]
    if lib.aol_abi_version() != ABI_VERSION:
        raise NativeLibraryError(f"{p}: ABI {lib.aol_abi_version()} != expected {ABI_VERSION}")
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != AOL_OK:
        raise AolError(rc, load().aol_last_error().decode(errors="replace"))


def device_count() -> int:
    n = C.c_int(0)
    check(load().aol_device_count(C.byref(n)))
    return n.value


def _ptrs(ptrs) -> C.Array:
    return (C.c_void_p * max(1, len(ptrs)))(*[C.c_void_p(int(p)) for p in ptrs])


def launch(task: AolTask, first: int, count: int, ports: list[int], scalars=(), stream: int = 0) -> None:
    sc = (C.c_double * max(1, len(scalars)))(*[float(s) for s in scalars])
    check(load().aol_launch(C.byref(task), int(first), int(count), _ptrs(ports), sc,
                            C.c_void_p(int(stream))))


def plan_name(task: AolTask, first: int, count: int, ports: list[int] | None = None) -> str:
    buf = C.create_string_buffer(128)
    pp = _ptrs(ports) if ports else None
    check(load().aol_plan_name(C.byref(task), int(first), int(count), pp, buf, 128))
    return buf.value.decode()


def validate(task: AolTask) -> None:
    check(load().aol_validate(C.byref(task)))


def tiler_offsets(bt: BoundTiler, first: int, count: int, out_ptr: int, stream: int = 0) -> None:
    t = pack_tiler(bt)
    check(load().aol_tiler_offsets(C.byref(t), int(first), int(count), C.c_void_p(int(out_ptr)),
                                   C.c_void_p(int(stream))))


def launch_fused2(producer: AolTask, consumer: AolTask, first: int, count: int, pports: list[int],
                  cports: list[int], stream: int = 0) -> bool:
    """True when the fused kernel ran; False when the pair is not fusable (nothing launched)."""
    rc = load().aol_launch_fused2(C.byref(producer), C.byref(consumer), int(first), int(count), _ptrs(pports),
                                  _ptrs(cports), C.c_void_p(int(stream)))
    if rc == AOL_EUNSUPPORTED:
        return False
    check(rc)
    return True


class AolLoopOp(C.Structure):
    _fields_ = [("op", C.c_int32), ("n_scalars", C.c_int32), ("part", C.c_int32), ("n_parts", C.c_int32),
                ("first", C.c_int64), ("count", C.c_int64), ("port", C.c_int32 * 6)]


def loop_op(op: str, ports: list[int], first: int = 0, count: int = 0, n_scalars: int = 0, part: int = 0,
            n_parts: int = 1) -> AolLoopOp:
    o = AolLoopOp(op=OP[op], n_scalars=n_scalars, part=part, n_parts=n_parts, first=int(first), count=int(count))
    for i, p in enumerate(list(ports) + [-1] * (6 - len(ports))):
        o.port[i] = p
    return o


def loop_persistent(ops: list[AolLoopOp], ports: list[int], dtype: str, index_dtype: str, relres_port: int,
                    tol: float, max_iter: int, stream: int = 0):
    """Run a LoopStep body as one persistent kernel: (iterations, relres, converged), or None
    when the body is outside the interpreter's op set (nothing launched)."""
    arr = (AolLoopOp * len(ops))(*ops)
    it, rr, cv = C.c_int64(), C.c_double(), C.c_int()
    rc = load().aol_loop_persistent(arr, len(ops), _ptrs(ports), len(ports), DTYPE[dtype], DTYPE[index_dtype],
                                    int(relres_port), float(tol), int(max_iter), C.c_void_p(int(stream)),
                                    C.byref(it), C.byref(rr), C.byref(cv))
    if rc == AOL_EUNSUPPORTED:
        return None
    check(rc)
    return it.value, rr.value, bool(cv.value)


def loop_begin(stream: int, relres_ptr: int, dtype: str, tol: float, max_iter: int) -> int:
    """Start capturing one LoopStep body on `stream` into a device-side WHILE loop; returns a handle."""
    h = C.c_void_p()
    check(load().aol_loop_begin(C.c_void_p(int(stream)), C.c_void_p(int(relres_ptr)), DTYPE[dtype], float(tol),
                                int(max_iter), C.byref(h)))
    return h.value


def loop_end(handle: int) -> None:
    check(load().aol_loop_end(C.c_void_p(handle)))


def loop_run(handle: int, stream: int) -> tuple[int, float, bool]:
    it, rr, cv = C.c_int64(), C.c_double(), C.c_int()
    check(load().aol_loop_run(C.c_void_p(handle), C.c_void_p(int(stream)), C.byref(it), C.byref(rr), C.byref(cv)))
    return it.value, rr.value, bool(cv.value)


def loop_destroy(handle: int) -> None:
    if handle:
        load().aol_loop_destroy(C.c_void_p(handle))


def ipc_export(ptr: int) -> bytes:
    """72-byte token (64-byte CUDA IPC handle + int64 offset) for the device buffer at ``ptr``."""
    h = (C.c_char * 64)()
    off = C.c_int64(0)
    check(load().aol_ipc_export(C.c_void_p(ptr), h, C.byref(off)))
    return bytes(h) + int(off.value).to_bytes(8, "little", signed=True)


def ipc_import(token: bytes) -> int:
    """Map a buffer another process exported with :func:`ipc_export`; returns the device pointer."""
    h = (C.c_char * 64).from_buffer_copy(token[:64])
    out = C.c_void_p(0)
    check(load().aol_ipc_import(h, int.from_bytes(token[64:72], "little", signed=True), C.byref(out)))
    return int(out.value)


def ipc_close(ptr: int) -> None:
    check(load().aol_ipc_close(C.c_void_p(ptr)))


def memcpy2d(dst: int, dpitch: int, src: int, spitch: int, width_bytes: int, height: int, stream: int) -> None:
    """Asynchronous strided copy (aol_memcpy2d): `height` rows of `width_bytes`, pitches in bytes."""
    check(load().aol_memcpy2d(C.c_void_p(dst), int(dpitch), C.c_void_p(src), int(spitch), int(width_bytes),
                              int(height), C.c_void_p(int(stream))))


def release_scratch() -> None:
    """Free the library's cached dot / loop scratch (aol_release_scratch)."""
    check(load().aol_release_scratch())


def launch_counter() -> int:
    return int(load().aol_launch_counter())

