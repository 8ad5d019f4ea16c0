"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker
or the timed CPU reference.  The product package (paper_1105_4424_b200)
never imports it; the product fails loudly when its CUDA library is absent.
House rule from the reference (pkg/tests/oracles.py:1): oracles never
share code with the library under test.

What it restates (file:line under /root/reference/pkg/src/gmodelc/):
  * schedule interpretation over flat row-major arrays, zero-initialised
    non-bound groups, one contiguous [offset, offset+count) range per
    simulated device ............................ refexec.py:375-412, :476-516
  * device partitioning ............................ partition.py:105-121
  * identity-tiler ops copy/sub/scale/axpy ......... refexec.py:504-514
  * spmv_csr strict left-to-right per row ......... refexec.py:111-121
  * dot_partial: per-launch dot, partials summed in ascending device
    order ........................................... refexec.py:478-487
  * the Array-OL tiler (not in the reference; SURVEY.md Appendix A,
    BASELINE.json north_star) and the tile intrinsics, accumulating in
    pattern order with each product and each sum rounded to the port
    dtype — the arithmetic order of the unmodified spmv_csr executor.

Parity pin: tests/golden/make_golden.py runs the UNMODIFIED reference
executor on selection / Kronecker / banded CSR matrices built from the
tiler index function and stores its outputs; tests
check this oracle against them bit for bit (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import numpy as np

CHUNK = 1 << 16   # repetitions per vectorised chunk


# -- partitioning (partition.py:105-121) ---------------------------------------

def partition_equally(total: int, devices: int) -> list[tuple[int, int]]:
    if total < 1 or devices < 1:
        raise ValueError("total_work and device_count must be positive")
    used = min(total, devices)
    counts = [total // used + (1 if d < total % used else 0) for d in range(used)]
    offs = [sum(counts[:d]) for d in range(used)]
    return list(zip(offs, counts))


# -- tiler index function ------------------------------------------------------

def _row_major_strides(shape):
    st = [1] * len(shape)
    for d in range(len(shape) - 2, -1, -1):
        st[d] = st[d + 1] * int(shape[d + 1])
    return st


def tiler_offsets_loop(tiler: dict, first: int, count: int) -> list[list[int]]:
    """Brute-force scalar restatement: one Python loop per (rho, iota). Small cases only."""
    arr, rep, pat = tiler["array"], tiler["rep"], tiler["pattern"]
    o, P, F = tiler["origin"], tiler["paving"], tiler["fitting"]
    ast = _row_major_strides(arr)
    out = []
    for rho in range(first, first + count):
        r, rem = [], rho
        for d in reversed(rep):
            r.append(rem % d)
            rem //= d
        r.reverse()
        row = []
        npat = 1
        for d in pat:
            npat *= d
        for iota in range(npat):
            i, rem = [], iota
            for d in reversed(pat):
                i.append(rem % d)
                rem //= d
            i.reverse()
            off = 0
            for a in range(len(arr)):
                e = o[a] + sum(P[a][j] * r[j] for j in range(len(rep))) \
                    + sum(F[a][k] * i[k] for k in range(len(pat)))
                off += (e % arr[a]) * ast[a]          # Python % is Euclidean for d > 0
            row.append(off)
        out.append(row)
    return out


def tiler_offsets(tiler: dict, first: int, count: int) -> np.ndarray:
    """Vectorised int64 [count, pattern_total] offsets (numpy, chunk-friendly)."""
    arr = np.asarray(tiler["array"], dtype=np.int64)
    rep, pat = tuple(tiler["rep"]), tuple(tiler["pattern"])
    o = np.asarray(tiler["origin"], dtype=np.int64)
    P = np.asarray(tiler["paving"], dtype=np.int64).reshape(len(arr), len(rep))
    F = np.asarray(tiler["fitting"], dtype=np.int64).reshape(len(arr), len(pat))
    ast = np.asarray(_row_major_strides(arr), dtype=np.int64)
    npat = int(np.prod(pat))
    rho = np.arange(first, first + count, dtype=np.int64)
    iota = np.arange(npat, dtype=np.int64)
    out = np.zeros((count, npat), dtype=np.int64)
    # build r and i coordinates by repeated divmod (row-major, last dim fastest)
    r = np.empty((len(rep), count), dtype=np.int64)
    rem = rho.copy()
    for j in range(len(rep) - 1, -1, -1):
        r[j] = rem % rep[j]
        rem //= rep[j]
    i = np.empty((len(pat), npat), dtype=np.int64)
    rem = iota.copy()
    for k in range(len(pat) - 1, -1, -1):
        i[k] = rem % pat[k]
        rem //= pat[k]
    for a in range(len(arr)):
        e_r = o[a] + (P[a][:, None] * r).sum(axis=0)        # count
        e_i = (F[a][:, None] * i).sum(axis=0)               # npat
        e = np.mod(e_r[:, None] + e_i[None, :], arr[a])
        out += e * ast[a]
    return out


def _chunks(first: int, count: int):
    lo = first
    while lo < first + count:
        n = min(CHUNK, first + count - lo)
        yield lo, n
        lo += n


# -- tile intrinsics (Array-OL) ------------------------------------------------

def tile_copy(src, dst, t_src: dict, t_dst: dict, first: int, count: int) -> None:
    """dst[off_dst(rho, iota)] = src[off_src(rho, iota)] for rho in [first, first+count)."""
    for lo, n in _chunks(first, count):
        dst[tiler_offsets(t_dst, lo, n).ravel()] = src[tiler_offsets(t_src, lo, n).ravel()]


def matmul(a, b, c, t_a: dict, t_b: dict, t_c: dict, first: int, count: int) -> None:
    """c[off_c(rho)] = sum_k a_pat[k]*b_pat[k]; k ascending, product and sum rounded separately."""
    for lo, n in _chunks(first, count):
        ia, ib = tiler_offsets(t_a, lo, n), tiler_offsets(t_b, lo, n)
        acc = np.zeros(n, dtype=c.dtype)
        for k in range(ia.shape[1]):
            acc += a[ia[:, k]] * b[ib[:, k]]
        c[tiler_offsets(t_c, lo, n)[:, 0]] = acc


def tile_filter(x, w, y, t_x: dict, t_y: dict, first: int, count: int) -> None:
    """y_pat[j] = sum_i w[j, i] * x_pat[i]; i ascending, product and sum rounded separately."""
    px = int(np.prod(t_x["pattern"]))
    py = int(np.prod(t_y["pattern"]))
    W = np.asarray(w).reshape(py, px)
    for lo, n in _chunks(first, count):
        xs = x[tiler_offsets(t_x, lo, n)]           # n x px
        oy = tiler_offsets(t_y, lo, n)              # n x py
        for j in range(py):
            acc = np.zeros(n, dtype=y.dtype)
            for i in range(px):
                acc += W[j, i] * xs[:, i]
            y[oy[:, j]] = acc


def tile_sum(x, s, t_x: dict, t_s: dict, first: int, count: int) -> None:
    for lo, n in _chunks(first, count):
        xs = x[tiler_offsets(t_x, lo, n)]
        acc = np.zeros(n, dtype=s.dtype)
        for i in range(xs.shape[1]):
            acc += xs[:, i]
        s[tiler_offsets(t_s, lo, n)[:, 0]] = acc


# -- identity-tiler reference ops (refexec.py:476-516) -------------------------

def spmv_rows(rowptr, colidx, values, x, y, lo: int, hi: int) -> None:
    """Rows lo..hi-1, each accumulated left to right in the value dtype (refexec.py:111-121)."""
    starts = rowptr[lo:hi].astype(np.int64)
    lens = rowptr[lo + 1:hi + 1].astype(np.int64) - starts
    acc = np.zeros(hi - lo, dtype=y.dtype)
    for j in range(int(lens.max()) if hi > lo else 0):
        rows = np.nonzero(lens > j)[0]
        idx = starts[rows] + j
        acc[rows] += values[idx] * x[colidx[idx]]
    y[lo:hi] = acc


def run_identity_op(op: str, arrays: dict, ranges, scalar_a: float | None = None) -> None:
    if op == "dot_partial":
        total = 0.0
        for lo, n in ranges:
            total += float(np.dot(arrays["a"][lo:lo + n], arrays["b"][lo:lo + n]))
        arrays["s"][0] = total
        return
    for lo, n in ranges:
        hi = lo + n
        if op == "copy":
            arrays["dst"][lo:hi] = arrays["src"][lo:hi]
        elif op == "sub":
            arrays["z"][lo:hi] = arrays["x"][lo:hi] - arrays["y"][lo:hi]
        elif op == "scale":
            arrays["y"][lo:hi] *= float(arrays["a"][0])
        elif op == "axpy":
            if "a" in arrays:
                arrays["y"][lo:hi] += float(arrays["a"][0]) * arrays["x"][lo:hi]
            else:
                arrays["y"][lo:hi] += arrays["x"][lo:hi]
        elif op == "spmv_csr":
            spmv_rows(arrays["rowptr"], arrays["colidx"], arrays["values"], arrays["x"],
                      arrays["y"], lo, hi)
        else:
            raise ValueError(f"oracle has no identity op '{op}'")


# -- single repetitive task, D simulated devices -------------------------------

def run_tile_task(op: str, tilers: dict, inputs: dict, outputs: dict, rep_total: int,
                  devices: int) -> dict:
    """Interpret one tile-intrinsic task over D contiguous shards.

    ``outputs`` maps out-port name -> (size, dtype); they start zeroed like
    non-bound storage groups (refexec.py:399-403).
    """
    res = {k: np.zeros(n, dtype=dt) for k, (n, dt) in outputs.items()}
    for lo, n in partition_equally(rep_total, devices):
        if op == "tile_copy":
            tile_copy(inputs["src"], res["dst"], tilers["src"], tilers["dst"], lo, n)
        elif op == "matmul":
            matmul(inputs["a"], inputs["b"], res["c"], tilers["a"], tilers["b"], tilers["c"], lo, n)
        elif op in ("tile_filter", "hfilter", "vfilter", "stencil"):
            tile_filter(inputs["x"], inputs["w"], res["y"], tilers["x"], tilers["y"], lo, n)
        elif op == "tile_sum":
            tile_sum(inputs["x"], res["s"], tilers["x"], tilers["s"], lo, n)
        else:
            raise ValueError(f"oracle has no tile op '{op}'")
    return res


# -- canonical tilers used by the configs ----------------

def gemm_tilers(M: int, N: int, K: int) -> dict:
    return {
        "a": dict(array=(M, K), rep=(M, N), pattern=(K,), origin=(0, 0),
                  paving=((1, 0), (0, 0)), fitting=((0,), (1,))),
        "b": dict(array=(K, N), rep=(M, N), pattern=(K,), origin=(0, 0),
                  paving=((0, 0), (0, 1)), fitting=((1,), (0,))),
        "c": dict(array=(M, N), rep=(M, N), pattern=(1,), origin=(0, 0),
                  paving=((1, 0), (0, 1)), fitting=((0,), (0,))),
    }


def stencil_tilers(H: int, W: int) -> dict:
    return {
        "x": dict(array=(H, W), rep=(H, W), pattern=(3, 3), origin=(H - 1, W - 1),
                  paving=((1, 0), (0, 1)), fitting=((1, 0), (0, 1))),
        "y": dict(array=(H, W), rep=(H, W), pattern=(1,), origin=(0, 0),
                  paving=((1, 0), (0, 1)), fitting=((0,), (0,))),
    }


def hfilter_tilers(F: int, H: int, W: int, taps: int = 13, step: int = 8, outs: int = 3) -> dict:
    Wo = W // step * outs
    return {
        "x": dict(array=(F, H, W), rep=(F, H, W // step), pattern=(taps,), origin=(0, 0, 0),
                  paving=((1, 0, 0), (0, 1, 0), (0, 0, step)), fitting=((0,), (0,), (1,))),
        "y": dict(array=(F, H, Wo), rep=(F, H, W // step), pattern=(outs,), origin=(0, 0, 0),
                  paving=((1, 0, 0), (0, 1, 0), (0, 0, outs)), fitting=((0,), (0,), (1,))),
    }


def vfilter_tilers(F: int, H: int, W: int, taps: int = 14, step: int = 9, outs: int = 4) -> dict:
    Ho = H // step * outs
    return {
        "x": dict(array=(F, H, W), rep=(F, H // step, W), pattern=(taps,), origin=(0, 0, 0),
                  paving=((1, 0, 0), (0, step, 0), (0, 0, 1)), fitting=((0,), (1,), (0,))),
        "y": dict(array=(F, Ho, W), rep=(F, H // step, W), pattern=(outs,), origin=(0, 0, 0),
                  paving=((1, 0, 0), (0, outs, 0), (0, 0, 1)), fitting=((0,), (1,), (0,))),
    }


def stencil_weights() -> np.ndarray:
    """[1,2,1]^T [1,2,1] / 16 — powers of two."""
    v = np.array([1.0, 2.0, 1.0])
    return (np.outer(v, v) / 16.0).astype(np.float32).ravel()


def hfilter_weights(taps: int = 13, outs: int = 3) -> np.ndarray:
    """Frozen downscaler weights: output j is a normalised triangle centred at 4*j+2 (spec decision)."""
    W = np.zeros((outs, taps))
    for j in range(outs):
        c = (taps - 1) * (j + 0.5) / outs
        for i in range(taps):
            W[j, i] = max(0.0, 3.0 - abs(i - c))
        W[j] /= W[j].sum()
    return W.astype(np.float32).ravel()


def vfilter_weights(taps: int = 14, outs: int = 4) -> np.ndarray:
    return hfilter_weights(taps, outs)
