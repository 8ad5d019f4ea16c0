"""Generate tests/golden/reference_golden.npz by running the UNMODIFIED reference executor.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py            # needs /root/reference

Every case is executed by ``gmodelc.refexec.execute_schedule``
(/root/reference/pkg/src/gmodelc/refexec.py:427-549) on a single-task
model written in the reference's own test-harness style
(pkg/tests/test_refexec.py:250-293).  Tile intrinsics do not exist in the
reference, so each linear tile task is expressed as ONE ``spmv_csr``
repetitive task over a CSR matrix built from the tiler index function
(SURVEY.md §8(c)):

  * tile_copy   -> 0/1 selection matrix  S[off_dst(r,i), off_src(r,i)] = 1
  * matmul      -> row off_c(r) holds a[off_a(r,k)] at column off_b(r,k), k ascending
                   (canonical tilers: the Kronecker matrix I (x) A of SURVEY.md §0.5)
  * tile_filter -> row off_y(r,j) holds w[j,i] at column off_x(r,i), i ascending
  * tile_sum    -> row off_s(r) holds 1.0 at columns off_x(r,i)

spmv_csr accumulates each row strictly left to right with the product and
the sum rounded separately (refexec.py:111-121), so the stored outputs pin
the oracle's "pattern order, no FMA" arithmetic bit for bit.  Rows with no
entries stay 0, which is the executor's zero-initialisation of unwritten
outputs (refexec.py:399-403).  The CSR matrix must be square for
``check_task_signature`` (intrinsics.py:138-146), so x and y are padded
to n = max(input size, output size).

The identity-tiler reference ops (copy/sub/scale/axpy/spmv/dot) are run
directly as reference tasks.  The tiler offsets are computed with the
brute-force loop of oracle/aol_oracle.py (tiler_offsets_loop), which is
the restatement under test; the golden outputs come from the reference.
"""

from __future__ import annotations

import json
import zlib
import os
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True          # never write __pycache__ into /root/reference
REF_SRC = Path(os.environ.get("GMODELC_SRC", "/root/reference/pkg/src"))
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(HERE.parent.parent))

import gmodelc                                          # noqa: E402
from gmodelc.partition import build_schedule, partition_equally   # noqa: E402
from gmodelc.refexec import execute_schedule, poisson_2d   # noqa: E402

from oracle import aol_oracle as orc                    # noqa: E402

SINGLE_TASK = """\
platform p {{
  component Host {{
    processor cpu : hwProcessor
    memory ram : hwMemory role=hostRam
  }}
  component Cu : hwProcessor {{
    processor pe : hwProcessor shaped [8]
  }}
  component Dev {{
    processor cu : Cu shaped [4]
    memory gmem : hwMemory role=deviceGlobal
  }}
  component p {{
    part host : Host
    part dev : Dev
  }}
}}
application m {{
  component T {{
{ports}
    repeat [{n}]
    deploy {op}
  }}
  component m {{
{root_ports}
    part t : T
{conns}
  }}
}}
{allocs}
"""


def single_task_model(op, ports, root_ports, conns, allocs, n):
    text = SINGLE_TASK.format(
        op=op, n=n, ports="\n".join(f"    port {p}" for p in ports),
        root_ports="\n".join(f"    port {p}" for p in root_ports),
        conns="\n".join(f"    connect {c}" for c in conns), allocs="\n".join(allocs))
    model = gmodelc.parse_model(text)
    assert gmodelc.validate_conformance(model) == [], text
    return model


def run_reference_spmv(rows: list[list[tuple[int, float]]], x: np.ndarray, dtype: str,
                       devices: int) -> np.ndarray:
    """y = A x through the unmodified executor; ``rows`` lists (column, value) in accumulation order."""
    n = len(rows)
    assert x.size == n
    rowptr = np.zeros(n + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum([len(r) for r in rows])
    nnz = int(rowptr[-1])
    colidx = np.fromiter((c for r in rows for c, _ in r), dtype=np.int32, count=nnz)
    values = np.fromiter((v for r in rows for _, v in r), dtype=np.float64, count=nnz)
    return run_reference_csr(rowptr, colidx, values, x, dtype, devices)


def run_reference_csr(rowptr, colidx, values, x, dtype, devices):
    n = rowptr.size - 1
    nnz = max(int(rowptr[-1]), 1)
    if rowptr[-1] == 0:                      # ports need >= 1 element
        colidx = np.zeros(1, np.int32)
        values = np.zeros(1)
    model = single_task_model(
        "spmv_csr",
        [f"rowptr in int32 [{n + 1}]", f"colidx in int32 [{nnz}]",
         f"values in {dtype} [{nnz}]", f"x in {dtype} [{n}]", f"y out {dtype} [{n}]"],
        [f"rp in int32 [{n + 1}]", f"ci in int32 [{nnz}]", f"va in {dtype} [{nnz}]",
         f"vx in {dtype} [{n}]", f"o out {dtype} [{n}]"],
        ["rp -> t.rowptr", "ci -> t.colidx", "va -> t.values", "vx -> t.x", "t.y -> o"],
        ["allocate data rp onto dev.gmem", "allocate data ci onto dev.gmem",
         "allocate data va onto dev.gmem", "allocate data vx onto dev.gmem",
         "allocate data t.y onto dev.gmem", "allocate task t onto dev.cu"], n)
    res = execute_schedule(model, build_schedule(model, devices),
                           {"rp": rowptr, "ci": colidx, "va": values, "vx": x}, devices)
    return res.outputs["o"]


def offsets(t, count=None):
    rep_total = int(np.prod(t["rep"]))
    return orc.tiler_offsets_loop(t, 0, rep_total if count is None else count)


def pad(x, n):
    out = np.zeros(n, dtype=x.dtype)
    out[:x.size] = x
    return out


# -- cases -------------------------------------------------------------------

def t1(array, rep, pattern, origin, paving, fitting):
    return dict(array=tuple(array), rep=tuple(rep), pattern=tuple(pattern), origin=tuple(origin),
                paving=tuple(map(tuple, paving)), fitting=tuple(map(tuple, fitting)))


COPY_CASES = {
    # dense 1-D gather of patterns of 4 into a dense output
    "copy_dense_1d": (t1([64], [16], [4], [0], [[4]], [[1]]),
                      t1([64], [16], [4], [0], [[4]], [[1]])),
    # overlapping input paving (stride 2 < pattern 4), toroidal wrap at the end
    "copy_overlap_wrap": (t1([40], [20], [4], [3], [[2]], [[1]]),
                          t1([80], [20], [4], [0], [[4]], [[1]])),
    # gaps: paving 6 > pattern 2, strided fitting
    "copy_gap_strided": (t1([100], [8], [2], [1], [[6]], [[3]]),
                         t1([16], [8], [2], [0], [[2]], [[1]])),
    # 2-D transpose through a [1] pattern
    "copy_transpose_2d": (t1([6, 10], [10, 6], [1], [0, 0], [[0, 1], [1, 0]], [[0], [0]]),
                          t1([10, 6], [10, 6], [1], [0, 0], [[1, 0], [0, 1]], [[0], [0]])),
    # 2-D box pattern, toroidal origin (-1,-1) == (H-1, W-1); sparse output (half unwritten)
    "copy_box_torus": (t1([5, 7], [5, 7], [3, 3], [4, 6], [[1, 0], [0, 1]], [[1, 0], [0, 1]]),
                       t1([5, 7, 9], [5, 7], [3, 3], [0, 0, 0],
                          [[1, 0], [0, 1], [0, 0]], [[0, 0], [0, 0], [3, 1]])),
    # negative paving (reverse) and rank-3 repetition
    "copy_reverse_rank3": (t1([24], [2, 3, 4], [1], [23], [[-12, -4, -1]], [[0]]),
                           t1([2, 3, 4], [2, 3, 4], [1], [0, 0, 0],
                              [[1, 0, 0], [0, 1, 0], [0, 0, 1]], [[0], [0], [0]])),
    # identity tiler (the reference's implicit one)
    "copy_identity": (t1([33], [33], [1], [0], [[1]], [[0]]),
                      t1([33], [33], [1], [0], [[1]], [[0]])),
}


def make_copy_case(name, ts, td, devices, store):
    nin = int(np.prod(ts["array"]))
    nout = int(np.prod(td["array"]))
    src = np.arange(nin, dtype=np.float32) + 1.0      # index-valued, no -0 / NaN
    os_, od = offsets(ts), offsets(td)
    n = max(nin, nout)
    rows = [[] for _ in range(n)]
    for rs, rd in zip(os_, od):
        for a, b in zip(rs, rd):
            rows[b].append((a, 1.0))
    y = run_reference_spmv(rows, pad(src, n), "float32", devices)[:nout]
    store[f"{name}/src"] = src
    store[f"{name}/out"] = y
    return dict(op="tile_copy", tilers={"src": ts, "dst": td}, devices=devices)


def make_matmul_case(name, ta, tb, tc, seed, devices, store, dtype="float32"):
    rng = np.random.default_rng(seed)
    na, nb, nc = (int(np.prod(t["array"])) for t in (ta, tb, tc))
    a = rng.standard_normal(na).astype(dtype)
    b = rng.standard_normal(nb).astype(dtype)
    oa, ob, oc = offsets(ta), offsets(tb), offsets(tc)
    n = max(nb, nc)
    rows = [[] for _ in range(n)]
    for ra, rb, rc in zip(oa, ob, oc):
        rows[rc[0]] = [(cb, float(a[ca])) for ca, cb in zip(ra, rb)]
    y = run_reference_spmv(rows, pad(b, n), dtype, devices)[:nc]
    store[f"{name}/a"], store[f"{name}/b"], store[f"{name}/out"] = a, b, y
    return dict(op="matmul", tilers={"a": ta, "b": tb, "c": tc}, devices=devices, seed=seed)


def make_filter_case(name, op, tx, ty, w, seed, devices, store):
    rng = np.random.default_rng(seed)
    nx, ny = int(np.prod(tx["array"])), int(np.prod(ty["array"]))
    x = rng.random(nx).astype(np.float32)
    ox, oy = offsets(tx), offsets(ty)
    px = len(ox[0])
    n = max(nx, ny)
    rows = [[] for _ in range(n)]
    for rx, ry in zip(ox, oy):
        for j, dst in enumerate(ry):
            rows[dst] = [(src, float(w[j * px + i])) for i, src in enumerate(rx)]
    y = run_reference_spmv(rows, pad(x, n), "float32", devices)[:ny]
    store[f"{name}/x"], store[f"{name}/w"], store[f"{name}/out"] = x, w, y
    return dict(op=op, tilers={"x": tx, "y": ty}, devices=devices, seed=seed)


def make_sum_case(name, tx, ts, devices, store):
    nx, ns = int(np.prod(tx["array"])), int(np.prod(ts["array"]))
    x = (np.arange(nx, dtype=np.float32) % 97) * 0.25 + 0.5
    ox, os_ = offsets(tx), offsets(ts)
    n = max(nx, ns)
    rows = [[] for _ in range(n)]
    for rx, rs in zip(ox, os_):
        rows[rs[0]] = [(c, 1.0) for c in rx]
    y = run_reference_spmv(rows, pad(x, n), "float32", devices)[:ns]
    store[f"{name}/x"], store[f"{name}/out"] = x, y
    return dict(op="tile_sum", tilers={"x": tx, "s": ts}, devices=devices)


def make_identity_cases(store, meta):
    """Reference ops through their own intrinsics (test_refexec.py:311-389 style)."""
    specs = {
        "copy": (["src in {t} [64]", "dst out {t} [64]"], ["i in {t} [64]", "o out {t} [64]"],
                 ["i -> t.src", "t.dst -> o"], ["i"]),
        "sub": (["x in {t} [64]", "y in {t} [64]", "z out {t} [64]"],
                ["i1 in {t} [64]", "i2 in {t} [64]", "o out {t} [64]"],
                ["i1 -> t.x", "i2 -> t.y", "t.z -> o"], ["i1", "i2"]),
        "scale": (["y inout {t} [64]", "a in {t} [1]"],
                  ["i in {t} [64]", "s in {t} [1]", "o out {t} [64]"],
                  ["i -> t.y", "s -> t.a", "t.y -> o"], ["i", "s"]),
        "axpy": (["y inout {t} [64]", "x in {t} [64]", "a in {t} [1]"],
                 ["i in {t} [64]", "v in {t} [64]", "s in {t} [1]", "o out {t} [64]"],
                 ["i -> t.y", "v -> t.x", "s -> t.a", "t.y -> o"], ["i", "v", "s"]),
        "dot_partial": (["a in {t} [4096]", "b in {t} [4096]", "s out {t} [1]"],
                        ["i1 in {t} [4096]", "i2 in {t} [4096]", "o out {t} [1]"],
                        ["i1 -> t.a", "i2 -> t.b", "t.s -> o"], ["i1", "i2"]),
    }
    for op, (ports, root_ports, conns, binds) in specs.items():
        for dt in ("float32", "float64"):
            n = 4096 if op == "dot_partial" else 64
            allocs = [f"allocate data {b} onto {'host.ram' if b == 's' else 'dev.gmem'}"
                      for b in binds]
            outp = conns[-1].split(" -> ")[0]
            if op == "dot_partial":
                allocs.append("allocate data t.s onto host.ram")
            elif op in ("copy", "sub"):
                allocs.append(f"allocate data {outp} onto dev.gmem")
            allocs.append("allocate task t onto dev.cu")
            model = single_task_model(op, [p.format(t=dt) for p in ports],
                                      [p.format(t=dt) for p in root_ports], conns, allocs, n)
            rng = np.random.default_rng(zlib.crc32(f"{op}{dt}".encode()))
            bindings = {b: rng.standard_normal(1 if b == "s" else n).astype(dt) for b in binds}
            for d in (1, 3, 5):
                res = execute_schedule(model, build_schedule(model, d), dict(bindings), d)
                key = f"ident_{op}_{dt}_d{d}"
                for b, v in bindings.items():
                    store[f"{key}/in_{b}"] = v
                store[f"{key}/out"] = res.outputs["o"]
                meta[key] = dict(op=op, dtype=dt, devices=d, n=n, bind=binds)
    # spmv_csr fp64 on poisson_2d(8) at D=1,3 (test_refexec.py:350-371)
    A = poisson_2d(8)
    rng = np.random.default_rng(5)
    x = rng.standard_normal(A.n)
    for d in (1, 3):
        y = run_reference_csr(A.row_ptr, A.col_idx, A.values, x, "float64", d)
        key = f"ident_spmv_poisson8_d{d}"
        store[f"{key}/rowptr"], store[f"{key}/colidx"] = A.row_ptr, A.col_idx
        store[f"{key}/values"], store[f"{key}/x"], store[f"{key}/out"] = A.values, x, y
        meta[key] = dict(op="spmv_csr", dtype="float64", devices=d, n=A.n)


def make_cg_case(store, meta):
    """The paper's case study: CG on poisson_2d(20) through the unmodified executor at D = 1, 2, 4."""
    from gmodelc.refexec import instantiate_for_matrix
    from paper_1105_4424_b200.model import model_to_dict
    model = gmodelc.parse_model(gmodelc.bundled_model_text())
    A = poisson_2d(20)
    sized = instantiate_for_matrix(model, A.n, A.nnz)
    assert gmodelc.validate_conformance(sized) == []
    b = np.ones(A.n)
    bind = {"rowptr": A.row_ptr, "colidx": A.col_idx, "values": A.values, "b": b}
    for k, v in bind.items():
        store[f"cg_k20/{k}"] = v
    meta["cg_k20"] = {"op": "cg", "model": model_to_dict(sized), "runs": {}}
    from gmodelc.memmap import build_memory_maps, emit_memory_map_report
    meta["cg_k20"]["memmap_report"] = emit_memory_map_report(build_memory_maps(sized))
    meta["cg_bundled"] = {"op": "memmap", "model": model_to_dict(model),
                          "memmap_report": emit_memory_map_report(build_memory_maps(model))}
    for d in (1, 2, 4):
        res = execute_schedule(sized, build_schedule(sized, d), dict(bind), d)
        store[f"cg_k20/x_d{d}"] = res.outputs["x"]
        meta["cg_k20"]["runs"][str(d)] = {"iterations": res.iterations, "final_relres": res.final_relres,
                                          "converged": res.converged}


def main():
    store: dict[str, np.ndarray] = {}
    meta: dict[str, dict] = {}
    make_cg_case(store, meta)
    for i, (name, (ts, td)) in enumerate(COPY_CASES.items()):
        meta[name] = make_copy_case(name, ts, td, (1, 3, 5)[i % 3], store)

    # C1: the paper-case-study MatMul 256x256 fp32 through the reference executor (Kronecker spmv)
    g = orc.gemm_tilers(256, 256, 256)
    meta["matmul_c1_256"] = make_matmul_case("matmul_c1_256", g["a"], g["b"], g["c"], 0, 1, store)
    y8 = make_matmul_case("tmp", g["a"], g["b"], g["c"], 0, 8, store)
    assert np.array_equal(store.pop("tmp/out"), store["matmul_c1_256/out"]), "C1 not D-invariant"
    store.pop("tmp/a"), store.pop("tmp/b")
    del y8
    # small canonical GEMM, unaligned shards (D=3), non-multiple-of-tile sizes
    g = orc.gemm_tilers(37, 23, 19)
    meta["matmul_small_d3"] = make_matmul_case("matmul_small_d3", g["a"], g["b"], g["c"], 11, 3, store)
    # B given transposed (b array [N,K]) and a toroidal shift of A's rows
    M, N, K = 12, 10, 7
    ta = t1([M, K], [M, N], [K], [5, 0], [[1, 0], [0, 0]], [[0], [1]])
    tb = t1([N, K], [M, N], [K], [0, 0], [[0, 1], [0, 0]], [[0], [1]])
    tc = t1([M, N], [M, N], [1], [0, 0], [[1, 0], [0, 1]], [[0], [0]])
    meta["matmul_bt_torus"] = make_matmul_case("matmul_bt_torus", ta, tb, tc, 12, 2, store)

    st = orc.stencil_tilers(32, 48)
    meta["stencil_32x48"] = make_filter_case("stencil_32x48", "stencil", st["x"], st["y"],
                                             orc.stencil_weights(), 13, 5, store)
    ht = orc.hfilter_tilers(2, 4, 64)
    meta["hfilter_2x4x64"] = make_filter_case("hfilter_2x4x64", "hfilter", ht["x"], ht["y"],
                                              orc.hfilter_weights(), 14, 3, store)
    vt = orc.vfilter_tilers(2, 27, 8)
    meta["vfilter_2x27x8"] = make_filter_case("vfilter_2x27x8", "vfilter", vt["x"], vt["y"],
                                              orc.vfilter_weights(), 15, 2, store)
    rng = np.random.default_rng(16)
    wr = rng.standard_normal(4 * 6).astype(np.float32)
    tx = t1([9, 11], [4, 5], [2, 3], [7, 9], [[2, 0], [0, 2]], [[1, 0], [0, 1]])
    ty = t1([4, 5, 4], [4, 5], [4], [0, 0, 0], [[1, 0], [0, 1], [0, 0]], [[0], [0], [1]])
    meta["filter_generic_torus"] = make_filter_case("filter_generic_torus", "tile_filter", tx, ty,
                                                    wr, 17, 3, store)
    tx = t1([6, 40], [6], [40], [0, 0], [[1], [0]], [[0], [1]])
    ts = t1([6], [6], [1], [0], [[1]], [[0]])
    meta["sum_rows"] = make_sum_case("sum_rows", tx, ts, 2, store)

    make_identity_cases(store, meta)

    parts = {f"{t},{d}": [(w.offset, w.count) for w in partition_equally(t, d)]
             for t, d in ((132651, 4), (10, 1), (7, 3), (3, 8), (67108864, 8), (265420800, 3),
                          (1000003, 7))}
    meta["_partition"] = parts
    meta["_generator"] = dict(reference=str(REF_SRC), numpy=np.__version__,
                              gmodelc=getattr(gmodelc, "__version__", "?"))
    np.savez_compressed(HERE / "reference_golden.npz", **store)
    (HERE / "reference_golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(store)} arrays, {len(meta)} cases")


if __name__ == "__main__":
    main()
