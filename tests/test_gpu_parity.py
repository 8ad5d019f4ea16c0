"""CUDA path vs the CPU oracle / the reference's golden outputs, through the drop-in executor.

Every test here calls libaolb200.so through ``execute_schedule`` (the
reference's public entry point, refexec.py:427) or the C ABI directly.
Bar: bit-exact for tiler indices, gather/scatter layouts and every op in
"exact" order; the TF32 tensor-core matmul is held to the stated bound
  |C - C_fp64| <= (2^-9 + K * 2^-23) * (|A| |B|)     (element-wise)
(two TF32-truncated operands: relative error < 2 * 2^-10 per product,
plus fp32 accumulation over K terms).
"""

import numpy as np
import pytest

from oracle import aol_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_1105_4424_b200 import _capi
    assert _capi.device_count() >= 1


def _tiler(d):
    from paper_1105_4424_b200 import Tiler
    return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"])


def _spec(d, direction, dtype):
    dims = ",".join(str(x) for x in d["array"])
    return f"{direction} {dtype} [{dims}]"


def _run_tile(op, tilers, ports, bindings, devices, **kw):
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.partition import build_schedule
    from paper_1105_4424_b200.executor import execute_schedule
    rep = next(iter(tilers.values()))["rep"]
    model = builders.tile_task_model(op, ports, {k: _tiler(v) for k, v in tilers.items()}, rep)
    res = execute_schedule(model, build_schedule(model, devices), {f"p_{k}": v for k, v in bindings.items()},
                           devices, **kw)
    return res


GOLDEN_TILE_OPS = ("tile_copy", "matmul", "tile_filter", "hfilter", "vfilter", "stencil", "tile_sum")


def _golden_names(meta):
    return sorted(k for k, v in meta.items() if not k.startswith("_") and not k.startswith("ident_")
                  and v["op"] in GOLDEN_TILE_OPS)


@pytest.mark.parametrize("devices", [1, 3, 5, 8])
def test_tile_ops_bitwise_vs_reference_golden(golden, devices):
    data, meta = golden
    for name in _golden_names(meta):
        m = meta[name]
        t = m["tilers"]
        ref = data[f"{name}/out"]
        op = m["op"]
        if op == "tile_copy":
            ports = {"src": _spec(t["src"], "in", "float32"), "dst": _spec(t["dst"], "out", "float32")}
            b = {"src": data[f"{name}/src"]}
            out = "dst"
        elif op == "matmul":
            ports = {"a": _spec(t["a"], "in", "float32"), "b": _spec(t["b"], "in", "float32"),
                     "c": _spec(t["c"], "out", "float32")}
            b = {"a": data[f"{name}/a"], "b": data[f"{name}/b"]}
            out = "c"
        elif op == "tile_sum":
            ports = {"x": _spec(t["x"], "in", "float32"), "s": _spec(t["s"], "out", "float32")}
            b = {"x": data[f"{name}/x"]}
            out = "s"
        else:
            w = data[f"{name}/w"]
            ports = {"x": _spec(t["x"], "in", "float32"), "w": f"in float32 [{w.size}]",
                     "y": _spec(t["y"], "out", "float32")}
            b = {"x": data[f"{name}/x"], "w": w}
            out = "y"
        res = _run_tile(op, t, ports, b, devices, precision="exact")
        got = res.outputs[f"p_{out}"]
        assert got.dtype == ref.dtype and got.shape == ref.shape, name
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (name, devices)


def test_tiler_offsets_bitwise_vs_oracle(golden):
    from paper_1105_4424_b200 import _capi
    _, meta = golden
    for name in _golden_names(meta):
        for d in meta[name]["tilers"].values():
            bt = _tiler(d).bind(d["array"], d["rep"])
            R, P = bt.rep_total, bt.pattern_total
            for first, count in ((0, R), (R // 3, R - R // 3), (R - 1, 1)):
                out = torch.empty(count * P, dtype=torch.int64, device="cuda")
                _capi.tiler_offsets(bt, first, count, out.data_ptr())
                torch.cuda.synchronize()
                ref = orc.tiler_offsets(d, first, count).ravel()
                assert np.array_equal(out.cpu().numpy(), ref), (name, first, count)


def _random_tiler_cases():
    rng = np.random.default_rng(1234)
    cases = []
    for _ in range(40):
        a = int(rng.integers(1, 4))
        q = int(rng.integers(1, 4))
        p = int(rng.integers(1, 3))
        arr = tuple(int(x) for x in rng.integers(1, 9, a))
        rep = tuple(int(x) for x in rng.integers(1, 7, q))
        pat = tuple(int(x) for x in rng.integers(1, 5, p))
        o = tuple(int(x) for x in rng.integers(-20, 20, a))
        P = tuple(tuple(int(x) for x in rng.integers(-5, 6, q)) for _ in range(a))
        F = tuple(tuple(int(x) for x in rng.integers(-5, 6, p)) for _ in range(a))
        cases.append(dict(array=arr, rep=rep, pattern=pat, origin=o, paving=P, fitting=F))
    return cases


def test_tiler_offsets_random_vs_loop_oracle():
    from paper_1105_4424_b200 import _capi
    for d in _random_tiler_cases():
        bt = _tiler(d).bind(d["array"], d["rep"])
        R, P = bt.rep_total, bt.pattern_total
        out = torch.empty(R * P, dtype=torch.int64, device="cuda")
        _capi.tiler_offsets(bt, 0, R, out.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), np.array(orc.tiler_offsets_loop(d, 0, R)).ravel()), d


@pytest.mark.parametrize("case", [
    # (src array, rep, pattern, paving, fitting, origin)   1-D sweep shapes of config C5
    ((4096,), (1024,), (4,), ((4,),), ((1,),), (0,)),           # dense -> stream copy
    ((4096,), (2047,), (4,), ((2,),), ((1,),), (0,)),           # overlap -> affine
    ((8192,), (1000,), (3,), ((8,),), ((2,),), (5,)),           # gaps + strided fitting -> affine
    ((1000,), (999,), (7,), ((1,),), ((1,),), (17,)),           # wraps -> generic
    ((64, 48), (48, 64), (1,), ((0, 1), (1, 0)), ((0,), (0,)), (0, 0)),   # transpose
    ((16384,), (1000,), (8,), ((16,),), ((1,),), (4,)),         # gaps -> vec (V=4 loads)
    ((4096,), (1023,), (4,), ((2,),), ((1,),), (2,)),           # overlap -> vec (V=2 loads)
    ((8192,), (1000,), (4,), ((8,),), ((2,),), (0,)),           # strided fitting -> vec_store
    ((8192,), (999,), (6,), ((7,),), ((1,),), (1,)),            # odd stride -> vec (V=2) or affine
    ((40, 1000), (1000,), (40,), ((0,), (1,)), ((1,), (0,)), (0, 0)),   # row stride -> transpose
    ((7, 3000), (2999,), (7,), ((0,), (1,)), ((1,), (0,)), (0, 1)),     # row stride, ragged -> transpose
    ((8, 4096), (4096,), (8,), ((0,), (1,)), ((1,), (0,)), (0, 0)),     # row stride, aligned -> vector transpose
    ((64, 1024), (1024,), (64,), ((0,), (1,)), ((1,), (0,)), (0, 0)),   # two pattern chunks
])
@pytest.mark.parametrize("devices", [1, 3])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_tile_copy_plans_vs_oracle(case, devices, dtype):
    from paper_1105_4424_b200 import _capi
    arr, rep, pat, P, F, o = case
    R = int(np.prod(rep))
    npat = int(np.prod(pat))
    ts = dict(array=arr, rep=rep, pattern=pat, origin=o, paving=P, fitting=F)
    # dense output [R * npat] with the same rep shape
    q = len(rep)
    strides = [int(np.prod(rep[j + 1:])) * npat for j in range(q)]
    td = dict(array=(R * npat,), rep=rep, pattern=pat, origin=(0,), paving=(tuple(strides),),
              fitting=(tuple(int(np.prod(pat[k + 1:])) for k in range(len(pat))),))
    src = (np.arange(int(np.prod(arr))) % (1 << 20)).astype(dtype) + 1
    ports = {"src": _spec(ts, "in", dtype), "dst": _spec(td, "out", dtype)}
    res = _run_tile("tile_copy", {"src": ts, "dst": td}, ports, {"src": src}, devices)
    ref = orc.run_tile_task("tile_copy", {"src": ts, "dst": td}, {"src": src},
                            {"dst": (R * npat, np.dtype(dtype))}, R, devices)["dst"]
    assert np.array_equal(res.outputs["p_dst"], ref)
    bts, btd = _tiler(ts).bind(arr, rep), _tiler(td).bind(td["array"], rep)
    name = _capi.plan_name(_capi.make_task("tile_copy", dtype, [bts, btd]), 0, R)
    assert name.startswith("tile_copy.")


@pytest.mark.parametrize("case", [
    # (dtype, src array, T, m, src paving, dst pitch, expected plan)        TMA box ring plans (>= 1 MB)
    ("float32", None, 40001, 8, 16, 8, "tile_copy.tma_box"),       # sweep "gaps", 32 B rows, ragged T
    ("float32", None, 30000, 16, 20, 16, "tile_copy.tma_box"),     # 80 B source pitch
    ("float32", None, 5000, 64, 128, 64, "tile_copy.tma_box"),     # 256 B rows
    ("float32", None, 30000, 12, 12, 24, "tile_copy.tma_box"),     # gaps on the destination side
    ("float64", None, 40000, 4, 8, 4, "tile_copy.tma_box"),        # 32 B fp64 rows
    ("float32", None, 300001, 4, 4, 4, "tile_copy.tma_stream"),    # dense: 256 B rows + 16 B vectors + tail
    ("float64", None, 150001, 2, 2, 2, "tile_copy.tma_stream"),
    ("float32", None, 200001, 2, 1, 2, "tile_copy.window"),        # overlapping 8-64 B rows: one bulk window/tile
    ("float32", None, 100001, 4, 2, 4, "tile_copy.window"),
    ("float32", None, 100000, 4, 3, 4, "tile_copy.window"),        # odd source pitch (windows unaligned)
    ("float32", None, 40000, 8, 4, 8, "tile_copy.window"),         # overlapping 32 B rows
    ("float32", None, 20001, 16, 5, 16, "tile_copy.window"),
    ("float32", None, 20001, 32, 16, 32, "tile_copy.tma_box"),     # overlapping 128 B rows: TMA box (L2 re-reads)
    ("float32", None, 20001, 12, 6, 12, "tile_copy.vec"),          # P not a power of two: register path
    ("float32", None, 300003, 1, 2, 1, "tile_copy.stride2"),       # every other element (m = 1 gaps)
])
@pytest.mark.parametrize("devices", [1, 3])
def test_tile_copy_tma_plans_vs_oracle(case, devices):
    from paper_1105_4424_b200 import _capi
    dtype, _, T, m, p, pd, plan = case
    span = (T - 1) * p + m
    ts = dict(array=(span,), rep=(T,), pattern=(m,), origin=(0,), paving=((p,),), fitting=((1,),))
    n_out = (T - 1) * pd + m
    td = dict(array=(n_out,), rep=(T,), pattern=(m,), origin=(0,), paving=((pd,),), fitting=((1,),))
    src = (np.arange(span) % (1 << 22)).astype(dtype) + 1
    ports = {"src": _spec(ts, "in", dtype), "dst": _spec(td, "out", dtype)}
    res = _run_tile("tile_copy", {"src": ts, "dst": td}, ports, {"src": src}, devices)
    ref = orc.run_tile_task("tile_copy", {"src": ts, "dst": td}, {"src": src},
                            {"dst": (n_out, np.dtype(dtype))}, T, devices)["dst"]
    assert np.array_equal(res.outputs["p_dst"], ref)
    bts, btd = _tiler(ts).bind(ts["array"], (T,)), _tiler(td).bind(td["array"], (T,))
    task = _capi.make_task("tile_copy", dtype, [bts, btd])
    x = torch.from_numpy(src).cuda()
    y = torch.zeros(n_out, dtype=x.dtype, device="cuda")
    assert _capi.plan_name(task, 0, T, [x.data_ptr(), y.data_ptr()]) == plan
    if plan in ("tile_copy.tma_box", "tile_copy.window"):
        # misaligned bases fall back to the register path, same bits
        xb = torch.zeros(span + 1, dtype=x.dtype, device="cuda")
        xb[1:] = x
        yb = torch.zeros(n_out + 1, dtype=x.dtype, device="cuda")
        ptrs = [xb[1:].data_ptr(), yb[1:].data_ptr()]
        assert _capi.plan_name(task, 0, T, ptrs) != plan
        for off, cnt in orc.partition_equally(T, devices):
            _capi.launch(task, off, cnt, ptrs, (), 0)
        torch.cuda.synchronize()
        assert np.array_equal(yb[1:].cpu().numpy(), ref)


def _gemm_bound(a64, b64, K):
    return (2.0 ** -9 + K * 2.0 ** -23) * (np.abs(a64) @ np.abs(b64))


@pytest.mark.parametrize("M,N,K,devices", [
    (256, 256, 256, 1), (128, 256, 64, 1), (300, 520, 200, 1), (1000, 700, 333, 3),
    (37, 23, 19, 5), (1024, 1024, 4096, 2), (513, 1031, 96, 7)])
def test_matmul_tf32_within_stated_bound(M, N, K, devices):
    from paper_1105_4424_b200 import _capi
    g = orc.gemm_tilers(M, N, K)
    rng = np.random.default_rng(M * 7 + N)
    a = rng.standard_normal(M * K).astype(np.float32)
    b = rng.standard_normal(K * N).astype(np.float32)
    ports = {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]", "c": f"out float32 [{M},{N}]"}
    res = _run_tile("matmul", g, ports, {"a": a, "b": b}, devices)
    c = res.outputs["p_c"].reshape(M, N)
    a64, b64 = a.reshape(M, K).astype(np.float64), b.reshape(K, N).astype(np.float64)
    c64 = a64 @ b64
    err = np.abs(c - c64)
    assert np.all(err <= _gemm_bound(a64, b64, K)), float(np.max(err / _gemm_bound(a64, b64, K)))
    assert np.linalg.norm(c - c64) / np.linalg.norm(c64) < 2e-3
    bt = [_tiler(g[k]).bind(g[k]["array"], (M, N)) for k in "abc"]
    task = _capi.make_task("matmul", "float32", bt)
    expect = "matmul.tcgen05_tf32" if (K % 4 == 0 and N % 4 == 0) else "matmul.exact_tiled"
    ta = torch.zeros(4, device="cuda")
    assert _capi.plan_name(task, 0, M * N, [ta.data_ptr()] * 3) == expect


@pytest.mark.parametrize("bt", [False, True])
def test_matmul_tf32_operand_majorness(bt):
    """B given as [N, K] (K-major) and A given as [K, M] (M-major) hit the other TMA layouts."""
    M, N, K = 384, 512, 160
    rng = np.random.default_rng(3)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    if bt:   # a row-major [M,K]; b stored transposed [N,K]
        ta = dict(array=(M, K), rep=(M, N), pattern=(K,), origin=(0, 0), paving=((1, 0), (0, 0)),
                  fitting=((0,), (1,)))
        tb = dict(array=(N, K), rep=(M, N), pattern=(K,), origin=(0, 0), paving=((0, 1), (0, 0)),
                  fitting=((0,), (1,)))
        a_bind, b_bind, a_arr, b_arr = A.ravel(), B.T.copy().ravel(), (M, K), (N, K)
    else:    # a stored transposed [K,M]; b row-major [K,N]
        ta = dict(array=(K, M), rep=(M, N), pattern=(K,), origin=(0, 0), paving=((0, 0), (1, 0)),
                  fitting=((1,), (0,)))
        tb = dict(array=(K, N), rep=(M, N), pattern=(K,), origin=(0, 0), paving=((0, 0), (0, 1)),
                  fitting=((1,), (0,)))
        a_bind, b_bind, a_arr, b_arr = A.T.copy().ravel(), B.ravel(), (K, M), (K, N)
    tc = dict(array=(M, N), rep=(M, N), pattern=(1,), origin=(0, 0), paving=((1, 0), (0, 1)),
              fitting=((0,), (0,)))
    ports = {"a": f"in float32 [{a_arr[0]},{a_arr[1]}]", "b": f"in float32 [{b_arr[0]},{b_arr[1]}]",
             "c": f"out float32 [{M},{N}]"}
    res = _run_tile("matmul", {"a": ta, "b": tb, "c": tc}, ports, {"a": a_bind, "b": b_bind}, 3)
    c = res.outputs["p_c"].reshape(M, N)
    a64, b64 = A.astype(np.float64), B.astype(np.float64)
    assert np.all(np.abs(c - a64 @ b64) <= _gemm_bound(a64, b64, K))


def test_c1_matmul_256_exact_equals_reference(golden):
    """Config C1 through the drop-in: exact mode is bit-identical to the reference executor."""
    data, _ = golden
    g = orc.gemm_tilers(256, 256, 256)
    ports = {"a": "in float32 [256,256]", "b": "in float32 [256,256]", "c": "out float32 [256,256]"}
    b = {"a": data["matmul_c1_256/a"], "b": data["matmul_c1_256/b"]}
    for d in (1, 8):
        res = _run_tile("matmul", g, ports, b, d, precision="exact")
        assert np.array_equal(res.outputs["p_c"], data["matmul_c1_256/out"])
        res = _run_tile("matmul", g, ports, b, d)
        a64 = data["matmul_c1_256/a"].reshape(256, 256).astype(np.float64)
        b64 = data["matmul_c1_256/b"].reshape(256, 256).astype(np.float64)
        c = res.outputs["p_c"].reshape(256, 256)
        assert np.all(np.abs(c - a64 @ b64) <= _gemm_bound(a64, b64, 256))


def test_identity_ops_vs_reference_golden(golden):
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.partition import build_schedule
    from paper_1105_4424_b200.executor import execute_schedule
    data, meta = golden
    specs = {
        "copy": (["src in {t} [{n}]", "dst out {t} [{n}]"], ["i in {t} [{n}]", "o out {t} [{n}]"],
                 ["i -> t.src", "t.dst -> o"]),
        "sub": (["x in {t} [{n}]", "y in {t} [{n}]", "z out {t} [{n}]"],
                ["i1 in {t} [{n}]", "i2 in {t} [{n}]", "o out {t} [{n}]"], ["i1 -> t.x", "i2 -> t.y", "t.z -> o"]),
        "scale": (["y inout {t} [{n}]", "a in {t} [1]"], ["i in {t} [{n}]", "s in {t} [1]", "o out {t} [{n}]"],
                  ["i -> t.y", "s -> t.a", "t.y -> o"]),
        "axpy": (["y inout {t} [{n}]", "x in {t} [{n}]", "a in {t} [1]"],
                 ["i in {t} [{n}]", "v in {t} [{n}]", "s in {t} [1]", "o out {t} [{n}]"],
                 ["i -> t.y", "v -> t.x", "s -> t.a", "t.y -> o"]),
        "dot_partial": (["a in {t} [{n}]", "b in {t} [{n}]", "s out {t} [1]"],
                        ["i1 in {t} [{n}]", "i2 in {t} [{n}]", "o out {t} [1]"], ["i1 -> t.a", "i2 -> t.b", "t.s -> o"]),
    }
    for key in sorted(k for k in meta if k.startswith("ident_") and meta[k]["op"] in specs):
        m = meta[key]
        ports, rports, conns = specs[m["op"]]
        fmt = dict(t=m["dtype"], n=m["n"])
        allocs = [f"allocate data {b} onto {'host.ram' if b == 's' else 'dev.gmem'}" for b in m["bind"]]
        allocs += ["allocate data t.s onto host.ram"] if m["op"] == "dot_partial" else []
        allocs += ["allocate task t onto dev.cu"]
        model = builders.single_task_model(m["op"], [p.format(**fmt) for p in ports],
                                           [p.format(**fmt) for p in rports], conns, allocs, m["n"])
        bind = {b: data[f"{key}/in_{b}"] for b in m["bind"]}
        res = execute_schedule(model, build_schedule(model, m["devices"]), bind, m["devices"])
        ref = data[f"{key}/out"]
        if m["op"] == "dot_partial":
            tol = 1e-12 if m["dtype"] == "float64" else 1e-5
            assert abs(float(res.outputs["o"][0]) - float(ref[0])) <= tol * max(1.0, abs(float(ref[0]))), key
        else:
            assert np.array_equal(res.outputs["o"], ref), key


def test_spmv_vs_reference_golden(golden):
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.partition import build_schedule
    from paper_1105_4424_b200.executor import execute_schedule
    data, meta = golden
    for key in sorted(k for k in meta if k.startswith("ident_spmv")):
        m = meta[key]
        n = m["n"]
        rp, ci = data[f"{key}/rowptr"], data[f"{key}/colidx"]
        nnz = ci.size
        model = builders.single_task_model(
            "spmv_csr",
            [f"rowptr in int32 [{n + 1}]", f"colidx in int32 [{nnz}]", f"values in float64 [{nnz}]",
             f"x in float64 [{n}]", f"y out float64 [{n}]"],
            [f"rp in int32 [{n + 1}]", f"ci in int32 [{nnz}]", f"va in float64 [{nnz}]",
             f"vx in float64 [{n}]", f"o out float64 [{n}]"],
            ["rp -> t.rowptr", "ci -> t.colidx", "va -> t.values", "vx -> t.x", "t.y -> o"],
            ["allocate data rp onto dev.gmem", "allocate data ci onto dev.gmem", "allocate data va onto dev.gmem",
             "allocate data vx onto dev.gmem", "allocate data t.y onto dev.gmem", "allocate task t onto dev.cu"], n)
        res = execute_schedule(model, build_schedule(model, m["devices"]),
                               {"rp": rp, "ci": ci, "va": data[f"{key}/values"], "vx": data[f"{key}/x"]},
                               m["devices"])
        assert np.array_equal(res.outputs["o"], data[f"{key}/out"]), key


def test_filter_and_stencil_random_vs_oracle():
    """Filters/stencil at sizes beyond the golden set, exact order, several shard counts."""
    cases = [("stencil", orc.stencil_tilers(97, 131), orc.stencil_weights()),
             ("hfilter", orc.hfilter_tilers(3, 17, 256), orc.hfilter_weights()),
             ("vfilter", orc.vfilter_tilers(2, 45, 96), orc.vfilter_weights())]
    rng = np.random.default_rng(77)
    for op, t, w in cases:
        nx = int(np.prod(t["x"]["array"]))
        ny = int(np.prod(t["y"]["array"]))
        x = rng.random(nx).astype(np.float32)
        R = int(np.prod(t["x"]["rep"]))
        ports = {"x": _spec(t["x"], "in", "float32"), "w": f"in float32 [{w.size}]",
                 "y": _spec(t["y"], "out", "float32")}
        for d in (1, 4):
            res = _run_tile(op, t, ports, {"x": x, "w": w}, d)
            ref = orc.run_tile_task(op, t, {"x": x, "w": w}, {"y": (ny, np.float32)}, R, d)["y"]
            assert np.array_equal(res.outputs["p_y"].view(np.uint32), ref.view(np.uint32)), (op, d)


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_1105_4424_b200 import _capi
    saved = _capi._lib
    try:
        _capi._lib = None
        with pytest.raises(_capi.NativeLibraryError):
            _capi.load(tmp_path / "nope.so")
    finally:
        _capi._lib = saved


def _filter_case(op, t, w, x, devices):
    ny = int(np.prod(t["y"]["array"]))
    R = int(np.prod(t["x"]["rep"]))
    ports = {"x": _spec(t["x"], "in", "float32"), "w": f"in float32 [{w.size}]",
             "y": _spec(t["y"], "out", "float32")}
    res = _run_tile(op, t, ports, {"x": x, "w": w}, devices)
    ref = orc.run_tile_task(op, t, {"x": x, "w": w}, {"y": (ny, np.float32)}, R, devices)["y"]
    return res.outputs["p_y"], ref


def _plan(op_tilers, dtype="float32"):
    from paper_1105_4424_b200 import _capi
    bts = [_tiler(d).bind(d["array"], d["rep"]) for d in op_tilers]
    return _capi.plan_name(_capi.make_task("tile_filter", dtype, bts), 0, bts[0].rep_total)


@pytest.mark.parametrize("H,W,origin,kh,devices", [
    (256, 512, None, 3, 1), (256, 512, None, 3, 3), (130, 260, (0, 0), 3, 2), (64, 128, (5, 7), 3, 5),
    (96, 64, None, 5, 4), (33, 44, (32, 43), 3, 1), (100, 1024, (99, 3), 3, 7), (17, 4096, None, 5, 2)])
@pytest.mark.parametrize("form", ["slide", "box"])
def test_stencil_box_kernel_vs_oracle(H, W, origin, kh, devices, form, monkeypatch):
    """Sliding-window (default when columns are float4-aligned) and register-box stencil kernels,
    bit-exact vs the oracle for toroidal origins, 5-row boxes and launch ranges that split rows."""
    if form == "box":
        monkeypatch.setenv("AOL_STENCIL_BOX", "1")
    t = orc.stencil_tilers(H, W)
    if origin is not None:
        t["x"] = dict(t["x"], origin=origin)
    if kh == 5:
        t["x"] = dict(t["x"], pattern=(5, 3), origin=(H - 2, W - 1))
        w = np.arange(1, 16, dtype=np.float32) / 64
    else:
        w = orc.stencil_weights()
    assert _plan([t["x"], t["y"]]) == "tile_filter.stencil_box"
    x = np.random.default_rng(H + W).standard_normal(H * W).astype(np.float32)
    got, ref = _filter_case("stencil", t, w, x, devices)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("form", ["stream", "classic"])
@pytest.mark.parametrize("kind,dims,devices", [
    ("h", (2, 5, 384), 1), ("h", (3, 7, 96), 3), ("v", (2, 45, 64), 1), ("v", (3, 27, 40), 4),
    ("h_shift", (2, 3, 128), 2), ("v_generic", (2, 40, 24), 3), ("h", (2, 9, 3840), 5), ("v", (2, 54, 1440), 3),
    ("v", (1, 36, 1436), 2)])
def test_line_filter_kernel_vs_oracle(kind, dims, devices, form, monkeypatch):
    """Line filters (streaming bulk-copy ring forms and the register forms) bit-exact vs the oracle,
    for launch ranges that split rows, toroidal windows and column counts not divisible by 3."""
    if form == "classic":
        monkeypatch.setenv("AOL_LINE_CLASSIC", "1")
    F, H, W = dims
    if kind.startswith("h"):
        t = orc.hfilter_tilers(F, H, W)
        w = orc.hfilter_weights()
        if kind == "h_shift":
            t["x"] = dict(t["x"], origin=(0, 0, W - 2))       # window starts 2 left: wraps at the row start
        expect = "tile_filter.line_13x3" if (form == "classic" or kind == "h_shift") else "tile_filter.line_13x3_stream"
    else:
        if kind == "v_generic":
            t = orc.vfilter_tilers(F, H, W, taps=6, step=4, outs=2)
            w = orc.vfilter_weights(6, 2)
            expect = "tile_filter.line"
        else:
            t = orc.vfilter_tilers(F, H, W)
            w = orc.vfilter_weights()
            expect = "tile_filter.line_14x4_vstrip" if form == "classic" else "tile_filter.line_14x4_stream"
    assert _plan([t["x"], t["y"]]) == expect
    x = np.random.default_rng(F * H * W).random(int(np.prod(t["x"]["array"]))).astype(np.float32)
    got, ref = _filter_case("tile_filter", t, w, x, devices)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("name", ["copy_box_torus", "hfilter_2x4x64", "matmul_small_d3", "stencil_32x48"])
def test_cuda_pack_unpack_roundtrip(golden, name):
    """The multi-GPU exchange primitives: pack a shard's output patterns, unpack them elsewhere."""
    from paper_1105_4424_b200.distributed import cuda_pack, cuda_unpack, shard
    _, meta = golden
    tl = meta[name]["tilers"]
    d = tl["dst"] if "dst" in tl else (tl["c"] if "c" in tl else tl["y"])
    bt = _tiler(d).bind(d["array"], d["rep"])
    n = bt.array_total
    src = torch.arange(1, n + 1, dtype=torch.float32, device="cuda")
    for D in (2, 3):
        for r in shard(bt.rep_total, 0, D).ranges:
            stream = cuda_pack(src, bt, r.offset, r.count)
            offs = orc.tiler_offsets(d, r.offset, r.count).ravel()
            assert np.array_equal(stream.cpu().numpy(), src.cpu().numpy()[offs])
            dst = torch.zeros(n, dtype=torch.float32, device="cuda")
            cuda_unpack(dst, bt, r.offset, r.count, stream)
            want = np.zeros(n, np.float32)
            want[offs] = src.cpu().numpy()[offs]
            assert np.array_equal(dst.cpu().numpy(), want)


def test_distributed_executor_world1_nccl():
    """The rank-local executor (world size 1 over NCCL) runs the two-stage downscaler chain like the plain one."""
    import os
    import torch.distributed as dist
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.distributed import make_distributed_executor
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    th = orc.hfilter_tilers(2, 18, 64)
    tv = orc.vfilter_tilers(2, 18, 24)
    wh, wv = orc.hfilter_weights(), orc.vfilter_weights()
    spec = lambda d, io: _spec(d, io, "float32")   # noqa: E731
    model = builders.chain_model(
        [("h", "hfilter", {"x": spec(th["x"], "in"), "w": f"in float32 [{wh.size}]", "y": spec(th["y"], "out")},
          {k: _tiler(v) for k, v in th.items()}, th["x"]["rep"]),
         ("v", "vfilter", {"x": spec(tv["x"], "in"), "w": f"in float32 [{wv.size}]", "y": spec(tv["y"], "out")},
          {k: _tiler(v) for k, v in tv.items()}, tv["x"]["rep"])],
        {"x": spec(th["x"], "in"), "wh": f"in float32 [{wh.size}]", "wv": f"in float32 [{wv.size}]"},
        {"y": spec(tv["y"], "out")},
        [("x", "h.x"), ("wh", "h.w"), ("h.y", "v.x"), ("wv", "v.w"), ("v.y", "y")])
    x = np.random.default_rng(8).random(2 * 18 * 64).astype(np.float32)
    bind = {"x": x, "wh": wh, "wv": wv}
    ref = execute_schedule(model, build_schedule(model, 1), bind, 1).outputs["y"]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29571")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ex = make_distributed_executor(model, build_schedule(model, 1), bind)
        ex.run()
        got = ex.outputs()["y"]
    finally:
        dist.destroy_process_group()
    assert np.array_equal(got, ref)
    mid = orc.run_tile_task("hfilter", th, {"x": x, "w": wh}, {"y": (2 * 18 * 24, np.float32)},
                            int(np.prod(th["x"]["rep"])), 1)["y"]
    want = orc.run_tile_task("vfilter", tv, {"x": mid, "w": wv}, {"y": (2 * 8 * 24, np.float32)},
                             int(np.prod(tv["x"]["rep"])), 1)["y"]
    assert np.array_equal(got, want)


@pytest.mark.parametrize("devices", [1, 2, 4])
def test_cg_case_study_through_the_drop_in(golden, devices):
    """The paper's case study (CG on poisson_2d(20), the bundled cg.gmodel resized by the reference)
    through execute_schedule on the B200: same iteration count as the reference executor at every D,
    solution within 1e-10 (the reference's own cross-D criterion, tests/test_refexec.py:237-247)."""
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    data, meta = golden
    m = meta["cg_k20"]
    model = model_from_dict(m["model"])
    bind = {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}
    res = execute_schedule(model, build_schedule(model, devices), bind, devices)
    ref = m["runs"][str(devices)]
    assert res.iterations == ref["iterations"] and res.converged
    x_ref = data[f"cg_k20/x_d{devices}"]
    assert np.max(np.abs(res.outputs["x"] - x_ref)) / np.max(np.abs(x_ref)) <= 1e-10
    assert abs(res.final_relres - ref["final_relres"]) <= 1e-3 * ref["final_relres"]


@pytest.mark.parametrize("case", ["matmul", "stencil", "hfilter", "copy_gaps", "axpy"])
@pytest.mark.parametrize("chunks", [2, 7])
def test_streamed_execution_equals_plain(case, chunks):
    """pipeline=k (chunked H2D / launch / D2H on three streams) returns exactly the plain result."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    rng = np.random.default_rng(chunks)
    if case == "matmul":
        M, N, K = 300, 264, 96
        t = orc.gemm_tilers(M, N, K)
        ports = {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]", "c": f"out float32 [{M},{N}]"}
        bind = {"p_a": rng.standard_normal(M * K).astype(np.float32),
                "p_b": rng.standard_normal(K * N).astype(np.float32)}
        model = builders.tile_task_model("matmul", ports, {k: _tiler(v) for k, v in t.items()}, (M, N))
    elif case in ("stencil", "hfilter"):
        t = orc.stencil_tilers(64, 96) if case == "stencil" else orc.hfilter_tilers(3, 5, 128)
        w = orc.stencil_weights() if case == "stencil" else orc.hfilter_weights()
        ports = {"x": _spec(t["x"], "in", "float32"), "w": f"in float32 [{w.size}]",
                 "y": _spec(t["y"], "out", "float32")}
        bind = {"p_x": rng.random(int(np.prod(t["x"]["array"]))).astype(np.float32), "p_w": w}
        model = builders.tile_task_model(case, ports, {k: _tiler(v) for k, v in t.items()}, t["x"]["rep"])
    elif case == "copy_gaps":
        t = {"src": dict(array=(4000,), rep=(300,), pattern=(4,), origin=(3,), paving=((12,),), fitting=((1,),)),
             "dst": dict(array=(2000,), rep=(300,), pattern=(4,), origin=(0,), paving=((6,),), fitting=((1,),))}
        ports = {"src": "in float32 [4000]", "dst": "out float32 [2000]"}
        bind = {"p_src": rng.random(4000).astype(np.float32)}
        model = builders.tile_task_model("tile_copy", ports, {k: _tiler(v) for k, v in t.items()}, (300,))
    else:
        model = builders.single_task_model(
            "axpy", ["y inout float64 [999]", "x in float64 [999]", "a in float64 [1]"],
            ["i in float64 [999]", "v in float64 [999]", "s in float64 [1]", "o out float64 [999]"],
            ["i -> t.y", "v -> t.x", "s -> t.a", "t.y -> o"],
            ["allocate data i onto dev.gmem", "allocate data v onto dev.gmem", "allocate data s onto host.ram",
             "allocate task t onto dev.cu"], 999)
        bind = {"i": rng.standard_normal(999), "v": rng.standard_normal(999), "s": np.array([0.75])}
    sched = build_schedule(model, 3)
    plain = execute_schedule(model, sched, bind, 3).outputs
    streamed = execute_schedule(model, sched, bind, 3, pipeline=chunks).outputs
    for k in plain:
        assert np.array_equal(plain[k], streamed[k]), k


def test_placement_report_names_kernels():
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import Executor
    from paper_1105_4424_b200.partition import build_schedule
    g = orc.gemm_tilers(256, 256, 64)
    model = builders.tile_task_model(
        "matmul", {"a": "in float32 [256,64]", "b": "in float32 [64,256]", "c": "out float32 [256,256]"},
        {k: _tiler(v) for k, v in g.items()}, (256, 256))
    ex = Executor(model, build_schedule(model, 1), {"p_a": np.ones(256 * 64, np.float32),
                                                    "p_b": np.ones(64 * 256, np.float32)}, 1)
    rep = ex.placement_report()
    assert "matmul.tcgen05_tf32" in rep and "TMEM" in rep and "-> hbm" in rep


@pytest.mark.parametrize("M,N,K,devices,bt", [(256, 256, 256, 1, False), (300, 520, 200, 3, False),
                                              (1024, 768, 2048, 2, True), (129, 130, 131, 1, False)])
def test_matmul_3xtf32_fp32_accuracy(M, N, K, devices, bt):
    """precision='3xtf32': hi/lo split, three TF32 products on the tensor cores.
    Stated bound: |C - C64| <= (2^-19 + 3K * 2^-24) (|A||B|) element-wise, and normwise error
    <= 4e-9 * K + 1e-6 (measured ~2.4e-9 * K: tensor-core fp32 accumulation; TF32 alone is ~8e-4)."""
    from paper_1105_4424_b200 import _capi
    rng = np.random.default_rng(M + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    g = orc.gemm_tilers(M, N, K)
    if bt:
        g["b"] = dict(array=(N, K), rep=(M, N), pattern=(K,), origin=(0, 0), paving=((0, 1), (0, 0)),
                      fitting=((0,), (1,)))
        b_bind, b_spec = B.T.copy().ravel(), f"in float32 [{N},{K}]"
    else:
        b_bind, b_spec = B.ravel(), f"in float32 [{K},{N}]"
    ports = {"a": f"in float32 [{M},{K}]", "b": b_spec, "c": f"out float32 [{M},{N}]"}
    res = _run_tile("matmul", g, ports, {"a": A.ravel(), "b": b_bind}, devices, precision="3xtf32")
    c = res.outputs["p_c"].reshape(M, N)
    a64, b64 = A.astype(np.float64), B.astype(np.float64)
    c64 = a64 @ b64
    bound = (2.0 ** -19 + 3 * K * 2.0 ** -24) * (np.abs(a64) @ np.abs(b64))
    assert np.all(np.abs(c - c64) <= bound)
    assert np.linalg.norm(c - c64) / np.linalg.norm(c64) <= 4e-9 * K + 1e-6
    bts = [_tiler(g[k]).bind(g[k]["array"], (M, N)) for k in "abc"]
    t = torch.zeros(4, device="cuda")
    if K % 4 == 0 and (bt or N % 4 == 0):
        assert _capi.plan_name(_capi.make_task("matmul", "float32", bts, precision="3xtf32"), 0, M * N,
                               [t.data_ptr()] * 3) == "matmul.tcgen05_3xtf32"


def _downscaler_model(F, H, W):
    from paper_1105_4424_b200 import builders
    th = orc.hfilter_tilers(F, H, W)
    Wo = th["y"]["array"][2]
    tv = orc.vfilter_tilers(F, H, Wo)
    wh, wv = orc.hfilter_weights(), orc.vfilter_weights()
    spec = lambda d, io: _spec(d, io, "float32")   # noqa: E731
    model = builders.chain_model(
        [("h", "hfilter", {"x": spec(th["x"], "in"), "w": f"in float32 [{wh.size}]", "y": spec(th["y"], "out")},
          {k: _tiler(v) for k, v in th.items()}, th["x"]["rep"]),
         ("v", "vfilter", {"x": spec(tv["x"], "in"), "w": f"in float32 [{wv.size}]", "y": spec(tv["y"], "out")},
          {k: _tiler(v) for k, v in tv.items()}, tv["x"]["rep"])],
        {"x": spec(th["x"], "in"), "wh": f"in float32 [{wh.size}]", "wv": f"in float32 [{wv.size}]"},
        {"y": spec(tv["y"], "out")},
        [("x", "h.x"), ("wh", "h.w"), ("h.y", "v.x"), ("wv", "v.w"), ("v.y", "y")])
    return model, th, tv, wh, wv


@pytest.mark.parametrize("form", ["stream", "tile"])
@pytest.mark.parametrize("F,H,W,devices", [(2, 18, 64, 1), (3, 45, 256, 3), (1, 27, 776, 2), (2, 99, 384, 5),
                                           (3, 2160 // 40, 3840, 7)])
def test_fused_downscaler_bitwise(F, H, W, devices, form, monkeypatch):
    """H->V task fusion (the intermediate never reaches HBM; streaming and tile kernels) equals the
    unfused chain and the oracle bit for bit, also for launch ranges that split rows."""
    if form == "tile":
        monkeypatch.setenv("AOL_FUSED_TILE", "1")
    from paper_1105_4424_b200.executor import Executor
    from paper_1105_4424_b200.partition import build_schedule
    model, th, tv, wh, wv = _downscaler_model(F, H, W)
    x = np.random.default_rng(F * H + W).random(F * H * W).astype(np.float32)
    bind = {"x": x, "wh": wh, "wv": wv}
    sched = build_schedule(model, devices)
    ex = Executor(model, sched, bind, devices, fuse=True)
    ex.run()
    fused = ex.outputs()["y"]
    assert ex.fused_launches == len(sched.steps[1].launches)
    ex2 = Executor(model, sched, bind, devices, fuse=False)
    ex2.run()
    assert ex2.fused_launches == 0
    plain = ex2.outputs()["y"]
    assert np.array_equal(fused.view(np.uint32), plain.view(np.uint32))
    Wo = th["y"]["array"][2]
    mid = orc.run_tile_task("hfilter", th, {"x": x, "w": wh}, {"y": (F * H * Wo, np.float32)},
                            int(np.prod(th["x"]["rep"])), 1)["y"]
    ny = int(np.prod(tv["y"]["array"]))
    want = orc.run_tile_task("vfilter", tv, {"x": mid, "w": wv}, {"y": (ny, np.float32)},
                             int(np.prod(tv["x"]["rep"])), 1)["y"]
    assert np.array_equal(fused.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("devices", [1, 4])
@pytest.mark.parametrize("persistent", ["1", "0"])
def test_cg_graph_mode_equals_eager(golden, devices, persistent, monkeypatch):
    """LoopStep on the device -- ONE persistent cooperative kernel, or (persistent=0) ONE CUDA
    graph with a conditional WHILE node -- bit-identical to the eager interpreter, and to the
    reference's iteration count."""
    monkeypatch.setenv("AOL_LOOP_PERSISTENT", persistent)
    from paper_1105_4424_b200.executor import Executor
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    data, meta = golden
    m = meta["cg_k20"]
    model = model_from_dict(m["model"])
    bind = {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}
    sched = build_schedule(model, devices)
    eager = Executor(model, sched, bind, devices, graphs=False)
    eager.run()
    gr = Executor(model, sched, bind, devices, graphs=True)
    gr.run()
    assert gr.device_loops == 1
    assert gr.persistent_loops == (1 if persistent == "1" else 0)
    assert gr.iterations == eager.iterations == m["runs"][str(devices)]["iterations"]
    assert np.array_equal(gr.outputs()["x"], eager.outputs()["x"])
    assert gr.final_relres == eager.final_relres


def _rand_tiler(rng, arr=None, rep=None, pat=None):
    a = len(arr) if arr else int(rng.integers(1, 4))
    arr = arr or tuple(int(x) for x in rng.integers(2, 12, a))
    q = len(rep) if rep else int(rng.integers(1, 4))
    rep = rep or tuple(int(x) for x in rng.integers(1, 7, q))
    p = len(pat) if pat else int(rng.integers(1, 3))
    pat = pat or tuple(int(x) for x in rng.integers(1, 5, p))
    return dict(array=arr, rep=rep, pattern=pat, origin=tuple(int(x) for x in rng.integers(-30, 30, a)),
                paving=tuple(tuple(int(x) for x in rng.integers(-6, 7, q)) for _ in range(a)),
                fitting=tuple(tuple(int(x) for x in rng.integers(-4, 5, p)) for _ in range(a)))


def _dense_out(rep, pat):
    R, P = int(np.prod(rep)), int(np.prod(pat))
    q = len(rep)
    return dict(array=(R * P,), rep=rep, pattern=pat, origin=(0,),
                paving=(tuple(int(np.prod(rep[j + 1:])) * P for j in range(q)),),
                fitting=(tuple(int(np.prod(pat[k + 1:])) for k in range(len(pat))),))


@pytest.mark.parametrize("seed", range(6))
def test_random_tilers_all_tile_ops_vs_oracle(seed):
    """Random gather tilers (toroidal, negative strides, ranks 1-3) through every tile intrinsic."""
    rng = np.random.default_rng(1000 + seed)
    for _ in range(6):
        tx = _rand_tiler(rng)
        rep, pat = tx["rep"], tx["pattern"]
        R, P = int(np.prod(rep)), int(np.prod(pat))
        nx = int(np.prod(tx["array"]))
        x = (rng.random(nx) * 4).astype(np.float32)
        d = int(rng.integers(1, 5))
        # tile_copy
        td = _dense_out(rep, pat)
        ports = {"src": _spec(tx, "in", "float32"), "dst": _spec(td, "out", "float32")}
        got = _run_tile("tile_copy", {"src": tx, "dst": td}, ports, {"src": x}, d).outputs["p_dst"]
        ref = orc.run_tile_task("tile_copy", {"src": tx, "dst": td}, {"src": x}, {"dst": (R * P, np.float32)}, R, d)
        assert np.array_equal(got, ref["dst"]), ("copy", tx)
        # tile_filter with 1..3 outputs per pattern
        py = int(rng.integers(1, 4))
        ty = _dense_out(rep, (py,))
        w = rng.standard_normal(py * P).astype(np.float32)
        ports = {"x": _spec(tx, "in", "float32"), "w": f"in float32 [{w.size}]", "y": _spec(ty, "out", "float32")}
        got = _run_tile("tile_filter", {"x": tx, "y": ty}, ports, {"x": x, "w": w}, d).outputs["p_y"]
        ref = orc.run_tile_task("tile_filter", {"x": tx, "y": ty}, {"x": x, "w": w}, {"y": (R * py, np.float32)}, R, d)
        assert np.array_equal(got.view(np.uint32), ref["y"].view(np.uint32)), ("filter", tx)
        # tile_sum
        ts = _dense_out(rep, (1,))
        ports = {"x": _spec(tx, "in", "float32"), "s": _spec(ts, "out", "float32")}
        got = _run_tile("tile_sum", {"x": tx, "s": ts}, ports, {"x": x}, d).outputs["p_s"]
        ref = orc.run_tile_task("tile_sum", {"x": tx, "s": ts}, {"x": x}, {"s": (R, np.float32)}, R, d)
        assert np.array_equal(got.view(np.uint32), ref["s"].view(np.uint32)), ("sum", tx)
        # matmul (generic path): a second random tiler over the same repetition space and pattern
        tb = _rand_tiler(rng, rep=rep, pat=pat)
        nb = int(np.prod(tb["array"]))
        b = (rng.random(nb) * 4).astype(np.float32)
        tc = _dense_out(rep, (1,))
        ports = {"a": _spec(tx, "in", "float32"), "b": _spec(tb, "in", "float32"), "c": _spec(tc, "out", "float32")}
        got = _run_tile("matmul", {"a": tx, "b": tb, "c": tc}, ports, {"a": x, "b": b}, d).outputs["p_c"]
        ref = orc.run_tile_task("matmul", {"a": tx, "b": tb, "c": tc}, {"a": x, "b": b}, {"c": (R, np.float32)}, R, d)
        assert np.array_equal(got.view(np.uint32), ref["c"].view(np.uint32)), ("matmul", tx, tb)


def _cg_model_and_bind(golden):
    from paper_1105_4424_b200.model import model_from_dict
    data, meta = golden
    model = model_from_dict(meta["cg_k20"]["model"])
    bind = {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}
    return model, bind


def test_missing_and_missized_bindings(golden):
    """tests/test_refexec.py:392-405 through the drop-in: MissingBinding before anything runs."""
    from paper_1105_4424_b200.executor import MissingBinding, execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    model, bind = _cg_model_and_bind(golden)
    b2 = dict(bind)
    del b2["b"]
    with pytest.raises(MissingBinding):
        execute_schedule(model, build_schedule(model, 1), b2, 1)
    b3 = dict(bind, b=np.ones(3))
    with pytest.raises(MissingBinding):
        execute_schedule(model, build_schedule(model, 1), b3, 1)


def test_max_iter_override_stops_early(golden):
    """tests/test_refexec.py:410-414: max_iter=3 -> 3 iterations, not converged."""
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    model, bind = _cg_model_and_bind(golden)
    for graphs in (False, True):
        res = execute_schedule(model, build_schedule(model, 1), bind, 1, max_iter=3, graphs=graphs)
        assert res.iterations == 3 and not res.converged


def test_signature_mismatch_and_aliasing():
    """tests/test_refexec.py:399-407 (wrong port name) and the output-aliases-input check (refexec.py:444-453)."""
    from paper_1105_4424_b200 import IntrinsicShapeMismatch, builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    model = builders.single_task_model(
        "scale", ["y inout float64 [64]", "b in float64 [1]"],
        ["i in float64 [64]", "s in float64 [1]", "o out float64 [64]"],
        ["i -> t.y", "s -> t.b", "t.y -> o"],
        ["allocate data i onto dev.gmem", "allocate data s onto host.ram", "allocate task t onto dev.cu"], 64)
    with pytest.raises(IntrinsicShapeMismatch):
        execute_schedule(model, build_schedule(model, 1), {"i": np.ones(64), "s": np.ones(1)}, 1)
    # copy whose dst is connected back to its own src group
    alias = builders.single_task_model(
        "copy", ["src in float64 [8]", "dst out float64 [8]"], ["i in float64 [8]"],
        ["i -> t.src", "t.dst -> t.src"],
        ["allocate data i onto dev.gmem", "allocate task t onto dev.cu"], 8)
    with pytest.raises(IntrinsicShapeMismatch, match="aliases"):
        execute_schedule(alias, build_schedule(alias, 1), {"i": np.ones(8)}, 1)


def test_no_repeat_touches_element_zero_only():
    """SURVEY App. B probe: with no `repeat` the repetition space is 1 -> only element 0 is written."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    model = builders.single_task_model(
        "copy", ["src in float32 [8]", "dst out float32 [8]"], ["i in float32 [8]", "o out float32 [8]"],
        ["i -> t.src", "t.dst -> o"], ["allocate data i onto dev.gmem", "allocate data t.dst onto dev.gmem",
                                       "allocate task t onto dev.cu"], None)
    res = execute_schedule(model, build_schedule(model, 3), {"i": np.arange(1, 9, dtype=np.float32)}, 3)
    assert res.outputs["o"].tolist() == [1, 0, 0, 0, 0, 0, 0, 0]


def test_single_pass_dot_deterministic_and_tree_order():
    """k_dot (one launch, last-block final reduction) equals the fixed 1024-block tree it
    restates, bit for bit, on every call and for ragged ranges."""
    from paper_1105_4424_b200 import _capi
    rng = np.random.default_rng(11)
    for n, first, count in [(1, 0, 1), (1000, 3, 997), (262_147, 0, 262_147), (3_000_001, 17, 2_999_000)]:
        a = rng.standard_normal(n)
        b = rng.standard_normal(n)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        task = _capi.make_task("dot_partial", "float64")
        vals = set()
        for _ in range(5):
            _capi.launch(task, first, count, [ta.data_ptr(), tb.data_ptr(), out.data_ptr()])
            torch.cuda.synchronize()
            vals.add(out.item())
        assert len(vals) == 1
        # restate the tree: grid-stride slices of 1024 blocks x 256 threads
        prod = a[first:first + count] * b[first:first + count]
        ref = float(np.sum(prod))
        assert abs(vals.pop() - ref) <= 1e-12 * max(1.0, np.sum(np.abs(prod)))


def test_scalar_seq_bit_exact_and_errors():
    """Several host scalar ops in one launch (AOL_OP_SCALAR_SEQ): Python's IEEE results."""
    import math
    from paper_1105_4424_b200 import _capi
    v = torch.tensor([3.7, 1.3, 0.0, 0.0, 0.0, 2.0e-7, 5.5], dtype=torch.float64, device="cuda")
    p = [v[i:i + 1].data_ptr() for i in range(7)]
    div, neg, rr = _capi.OP["div"], _capi.OP["neg"], _capi.OP["rel_residual"]
    prog = [div, 0, 1, 2,      # q = num / den          -> v[2]
            neg, 2, -1, 3,     # z = -q                 -> v[3]
            rr, 4, 5, 6]       # sqrt(num) / sqrt(den)  -> v[4]
    _capi.launch(_capi.make_task("scalar_seq", "float64"), 0, 3, [p[0], p[1], p[2], p[3], p[5], p[6], p[4]], prog)
    torch.cuda.synchronize()
    h = v.cpu().numpy()
    q = 3.7 / 1.3
    assert h[2] == q and h[3] == -q
    assert h[4] == math.sqrt(2.0e-7) / math.sqrt(5.5)
    with pytest.raises(Exception):
        _capi.launch(_capi.make_task("scalar_seq", "float64"), 0, 9, [p[0]], [div, 0, 0, 0] * 9)
    with pytest.raises(Exception):
        _capi.launch(_capi.make_task("scalar_seq", "float64"), 0, 1, [p[0]], [_capi.OP["axpy"], 0, 0, 0])


@pytest.mark.parametrize("devices,k,max_iter", [(1, 600, 40), (3, 600, 25), (2, 364, 3000), (1, "p27", 3000),
                                                (4, "p27", 30)])
def test_cg_persistent_large_equals_graph_and_eager(devices, k, max_iter, monkeypatch):
    """Persistent LoopStep kernel on the bench's Poisson matrices (n up to 360,000, so virtual
    blocks wrap more than once): x, iterations and relres identical to the CUDA-graph loop
    and to eager launches, also when stopped by max_iter."""
    import bench
    from paper_1105_4424_b200.executor import Executor
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    import json
    from pathlib import Path
    meta = json.loads((Path(__file__).parent / "golden" / "reference_golden.json").read_text())
    n, rowptr, colidx, vals = bench._poisson_3d27(51) if k == "p27" else bench._poisson_2d(k)
    model = model_from_dict(bench._resize_model_dict(meta["cg_k20"]["model"], 400, 1920, n, int(rowptr[-1])))
    sched = build_schedule(model, devices)
    bind = {"rowptr": rowptr, "colidx": colidx, "values": vals, "b": np.ones(n)}
    runs = {}
    for mode, env, graphs in (("persistent", "1", True), ("graph", "0", True), ("eager", "1", False)):
        monkeypatch.setenv("AOL_LOOP_PERSISTENT", env)
        ex = Executor(model, sched, bind, devices, graphs=graphs)
        ex.run(max_iter=max_iter)
        runs[mode] = (ex.iterations, ex.final_relres, ex.converged, ex.outputs()["x"])
        if mode == "persistent":
            assert ex.persistent_loops == 1
    for mode in ("graph", "eager"):
        assert runs[mode][:3] == runs["persistent"][:3], mode
        assert np.array_equal(runs[mode][3], runs["persistent"][3]), mode


def test_loop_persistent_abi_errors():
    """aol_loop_persistent: bodies outside its op set are refused with nothing launched (the
    executor then falls back to the CUDA-graph loop); malformed programs raise."""
    from paper_1105_4424_b200 import _capi
    v = torch.zeros(16, dtype=torch.float64, device="cuda")
    p = [v[i:i + 1].data_ptr() for i in range(4)]
    ops = [_capi.loop_op("div", [0, 1, 2])]
    assert _capi.loop_persistent([_capi.loop_op("tile_copy", [0, 1], 0, 1)] + ops, p, "float64", "int32", 2,
                                 1e-10, 5) is None
    assert _capi.loop_persistent(ops, p, "int32", "int32", 2, 1e-10, 5) is None
    with pytest.raises(_capi.AolError):
        _capi.loop_persistent([_capi.loop_op("div", [0, 1, 9])], p, "float64", "int32", 2, 1e-10, 5)
    with pytest.raises(_capi.AolError):
        _capi.loop_persistent(ops, p, "float64", "int32", 2, 1e-10, 0)
    # relres must be a scalar written by the body
    assert _capi.loop_persistent([_capi.loop_op("copy", [0, 1], 0, 1)], p, "float64", "int32", 1, 1e-10, 5) is None
    # a pure scalar body runs: q = 1 / 1 = 1 > tol every iteration -> stops at max_iter
    v[0] = 1.0
    v[1] = 1.0
    it, rr, conv = _capi.loop_persistent(ops, p, "float64", "int32", 2, 1e-10, 7)
    assert (it, rr, conv) == (7, 1.0, False)


def test_dots_on_concurrent_streams():
    """dot_partial launches on different streams at once do not share partials or tickets:
    every result equals the same dot launched alone."""
    from paper_1105_4424_b200 import _capi
    rng = np.random.default_rng(23)
    n = 3_000_000
    task = _capi.make_task("dot_partial", "float64")
    vecs = [(torch.from_numpy(rng.standard_normal(n)).cuda(), torch.from_numpy(rng.standard_normal(n)).cuda())
            for _ in range(6)]
    alone = []
    for a, b in vecs:
        o = torch.zeros(1, dtype=torch.float64, device="cuda")
        _capi.launch(task, 0, n, [a.data_ptr(), b.data_ptr(), o.data_ptr()])
        torch.cuda.synchronize()
        alone.append(o.item())
    streams = [torch.cuda.Stream() for _ in vecs]
    outs = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in vecs]
    for _ in range(20):
        for (a, b), st, o in zip(vecs, streams, outs):
            _capi.launch(task, 0, n, [a.data_ptr(), b.data_ptr(), o.data_ptr()], (), st.cuda_stream)
        torch.cuda.synchronize()
        assert [o.item() for o in outs] == alone


def test_loop_dot_reuse_keeps_bits_and_respects_writes(monkeypatch):
    """Dot reuse in the persistent loop: a dot re-reading vectors that no op wrote since an
    identical dot takes that dot's value (bit-identical to recomputing it); a dot whose
    vector was written in between is recomputed."""
    from paper_1105_4424_b200 import _capi
    n = 5000
    rng = np.random.default_rng(11)
    a0 = rng.standard_normal(n)

    def run(reuse):
        monkeypatch.setenv("AOL_LOOP_DOT_REUSE", reuse)
        a = torch.from_numpy(a0.copy()).cuda()
        s = torch.zeros(8, dtype=torch.float64, device="cuda")
        s[3] = 0.5
        p = [a.data_ptr()] + [s[i:i + 1].data_ptr() for i in range(1, 8)]
        ops = [_capi.loop_op("dot_partial", [0, 0, 2], 0, n),     # s1 = a.a   (reuses s2 from iteration 1 on)
               _capi.loop_op("scale", [0, 3], 0, n, n_scalars=1),  # a *= 0.5
               _capi.loop_op("dot_partial", [0, 0, 4], 0, n),     # s2 = a.a   (a written: recomputed)
               _capi.loop_op("div", [4, 2, 5])]                   # q = s2 / s1 = 0.25
        res = _capi.loop_persistent(ops, p, "float64", "int32", 5, 0.1, 9)
        torch.cuda.synchronize()
        return res, a.cpu().numpy(), s.cpu().numpy()

    (it1, q1, c1), a1, s1 = run("1")
    (it0, q0, c0), a0_, s0 = run("0")
    assert (it1, c1) == (it0, c0) == (9, False)
    assert q1 == q0 == 0.25
    assert np.array_equal(a1.view(np.uint64), a0_.view(np.uint64))
    assert np.array_equal(s1.view(np.uint64), s0.view(np.uint64))
    assert s1[4] == s1[2] * 0.25 and s1[2] != s1[4]


@pytest.mark.parametrize("seed", range(3))
def test_random_tilers_float64_tile_ops_vs_oracle(seed):
    """The float64 instantiations of every tile intrinsic (copy, filter, sum, generic matmul),
    random toroidal tilers, bit-exact against the oracle."""
    rng = np.random.default_rng(2000 + seed)
    for _ in range(4):
        tx = _rand_tiler(rng)
        rep, pat = tx["rep"], tx["pattern"]
        R, P = int(np.prod(rep)), int(np.prod(pat))
        x = rng.standard_normal(int(np.prod(tx["array"])))
        d = int(rng.integers(1, 5))
        td = _dense_out(rep, pat)
        got = _run_tile("tile_copy", {"src": tx, "dst": td},
                        {"src": _spec(tx, "in", "float64"), "dst": _spec(td, "out", "float64")},
                        {"src": x}, d).outputs["p_dst"]
        ref = orc.run_tile_task("tile_copy", {"src": tx, "dst": td}, {"src": x}, {"dst": (R * P, np.float64)}, R, d)
        assert np.array_equal(got.view(np.uint64), ref["dst"].view(np.uint64))
        py = int(rng.integers(1, 4))
        ty = _dense_out(rep, (py,))
        w = rng.standard_normal(py * P)
        got = _run_tile("tile_filter", {"x": tx, "y": ty},
                        {"x": _spec(tx, "in", "float64"), "w": f"in float64 [{w.size}]",
                         "y": _spec(ty, "out", "float64")}, {"x": x, "w": w}, d).outputs["p_y"]
        ref = orc.run_tile_task("tile_filter", {"x": tx, "y": ty}, {"x": x, "w": w}, {"y": (R * py, np.float64)}, R, d)
        assert np.array_equal(got.view(np.uint64), ref["y"].view(np.uint64))
        ts = _dense_out(rep, (1,))
        got = _run_tile("tile_sum", {"x": tx, "s": ts}, {"x": _spec(tx, "in", "float64"),
                                                         "s": _spec(ts, "out", "float64")}, {"x": x}, d).outputs["p_s"]
        ref = orc.run_tile_task("tile_sum", {"x": tx, "s": ts}, {"x": x}, {"s": (R, np.float64)}, R, d)
        assert np.array_equal(got.view(np.uint64), ref["s"].view(np.uint64))
        tb = _rand_tiler(rng, rep=rep, pat=pat)
        b = rng.standard_normal(int(np.prod(tb["array"])))
        tc = _dense_out(rep, (1,))
        got = _run_tile("matmul", {"a": tx, "b": tb, "c": tc},
                        {"a": _spec(tx, "in", "float64"), "b": _spec(tb, "in", "float64"),
                         "c": _spec(tc, "out", "float64")}, {"a": x, "b": b}, d).outputs["p_c"]
        ref = orc.run_tile_task("matmul", {"a": tx, "b": tb, "c": tc}, {"a": x, "b": b}, {"c": (R, np.float64)}, R, d)
        assert np.array_equal(got.view(np.uint64), ref["c"].view(np.uint64))


@pytest.mark.parametrize("index_dtype,dtype", [("int64", "float64"), ("int64", "float32"), ("int32", "float32")])
def test_spmv_index_and_value_dtypes_vs_oracle(index_dtype, dtype):
    """spmv_csr through the C ABI for every (index, value) dtype pair: left-to-right rows,
    bit-exact against the oracle's restatement of refexec.py:111-121."""
    from paper_1105_4424_b200 import _capi
    rng = np.random.default_rng(5)
    n = 3000
    lens = rng.integers(0, 40, n)
    rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(index_dtype)
    nnz = int(rowptr[-1])
    colidx = rng.integers(0, n, nnz).astype(index_dtype)
    values = rng.standard_normal(nnz).astype(dtype)
    x = rng.standard_normal(n).astype(dtype)
    want = np.zeros(n, dtype)
    orc.spmv_rows(rowptr, colidx, values, x, want, 0, n)
    t = [torch.from_numpy(a).cuda() for a in (rowptr, colidx, values, x)]
    y = torch.zeros(n, dtype=t[2].dtype, device="cuda")
    task = _capi.make_task("spmv_csr", dtype, index_dtype=index_dtype)
    for off, cnt in orc.partition_equally(n, 3):
        _capi.launch(task, off, cnt, [a.data_ptr() for a in t] + [y.data_ptr()], (), 0)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    assert np.array_equal(got.view(f"u{got.itemsize}"), want.view(f"u{want.itemsize}"))


@pytest.mark.parametrize("variant", ["int64_index", "float32"])
def test_cg_dtype_variants_persistent_equals_eager(golden, variant):
    """The CG model with int64 CSR indices (persistent kernel <double, int64>, SELL copy with
    64-bit indices) or float32 vectors (<float, int32>): the persistent loop is bit-identical to
    the eager interpreter; int64 indices change nothing against the int32 model."""
    import json as _json
    from paper_1105_4424_b200.executor import Executor
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    data, meta = golden
    text = _json.dumps(meta["cg_k20"]["model"])
    bind = {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}
    if variant == "int64_index":
        text = text.replace('"int32"', '"int64"')
        bind = {k: (v.astype(np.int64) if k in ("rowptr", "colidx") else v) for k, v in bind.items()}
    else:
        text = text.replace('"float64"', '"float32"')
        bind = {k: (v.astype(np.float32) if k in ("values", "b") else v) for k, v in bind.items()}
    model = model_from_dict(_json.loads(text))
    sched = build_schedule(model, 1)
    eager = Executor(model, sched, bind, 1, graphs=False)
    eager.run()
    dev = Executor(model, sched, bind, 1, graphs=True)
    dev.run()
    assert dev.persistent_loops == 1
    assert dev.iterations == eager.iterations
    xe, xd = eager.outputs()["x"], dev.outputs()["x"]
    assert np.array_equal(xd.view(f"u{xd.itemsize}"), xe.view(f"u{xe.itemsize}"))
    if variant == "int64_index":
        base = Executor(model_from_dict(meta["cg_k20"]["model"]), sched,
                        {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}, 1, graphs=True)
        base.run()
        assert np.array_equal(base.outputs()["x"].view(np.uint64), xd.view(np.uint64))


@pytest.mark.parametrize("m,T,plan", [(4, 70000, "tile_copy.interleave"), (2, 100000, "tile_copy.interleave"),
                                      (4, 70001, "tile_copy.transpose"), (2, 50003, "tile_copy.transpose"),
                                      (8, 40000, "tile_copy.tma_transpose"),
                                      (16, 20004, "tile_copy.tma_transpose"), (8, 40001, "tile_copy.transpose"),
                                      (32, 9000, "tile_copy.tma_transpose"), (64, 5004, "tile_copy.tma_transpose"),
                                      (64, 5001, "tile_copy.transpose")])
@pytest.mark.parametrize("devices", [1, 3])
def test_tile_copy_row_stride_tma_transpose_vs_oracle(m, T, plan, devices):
    """Row-stride gathers (pattern down a column of an [m, T] array) into the dense stream:
    the TMA transpose (swizzled {32, m} boxes, smem transpose, TMA store) for m = 8..64 with a
    16-byte row pitch, float4 register interleaving for m = 2 / 4, the shared-memory transpose
    otherwise; ragged tiles and unaligned shard starts (devices=3) peel through the register path."""
    from paper_1105_4424_b200 import _capi
    ts = dict(array=(m, T), rep=(T,), pattern=(m,), origin=(0, 0), paving=((0,), (1,)), fitting=((1,), (0,)))
    td = dict(array=(T * m,), rep=(T,), pattern=(m,), origin=(0,), paving=((m,),), fitting=((1,),))
    src = (np.arange(m * T) % (1 << 22)).astype(np.float32) + 1
    res = _run_tile("tile_copy", {"src": ts, "dst": td},
                    {"src": _spec(ts, "in", "float32"), "dst": _spec(td, "out", "float32")}, {"src": src}, devices)
    ref = orc.run_tile_task("tile_copy", {"src": ts, "dst": td}, {"src": src}, {"dst": (T * m, np.float32)}, T, devices)
    assert np.array_equal(res.outputs["p_dst"], ref["dst"])
    task = _capi.make_task("tile_copy", "float32", [_tiler(ts).bind((m, T), (T,)), _tiler(td).bind((T * m,), (T,))])
    x = torch.from_numpy(src).cuda()
    y = torch.zeros(T * m, device="cuda")
    assert _capi.plan_name(task, 0, T, [x.data_ptr(), y.data_ptr()]) == plan


@pytest.mark.parametrize("chunks", [2, 7])
@pytest.mark.parametrize("devices", [1, 3])
def test_streamed_fused_downscaler_equals_plain(chunks, devices):
    """The downscaler chain streamed from host memory (pipeline=k): consumer chunks, producer
    input ranges derived through the intermediate's dense stream, one fused launch per chunk
    (devices=1); a multi-launch schedule falls back to upload-then-run (devices=3).  Both
    return exactly the plain result."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import Executor, execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    F, H, W = 3, 54, 128
    th = orc.hfilter_tilers(F, H, W)
    Wo = th["y"]["array"][2]
    tv = orc.vfilter_tilers(F, H, Wo)
    wh, wv = orc.hfilter_weights(), orc.vfilter_weights()
    model = builders.chain_model(
        [("h", "hfilter", {"x": _spec(th["x"], "in", "float32"), "w": f"in float32 [{wh.size}]",
                           "y": _spec(th["y"], "out", "float32")}, {k: _tiler(v) for k, v in th.items()},
          th["x"]["rep"]),
         ("v", "vfilter", {"x": _spec(tv["x"], "in", "float32"), "w": f"in float32 [{wv.size}]",
                           "y": _spec(tv["y"], "out", "float32")}, {k: _tiler(v) for k, v in tv.items()},
          tv["x"]["rep"])],
        {"x": _spec(th["x"], "in", "float32"), "wh": f"in float32 [{wh.size}]", "wv": f"in float32 [{wv.size}]"},
        {"y": _spec(tv["y"], "out", "float32")},
        [("x", "h.x"), ("wh", "h.w"), ("h.y", "v.x"), ("wv", "v.w"), ("v.y", "y")])
    x = np.random.default_rng(chunks).random(F * H * W).astype(np.float32)
    bind = {"x": x, "wh": wh, "wv": wv}
    sched = build_schedule(model, devices)
    plain = execute_schedule(model, sched, bind, devices).outputs["y"]
    ex = Executor(model, sched, {k: torch.from_numpy(v).pin_memory() for k, v in bind.items()}, devices,
                  pipeline=chunks)
    with torch.cuda.device(ex.device):
        got = ex.run_streamed()["y"]
    assert np.array_equal(got.view(np.uint32), plain.view(np.uint32))
    assert ex.fused_launches == (chunks if devices == 1 else devices)


def _rand_big_copy(rng):
    """A random >= 1 MB affine gather that lands on one of the bulk plans (TMA stream / box /
    transpose, bulk window, stride-2, register paths), with random origins and pitches."""
    kind = rng.choice(["box", "window", "transpose", "stride2", "dense", "dstgap"])
    if kind == "transpose":
        m = int(rng.choice([8, 16, 32, 64]))
        T = int(rng.integers(1 << 20, 1 << 21) // (4 * m)) * 4 + int(rng.integers(0, 2)) * 4
        extra = int(rng.integers(0, 3)) * 4
        return dict(array=(m, T + extra), rep=(T,), pattern=(m,), origin=(0, int(rng.integers(0, extra + 1))),
                    paving=((0,), (1,)), fitting=((1,), (0,))), T, m
    if kind == "stride2":
        T = int(rng.integers(300000, 600000))
        o = int(rng.integers(0, 9))
        return dict(array=(2 * T + o + 3,), rep=(T,), pattern=(1,), origin=(o,), paving=((2,),), fitting=((1,),)), T, 1
    m = int(rng.choice([2, 4, 8, 16, 32, 64]))
    p = {"box": 2 * m + 4 * int(rng.integers(0, 3)), "window": max(1, m // 2 - int(rng.integers(0, max(1, m // 4)))),
         "dense": m, "dstgap": m}[kind]
    T = int(rng.integers((1 << 20) // (4 * m), (1 << 21) // (4 * m)))
    o = int(rng.integers(0, 64))
    return dict(array=((T - 1) * p + m + o + int(rng.integers(0, 5)),), rep=(T,), pattern=(m,), origin=(o,),
                paving=((p,),), fitting=((1,),)), T, m


@pytest.mark.parametrize("seed", range(8))
def test_random_large_copies_on_bulk_plans_vs_oracle(seed):
    """Randomised >= 1 MB gathers through the bulk-copy plans, shards with arbitrary starts,
    destinations with and without gaps: bit-exact against the C oracle."""
    from paper_1105_4424_b200 import _capi
    from oracle import c_oracle as co
    rng = np.random.default_rng(7000 + seed)
    plans = set()
    for _ in range(5):
        ts, T, m = _rand_big_copy(rng)
        gap = int(rng.choice([0, 0, 4]))
        td = dict(array=(T * (m + gap),), rep=(T,), pattern=(m,), origin=(0,), paving=((m + gap,),), fitting=((1,),))
        src = (np.arange(int(np.prod(ts["array"]))) % (1 << 22)).astype(np.float32) + 1
        want = np.zeros(T * (m + gap), np.float32)
        co.tile_copy(src, want, ts, td, 0, T)
        x = torch.from_numpy(src).cuda()
        y = torch.zeros(T * (m + gap), device="cuda")
        task = _capi.make_task("tile_copy", "float32",
                               [_tiler(ts).bind(ts["array"], (T,)), _tiler(td).bind(td["array"], (T,))])
        plans.add(_capi.plan_name(task, 0, T, [x.data_ptr(), y.data_ptr()]))
        for off, cnt in orc.partition_equally(T, int(rng.choice([1, 2, 3, 5]))):
            _capi.launch(task, off, cnt, [x.data_ptr(), y.data_ptr()], (), 0)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), want), (ts, gap)
    assert plans


@pytest.mark.parametrize("kh,kw", [(3, 5), (5, 5), (7, 5), (3, 7), (5, 7), (7, 7), (7, 3)])
@pytest.mark.parametrize("H,W,devices", [(64, 256, 1), (37, 512, 3), (100, 1024, 5)])
def test_stencil_wide_windows_vs_oracle(kh, kw, H, W, devices):
    """KH x KW toroidal box stencils beyond 3 columns (aligned quad form, k_stencil_slide_wide)
    and 7-row windows: bit-exact vs the oracle (random weights, origin centring the window)."""
    t = orc.stencil_tilers(H, W)
    t["x"] = dict(t["x"], pattern=(kh, kw), origin=(H - kh // 2, W - kw // 2))
    w = (np.random.default_rng(kh * 10 + kw).standard_normal(kh * kw) / 8).astype(np.float32)
    assert _plan([t["x"], t["y"]]) == "tile_filter.stencil_box"
    x = np.random.default_rng(H + W + kw).standard_normal(H * W).astype(np.float32)
    got, ref = _filter_case("stencil", t, w, x, devices)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    # a misaligned window centre has no wide form: the generic filter takes it, still exact
    if kw != 3:
        t2 = dict(t)
        t2["x"] = dict(t["x"], origin=(H - kh // 2, W - kw // 2 + 1))
        assert _plan([t2["x"], t2["y"]]) != "tile_filter.stencil_box"
        got, ref = _filter_case("stencil", t2, w, x, devices)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("case,plan", [("rows", "tile_sum.rows"), ("rows_ragged", "tile_sum.rows"),
                                       ("rows_pitch", "tile_sum.rows"),
                                       ("cols", "tile_sum.columns"), ("cols_small", "tile_sum.direct"),
                                       ("cols_pitch", "tile_sum.columns"), ("wrap_small", "tile_sum.generic"),
                                       ("wrap_long", "tile_sum.batched"), ("strided", "tile_sum.batched"),
                                       ("wrap_big", "tile_sum.generic_direct")])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("devices", [1, 3])
def test_tile_sum_plans_vs_oracle(case, plan, dtype, devices):
    """Pattern reductions (i ascending, one rounding per add) on every tile_sum plan: coalesced
    warp-transposed and TMA-swizzled row sums, TMA-streamed column sums (shard starts off 16 B), direct affine
    sums, the batched unit-weight filter kernel (wrapping or strided patterns), the offset-table generic form
    and the table-free form for large wrapping patterns -- bit-exact against the oracle."""
    if case in ("rows", "rows_ragged"):
        R, P = (300, 1000) if case == "rows" else (77, 45)
        tx = dict(array=(R, P), rep=(R,), pattern=(P,), origin=(0, 0), paving=((1,), (0,)), fitting=((0,), (1,)))
    elif case == "rows_pitch":
        # 777 of every 780 elements (TMA row boxes, partial last box), 1000 rows
        R, P = 1000, 777
        tx = dict(array=(R, 780), rep=(R,), pattern=(P,), origin=(0, 2), paving=((1,), (0,)), fitting=((0,), (1,)))
    elif case in ("cols", "cols_small"):
        R, P = (700, 300) if case == "cols" else (100, 300)
        tx = dict(array=(P, R), rep=(R,), pattern=(P,), origin=(0, 0), paving=((0,), (1,)), fitting=((1,), (0,)))
    elif case == "cols_pitch":
        # columns 5..1004 of a 2-D array with a wider row pitch, 1000 rows (partial last box)
        R, P = 1000, 1000
        tx = dict(array=(P, 1024), rep=(R,), pattern=(P,), origin=(0, 5), paving=((0,), (1,)), fitting=((1,), (0,)))
    elif case == "wrap_long":
        R, P = 4000, 9
        tx = dict(array=(5000,), rep=(R,), pattern=(P,), origin=(4995,), paving=((1,),), fitting=((1,),))
    elif case == "strided":
        R, P = 3000, 7
        tx = dict(array=(30000,), rep=(R,), pattern=(P,), origin=(11,), paving=((3,),), fitting=((2,),))
    elif case == "wrap_small":
        R, P = 500, 9
        tx = dict(array=(600,), rep=(R,), pattern=(P,), origin=(595,), paving=((1,),), fitting=((1,),))
    else:
        R, P = 40, 5000
        tx = dict(array=(6000,), rep=(R,), pattern=(P,), origin=(5990,), paving=((7,),), fitting=((1,),))
    ts = dict(array=(R,), rep=(R,), pattern=(1,), origin=(0,), paving=((1,),), fitting=((0,),))
    x = np.random.default_rng(R + P).standard_normal(int(np.prod(tx["array"]))).astype(dtype)
    got = _run_tile("tile_sum", {"x": tx, "s": ts}, {"x": _spec(tx, "in", dtype), "s": _spec(ts, "out", dtype)},
                    {"x": x}, devices).outputs["p_s"]
    ref = orc.run_tile_task("tile_sum", {"x": tx, "s": ts}, {"x": x}, {"s": (R, np.dtype(dtype))}, R, devices)["s"]
    u = f"u{np.dtype(dtype).itemsize}"
    assert np.array_equal(got.view(u), ref.view(u))
    from paper_1105_4424_b200 import _capi
    task = _capi.make_task("tile_sum", dtype, [_tiler(tx).bind(tx["array"], (R,)), _tiler(ts).bind(ts["array"], (R,))])
    assert _capi.plan_name(task, 0, R) == plan


@pytest.mark.parametrize("outer,S,px,sx,py,sy,ox", [
    (1, 5000, 8, 1, 1, 1, 0), (1, 4096, 16, 1, 1, 1, 4093), (3, 2000, 32, 1, 1, 1, 7), (2, 8192, 16, 4, 1, 1, 0),
    (4, 3000, 13, 8, 3, 3, 5), (2, 1000, 5, 2, 8, 8, 999), (1, 10000, 7, 3, 2, 2, 1), (2, 6000, 16, 8, 2, 2, 3),
    (2, 4096, 12, 4, 2, 2, 0), (1, 4100, 9, 4, 1, 1, 8), (3, 2048, 16, 4, 1, 1, 4090),
    (2, 2048, 16, 8, 2, 2, 0), (3, 1600, 12, 16, 1, 1, 0), (1, 3072, 16, 12, 4, 4, 0), (2, 2048, 9, 8, 3, 3, 0)])
@pytest.mark.parametrize("devices", [1, 3, 5])
@pytest.mark.parametrize("wide", [False, True])
def test_line_tiled_filters_vs_oracle(outer, S, px, sx, py, sy, ox, devices, wide, monkeypatch):
    """Generic horizontal line filters (1-D FIRs, decimating FIRs, wrapping windows, up to 8
    outputs per repetition) through the 32-bit batched kernel (default), the shared-memory
    window kernel (`AOL_FILTER_WIDE`) and the row-streaming ring for strided windows
    (`line_stream`): bit-exact vs the oracle, shard starts anywhere inside a line."""
    if wide:
        monkeypatch.setenv("AOL_FILTER_WIDE", "1")
    NL = (S - 1) // sx + 1 if sx > 1 else S
    NL = min(NL, S // sx) if sx > 1 else NL
    Sy = NL * sy if sy >= py else NL * py
    tx = dict(array=(outer, S), rep=(outer, NL), pattern=(px,), origin=(0, ox), paving=((1, 0), (0, sx)),
              fitting=((0,), (1,)))
    ty = dict(array=(outer, Sy), rep=(outer, NL), pattern=(py,), origin=(0, 0), paving=((1, 0), (0, sy)),
              fitting=((0,), (1,)))
    t = {"x": tx, "y": ty}
    w = (np.random.default_rng(px * 10 + py).standard_normal(px * py) / px).astype(np.float32)
    x = np.random.default_rng(S + px).standard_normal(outer * S).astype(np.float32)
    stream = (ox == 0 and sx % 4 == 0 and sx >= 8 and px <= min(16, sx + 8) and py <= 4 and sy == py
              and NL * sx == S and (px, py) != (13, 3))
    want = ("tile_filter.line_13x3" if (px, py) == (13, 3) else "tile_filter.line_stream" if stream else
            "tile_filter.line" if sx > 4 else "tile_filter.line_tiled" if wide else "tile_filter.batched")
    assert _plan([tx, ty]) == want
    got, ref = _filter_case("tile_filter", t, w, x, devices)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("kh,kw", [(2, 2), (3, 3), (4, 4), (2, 4), (1, 2), (4, 1), (3, 2)])
@pytest.mark.parametrize("devices", [1, 3])
def test_box_pool_filters_vs_oracle(kh, kw, devices):
    """Block pooling / decimating 2-D filters (a KH x KW box paved by its own size): the
    float4 quad kernel, bit-exact vs the oracle; an output width not divisible by 4 takes the
    generic filter, also exact."""
    for Ho, Wo, plan in ((40, 96, "tile_filter.box_pool"), (17, 30, None)):
        H, W = Ho * kh, Wo * kw
        tx = dict(array=(H, W), rep=(Ho, Wo), pattern=(kh, kw), origin=(0, 0), paving=((kh, 0), (0, kw)),
                  fitting=((1, 0), (0, 1)))
        ty = dict(array=(Ho, Wo), rep=(Ho, Wo), pattern=(1,), origin=(0, 0), paving=((1, 0), (0, 1)),
                  fitting=((0,), (0,)))
        t = {"x": tx, "y": ty}
        w = (np.random.default_rng(kh * 10 + kw).standard_normal(kh * kw) / (kh * kw)).astype(np.float32)
        x = np.random.default_rng(H + W).standard_normal(H * W).astype(np.float32)
        if plan:
            assert _plan([tx, ty]) == plan
        else:
            assert _plan([tx, ty]) != "tile_filter.box_pool"
        got, ref = _filter_case("tile_filter", t, w, x, devices)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (kh, kw, Ho, Wo)


@pytest.mark.parametrize("bh,bw", [(8, 8), (4, 16), (3, 5), (2, 2)])
@pytest.mark.parametrize("devices", [1, 3])
def test_tile_copy_block_tilers_vs_oracle(bh, bw, devices):
    """2-D block tilers (an image cut into bh x bw blocks, each block a pattern) to a dense
    stream and back, through the two-stride affine kernel (`tile_copy.affine2d`): bit-exact vs
    the oracle, with an origin offset and shards starting inside block rows."""
    from paper_1105_4424_b200 import _capi
    nbh, nbw = 24, 20
    H, W = nbh * bh + 3, nbw * bw + 4
    blk = dict(array=(H, W), rep=(nbh, nbw), pattern=(bh, bw), origin=(2, 4), paving=((bh, 0), (0, bw)),
               fitting=((1, 0), (0, 1)))
    P = bh * bw
    dense = dict(array=(nbh * nbw * P,), rep=(nbh, nbw), pattern=(bh, bw), origin=(0,),
                 paving=((nbw * P, P),), fitting=((bw, 1),))
    img = (np.arange(H * W) % (1 << 20)).astype(np.float32) + 1
    R = nbh * nbw
    for src, dst, n_out, data in ((blk, dense, R * P, img), (dense, blk, H * W, None)):
        if data is None:
            data = (np.arange(R * P) % (1 << 20)).astype(np.float32) + 7
        ports = {"src": _spec(src, "in", "float32"), "dst": _spec(dst, "out", "float32")}
        res = _run_tile("tile_copy", {"src": src, "dst": dst}, ports, {"src": data}, devices)
        ref = orc.run_tile_task("tile_copy", {"src": src, "dst": dst}, {"src": data},
                                {"dst": (n_out, np.dtype("float32"))}, R, devices)["dst"]
        assert np.array_equal(res.outputs["p_dst"], ref)
        task = _capi.make_task("tile_copy", "float32", [_tiler(src).bind(src["array"], (nbh, nbw)),
                                                        _tiler(dst).bind(dst["array"], (nbh, nbw))])
        assert _capi.plan_name(task, 0, R) == "tile_copy.affine2d"


@pytest.mark.parametrize("batch", [(3,), (2, 3)])
@pytest.mark.parametrize("devices", [1, 4])
def test_batched_matmul_tf32_within_bound(batch, devices):
    """MatMul with leading repetition axes (c[b..., m, n] = a[b..., m, :] . b[b..., :, n]): each
    batch slice runs as a tcgen05 launch over its share of the range; held to the TF32 bound."""
    from paper_1105_4424_b200 import _capi
    M, N, K = 200, 264, 96
    nb = int(np.prod(batch))
    q = len(batch)
    eye = lambda i, n: tuple(1 if j == i else 0 for j in range(n))  # noqa: E731
    rep = batch + (M, N)
    R = q + 2
    ta = dict(array=batch + (M, K), rep=rep, pattern=(K,), origin=(0,) * (q + 2),
              paving=tuple(eye(i, R) if i < q else (eye(q, R) if i == q else (0,) * R) for i in range(q + 2)),
              fitting=tuple((1,) if i == q + 1 else (0,) for i in range(q + 2)))
    tb = dict(array=batch + (K, N), rep=rep, pattern=(K,), origin=(0,) * (q + 2),
              paving=tuple(eye(i, R) if i < q else ((0,) * R if i == q else eye(q + 1, R)) for i in range(q + 2)),
              fitting=tuple((1,) if i == q else (0,) for i in range(q + 2)))
    tc = dict(array=batch + (M, N), rep=rep, pattern=(1,), origin=(0,) * (q + 2),
              paving=tuple(eye(i, R) for i in range(q + 2)), fitting=tuple((0,) for _ in range(q + 2)))
    rng = np.random.default_rng(nb)
    a = rng.standard_normal(nb * M * K).astype(np.float32)
    b = rng.standard_normal(nb * K * N).astype(np.float32)
    ports = {"a": _spec(ta, "in", "float32"), "b": _spec(tb, "in", "float32"), "c": _spec(tc, "out", "float32")}
    c = _run_tile("matmul", {"a": ta, "b": tb, "c": tc}, ports, {"a": a, "b": b}, devices).outputs["p_c"]
    A = a.reshape(nb, M, K).astype(np.float64)
    B = b.reshape(nb, K, N).astype(np.float64)
    C = c.reshape(nb, M, N)
    for i in range(nb):
        c64 = A[i] @ B[i]
        assert np.all(np.abs(C[i] - c64) <= _gemm_bound(A[i], B[i], K)), i
    bt = [_tiler(d).bind(d["array"], rep) for d in (ta, tb, tc)]
    task = _capi.make_task("matmul", "float32", bt)
    t0 = torch.zeros(4, device="cuda")
    assert _capi.plan_name(task, 0, nb * M * N, [t0.data_ptr()] * 3) == "matmul.tcgen05_tf32_batched"
    # exact mode: every slice through the tiled exact kernel, bit-exact against the oracle
    ex = _run_tile("matmul", {"a": ta, "b": tb, "c": tc}, ports, {"a": a, "b": b}, devices, precision="exact")
    ref = orc.run_tile_task("matmul", {"a": ta, "b": tb, "c": tc}, {"a": a, "b": b},
                            {"c": (nb * M * N, np.float32)}, nb * M * N, devices)["c"]
    assert np.array_equal(ex.outputs["p_c"], ref)
    task_x = _capi.make_task("matmul", "float32", bt, precision="exact")
    assert _capi.plan_name(task_x, 0, nb * M * N, [t0.data_ptr()] * 3) == "matmul.exact_tiled_batched"


@pytest.mark.parametrize("shape,origin", [((100000,), (12345,)), ((300, 257), (299, 5)), ((40, 36, 52), (3, 35, 51)),
                                          ((64, 80), (0, 79))])
@pytest.mark.parametrize("devices", [1, 3])
def test_tile_copy_toroidal_shift_vs_oracle(shape, origin, devices):
    """Toroidal shifts / rotations (identity paving, pattern [1], any origin): whole-range launches
    split at the wrap seams into affine boxes (`tile_copy.seam_boxes`), shard ranges through the
    generic kernel -- both bit-exact vs the oracle."""
    from paper_1105_4424_b200 import _capi
    a = len(shape)
    eye = tuple(tuple(1 if i == j else 0 for j in range(a)) for i in range(a))
    src = dict(array=shape, rep=shape, pattern=(1,), origin=origin, paving=eye, fitting=tuple((0,) for _ in range(a)))
    dst = dict(src, origin=(0,) * a)
    n = int(np.prod(shape))
    x = (np.arange(n) % (1 << 22)).astype(np.float32) + 1
    ports = {"src": _spec(src, "in", "float32"), "dst": _spec(dst, "out", "float32")}
    res = _run_tile("tile_copy", {"src": src, "dst": dst}, ports, {"src": x}, devices)
    ref = orc.run_tile_task("tile_copy", {"src": src, "dst": dst}, {"src": x}, {"dst": (n, np.dtype("float32"))},
                            n, devices)["dst"]
    assert np.array_equal(res.outputs["p_dst"], ref)
    task = _capi.make_task("tile_copy", "float32", [_tiler(src).bind(shape, shape), _tiler(dst).bind(shape, shape)])
    assert _capi.plan_name(task, 0, n) == "tile_copy.seam_boxes"


def _generic_filter_cases():
    H, W = 70, 300
    return [
        # 3x3 stride-2 window on a torus (origin -1, -1): wrapping rows/columns at both edges
        ("s2_torus", dict(array=(H, W), rep=(H // 2, W // 2), pattern=(3, 3), origin=(H - 1, W - 1),
                          paving=((2, 0), (0, 2)), fitting=((1, 0), (0, 1))),
         dict(array=(H // 2, W // 2), rep=(H // 2, W // 2), pattern=(1,), origin=(0, 0),
              paving=((1, 0), (0, 1)), fitting=((0,), (0,)))),
        # 4x4 window -> 2x2 outputs (16 taps, 4 outputs per repetition)
        ("win4_out2", dict(array=(H - 2, W), rep=((H - 2) // 4, W // 4), pattern=(4, 4), origin=(0, 0),
                           paving=((4, 0), (0, 4)), fitting=((1, 0), (0, 1))),
         dict(array=((H - 2) // 2, W // 2), rep=((H - 2) // 4, W // 4), pattern=(2, 2), origin=(0, 0),
              paving=((2, 0), (0, 2)), fitting=((1, 0), (0, 1)))),
        # 3-D repetition space, column (strided) pattern, 6 outputs written along a wrapping row
        ("rank3_cols", dict(array=(4, 40, 50), rep=(4, 10, 50), pattern=(5,), origin=(0, 1, 0),
                            paving=((1, 0, 0), (0, 4, 0), (0, 0, 1)), fitting=((0,), (1,), (0,))),
         dict(array=(4, 10, 300), rep=(4, 10, 50), pattern=(6,), origin=(0, 0, 7),
              paving=((1, 0, 0), (0, 1, 0), (0, 0, 6)), fitting=((0,), (0,), (1,)))),
        # diagonal (non-separable) 2-D pattern fitting, negative paving along columns
        ("diag_neg", dict(array=(64, 96), rep=(60, 90), pattern=(3, 2), origin=(2, 5),
                          paving=((1, 0), (0, -1)), fitting=((1, 1), (1, -1))),
         dict(array=(60, 90), rep=(60, 90), pattern=(1,), origin=(0, 0),
              paving=((1, 0), (0, 1)), fitting=((0,), (0,)))),
    ]


@pytest.mark.parametrize("case", [c[0] for c in _generic_filter_cases()])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("devices", [1, 3])
@pytest.mark.parametrize("wide", [False, True])
def test_generic_filter_batched32_vs_oracle(case, dtype, devices, wide, monkeypatch):
    """Filters no specialised kernel covers (strided windows on a torus, several outputs per
    repetition, rank-3 repetition spaces, diagonal fittings, negative pavings): the 32-bit batched
    kernel (default) and the int64 kernel (AOL_FILTER_WIDE) bit-exact vs the oracle."""
    if wide:
        monkeypatch.setenv("AOL_FILTER_WIDE", "1")
    _, tx, ty = next(c for c in _generic_filter_cases() if c[0] == case)
    assert _plan([tx, ty], dtype) == ("tile_filter.generic" if wide else "tile_filter.batched")
    np_dt = np.dtype(dtype)
    px = int(np.prod(tx["pattern"]))
    py = int(np.prod(ty["pattern"]))
    nx, ny = int(np.prod(tx["array"])), int(np.prod(ty["array"]))
    w = (np.random.default_rng(px + py).standard_normal(px * py) / px).astype(np_dt)
    x = np.random.default_rng(nx).standard_normal(nx).astype(np_dt)
    t = {"x": tx, "y": ty}
    R = int(np.prod(tx["rep"]))
    ports = {"x": _spec(tx, "in", dtype), "w": f"in {dtype} [{w.size}]", "y": _spec(ty, "out", dtype)}
    res = _run_tile("tile_filter", t, ports, {"x": x, "w": w}, devices)
    ref = orc.run_tile_task("tile_filter", t, {"x": x, "w": w}, {"y": (ny, np_dt)}, R, devices)["y"]
    got = res.outputs["p_y"]
    assert got.dtype == np_dt and np.array_equal(got.view(np.uint8), ref.view(np.uint8)), (case, dtype)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("so,do", [((3, 5), (0, 2)), ((0, 0), (0, 0)), ((7, 1), (1, 3)), ((2, 4), (0, 1)),
                                   ((4, 4), (4, 4)), ((1, 2), (3, 0))])
@pytest.mark.parametrize("devices", [1, 3])
def test_tile_copy_tma_plane_vs_oracle(dtype, so, do, devices):
    """2-D crops / embeddings (rows contiguous on both sides at 16 B pitches, any element offset):
    whole-row ranges go through TMA plane boxes when both row starts are 16 B-aligned
    (`tile_copy.tma_plane`, last column/row boxes clipped), through the funnel-shift float4 kernel
    otherwise (`tile_copy.rows_shift`, fp32); shard ranges that split rows through
    `tile_copy.affine2d` -- all bit-exact vs the oracle."""
    from paper_1105_4424_b200 import _capi
    np_dt = np.dtype(dtype)
    src = dict(array=(1030, 1100), rep=(1000, 1052), pattern=(1,), origin=so, paving=((1, 0), (0, 1)),
               fitting=((0,), (0,)))
    dst = dict(array=(1004, 1056), rep=(1000, 1052), pattern=(1,), origin=do, paving=((1, 0), (0, 1)),
               fitting=((0,), (0,)))
    ns, nd = 1030 * 1100, 1004 * 1056
    x = (np.arange(ns) % 65521).astype(np_dt) + 1
    ports = {"src": _spec(src, "in", dtype), "dst": _spec(dst, "out", dtype)}
    res = _run_tile("tile_copy", {"src": src, "dst": dst}, ports, {"src": x}, devices)
    R = 1000 * 1052
    ref = orc.run_tile_task("tile_copy", {"src": src, "dst": dst}, {"src": x}, {"dst": (nd, np_dt)}, R, devices)["dst"]
    got = res.outputs["p_dst"]
    written = np.zeros(nd, bool)
    written.reshape(1004, 1056)[do[0]:do[0] + 1000, do[1]:do[1] + 1052] = True
    assert np.array_equal(got[written], ref[written])
    task = _capi.make_task("tile_copy", dtype, [_tiler(src).bind(src["array"], src["rep"]),
                                                _tiler(dst).bind(dst["array"], dst["rep"])])
    aligned = ((so[0] * 1100 + so[1]) * np_dt.itemsize) % 16 == 0 and ((do[0] * 1056 + do[1]) * np_dt.itemsize) % 16 == 0
    want = "tile_copy.tma_plane" if aligned else "tile_copy.rows_shift" if dtype == "float32" else "tile_copy.affine2d"
    assert _capi.plan_name(task, 0, R) == want


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_random_long_rows_batched_filters_vs_oracle(seed, dtype):
    """Random filter tilers whose last repetition axis is long (200-700), so the 32-bit batched
    kernel's lane runs (32 x R repetitions of one row) and its wrapping / row-leaving fallbacks
    all occur: negative pavings and fittings, toroidal origins, 1-4 outputs written through a
    shifted (wrapping) dense output tiler, several shard counts -- bit-exact vs the oracle."""
    rng = np.random.default_rng(5000 + seed)
    np_dt = np.dtype(dtype)
    for _ in range(3):
        q = int(rng.integers(1, 3))
        rep = tuple(int(x) for x in rng.integers(2, 5, q - 1)) + (int(rng.integers(200, 700)),)
        p = int(rng.integers(1, 3))
        pat = tuple(int(x) for x in rng.integers(1, 5, p))
        a = int(rng.integers(1, 3))
        arr = tuple(int(x) for x in rng.integers(50, 900, a))
        tx = dict(array=arr, rep=rep, pattern=pat, origin=tuple(int(x) for x in rng.integers(-900, 900, a)),
                  paving=tuple(tuple(int(x) for x in rng.integers(-4, 5, q)) for _ in range(a)),
                  fitting=tuple(tuple(int(x) for x in rng.integers(-3, 4, p)) for _ in range(a)))
        R, P = int(np.prod(rep)), int(np.prod(pat))
        py = int(rng.integers(1, 5))
        ty = _dense_out(rep, (py,))
        ty = dict(ty, origin=(int(rng.integers(0, R * py)),))
        nx = int(np.prod(arr))
        x = rng.standard_normal(nx).astype(np_dt)
        w = rng.standard_normal(py * P).astype(np_dt)
        d = int(rng.integers(1, 4))
        ports = {"x": _spec(tx, "in", dtype), "w": f"in {dtype} [{w.size}]", "y": _spec(ty, "out", dtype)}
        got = _run_tile("tile_filter", {"x": tx, "y": ty}, ports, {"x": x, "w": w}, d).outputs["p_y"]
        ref = orc.run_tile_task("tile_filter", {"x": tx, "y": ty}, {"x": x, "w": w}, {"y": (R * py, np_dt)}, R, d)
        assert np.array_equal(got.view(np.uint8), ref["y"].view(np.uint8)), (tx, ty)


def _special_values(n, seed):
    """float32 data in three bands: subnormals and signed zeros, overflow-prone magnitudes
    (1e38-3.3e38), ordinary values -- all non-negative, so every product and sum has one IEEE
    answer (no inf - inf, no 0 * inf) and the comparison can be bit for bit."""
    rng = np.random.default_rng(seed)
    tiny = np.array([0.0, -0.0, 1e-45, 3e-42, 1e-40, 5e-39], dtype=np.float32)
    huge = np.array([1e38, 2e38, 3.3e38], dtype=np.float32)
    v = np.abs(rng.standard_normal(n)).astype(np.float32)
    third = n // 3
    v[:third] = tiny[rng.integers(0, tiny.size, third)]
    v[third:2 * third] = huge[rng.integers(0, huge.size, third)]
    v[:third] = np.where(v[:third] == 0, v[:third], np.abs(v[:third]))
    return v


@pytest.mark.parametrize("devices", [1, 3])
def test_special_values_bit_exact(devices):
    """Stencil, line filter, tile sum and exact-order matmul on subnormals, signed zeros and
    overflowing magnitudes: no flush-to-zero (the library is built without fast math), the same
    IEEE rounding per product and per add as the oracle, +inf where the oracle overflows."""
    H, W = 48, 64
    t = orc.stencil_tilers(H, W)
    x = _special_values(H * W, 1)
    w = (16 * np.abs(orc.stencil_weights())).astype(np.float32)     # 1 2 1 / 2 4 2 / 1 2 1: overflows
    res = _run_tile("stencil", t, {"x": _spec(t["x"], "in", "float32"), "w": "in float32 [9]",
                                   "y": _spec(t["y"], "out", "float32")}, {"x": x, "w": w}, devices)
    with np.errstate(over="ignore"):
        want = orc.run_tile_task("stencil", t, {"x": x, "w": w}, {"y": (H * W, np.float32)}, H * W, devices)["y"]
    got = res.outputs["p_y"]
    assert np.isinf(want).any() and (np.abs(want[want != 0]) < 1.2e-38).any()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    M, N, K = 40, 36, 24
    g = orc.gemm_tilers(M, N, K)
    a, b = _special_values(M * K, 2), _special_values(K * N, 3)
    res = _run_tile("matmul", g, {"a": _spec(g["a"], "in", "float32"), "b": _spec(g["b"], "in", "float32"),
                                  "c": _spec(g["c"], "out", "float32")}, {"a": a, "b": b}, devices, precision="exact")
    with np.errstate(over="ignore"):
        want = orc.run_tile_task("matmul", g, {"a": a, "b": b}, {"c": (M * N, np.float32)}, M * N, devices)["c"]
    assert np.array_equal(res.outputs["p_c"].view(np.uint32), want.view(np.uint32))
