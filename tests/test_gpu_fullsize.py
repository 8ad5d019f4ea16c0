"""Parity at BASELINE.json's full sizes (C2-C5) through size-independent properties.

The CPU oracle cannot redo a whole 8192^3 matmul or a 256-frame downscaler
in seconds, so each config is run at its full size on the B200 and checked by
properties that do not depend on the size:

- C4 stencil 16384^2: the whole torus, bit-exact against the C oracle
  (oracle/aol_oracle.c, every row; weights are powers of two so every
  product is exact and the tap-order sum pins the bits).
- C3 downscaler 256x2160x3840: frames are independent repetitions of both
  tilers (the H wrap stays inside a row, the V wrap inside a frame), so a
  spread sample of frames (first, last, and interior ones) is compared
  bit-exact with the oracle's two-filter chain on those frames.
- C2 matmul 8192^3: sampled rows against the fp64 product under the stated
  TF32 element-wise bound, plus the row-sum checksum C.1 = A.(B.1) (linearity)
  under the normwise bound.
- C5 tile_copy at T = 1e9: index-valued inputs make the output
  self-verifying: dst[r*m + i] must equal src[o + p*r + f*i] exactly, checked
  on the device chunk by chunk.
"""

import numpy as np
import pytest

from oracle import aol_oracle as orc
from oracle import c_oracle as co

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_1105_4424_b200 import _capi
    _capi.load()
    yield
    torch.cuda.empty_cache()


def _tiler(d):
    from paper_1105_4424_b200 import Tiler
    return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"])


def _spec(d, direction):
    return f"{direction} float32 [{','.join(str(x) for x in d['array'])}]"


def _executor(model, bindings, devices, **kw):
    from paper_1105_4424_b200.executor import Executor
    from paper_1105_4424_b200.partition import build_schedule
    ex = Executor(model, build_schedule(model, devices), bindings, devices, **kw)
    ex.run()
    torch.cuda.synchronize()
    return ex


def test_c4_stencil_16384_full_torus_bitexact():
    from paper_1105_4424_b200 import builders
    n = 16384
    t = orc.stencil_tilers(n, n)
    w = orc.stencil_weights()
    model = builders.tile_task_model(
        "stencil", {"x": _spec(t["x"], "in"), "w": "in float32 [9]", "y": _spec(t["y"], "out")},
        {k: _tiler(v) for k, v in t.items()}, (n, n))
    x = np.random.default_rng(5).standard_normal(n * n, dtype=np.float32)
    for devices in (1, 8):       # 8 contiguous shards of the repetition space on one device
        ex = _executor(model, {"p_x": torch.from_numpy(x).cuda(), "p_w": torch.from_numpy(w).cuda()}, devices)
        got = ex.outputs(on_device=True)["p_y"].cpu().numpy()
        del ex
        want = np.zeros_like(x)
        co.stencil_rows(x, w, want, n, n, 0, n)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), devices


def test_c3_downscaler_256_frames_sampled_bitexact():
    from paper_1105_4424_b200 import builders
    frames, H, W = 256, 2160, 3840
    th = orc.hfilter_tilers(frames, H, W)
    Wo = th["y"]["array"][2]
    tv = orc.vfilter_tilers(frames, H, Wo)
    Ho = tv["y"]["array"][1]
    wh, wv = orc.hfilter_weights(), orc.vfilter_weights()
    model = builders.chain_model(
        [("h", "hfilter", {"x": _spec(th["x"], "in"), "w": f"in float32 [{wh.size}]", "y": _spec(th["y"], "out")},
          {k: _tiler(v) for k, v in th.items()}, th["x"]["rep"]),
         ("v", "vfilter", {"x": _spec(tv["x"], "in"), "w": f"in float32 [{wv.size}]", "y": _spec(tv["y"], "out")},
          {k: _tiler(v) for k, v in tv.items()}, tv["x"]["rep"])],
        {"x": _spec(th["x"], "in"), "wh": f"in float32 [{wh.size}]", "wv": f"in float32 [{wv.size}]"},
        {"y": _spec(tv["y"], "out")},
        [("x", "h.x"), ("wh", "h.w"), ("h.y", "v.x"), ("wv", "v.w"), ("v.y", "y")])
    fpx, fpy = H * W, Ho * Wo
    gen = torch.Generator(device="cuda").manual_seed(4)
    x = torch.rand(frames * fpx, device="cuda", generator=gen)
    ex = _executor(model, {"x": x, "wh": torch.from_numpy(wh).cuda(), "wv": torch.from_numpy(wv).cuda()}, 1)
    assert ex.fused_launches > 0, "the default path for C3 is the fused H->V kernel"
    y = ex.outputs(on_device=True)["y"]
    assert y.numel() == frames * fpy
    # one-frame oracle chain
    th1, tv1 = orc.hfilter_tilers(1, H, W), orc.vfilter_tilers(1, H, Wo)
    rh, rv = int(np.prod(th1["x"]["rep"])), int(np.prod(tv1["x"]["rep"]))
    for f in (0, 1, 97, 128, 200, 255):
        xf = x[f * fpx:(f + 1) * fpx].cpu().numpy()
        mid = np.zeros(H * Wo, np.float32)
        want = np.zeros(fpy, np.float32)
        co.tile_filter(xf, wh, mid, th1["x"], th1["y"], 0, rh)
        co.tile_filter(mid, wv, want, tv1["x"], tv1["y"], 0, rv)
        got = y[f * fpy:(f + 1) * fpy].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f


def test_c2_matmul_8192_sampled_rows_and_checksum():
    from paper_1105_4424_b200 import builders
    M = N = K = 8192
    g = orc.gemm_tilers(M, N, K)
    model = builders.tile_task_model(
        "matmul", {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]", "c": f"out float32 [{M},{N}]"},
        {k: _tiler(v) for k, v in g.items()}, (M, N))
    a = torch.randn(M * K, device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    b = torch.randn(K * N, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    for devices in (1, 8):
        ex = _executor(model, {"p_a": a, "p_b": b}, devices)
        c = ex.outputs(on_device=True)["p_c"].view(M, N)
        A, B = a.view(M, K), b.view(K, N)
        rows = torch.tensor([0, 1, 127, 128, 1023, 1024, 4095, 4096, 5000, 8190, 8191], device="cuda")
        a64, b64 = A[rows].double(), B.double()
        c64 = a64 @ b64
        bound = (2.0 ** -9 + K * 2.0 ** -23) * (a64.abs() @ b64.abs())
        err = (c[rows].double() - c64).abs()
        assert bool((err <= bound).all()), float((err / bound).max())
        # linearity checksum over the whole product: C.1 == A.(B.1)
        ones = torch.ones(N, 1, device="cuda", dtype=torch.float64)
        lhs = c.double() @ ones
        rhs = A.double() @ (B.double() @ ones)
        rel = float(torch.linalg.norm(lhs - rhs) / torch.linalg.norm(rhs))
        assert rel < 2e-3, rel
        del ex, c, lhs, rhs, a64, b64, c64, bound, err


def _index_values(off):
    return (off % (1 << 24)).to(torch.float32)


@pytest.mark.parametrize("m,kind,T", [(1, "dense", 10 ** 9), (1, "gaps", 10 ** 9), (2, "overlap", 10 ** 9),
                                      (2, "strided", 10 ** 9), (8, "rowstride", 10 ** 8)])
def test_c5_tile_copy_full_T_self_verifying(m, kind, T):
    from paper_1105_4424_b200 import Tiler, _capi
    if kind == "rowstride":
        span = m * T
        src = Tiler((0, 0), ((0,), (1,)), ((1,), (0,)), (m,)).bind((m, T), (T,))
    else:
        p = {"dense": m, "overlap": max(1, m // 2), "gaps": 2 * m, "strided": 2 * m}[kind]
        f = 2 if kind == "strided" else 1
        span = (T - 1) * p + (m - 1) * f + 1
        src = Tiler((0,), ((p,),), ((f,),), (m,)).bind((span,), (T,))
    dst = Tiler((0,), ((m,),), ((1,),), (m,)).bind((T * m,), (T,))
    x = torch.empty(span, device="cuda")
    chunk = 1 << 28
    for lo in range(0, span, chunk):
        hi = min(span, lo + chunk)
        x[lo:hi] = _index_values(torch.arange(lo, hi, device="cuda"))
    y = torch.full((T * m,), -1.0, device="cuda")
    task = _capi.make_task("tile_copy", "float32", [src, dst])
    for devices in (1, 3):
        y.fill_(-1.0)
        for (off, cnt) in orc.partition_equally(T, devices):
            _capi.launch(task, off, cnt, [x.data_ptr(), y.data_ptr()], (), torch.cuda.current_stream().cuda_stream)
        rc = chunk // m
        for r0 in range(0, T, rc):
            r1 = min(T, r0 + rc)
            r = torch.arange(r0, r1, device="cuda").view(-1, 1)
            i = torch.arange(m, device="cuda").view(1, -1)
            off = (i * T + r) if kind == "rowstride" else (p * r + f * i)
            assert torch.equal(y[r0 * m:r1 * m].view(-1, m), _index_values(off)), (devices, r0)
    del x, y


def test_zero_count_launch_is_a_noop():
    """count == 0 returns success and touches nothing (partition ranges can be empty only past T)."""
    from paper_1105_4424_b200 import Tiler, _capi
    src = Tiler((0,), ((2,),), ((1,),), (2,)).bind((64,), (32,))
    dst = Tiler((0,), ((2,),), ((1,),), (2,)).bind((64,), (32,))
    x = torch.arange(64, dtype=torch.float32, device="cuda")
    y = torch.full((64,), 7.0, device="cuda")
    task = _capi.make_task("tile_copy", "float32", [src, dst])
    before = _capi.launch_counter()
    for first in (0, 5, 32):
        _capi.launch(task, first, 0, [x.data_ptr(), y.data_ptr()], (), 0)
    torch.cuda.synchronize()
    assert bool((y == 7.0).all())
    assert _capi.launch_counter() == before
    with pytest.raises(Exception):
        _capi.launch(task, 31, 2, [x.data_ptr(), y.data_ptr()], (), 0)   # past the repetition space


def test_c2_matmul_8192_3xtf32_fp32_faithful():
    """C2 in precision='3xtf32' at full size: normwise error on sampled rows <= 1e-6 and below
    cuBLAS SIMT fp32 (allow_tf32=False) on the same rows."""
    from paper_1105_4424_b200 import builders
    M = N = K = 8192
    model = builders.matmul_model(M, N, K)
    a = torch.randn(M * K, device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    b = torch.randn(K * N, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    from paper_1105_4424_b200.executor import Executor
    from paper_1105_4424_b200.partition import build_schedule
    ex = Executor(model, build_schedule(model, 3), {"p_a": a, "p_b": b}, 3, precision="3xtf32")
    ex.run()
    c = ex.outputs(on_device=True)["p_c"].view(M, N)
    A, B = a.view(M, K), b.view(K, N)
    rows = torch.tensor([0, 1, 255, 256, 2730, 2731, 5461, 5462, 8191], device="cuda")
    c64 = A[rows].double() @ B.double()
    ours = float(torch.linalg.norm(c[rows].double() - c64) / torch.linalg.norm(c64))
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        simt = float(torch.linalg.norm((A @ B)[rows].double() - c64) / torch.linalg.norm(c64))
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    assert ours <= 1e-6 and ours <= simt, (ours, simt)


@pytest.mark.parametrize("precision", ["default", "3xtf32", "exact"])
def test_matmul_output_beyond_2_31_elements(precision):
    """C with 65536 x 36864 = 2.4e9 elements (9.7 GB): every tile's store offset passes 2^31, on
    three unaligned shards; sampled rows at both ends against fp64 (TF32 bound / 3xTF32 1e-6)."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    M, N, K, D = 65536, 36864, 32, 3
    g = torch.Generator(device="cuda").manual_seed(11)
    a = torch.randn(M * K, device="cuda", generator=g)
    b = torch.randn(K * N, device="cuda", generator=g)
    model = builders.matmul_model(M, N, K)
    c = execute_schedule(model, build_schedule(model, D), {"p_a": a, "p_b": b}, D, precision=precision,
                         device_outputs=True).outputs["p_c"].view(M, N)
    rows = torch.tensor([0, 1, 21845, 21846, 43690, 43691, M - 2, M - 1], device="cuda")
    A, B = a.view(M, K), b.view(K, N)
    ref = A[rows].double() @ B.double()
    got = c[rows].double()
    if precision == "default":
        bound = (2.0 ** -9 + K * 2.0 ** -23) * (A[rows].double().abs() @ B.double().abs())
        assert bool(((got - ref).abs() <= bound).all())
    elif precision == "exact":                       # k ascending, a rounding per product and per add
        an, bn = A[rows].cpu().numpy(), B.cpu().numpy()
        want = np.zeros((len(rows), N), dtype=np.float32)
        for k in range(K):
            want = want + an[:, k:k + 1] * bn[k:k + 1, :]
        assert np.array_equal(c[rows].cpu().numpy(), want)
    else:
        assert float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref)) <= 1e-6
    del c, a, b
    torch.cuda.empty_cache()


def test_stencil_beyond_2_31_elements_sampled_rows():
    """A 65536 x 36864 torus (2.4e9 elements, 9.7 GB each way) on three shards: offsets past 2^31
    in the stencil kernel; the wrap rows, the shard seams and the middle against the oracle order
    (`_stencil_rows_np`, equal to oracle/aol_oracle.c stencil_rows on a small torus)."""
    from paper_1105_4424_b200 import builders
    H, W, D = 65536, 36864, 3
    t = orc.stencil_tilers(H, W)
    w = orc.stencil_weights()
    model = builders.tile_task_model(
        "stencil", {"x": _spec(t["x"], "in"), "w": "in float32 [9]", "y": _spec(t["y"], "out")},
        {k: _tiler(v) for k, v in t.items()}, (H, W))
    xd = torch.randn(H * W, device="cuda", generator=torch.Generator(device="cuda").manual_seed(13))
    ex = _executor(model, {"p_x": xd, "p_w": torch.from_numpy(w).cuda()}, D)
    got = ex.outputs(on_device=True)["p_y"].view(H, W)
    del ex
    x = xd.cpu().numpy()
    for lo in (0, H // 3 - 1, H // 2, 2 * H // 3, H - 2):
        want = _stencil_rows_np(x, w, H, W, lo, lo + 2)
        assert np.array_equal(got[lo:lo + 2].cpu().numpy().view(np.uint32), want.view(np.uint32)), lo
    del got, xd
    torch.cuda.empty_cache()


def _stencil_rows_np(x, w, H, W, lo, hi):
    """Oracle rows lo..hi-1 of the toroidal 3x3 stencil, taps row-major, each product and each
    add rounded in float32 (the order orc.stencil_tilers' pattern walks)."""
    x2 = x.reshape(H, W)
    acc = np.zeros((hi - lo, W), dtype=np.float32)
    for i in range(3):
        rows = x2[[(r + i - 1) % H for r in range(lo, hi)]]
        for j in range(3):
            acc = acc + np.float32(w[i * 3 + j]) * np.roll(rows, 1 - j, axis=1)
    return acc
