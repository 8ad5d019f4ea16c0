"""Round-2 GPU checks: streamed-path gating, fused-pair fallback, caller streams.

Each case runs through ``execute_schedule`` (refexec.py:427) on the B200 and is
compared with the plain (unstreamed) run and with the CPU oracle.
"""

import numpy as np
import pytest

from oracle import aol_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200"


def _tiler(d):
    from paper_1105_4424_b200 import Tiler
    return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"])


def _spmv_model(n, nnz, dt="float64"):
    from paper_1105_4424_b200 import builders
    return builders.single_task_model(
        "spmv_csr",
        [f"rowptr in int32 [{n + 1}]", f"colidx in int32 [{nnz}]", f"values in {dt} [{nnz}]",
         f"x in {dt} [{n}]", f"y out {dt} [{n}]"],
        [f"rp in int32 [{n + 1}]", f"ci in int32 [{nnz}]", f"va in {dt} [{nnz}]",
         f"vx in {dt} [{n}]", f"o out {dt} [{n}]"],
        ["rp -> t.rowptr", "ci -> t.colidx", "va -> t.values", "vx -> t.x", "t.y -> o"],
        ["allocate data rp onto dev.gmem", "allocate data ci onto dev.gmem", "allocate data va onto dev.gmem",
         "allocate data vx onto dev.gmem", "allocate data t.y onto dev.gmem", "allocate task t onto dev.cu"], n)


def _random_csr(rng, n, per_row=7):
    cols = [np.sort(rng.choice(n, size=int(rng.integers(0, per_row + 1)), replace=False)) for _ in range(n)]
    rowptr = np.zeros(n + 1, np.int32)
    rowptr[1:] = np.cumsum([c.size for c in cols])
    colidx = np.concatenate(cols).astype(np.int32)
    return rowptr, colidx, rng.standard_normal(colidx.size)


@pytest.mark.parametrize("chunks", [2, 7])
@pytest.mark.parametrize("devices", [1, 3])
def test_streamed_spmv_equals_plain_and_oracle(chunks, devices):
    """pipeline>1 on a spmv_csr schedule: rowptr/colidx/values are gathered whole, so the
    executor must not stream it chunk-wise -- results equal the plain run."""
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    rng = np.random.default_rng(11)
    n = 1500
    rp, ci, va = _random_csr(rng, n)
    x = rng.standard_normal(n)
    model = _spmv_model(n, ci.size)
    sched = build_schedule(model, devices)
    bind = {"rp": rp, "ci": ci, "va": va, "vx": x}
    plain = execute_schedule(model, sched, bind, devices).outputs["o"]
    streamed = execute_schedule(model, sched, bind, devices, pipeline=chunks).outputs["o"]
    ref = np.zeros(n)
    orc.spmv_rows(rp, ci, va, x, ref, 0, n)
    assert np.array_equal(plain, ref)
    assert np.array_equal(streamed, ref)


@pytest.mark.parametrize("chunks", [2, 5])
@pytest.mark.parametrize("devices", [1, 4])
def test_streamed_dot_equals_plain(chunks, devices):
    """pipeline>1 on dot_partial: one partial per launch summed in device order, not the last chunk's."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    n = 10007
    model = builders.single_task_model(
        "dot_partial", [f"a in float64 [{n}]", f"b in float64 [{n}]", "s out float64 [1]"],
        [f"i1 in float64 [{n}]", f"i2 in float64 [{n}]", "o out float64 [1]"],
        ["i1 -> t.a", "i2 -> t.b", "t.s -> o"],
        ["allocate data i1 onto dev.gmem", "allocate data i2 onto dev.gmem", "allocate data t.s onto host.ram",
         "allocate task t onto dev.cu"], n)
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    sched = build_schedule(model, devices)
    plain = execute_schedule(model, sched, {"i1": a, "i2": b}, devices).outputs["o"]
    streamed = execute_schedule(model, sched, {"i1": a, "i2": b}, devices, pipeline=chunks).outputs["o"]
    assert np.array_equal(plain, streamed)
    assert abs(float(plain[0]) - float(a @ b)) <= 1e-12 * max(1.0, abs(float(a @ b)))


@pytest.mark.parametrize("chunks", [2, 6])
def test_streamed_unfusable_filter_pair_falls_back(chunks):
    """Two chained 1-D FIRs (not the 13x3 -> 14x4 geometry the fused kernel exists for) with
    pipeline>1: the streamed pair path must fall back to unfused launches."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    n = 4096
    taps1, taps2 = 5, 3
    t1 = {"x": dict(array=(n,), rep=(n,), pattern=(taps1,), origin=(0,), paving=((1,),), fitting=((1,),)),
          "y": dict(array=(n,), rep=(n,), pattern=(1,), origin=(0,), paving=((1,),), fitting=((0,),))}
    t2 = {"x": dict(array=(n,), rep=(n,), pattern=(taps2,), origin=(n - 1,), paving=((1,),), fitting=((1,),)),
          "y": dict(array=(n,), rep=(n,), pattern=(1,), origin=(0,), paving=((1,),), fitting=((0,),))}
    w1 = np.array([1, 2, 4, 2, 1], np.float32) / 8
    w2 = np.array([1, 2, 1], np.float32) / 4
    model = builders.chain_model(
        [("f", "tile_filter", {"x": f"in float32 [{n}]", "w": "in float32 [5]", "y": f"out float32 [{n}]"},
          {k: _tiler(v) for k, v in t1.items()}, (n,)),
         ("g", "tile_filter", {"x": f"in float32 [{n}]", "w": "in float32 [3]", "y": f"out float32 [{n}]"},
          {k: _tiler(v) for k, v in t2.items()}, (n,))],
        {"x": f"in float32 [{n}]", "w1": "in float32 [5]", "w2": "in float32 [3]"}, {"y": f"out float32 [{n}]"},
        [("x", "f.x"), ("w1", "f.w"), ("f.y", "g.x"), ("w2", "g.w"), ("g.y", "y")])
    x = np.random.default_rng(5).random(n).astype(np.float32)
    sched = build_schedule(model, 2)
    bind = {"x": x, "w1": w1, "w2": w2}
    plain = execute_schedule(model, sched, bind, 2).outputs["y"]
    streamed = execute_schedule(model, sched, bind, 2, pipeline=chunks).outputs["y"]
    mid = np.zeros(n, np.float32)
    orc.tile_filter(x, w1, mid, t1["x"], t1["y"], 0, n)
    ref = np.zeros(n, np.float32)
    orc.tile_filter(mid, w2, ref, t2["x"], t2["y"], 0, n)
    assert np.array_equal(plain, ref)
    assert np.array_equal(streamed, ref)


def test_caller_stream_orders_uploads_kernels_and_downloads():
    """stream= kwarg: storage uploads, kernels and the output copy all run on the caller's
    stream.  A busy default stream must not be raced."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    M, N, K = 512, 384, 256
    g = orc.gemm_tilers(M, N, K)
    model = builders.tile_task_model(
        "matmul", {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]", "c": f"out float32 [{M},{N}]"},
        {k: _tiler(v) for k, v in g.items()}, (M, N))
    rng = np.random.default_rng(8)
    a = torch.from_numpy(rng.standard_normal(M * K).astype(np.float32)).pin_memory()
    b = torch.from_numpy(rng.standard_normal(K * N).astype(np.float32)).pin_memory()
    s = torch.cuda.Stream()
    ref = execute_schedule(model, build_schedule(model, 2), {"p_a": a, "p_b": b}, 2,
                           precision="exact").outputs["p_c"]
    for _ in range(3):
        busy = torch.empty(1 << 26, device="cuda")
        busy.normal_()                                   # keep the default stream occupied
        res = execute_schedule(model, build_schedule(model, 2), {"p_a": a, "p_b": b}, 2, precision="exact",
                               stream=s).outputs["p_c"]
        assert np.array_equal(res, ref)
        dev = execute_schedule(model, build_schedule(model, 2), {"p_a": a.cuda(), "p_b": b.cuda()}, 2,
                               precision="exact", stream=s, device_outputs=True).outputs["p_c"]
        s.synchronize()
        assert np.array_equal(dev.cpu().numpy(), ref)


# -- fp32-faithful matmul (precision="3xtf32", the fused tcgen05 kernel) --------------------

def _gemm_case(M, N, K, a_mn, b_k, seed):
    """(tilers, ports, bindings, A, B) with A stored [M,K] or transposed [K,M], B [K,N] or [N,K]."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    if a_mn:
        ta = dict(array=(K, M), rep=(M, N), pattern=(K,), origin=(0, 0), paving=((0, 0), (1, 0)),
                  fitting=((1,), (0,)))
        a_bind, a_arr = A.T.copy().ravel(), (K, M)
    else:
        ta = dict(array=(M, K), rep=(M, N), pattern=(K,), origin=(0, 0), paving=((1, 0), (0, 0)),
                  fitting=((0,), (1,)))
        a_bind, a_arr = A.ravel(), (M, K)
    if b_k:
        tb = dict(array=(N, K), rep=(M, N), pattern=(K,), origin=(0, 0), paving=((0, 1), (0, 0)),
                  fitting=((0,), (1,)))
        b_bind, b_arr = B.T.copy().ravel(), (N, K)
    else:
        tb = dict(array=(K, N), rep=(M, N), pattern=(K,), origin=(0, 0), paving=((0, 0), (0, 1)),
                  fitting=((1,), (0,)))
        b_bind, b_arr = B.ravel(), (K, N)
    tc = dict(array=(M, N), rep=(M, N), pattern=(1,), origin=(0, 0), paving=((1, 0), (0, 1)),
              fitting=((0,), (0,)))
    ports = {"a": f"in float32 [{a_arr[0]},{a_arr[1]}]", "b": f"in float32 [{b_arr[0]},{b_arr[1]}]",
             "c": f"out float32 [{M},{N}]"}
    return {"a": ta, "b": tb, "c": tc}, ports, {"p_a": a_bind, "p_b": b_bind}, A, B


@pytest.mark.parametrize("M,N,K,devices", [(256, 128, 64, 1), (300, 520, 200, 3), (1024, 768, 2048, 2),
                                           (129, 132, 96, 5), (777, 1000, 1500, 7)])
@pytest.mark.parametrize("a_mn,b_k", [(False, False), (False, True), (True, False), (True, True)])
def test_matmul_3xtf32_fused_accuracy(M, N, K, devices, a_mn, b_k):
    """Stated tolerance of precision='3xtf32' (fused kernel, K-chunked accumulation):
    element-wise |C - C64| <= (2^-20 + 2^-21 * sqrt(K)) * (|A||B|) and normwise <= 1e-6
    (cuBLAS SIMT fp32 measures 1.6e-6 normwise at 8192^3; TF32 alone ~8e-4)."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    t, ports, bind, A, B = _gemm_case(M, N, K, a_mn, b_k, M + K)
    model = builders.tile_task_model("matmul", ports, {k: _tiler(v) for k, v in t.items()}, (M, N))
    c = execute_schedule(model, build_schedule(model, devices), bind, devices,
                         precision="3xtf32").outputs["p_c"].reshape(M, N)
    a64, b64 = A.astype(np.float64), B.astype(np.float64)
    c64 = a64 @ b64
    bound = (2.0 ** -20 + 2.0 ** -21 * np.sqrt(K)) * (np.abs(a64) @ np.abs(b64))
    assert np.all(np.abs(c - c64) <= bound), float(np.max(np.abs(c - c64) / bound))
    assert np.linalg.norm(c - c64) / np.linalg.norm(c64) <= 1e-6


def test_matmul_3xtf32_split_form_still_matches(monkeypatch):
    """AOL_3XTF32_SPLIT=1 keeps the round-1 form (hi/lo copies in HBM, one accumulation)."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    monkeypatch.setenv("AOL_3XTF32_SPLIT", "1")
    M, N, K = 320, 256, 512
    t, ports, bind, A, B = _gemm_case(M, N, K, False, False, 9)
    model = builders.tile_task_model("matmul", ports, {k: _tiler(v) for k, v in t.items()}, (M, N))
    c = execute_schedule(model, build_schedule(model, 2), bind, 2, precision="3xtf32").outputs["p_c"]
    c64 = A.astype(np.float64) @ B.astype(np.float64)
    assert np.linalg.norm(c.reshape(M, N) - c64) / np.linalg.norm(c64) <= 4e-9 * K + 1e-6


# -- placement drives execution (rows a9 / f3) ---------------------------------------------

def test_memory_role_selects_the_kernel_staging():
    """Two FIR models that differ only in where the input is allocated: deviceGlobal runs the
    register-window batched kernel, deviceLocal the shared-memory-staged line window; both
    equal the oracle bit for bit, and the deviceGlobal groups live in one arena at the
    placement's offsets."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from _sharded_cases import fir_model
    from paper_1105_4424_b200 import _capi
    from paper_1105_4424_b200.executor import Executor
    from paper_1105_4424_b200.partition import build_schedule
    plans = {}
    for mem in ("dev.gmem", "dev.cu.lmem"):
        model, bind, out, ref = fir_model(memory=mem)
        for D in (1, 3):
            ex = Executor(model, build_schedule(model, D), bind, D)
            ex.run()
            got = ex.outputs()[out]
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (mem, D)
        t = ex.task("t")
        ptrs = [ex.storage.array(t.nodes[n]).data_ptr() for n in t.port_order]
        plans[mem] = _capi.plan_name(t.ctask, 0, 16384, ptrs)
        arena = ex.storage.arenas["dev.gmem"]
        for g, pl in ex.storage.placement.items():
            if pl.tier == "hbm":
                assert ex.storage.arrays[g].data_ptr() == arena.data_ptr() + pl.b200_offset
        assert "line_tiled" in ex.placement_report() or mem == "dev.gmem"
    assert plans == {"dev.gmem": "tile_filter.batched", "dev.cu.lmem": "tile_filter.line_tiled"}


# -- stream-K tail of the TF32 pair kernel -----------------------------------------------------

@pytest.mark.parametrize("M,N,K,devices,a_mn,b_k", [
    (1024, 8192, 8192, 1, False, False),   # C2's 8-rank shard: 128 tiles = 1 wave + 54 (no split)
    (2048, 8192, 8192, 1, False, False),   # C2's 4-rank shard: 256 tiles = 3 waves + 34 tail tiles, s = 2
    (2048, 8192, 2048, 1, False, True),    # the same tail, 64 k-blocks: pieces of 32
    (768, 10496, 3072, 1, True, False),    # 123 tiles = 1 wave + 49 tail tiles (s = 3 forced below)
    (256, 256, 4096, 1, True, False),      # one tile (s = 2: two pieces of 64 k-blocks)
    (300, 520, 200, 3, False, False),      # ragged shards, few k-blocks
    (777, 1000, 1500, 7, True, True),
    (2304, 2560, 768, 2, False, False)])   # 2 shards of 1152 rows: 50 tiles each
@pytest.mark.parametrize("force", [None, "3", "4", "8"])
def test_matmul_stream_k_tail(M, N, K, devices, a_mn, b_k, force, monkeypatch):
    """Tiles of the last partial wave are cut into s k-ranges dealt to every pair and summed in
    k order by the last piece to arrive: inside the stated TF32 bound, and bit-identical from
    run to run (fixed summation order, counters reset by the last arriver)."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    if force is not None:
        if M * N * K > 2 ** 34:
            pytest.skip("forced splits are checked on the smaller shapes")
        monkeypatch.setenv("AOL_GEMM_SPLIT", force)      # read per launch
    t, ports, bind, A, B = _gemm_case(M, N, K, a_mn, b_k, M + N + K)
    model = builders.tile_task_model("matmul", ports, {k: _tiler(v) for k, v in t.items()}, (M, N))
    sched = build_schedule(model, devices)
    c1 = execute_schedule(model, sched, bind, devices).outputs["p_c"].reshape(M, N)
    c2 = execute_schedule(model, sched, bind, devices).outputs["p_c"].reshape(M, N)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    a64, b64 = A.astype(np.float64), B.astype(np.float64)
    if M * N * K > 2 ** 34:                  # check 64 sampled rows of the big case
        rows = np.random.default_rng(1).choice(M, 64, replace=False)
        a64, c1 = a64[rows], c1[rows]
    bound = (2.0 ** -9 + K * 2.0 ** -23) * (np.abs(a64) @ np.abs(b64))
    assert np.all(np.abs(c1 - a64 @ b64) <= bound)


# -- more simulated devices than repetitions (partition.py:105-121: only T ranges) -------------

@pytest.mark.parametrize("D", [5, 8, 13])
def test_more_devices_than_repetitions_vs_oracle(D):
    """partition_equally(T, D) with D > T yields T one-repetition launches (refexec.py:488);
    tile_copy, the stencil and the TF32 matmul then run T tiny launches and still match the
    oracle (matmul: the TF32 bound), on one device and sharded over local replicas."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    rng = np.random.default_rng(D)
    # tile_copy: 3 repetitions of a 4-element reversed pattern
    ts = dict(array=(12,), rep=(3,), pattern=(4,), origin=(3,), paving=((4,),), fitting=((-1,),))
    td = dict(array=(12,), rep=(3,), pattern=(4,), origin=(0,), paving=((4,),), fitting=((1,),))
    m = builders.tile_task_model("tile_copy", {"src": "in float32 [12]", "dst": "out float32 [12]"},
                                 {"src": _tiler(ts), "dst": _tiler(td)}, (3,))
    x = (np.arange(12) + 1).astype(np.float32)
    want = orc.run_tile_task("tile_copy", {"src": ts, "dst": td}, {"src": x}, {"dst": (12, np.float32)}, 3, D)["dst"]
    sched = build_schedule(m, D)
    assert len(sched.device_steps()[0].launches) == 3
    for devices in (None, [0, 0]):
        got = execute_schedule(m, sched, {"p_src": x}, D, devices=devices).outputs["p_dst"]
        assert np.array_equal(got, want)
    # 2x2 toroidal stencil: 4 repetitions
    t = orc.stencil_tilers(2, 2)
    m = builders.tile_task_model("stencil", {"x": "in float32 [2,2]", "w": "in float32 [9]", "y": "out float32 [2,2]"},
                                 {k: _tiler(v) for k, v in t.items()}, (2, 2))
    xs = rng.random(4).astype(np.float32)
    want = orc.run_tile_task("stencil", t, {"x": xs, "w": orc.stencil_weights()}, {"y": (4, np.float32)}, 4, D)["y"]
    got = execute_schedule(m, build_schedule(m, D), {"p_x": xs, "p_w": orc.stencil_weights()}, D).outputs["p_y"]
    assert np.array_equal(got, want)
    # 1x2 matmul with K = 96: 2 repetitions
    M, N, K = 1, 2, 96
    g = orc.gemm_tilers(M, N, K)
    m = builders.tile_task_model("matmul", {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]",
                                            "c": f"out float32 [{M},{N}]"}, {k: _tiler(v) for k, v in g.items()}, (M, N))
    a = rng.standard_normal(M * K).astype(np.float32)
    b = rng.standard_normal(K * N).astype(np.float32)
    c = execute_schedule(m, build_schedule(m, D), {"p_a": a, "p_b": b}, D).outputs["p_c"].reshape(M, N)
    a64, b64 = a.reshape(M, K).astype(np.float64), b.reshape(K, N).astype(np.float64)
    assert np.all(np.abs(c - a64 @ b64) <= (2.0 ** -9 + K * 2.0 ** -23) * (np.abs(a64) @ np.abs(b64)))


# -- mixed-width column tiles of the TF32 pair kernel -------------------------------------------

@pytest.mark.parametrize("M,N,K,devices,a_mn,b_k", [
    (1024, 8192, 2048, 1, False, False),   # the 8-rank C2 shard shape: 17 x 256 + 20 x 192 per row
    (1024, 8192, 1024, 1, False, True),    # the same with K-major B (full 128-row boxes, 96 used)
    (1024, 8000, 512, 1, True, False),     # ragged N: the last narrow tile runs past N (masked)
    (300, 520, 200, 3, False, False),      # ragged shards: 128-column tiles
    (256, 256, 4096, 1, False, True),      # one tile -> two 128-column tiles
    (2304, 2560, 768, 2, True, True)])     # 192-column tiles only
@pytest.mark.parametrize("narrow", ["1", "0"])
def test_matmul_mixed_width_tiles(M, N, K, devices, a_mn, b_k, narrow, monkeypatch):
    """Opt-in mixed-width plan (AOL_GEMM_NARROW=1): whole 256-column tiles that would leave the
    last wave partly idle are replaced by 256- and 192/128-column tiles (tcgen05 N from the
    instruction descriptor at run time): inside the TF32 bound either way."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    monkeypatch.setenv("AOL_GEMM_NARROW", narrow)          # read per launch
    monkeypatch.setenv("AOL_GEMM_STREAMK", "0")            # the split-K tail would take precedence
    t, ports, bind, A, B = _gemm_case(M, N, K, a_mn, b_k, M * 7 + N + K)
    model = builders.tile_task_model("matmul", ports, {k: _tiler(v) for k, v in t.items()}, (M, N))
    c = execute_schedule(model, build_schedule(model, devices), bind, devices).outputs["p_c"].reshape(M, N)
    a64, b64 = A.astype(np.float64), B.astype(np.float64)
    bound = (2.0 ** -9 + K * 2.0 ** -23) * (np.abs(a64) @ np.abs(b64))
    assert np.all(np.abs(c - a64 @ b64) <= bound)


def test_ipc_abi_errors():
    """aol_ipc_*: exporting a device pointer gives a 72-byte token (handle + offset inside the
    allocation); closing a pointer that was never imported, or exporting host memory, fails
    with an error status instead of crashing."""
    from paper_1105_4424_b200 import _capi
    t = torch.zeros(1 << 20, device="cuda")
    tok = _capi.ipc_export(t.data_ptr() + 4096)
    assert len(tok) == 72 and int.from_bytes(tok[64:], "little") >= 4096
    with pytest.raises(_capi.AolError):
        _capi.ipc_close(t.data_ptr())
    host = np.zeros(16, np.float32)
    with pytest.raises(_capi.AolError):
        _capi.ipc_export(host.ctypes.data)


# -- 2-D streamed MatMul from pinned host memory ------------------------------------------------

@pytest.mark.parametrize("M,N,K,precision", [(2304, 2560, 512, "default"), (1024, 1024, 256, "exact"),
                                             (4096, 4096, 1024, "default"), (1536, 2048, 512, "3xtf32")])
def test_streamed_gemm2d_equals_plain(M, N, K, precision):
    """pipeline > 1 with pinned torch host tensors takes the 2-D block path (B and C moved in
    column blocks by aol_memcpy2d, each C block a derived GEMM over the same arrays launched
    as soon as its operands landed): bit-identical to the plain run (the same per-element
    accumulation), and for precision="exact" to the oracle."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    model = builders.matmul_model(M, N, K)
    sched = build_schedule(model, 1)
    g = torch.Generator().manual_seed(M + N + K)
    ha = torch.randn(M * K, generator=g).pin_memory()
    hb = torch.randn(K * N, generator=g).pin_memory()
    hc = torch.empty(M * N).pin_memory()
    plain = execute_schedule(model, sched, {"p_a": ha.numpy(), "p_b": hb.numpy()}, 1,
                             precision=precision).outputs["p_c"]
    res = execute_schedule(model, sched, {"p_a": ha, "p_b": hb}, 1, precision=precision, pipeline=8,
                           out={"p_c": hc})
    assert res.outputs["p_c"] is hc
    assert np.array_equal(hc.numpy().view(np.uint32), plain.view(np.uint32))
    fresh = execute_schedule(model, sched, {"p_a": ha, "p_b": hb}, 1, precision=precision, pipeline=8).outputs["p_c"]
    assert np.array_equal(fresh.view(np.uint32), plain.view(np.uint32))
    # pageable numpy sources (the reference's call) take the same path through the staging ring
    na, nb = ha.numpy().copy(), hb.numpy().copy()
    paged = execute_schedule(model, sched, {"p_a": na, "p_b": nb}, 1, precision=precision, pipeline=8).outputs["p_c"]
    assert np.array_equal(paged.view(np.uint32), plain.view(np.uint32))
    if precision == "exact":
        want = orc.run_tile_task("matmul", orc.gemm_tilers(M, N, K), {"a": ha.numpy(), "b": hb.numpy()},
                                 {"c": (M * N, np.float32)}, M * N, 1)["c"]
        assert np.array_equal(plain.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("M,N,K,devices", [(2048, 264, 2048, 3), (2048, 1000, 512, 7), (1024, 520, 256, 5)])
def test_matmul_mn_major_a_unaligned_shards(M, N, K, devices):
    """MN-major A with shards that start mid-matrix (m_lo not a multiple of 32): the TF32 kernel
    tiles from m_lo aligned down to a 128 B swizzle atom and masks the rows before m_lo
    (a TMA box starting off the atom raised an illegal-instruction fault)."""
    from paper_1105_4424_b200 import _capi, builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    t, ports, bind, A, B = _gemm_case(M, N, K, True, False, M + N + K + devices)
    model = builders.tile_task_model("matmul", ports, {k: _tiler(v) for k, v in t.items()}, (M, N))
    sched = build_schedule(model, devices)
    assert any((l.range.offset // N) % 32 for l in sched.device_steps()[0].launches)   # really unaligned
    c = execute_schedule(model, sched, bind, devices).outputs["p_c"].reshape(M, N)
    a64, b64 = A.astype(np.float64), B.astype(np.float64)
    assert np.all(np.abs(c - a64 @ b64) <= (2.0 ** -9 + K * 2.0 ** -23) * (np.abs(a64) @ np.abs(b64)))
    c3 = execute_schedule(model, sched, bind, devices, precision="3xtf32").outputs["p_c"].reshape(M, N)
    assert np.linalg.norm(c3 - a64 @ b64) / np.linalg.norm(a64 @ b64) <= 1e-6


@pytest.mark.parametrize("chunks", [2, 5])
def test_streamed_inout_keeps_bound_values_outside_the_repetitions(chunks):
    """axpy with no `repeat` (repetition space 1: only element 0 is touched) on
    999-element vectors: the streamed path uploads y only where a chunk reads it, so every other
    element must come back as the caller's bound value, exactly as the plain run returns it."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    model = builders.single_task_model(
        "axpy", ["y inout float64 [999]", "x in float64 [999]", "a in float64 [1]"],
        ["i in float64 [999]", "v in float64 [999]", "s in float64 [1]", "o out float64 [999]"],
        ["i -> t.y", "v -> t.x", "s -> t.a", "t.y -> o"],
        ["allocate data i onto dev.gmem", "allocate data v onto dev.gmem", "allocate data s onto host.ram",
         "allocate task t onto dev.cu"], None)
    rng = np.random.default_rng(chunks)
    bind = {"i": rng.standard_normal(999), "v": rng.standard_normal(999), "s": np.array([0.75])}
    sched = build_schedule(model, 3)
    plain = execute_schedule(model, sched, bind, 3).outputs["o"]
    streamed = execute_schedule(model, sched, bind, 3, pipeline=chunks).outputs["o"]
    want = bind["i"].copy()
    want[0] += 0.75 * bind["v"][0]
    assert np.array_equal(plain, want)
    assert np.array_equal(streamed, want)


@pytest.mark.parametrize("n", [1, 1000, 4096, 100_003])
def test_host_stager_download_pieces(n):
    """HostStager.download through a 4 KiB x 2-slot ring: pieces alternate slots, the host copy
    of piece k overlaps the DMA of piece k+1, the result equals the device data bit for bit."""
    import torch
    from paper_1105_4424_b200.executor import HostStager
    st = HostStager(slot_bytes=4096, slots=2)
    src = torch.randn(n, device="cuda", dtype=torch.float32)
    dst = torch.empty(n, dtype=torch.float32)
    st.download(dst, src, torch.cuda.current_stream())
    assert torch.equal(dst, src.cpu())


def test_numpy_outputs_pinned_and_staged_forms(monkeypatch):
    """Numpy outputs come back through a pinned block (small) or the staging ring (large):
    both forms equal the device-resident result."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import Executor, execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    n = 192
    model = builders.matmul_model(n, n, n)
    sched = build_schedule(model, 2)
    rng = np.random.default_rng(0)
    bind = {"p_a": rng.standard_normal(n * n, dtype=np.float32), "p_b": rng.standard_normal(n * n, dtype=np.float32)}
    dev = execute_schedule(model, sched, bind, 2, device_outputs=True).outputs["p_c"].cpu().numpy()
    pinned = execute_schedule(model, sched, bind, 2).outputs["p_c"]
    assert isinstance(pinned, np.ndarray) and np.array_equal(pinned, dev)
    monkeypatch.setattr(Executor, "PINNED_OUTPUT_BYTES", 0)
    staged = execute_schedule(model, sched, bind, 2).outputs["p_c"]
    assert isinstance(staged, np.ndarray) and np.array_equal(staged, dev)


_X3_FORM_SCRIPT = """
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1105_4424_b200 import builders
from paper_1105_4424_b200.executor import execute_schedule
from paper_1105_4424_b200.partition import build_schedule
M, N, K, D = 300, 520, 1000, 3
rng = np.random.default_rng(5)
bind = {"p_a": rng.standard_normal(M * K, dtype=np.float32), "p_b": rng.standard_normal(K * N, dtype=np.float32)}
model = builders.matmul_model(M, N, K)
np.save(sys.argv[2], execute_schedule(model, build_schedule(model, D), bind, D, precision="3xtf32").outputs["p_c"])
"""


def test_matmul_3xtf32_forms_are_bit_identical(tmp_path):
    """The three fused 3xTF32 kernels -- regs (default: 256x256 tiles, running sum in registers),
    wide (256x256, one accumulator + running sum in TMEM) and narrow (256x128) -- use the same
    64-deep chunks and add order: bit-identical C on unaligned shards (the form is read once per
    process, so each runs in its own interpreter)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    outs = {}
    for form, env in (("regs", {}), ("wide", {"AOL_3XTF32_FORM": "wide"}), ("narrow", {"AOL_3XTF32_WIDE": "0"})):
        out = tmp_path / f"{form}.npy"
        subprocess.run([sys.executable, "-c", _X3_FORM_SCRIPT, root, str(out)],
                       env={**os.environ, **env}, check=True, timeout=300)
        outs[form] = np.load(out)
    assert np.array_equal(outs["regs"], outs["narrow"])
    assert np.array_equal(outs["wide"], outs["narrow"])


def test_prepared_executor_reuse_is_isolated():
    """Repeated calls on one (model, schedule) reuse a prepared executor: results follow each
    call's bindings, device outputs from an earlier call are not overwritten by a later one,
    and a partially written output (gaps) keeps zeros outside the written elements."""
    import torch
    from paper_1105_4424_b200 import Tiler, builders
    from paper_1105_4424_b200 import executor as exm
    from paper_1105_4424_b200.partition import build_schedule
    n = 96
    model = builders.matmul_model(n, n, n)
    sched = build_schedule(model, 2)
    rng = np.random.default_rng(1)
    exm.clear_prepared()
    results, devs = [], []
    for i in range(4):
        a = rng.standard_normal(n * n, dtype=np.float32)
        b = rng.standard_normal(n * n, dtype=np.float32)
        want = exm.execute_schedule(model, sched, {"p_a": a, "p_b": b}, 2, precision="exact").outputs["p_c"]
        dev = exm.execute_schedule(model, sched, {"p_a": torch.from_numpy(a).cuda(), "p_b": torch.from_numpy(b).cuda()},
                                   2, precision="exact", device_outputs=True).outputs["p_c"]
        results.append(want)
        devs.append(dev)
    assert any(k[0] == id(model) for k in exm._PREPARED)
    for want, dev in zip(results, devs):
        assert np.array_equal(dev.cpu().numpy(), want)
    assert not np.array_equal(results[0], results[1])
    # gaps: dst written at every other element, the rest must read back zero on every call
    T = 1000
    src = Tiler((0,), ((1,),), ((1,),), (1,))
    dst = Tiler((0,), ((2,),), ((1,),), (1,))
    gm = builders.tile_task_model("tile_copy", {"src": f"in float32 [{T}]", "dst": f"out float32 [{2 * T}]"},
                                  {"src": src, "dst": dst}, (T,))
    gs = build_schedule(gm, 3)
    for i in range(3):
        x = rng.standard_normal(T).astype(np.float32) + 10.0
        y = exm.execute_schedule(gm, gs, {"p_src": x}, 3).outputs["p_dst"]
        assert np.array_equal(y[0::2], x) and not y[1::2].any()
    exm.clear_prepared()


def test_prepared_executor_busy_entry_is_bypassed():
    """A call that finds the cached executor in use (another thread) builds its own."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200 import executor as exm
    from paper_1105_4424_b200.partition import build_schedule
    n = 64
    model = builders.matmul_model(n, n, n)
    sched = build_schedule(model, 1)
    rng = np.random.default_rng(2)
    a = rng.standard_normal(n * n, dtype=np.float32)
    b = rng.standard_normal(n * n, dtype=np.float32)
    exm.clear_prepared()
    first = exm.execute_schedule(model, sched, {"p_a": a, "p_b": b}, 1, precision="exact").outputs["p_c"]
    (_, _, _, lock), = exm._PREPARED.values()
    assert lock.acquire(blocking=False)                  # simulate a concurrent user
    try:
        again = exm.execute_schedule(model, sched, {"p_a": a, "p_b": b}, 1, precision="exact").outputs["p_c"]
    finally:
        lock.release()
    assert np.array_equal(first, again)
    exm.clear_prepared()


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("a_mn,b_k", [(False, False), (True, True), (False, True)])
def test_matmul_exact_128_tiles_bit_exact(dtype, a_mn, b_k):
    """precision="exact" at sizes that take the 128 x 128 double-buffered kernel (>= 2 tiles per
    SM), K not a multiple of the 8-deep slab, unaligned shards: every output equals the k-ascending
    product with a rounding per product and per add (numpy elementwise arithmetic in that order)."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.partition import build_schedule
    M, N, K, D = 2200, 2100, 45, 3
    t, ports, bind, A, B = _gemm_case(M, N, K, a_mn, b_k, 17)
    ports = {k: v.replace("float32", dtype) for k, v in ports.items()}
    bind = {k: np.asarray(v).astype(dtype) for k, v in bind.items()}
    model = builders.tile_task_model("matmul", ports, {k: _tiler(v) for k, v in t.items()}, (M, N))
    sched = build_schedule(model, D)
    c = execute_schedule(model, sched, bind, D, precision="exact").outputs["p_c"].reshape(M, N)
    A, B = A.astype(dtype), B.astype(dtype)
    want = np.zeros((M, N), dtype=dtype)
    for k in range(K):
        want = want + A[:, k:k + 1] * B[k:k + 1, :]
    assert c.dtype == want.dtype and np.array_equal(c, want)


@pytest.mark.parametrize("persistent", ["1", "0"])
@pytest.mark.parametrize("D", [1, 5, 8])
def test_cg_with_caller_stream_matches_default(golden, persistent, D, monkeypatch):
    """A LoopStep run with execute_schedule(stream=...) equals the default-stream run bit for bit,
    on the persistent interpreter (D up to 8 now fits it) and on the CUDA-graph WHILE path
    (AOL_LOOP_PERSISTENT=0), whose capture must take the body's launches even when the caller
    named a stream (they used to run once, eagerly, outside the graph: 400 iterations, no
    convergence)."""
    import torch
    from paper_1105_4424_b200.executor import Executor, execute_schedule
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    monkeypatch.setenv("AOL_LOOP_PERSISTENT", persistent)
    data, meta = golden
    model = model_from_dict(meta["cg_k20"]["model"])
    bind = {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}
    sched = build_schedule(model, D)
    plain = execute_schedule(model, sched, bind, D)
    s = torch.cuda.Stream()
    res = execute_schedule(model, sched, bind, D, stream=s)
    torch.cuda.synchronize()
    assert res.iterations == plain.iterations
    assert np.array_equal(np.asarray(res.outputs["x"]), np.asarray(plain.outputs["x"]))
    if persistent == "1":
        ex = Executor(model, sched, bind, D)
        ex.run()
        assert ex.persistent_loops == 1


def test_concurrent_calls_from_threads():
    """Four host threads calling execute_schedule on shared (model, schedule) objects at once --
    two of them on their own streams -- all get the single-threaded results (the prepared-executor
    cache's dict is locked; a busy entry is bypassed)."""
    import threading
    import torch
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200 import executor as exm
    from paper_1105_4424_b200.partition import build_schedule
    rng = np.random.default_rng(4)
    cases = []
    for n, D in ((96, 1), (160, 3)):
        model = builders.matmul_model(n, n, n)
        sched = build_schedule(model, D)
        bind = {"p_a": rng.standard_normal(n * n, dtype=np.float32), "p_b": rng.standard_normal(n * n, dtype=np.float32)}
        want = exm.execute_schedule(model, sched, bind, D, precision="exact").outputs["p_c"]
        cases.append((model, sched, bind, D, want))
    exm.clear_prepared()
    errors = []

    def work(tid):
        s = torch.cuda.Stream() if tid % 2 else None
        for c in range(30):
            model, sched, bind, D, want = cases[(tid + c) % len(cases)]
            kw = {"stream": s} if s is not None else {}
            try:
                got = exm.execute_schedule(model, sched, bind, D, precision="exact", **kw).outputs["p_c"]
                if not np.array_equal(got, want):
                    errors.append((tid, c, "mismatch"))
            except Exception as e:  # noqa: BLE001
                errors.append((tid, c, repr(e)))

    ts = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    exm.clear_prepared()
    assert not errors, errors[:5]


def test_prepared_executor_survives_a_failed_call():
    """A call whose binding is the wrong size raises MissingBinding from the prepared executor's
    rebind; the entry's lock is released, and the next good call on the same cached executor
    returns the right result."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200 import executor as exm
    from paper_1105_4424_b200.partition import build_schedule
    n = 80
    model = builders.matmul_model(n, n, n)
    sched = build_schedule(model, 2)
    rng = np.random.default_rng(6)
    bind = {"p_a": rng.standard_normal(n * n, dtype=np.float32), "p_b": rng.standard_normal(n * n, dtype=np.float32)}
    exm.clear_prepared()
    want = exm.execute_schedule(model, sched, bind, 2, precision="exact").outputs["p_c"]
    with pytest.raises(exm.MissingBinding):
        exm.execute_schedule(model, sched, {"p_a": bind["p_a"][:-1], "p_b": bind["p_b"]}, 2, precision="exact")
    (_, _, _, lock), = exm._PREPARED.values()
    assert not lock.locked()
    again = exm.execute_schedule(model, sched, bind, 2, precision="exact").outputs["p_c"]
    assert np.array_equal(again, want)
    exm.clear_prepared()
