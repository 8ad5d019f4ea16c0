"""Host-side logic and the C ABI surface — runs without a GPU."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import aol_oracle as orc
from paper_1105_4424_b200 import (INTRINSICS, IntrinsicShapeMismatch, Tiler, TilerError, UnknownIntrinsic,
                                  WorkRange, builders, build_schedule, check_task_signature, partition_equally)
from paper_1105_4424_b200 import _capi

ROOT = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg/src")


# -- C ABI -------------------------------------------------------------------

def header_functions():
    text = (ROOT / "include" / "aol_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(aol_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(_capi.LIB_PATH))
    names = header_functions()
    assert len(names) >= 8
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_capi.EXPORTS)
    assert _capi.load().aol_abi_version() == _capi.ABI_VERSION


def test_struct_layout_matches_header():
    assert ctypes.sizeof(_capi.AolTiler) == 16 + 4 * 4 * 8 + 2 * 16 * 8
    assert ctypes.sizeof(_capi.AolTask) == 32 + 4 * ctypes.sizeof(_capi.AolTiler)


def _bt(d):
    return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"]).bind(d["array"], d["rep"])


def test_validate_and_plan_without_gpu():
    g = orc.gemm_tilers(64, 64, 32)
    task = _capi.make_task("matmul", "float32", [_bt(g[k]) for k in "abc"])
    _capi.validate(task)
    assert _capi.plan_name(task, 0, 64 * 64) == "matmul.exact_tiled"        # no ports -> no TMA check
    bad = _capi.make_task("matmul", "float32", [_bt(g[k]) for k in "ab"])
    with pytest.raises(_capi.AolError, match="tilers"):
        _capi.validate(bad)
    cp = dict(array=(100,), rep=(25,), pattern=(4,), origin=(0,), paving=((4,),), fitting=((1,),))
    t = _capi.make_task("tile_copy", "float32", [_bt(cp), _bt(cp)])
    assert _capi.plan_name(t, 0, 25) == "tile_copy.stream16"
    ov = dict(cp, rep=(49,), paving=((2,),))
    dst = dict(array=(196,), rep=(49,), pattern=(4,), origin=(0,), paving=((4,),), fitting=((1,),))
    assert _capi.plan_name(_capi.make_task("tile_copy", "float32", [_bt(ov), _bt(dst)]), 0, 49) == "tile_copy.vec"
    st = dict(cp, rep=(24,), paving=((4,),), fitting=((2,),))
    dst2 = dict(dst, array=(96,), rep=(24,))
    assert _capi.plan_name(_capi.make_task("tile_copy", "float32", [_bt(st), _bt(dst2)]), 0, 24) == "tile_copy.vec_store"
    od = dict(cp, array=(75,), rep=(25,), pattern=(3,), paving=((3,),), fitting=((1,),))
    odd = dict(od, origin=(0,), array=(80,), paving=((3,),), fitting=((1,),))
    assert _capi.plan_name(_capi.make_task("tile_copy", "float32", [_bt(dict(od, paving=((2,),), array=(60,))), _bt(odd)]), 0, 25) == "tile_copy.affine"
    wr = dict(cp, origin=(99,))
    assert _capi.plan_name(_capi.make_task("tile_copy", "float32", [_bt(wr), _bt(cp)]), 0, 25) == "tile_copy.generic"
    mism = dict(cp, pattern=(2,), array=(50,), paving=((2,),))
    with pytest.raises(_capi.AolError, match="pattern"):
        _capi.validate(_capi.make_task("tile_copy", "float32", [_bt(cp), _bt(mism)]))


def _copy_plan(src, dst, dtype="float32"):
    T = src["rep"][0]
    return _capi.plan_name(_capi.make_task("tile_copy", dtype, [_bt(src), _bt(dst)]), 0, T)


def _dense(T, m):
    return dict(array=(T * m,), rep=(T,), pattern=(m,), origin=(0,), paving=((m,),), fitting=((1,),))


def test_tile_copy_plan_dispatch_rules_without_gpu():
    """Which kernel each tile_copy geometry selects (host-side planning, no device): TMA box
    rings from 1 MB on, 16-byte pitches and >= 32 B rows; bulk windows for overlapping 8-16 B
    rows; the TMA transpose for row-stride gathers with 32-256 B pattern columns."""
    def row1d(T, m, p, f=1):
        return dict(array=((T - 1) * p + (m - 1) * f + 1,), rep=(T,), pattern=(m,), origin=(0,), paving=((p,),),
                    fitting=((f,),))
    big = 1 << 20
    assert _copy_plan(row1d(big // 8, 2, 2), _dense(big // 8, 2)) == "tile_copy.tma_stream"       # dense, 1 MB
    assert _copy_plan(row1d(1000, 2, 2), _dense(1000, 2)) == "tile_copy.stream16"                 # dense, small
    assert _copy_plan(row1d(40000, 8, 16), _dense(40000, 8)) == "tile_copy.tma_box"               # 32 B rows, gaps
    assert _copy_plan(row1d(40000, 4, 8), _dense(40000, 4)) == "tile_copy.vec"                    # 16 B rows
    assert _copy_plan(row1d(40000, 8, 18), _dense(40000, 8)) == "tile_copy.vec"                   # 72 B pitch
    assert _copy_plan(row1d(20000, 32, 16), _dense(20000, 32)) == "tile_copy.tma_box"             # overlap, 128 B
    assert _copy_plan(row1d(40000, 8, 4), _dense(40000, 8)) == "tile_copy.window"                 # overlap, 32 B
    assert _copy_plan(row1d(200000, 2, 1), _dense(200000, 2)) == "tile_copy.window"               # overlap, 8 B
    assert _copy_plan(row1d(100000, 4, 3), _dense(100000, 4)) == "tile_copy.window"
    assert _copy_plan(row1d(40000, 8, 16, f=2), _dense(40000, 8)) == "tile_copy.vec_store"        # strided fitting
    assert _copy_plan(row1d(1000, 1, 2), _dense(1000, 1)) == "tile_copy.stride2"                  # m = 1 gaps
    assert _copy_plan(row1d(1000, 1, 3), _dense(1000, 1)) == "tile_copy.affine"
    assert _copy_plan(row1d(40000, 4, 8), _dense(40000, 4), "float64") == "tile_copy.tma_box"    # 32 B fp64 rows

    def rowstride(m, T):
        return dict(array=(m, T), rep=(T,), pattern=(m,), origin=(0, 0), paving=((0,), (1,)), fitting=((1,), (0,)))
    assert _copy_plan(rowstride(8, 40000), _dense(40000, 8)) == "tile_copy.tma_transpose"
    assert _copy_plan(rowstride(64, 5004), _dense(5004, 64)) == "tile_copy.tma_transpose"
    assert _copy_plan(rowstride(8, 40001), _dense(40001, 8)) == "tile_copy.transpose"             # pitch % 16 B
    assert _copy_plan(rowstride(4, 80000), _dense(80000, 4)) == "tile_copy.interleave"            # 16 B columns
    assert _copy_plan(rowstride(4, 80001), _dense(80001, 4)) == "tile_copy.transpose"             # pitch % 16 B
    assert _copy_plan(rowstride(8, 40000), _dense(40000, 8), "float64") == "tile_copy.transpose"
    blk = dict(array=(64, 64), rep=(8, 8), pattern=(8, 8), origin=(0, 0), paving=((8, 0), (0, 8)),
               fitting=((1, 0), (0, 1)))
    dense = dict(array=(4096,), rep=(8, 8), pattern=(8, 8), origin=(0,), paving=((512, 64),), fitting=((8, 1),))
    assert _capi.plan_name(_capi.make_task("tile_copy", "float32", [_bt(blk), _bt(dense)]), 0, 64) == \
        "tile_copy.affine2d"                                                                     # block tilers


# -- partitioning (partition.py:105-121) ---------------------------------------

def test_partition_paper_scale():
    ranges = partition_equally(132651, 4)
    assert [r.count for r in ranges] == [33163, 33163, 33163, 33162]
    assert [r.offset for r in ranges] == [0, 33163, 66326, 99489]
    assert partition_equally(10, 1) == [WorkRange(0, 10)]
    assert len(partition_equally(3, 8)) == 3
    with pytest.raises(ValueError):
        partition_equally(0, 4)


@settings(max_examples=300, deadline=None)
@given(st.integers(1, 100000), st.integers(1, 16))
def test_partition_matches_oracle(total, devices):
    assert [(r.offset, r.count) for r in partition_equally(total, devices)] == orc.partition_equally(total, devices)


def test_partition_golden(golden):
    _, meta = golden
    for key, ranges in meta["_partition"].items():
        t, d = map(int, key.split(","))
        assert [[r.offset, r.count] for r in partition_equally(t, d)] == ranges


# -- tilers -------------------------------------------------------------------

def test_tiler_bind_errors():
    with pytest.raises(TilerError):
        Tiler([0], [[1]], [[1]], [2]).bind((4, 4), (4,))        # origin rank != array rank
    with pytest.raises(TilerError):
        Tiler([0], [[1, 0]], [[1]], [2]).bind((4,), (4,))       # paving not a x q
    with pytest.raises(TilerError):
        Tiler([0], [[1]], [[1]], [0]).bind((4,), (4,))          # zero pattern dim
    with pytest.raises(TilerError):
        Tiler([0] * 5, [[1]] * 5, [[1]] * 5, [1]).bind((2,) * 5, (1,))


def test_tiler_affine_and_wrap():
    g = orc.gemm_tilers(8, 6, 5)
    a = _bt(g["a"])
    assert not a.wraps and a.affine == (0, (5, 0), (1,))
    s = _bt(orc.stencil_tilers(8, 8)["x"])
    assert s.wraps and s.affine is None


def test_tiler_offsets_match_oracle_loop():
    rng = np.random.default_rng(5)
    for _ in range(60):
        a, q, p = (int(x) for x in rng.integers(1, 4, 3))
        d = dict(array=tuple(int(x) for x in rng.integers(1, 7, a)), rep=tuple(int(x) for x in rng.integers(1, 5, q)),
                 pattern=tuple(int(x) for x in rng.integers(1, 4, p)),
                 origin=tuple(int(x) for x in rng.integers(-9, 9, a)),
                 paving=tuple(tuple(int(x) for x in rng.integers(-4, 5, q)) for _ in range(a)),
                 fitting=tuple(tuple(int(x) for x in rng.integers(-4, 5, p)) for _ in range(a)))
        bt = _bt(d)
        assert np.array_equal(bt.offsets(), np.array(orc.tiler_offsets_loop(d, 0, bt.rep_total)))


def test_injectivity():
    _bt(orc.gemm_tilers(64, 32, 8)["c"]).check_injective()
    _bt(orc.stencil_tilers(16, 16)["y"]).check_injective()
    big = dict(array=(1 << 30,), rep=(1 << 28,), pattern=(4,), origin=(0,), paving=((4,),), fitting=((1,),))
    _bt(big).check_injective()                                  # mixed-radix proof, no enumeration
    with pytest.raises(TilerError):
        _bt(dict(array=(100,), rep=(20,), pattern=(4,), origin=(0,), paving=((2,),), fitting=((1,),))).check_injective()
    with pytest.raises(TilerError):   # wraps onto itself
        _bt(dict(array=(10,), rep=(10,), pattern=(1,), origin=(0,), paving=((2,),), fitting=((0,),))).check_injective()


# -- registry / signature checks ------------------------------------------------

def _copy_model(op="copy", ports=("src in float64 [64]", "dst out float64 [64]")):
    return builders.single_task_model(
        op, list(ports), ["i in float64 [64]", "o out float64 [64]"], ["i -> t.src", "t.dst -> o"],
        ["allocate data i onto dev.gmem", "allocate data t.dst onto dev.gmem", "allocate task t onto dev.cu"], 64)


def test_signature_checks():
    m = _copy_model()
    assert check_task_signature("t", m.application_components["T"]).name == "copy"
    with pytest.raises(UnknownIntrinsic):
        check_task_signature("t", _copy_model(op="nope").application_components["T"])
    with pytest.raises(IntrinsicShapeMismatch, match="expects ports"):
        check_task_signature("t", _copy_model(ports=("src in float64 [64]", "z out float64 [64]"))
                             .application_components["T"])
    tm = builders.tile_task_model("tile_copy", {"src": "in float32 [64]", "dst": "out float32 [64]"}, {}, (16,))
    with pytest.raises(IntrinsicShapeMismatch, match="no tiler"):
        check_task_signature("t", tm.application_components["T"])
    cp = Tiler([0], [[4]], [[1]], [4])
    tm = builders.tile_task_model("tile_copy", {"src": "in float32 [64]", "dst": "out float32 [64]"},
                                  {"src": cp, "dst": cp}, (16,))
    assert check_task_signature("t", tm.application_components["T"]).tile
    ov = Tiler([0], [[2]], [[1]], [4])
    tm = builders.tile_task_model("tile_copy", {"src": "in float32 [64]", "dst": "out float32 [64]"},
                                  {"src": cp, "dst": ov}, (16,))
    with pytest.raises(IntrinsicShapeMismatch, match="injective"):
        check_task_signature("t", tm.application_components["T"])


def test_schedule_mirror():
    m = _copy_model()
    s = build_schedule(m, 3)
    (step,) = s.steps
    assert [(l.range.offset, l.range.count, l.global_size, l.local_size) for l in step.launches] == \
        [(0, 22, 24, 8), (22, 21, 24, 8), (43, 21, 24, 8)]


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference not present (GPU box)")
def test_reference_models_drive_the_mirror(monkeypatch):
    """A model parsed by the unmodified reference front-end is accepted by the host mirror."""
    import sys
    sys.dont_write_bytecode = True
    monkeypatch.syspath_prepend(str(REF_SRC))
    import gmodelc
    from paper_1105_4424_b200.model import connected_port_groups
    text = gmodelc.bundled_model_text()
    model = gmodelc.parse_model(text)
    for d in (1, 4):
        ref = gmodelc.build_schedule(model, d)
        mine = build_schedule(model, d)

        def flat(steps):
            out = []
            for s in steps:
                if hasattr(s, "launches"):
                    out.append(("D", s.task_path, s.op, tuple((l.device_index, l.range.offset, l.range.count,
                                                               l.global_size, l.local_size) for l in s.launches)))
                elif hasattr(s, "body"):
                    out.append(("L", s.task_path, s.tolerance, s.max_iterations, s.relres_port, tuple(flat(s.body))))
                else:
                    out.append(("H", s.task_path, s.op))
            return out
        assert flat(ref.steps) == flat(mine.steps)
    assert connected_port_groups(model) == gmodelc.metamodel.connected_port_groups(model)
    for comp in model.application_components.values():
        if comp.elementary_op:
            assert check_task_signature("x", comp).name == gmodelc.intrinsics.check_task_signature("x", comp).name
    reg = dict(gmodelc.intrinsics.INTRINSICS)
    from paper_1105_4424_b200 import register_into
    register_into(reg)
    assert "matmul" in reg and reg["copy"] is gmodelc.intrinsics.INTRINSICS["copy"]


def test_registry_has_reference_and_tile_ops():
    for op in ("spmv_csr", "dot_partial", "axpy", "scale", "copy", "sub", "div", "neg", "rel_residual",
               "tile_copy", "matmul", "tile_filter", "hfilter", "vfilter", "stencil", "tile_sum"):
        assert op in INTRINSICS


def test_model_json_roundtrip(golden):
    from paper_1105_4424_b200.model import model_from_dict, model_to_dict
    _, meta = golden
    d = meta["cg_k20"]["model"]
    m = model_from_dict(d)
    assert model_to_dict(m) == d
    s = build_schedule(m, 4)
    assert len(s.steps) == 4 and hasattr(s.steps[-1], "body") and len(s.steps[-1].body) == 12


def test_model_memo_per_object_and_evicted():
    """Derived per-model structures are computed once per model object and dropped with it."""
    import gc
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.model import _MODEL_MEMO, connected_port_groups, model_memo
    g = orc.gemm_tilers(8, 8, 4)
    mk = lambda: builders.tile_task_model(  # noqa: E731
        "matmul", {"a": "in float32 [8,4]", "b": "in float32 [4,8]", "c": "out float32 [8,8]"},
        {k: Tiler(v["origin"], v["paving"], v["fitting"], v["pattern"]) for k, v in g.items()}, (8, 8))
    m1, m2 = mk(), mk()
    calls = []
    assert model_memo(m1, "k", lambda m: calls.append(1) or 7) == 7
    assert model_memo(m1, "k", lambda m: calls.append(1) or 8) == 7
    assert model_memo(m2, "k", lambda m: calls.append(1) or 9) == 9
    assert len(calls) == 2
    assert connected_port_groups(m1) is connected_port_groups(m1)
    key = id(m1)
    assert key in _MODEL_MEMO
    del m1
    gc.collect()
    assert key not in _MODEL_MEMO


def test_config_builders_equal_the_oracle_tilers():
    """The package's config models (used by bench.py) carry the same tilers and weights as
    the oracle's independent restatement of SURVEY.md Appendix A."""
    import numpy as np
    from oracle import aol_oracle as orc
    from paper_1105_4424_b200 import builders

    def same(t, d):
        return (tuple(t.origin) == tuple(d["origin"]) and tuple(map(tuple, t.paving)) == tuple(map(tuple, d["paving"]))
                and tuple(map(tuple, t.fitting)) == tuple(map(tuple, d["fitting"]))
                and tuple(t.pattern) == tuple(d["pattern"]))
    for M, N, K in ((256, 256, 256), (13, 7, 5)):
        o = orc.gemm_tilers(M, N, K)
        assert all(same(builders.gemm_tilers(M, N, K)[k], o[k]) for k in "abc")
    o = orc.stencil_tilers(33, 45)
    assert all(same(builders.stencil_tilers(33, 45)[k], o[k]) for k in "xy")
    assert np.array_equal(builders.stencil_weights(), orc.stencil_weights())
    oh = orc.hfilter_tilers(2, 18, 64)
    th, rep, arr = builders.line_filter_tilers(2, 18, 64, 2, 13, 8, 3)
    assert all(same(th[k], oh[k]) for k in "xy") and rep == tuple(oh["x"]["rep"]) and arr == tuple(oh["y"]["array"])
    ov = orc.vfilter_tilers(2, 18, 24)
    tv, rep, arr = builders.line_filter_tilers(2, 18, 24, 1, 14, 9, 4)
    assert all(same(tv[k], ov[k]) for k in "xy") and rep == tuple(ov["x"]["rep"]) and arr == tuple(ov["y"]["array"])
    assert np.array_equal(builders.downscaler_weights(13, 3), orc.hfilter_weights())
    assert np.array_equal(builders.downscaler_weights(14, 4), orc.vfilter_weights())
    m = builders.downscaler_model(2, 18, 64)
    assert set(m.application_components) >= {"HT", "VT", "m"}


def test_launch_rejects_null_ports_without_gpu():
    """aol_launch refuses a null pointer in any port the op dereferences (AOL_EINVAL, nothing
    launched) -- checked before any CUDA call, so it runs here."""
    cp = dict(array=(100,), rep=(25,), pattern=(4,), origin=(0,), paving=((4,),), fitting=((1,),))
    t = _capi.make_task("tile_copy", "float32", [_bt(cp), _bt(cp)])
    with pytest.raises(_capi.AolError, match="null port 1"):
        _capi.launch(t, 0, 25, [0x1000, 0], (), 0)
    g = orc.gemm_tilers(64, 64, 32)
    mm = _capi.make_task("matmul", "float32", [_bt(g[k]) for k in "abc"])
    with pytest.raises(_capi.AolError, match="null port 0"):
        _capi.launch(mm, 0, 64 * 64, [0, 0x1000, 0x2000], (), 0)
    with pytest.raises(_capi.AolError, match="outside the repetition space"):
        _capi.launch(mm, 0, 64 * 64 + 1, [0x1000, 0x1000, 0x2000], (), 0)
