"""The CPU oracle against the UNMODIFIED reference executor's outputs (tests/golden/make_golden.py).

Pins the oracle before it is trusted as the checker of the CUDA path.
"""

import numpy as np
import pytest

from oracle import aol_oracle as orc


def _cases(meta, op_prefixes):
    return sorted(k for k, v in meta.items() if not k.startswith("_")
                  and not k.startswith("ident_") and v["op"] in op_prefixes)


def test_partition_known_answers(golden):
    _, meta = golden
    for key, ranges in meta["_partition"].items():
        t, d = map(int, key.split(","))
        assert [list(r) for r in orc.partition_equally(t, d)] == ranges


def test_tiler_vectorised_equals_loop(golden):
    _, meta = golden
    for name in _cases(meta, {"tile_copy", "matmul", "tile_filter", "hfilter", "vfilter",
                              "stencil", "tile_sum"}):
        for t in meta[name]["tilers"].values():
            rep = int(np.prod(t["rep"]))
            n = min(rep, 300)
            assert np.array_equal(orc.tiler_offsets(t, 0, n), np.array(orc.tiler_offsets_loop(t, 0, n)))
            lo = rep - n
            assert np.array_equal(orc.tiler_offsets(t, lo, n), np.array(orc.tiler_offsets_loop(t, lo, n)))


@pytest.mark.parametrize("kind", ["tile_copy", "matmul", "filter", "tile_sum"])
def test_oracle_matches_reference_bitwise(golden, kind):
    data, meta = golden
    ops = {"filter": {"tile_filter", "hfilter", "vfilter", "stencil"}}.get(kind, {kind})
    names = _cases(meta, ops)
    assert names
    for name in names:
        m = meta[name]
        t = m["tilers"]
        ref = data[f"{name}/out"]
        if m["op"] == "tile_copy":
            ins = {"src": data[f"{name}/src"]}
            outs = {"dst": (ref.size, ref.dtype)}
            rep = int(np.prod(t["src"]["rep"]))
        elif m["op"] == "matmul":
            ins = {"a": data[f"{name}/a"], "b": data[f"{name}/b"]}
            outs = {"c": (ref.size, ref.dtype)}
            rep = int(np.prod(t["c"]["rep"]))
        elif m["op"] == "tile_sum":
            ins = {"x": data[f"{name}/x"]}
            outs = {"s": (ref.size, ref.dtype)}
            rep = int(np.prod(t["x"]["rep"]))
        else:
            ins = {"x": data[f"{name}/x"], "w": data[f"{name}/w"]}
            outs = {"y": (ref.size, ref.dtype)}
            rep = int(np.prod(t["x"]["rep"]))
        for d in (1, m["devices"], 7):
            got = orc.run_tile_task(m["op"], t, ins, outs, rep, d)
            out = next(iter(got.values()))
            assert out.dtype == ref.dtype
            assert np.array_equal(out.view(np.uint32), ref.view(np.uint32)), (name, d)


def test_c1_matmul_is_kahan_free_k_ascending(golden):
    """C1 via the reference equals the plain fp32 k-ascending loop, and is close to fp64."""
    data, _ = golden
    a = data["matmul_c1_256/a"].reshape(256, 256)
    b = data["matmul_c1_256/b"].reshape(256, 256)
    c = data["matmul_c1_256/out"].reshape(256, 256)
    acc = np.zeros((256, 256), np.float32)
    for k in range(256):
        acc += a[:, k:k + 1] * b[k:k + 1, :]
    assert np.array_equal(acc, c)
    c64 = a.astype(np.float64) @ b.astype(np.float64)
    assert np.linalg.norm(c - c64) / np.linalg.norm(c64) < 1e-6


def test_identity_ops_match_reference(golden):
    data, meta = golden
    for key in sorted(k for k in meta if k.startswith("ident_")):
        m = meta[key]
        ref = data[f"{key}/out"]
        if m["op"] == "spmv_csr":
            y = np.zeros(m["n"])
            for lo, n in orc.partition_equally(m["n"], m["devices"]):
                orc.spmv_rows(data[f"{key}/rowptr"], data[f"{key}/colidx"], data[f"{key}/values"],
                              data[f"{key}/x"], y, lo, lo + n)
            assert np.array_equal(y, ref), key
            continue
        op, n, dt = m["op"], m["n"], m["dtype"]
        ins = {b: data[f"{key}/in_{b}"] for b in m["bind"]}
        names = {"copy": (["src"], "dst"), "sub": (["x", "y"], "z"), "scale": (["y", "a"], "y"),
                 "axpy": (["y", "x", "a"], "y"), "dot_partial": (["a", "b"], "s")}[op]
        arrays = {p: ins[b].copy() for p, b in zip(names[0], m["bind"])}
        outn = names[1]
        if outn not in arrays:
            arrays[outn] = np.zeros(1 if op == "dot_partial" else n, dtype=dt)
        orc.run_identity_op(op, arrays, orc.partition_equally(n, m["devices"]))
        if op == "dot_partial":
            assert abs(arrays["s"][0] - ref[0]) <= 1e-12 * max(1.0, abs(ref[0])) * (1e5 if dt == "float32" else 1)
        else:
            assert np.array_equal(arrays[outn], ref), key


def test_c_oracle_matches_numpy_oracle_and_reference(golden):
    """The C restatement (bench CPU baseline, big checks) agrees bit for bit with the pinned numpy oracle."""
    from oracle import c_oracle as co
    data, meta = golden
    for name in _cases(meta, {"tile_copy", "matmul", "tile_filter", "hfilter", "vfilter", "stencil"}):
        m = meta[name]
        t = m["tilers"]
        ref = data[f"{name}/out"]
        for tl in t.values():
            R = int(np.prod(tl["rep"]))
            assert np.array_equal(co.tiler_offsets(tl, 0, R), orc.tiler_offsets(tl, 0, R))
        out = np.zeros_like(ref)
        if m["op"] == "tile_copy":
            R = int(np.prod(t["src"]["rep"]))
            co.tile_copy(data[f"{name}/src"], out, t["src"], t["dst"], 0, R)
        elif m["op"] == "matmul":
            R = int(np.prod(t["c"]["rep"]))
            co.matmul(data[f"{name}/a"], data[f"{name}/b"], out, t["a"], t["b"], t["c"], 0, R)
        else:
            R = int(np.prod(t["x"]["rep"]))
            co.tile_filter(data[f"{name}/x"], data[f"{name}/w"], out, t["x"], t["y"], 0, R)
        assert np.array_equal(out.view(np.uint32), ref.view(np.uint32)), name
    a = data["matmul_c1_256/a"]
    b = data["matmul_c1_256/b"]
    c = np.zeros(256 * 256, np.float32)
    co.gemm_rows(a, b, c, 256, 256, 0, 256)
    assert np.array_equal(c, data["matmul_c1_256/out"])
    x = data["stencil_32x48/x"]
    y = np.zeros_like(x)
    co.stencil_rows(x, data["stencil_32x48/w"], y, 32, 48, 0, 32)
    assert np.array_equal(y, data["stencil_32x48/out"])


def test_fullsize_stencil_row_restatement_equals_c_oracle():
    """tests/test_gpu_fullsize.py checks a 2.4e9-element torus on sampled rows with a numpy
    restatement (`_stencil_rows_np`); pin it to the C oracle's stencil_rows on a small torus,
    including the wrap rows and columns."""
    from pathlib import Path
    from oracle import c_oracle as co
    path = Path(__file__).resolve().parent / "test_gpu_fullsize.py"
    src = path.read_text()
    ns = {}
    exec(src[src.index("def _stencil_rows_np"):], {"np": np}, ns)
    H, W = 37, 52
    x = np.random.default_rng(2).standard_normal(H * W).astype(np.float32)
    w = orc.stencil_weights()
    want = np.zeros(H * W, np.float32)
    co.stencil_rows(x, w, want, H, W, 0, H)
    got = ns["_stencil_rows_np"](x, w, H, W, 0, H)
    assert np.array_equal(got.ravel().view(np.uint32), want.view(np.uint32))
