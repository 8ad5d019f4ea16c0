"""Models + bindings + oracle answers shared by the sharded-execution tests (CPU and GPU).

Each case returns (model, bindings, output port, oracle result) at a size the oracle
finishes in well under a second.  Used by tests/test_gpu_sharded.py (replicas in one
process and two torch.distributed ranks sharing cuda:0) and tests/test_sharded_plan.py.
"""

import numpy as np

from oracle import aol_oracle as orc


def _tiler(d):
    from paper_1105_4424_b200 import Tiler
    return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"])


def _spec(d, direction, dtype="float32"):
    return f"{direction} {dtype} [{','.join(str(x) for x in d['array'])}]"


def matmul_case(M=200, N=136, K=72, seed=2):
    """C1-style GEMM with unaligned row shards; precision='exact' gives the oracle's order."""
    from paper_1105_4424_b200 import builders
    g = orc.gemm_tilers(M, N, K)
    model = builders.tile_task_model(
        "matmul", {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]", "c": f"out float32 [{M},{N}]"},
        {k: _tiler(v) for k, v in g.items()}, (M, N))
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(M * K).astype(np.float32)
    b = rng.standard_normal(K * N).astype(np.float32)
    ref = orc.run_tile_task("matmul", g, {"a": a, "b": b}, {"c": (M * N, np.float32)}, M * N, 1)["c"]
    return model, {"p_a": a, "p_b": b}, "p_c", ref


def stencil_chain_case(H=48, W=80, seed=5):
    """Two toroidal 3x3 stencils back to back: the second reads the first's output one row
    across every shard seam (and across the torus wrap), so the exchange is exercised."""
    from paper_1105_4424_b200 import builders
    t = orc.stencil_tilers(H, W)
    w = orc.stencil_weights()
    tl = {k: _tiler(v) for k, v in t.items()}
    model = builders.chain_model(
        [("s1", "stencil", {"x": _spec(t["x"], "in"), "w": "in float32 [9]", "y": _spec(t["y"], "out")}, tl, (H, W)),
         ("s2", "stencil", {"x": _spec(t["x"], "in"), "w": "in float32 [9]", "y": _spec(t["y"], "out")}, tl, (H, W))],
        {"x": _spec(t["x"], "in"), "w": "in float32 [9]"}, {"y": _spec(t["y"], "out")},
        [("x", "s1.x"), ("w", "s1.w"), ("s1.y", "s2.x"), ("w", "s2.w"), ("s2.y", "y")])
    x = np.random.default_rng(seed).random(H * W).astype(np.float32)
    mid = orc.run_tile_task("stencil", t, {"x": x, "w": w}, {"y": (H * W, np.float32)}, H * W, 1)["y"]
    ref = orc.run_tile_task("stencil", t, {"x": mid, "w": w}, {"y": (H * W, np.float32)}, H * W, 1)["y"]
    return model, {"x": x, "w": w}, "y", ref


def downscaler_case(F=2, H=36, W=128, seed=8):
    from paper_1105_4424_b200 import builders
    th = orc.hfilter_tilers(F, H, W)
    Wo = th["y"]["array"][2]
    tv = orc.vfilter_tilers(F, H, Wo)
    wh, wv = orc.hfilter_weights(), orc.vfilter_weights()
    model = builders.chain_model(
        [("h", "hfilter", {"x": _spec(th["x"], "in"), "w": f"in float32 [{wh.size}]", "y": _spec(th["y"], "out")},
          {k: _tiler(v) for k, v in th.items()}, th["x"]["rep"]),
         ("v", "vfilter", {"x": _spec(tv["x"], "in"), "w": f"in float32 [{wv.size}]", "y": _spec(tv["y"], "out")},
          {k: _tiler(v) for k, v in tv.items()}, tv["x"]["rep"])],
        {"x": _spec(th["x"], "in"), "wh": f"in float32 [{wh.size}]", "wv": f"in float32 [{wv.size}]"},
        {"y": _spec(tv["y"], "out")},
        [("x", "h.x"), ("wh", "h.w"), ("h.y", "v.x"), ("wv", "v.w"), ("v.y", "y")])
    x = np.random.default_rng(seed).random(F * H * W).astype(np.float32)
    mid = orc.run_tile_task("hfilter", th, {"x": x, "w": wh}, {"y": (F * H * Wo, np.float32)},
                            int(np.prod(th["x"]["rep"])), 1)["y"]
    ny = int(np.prod(tv["y"]["array"]))
    ref = orc.run_tile_task("vfilter", tv, {"x": mid, "w": wv}, {"y": (ny, np.float32)},
                            int(np.prod(tv["x"]["rep"])), 1)["y"]
    return model, {"x": x, "wh": wh, "wv": wv}, "y", ref


def transpose_chain_case(R=24, C=40, seed=3):
    """tile_copy transposing into a non-dense output tiler, then a dense copy of the result:
    the first step's output has no dense-stream form, so the packed-pattern all-gather runs."""
    from paper_1105_4424_b200 import Tiler, builders
    # step 1: rep [R, C]; src[r, c] -> dst[c, r]  (dst written with stride R: not a dense stream)
    t1s = Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,))
    t1d = Tiler((0, 0), ((0, 1), (1, 0)), ((0,), (0,)), (1,))
    # step 2: rep [C*R] dense copy of the transposed array, shifted by 5 (reads across shards)
    t2s = Tiler((5,), ((1,),), ((0,),), (1,))
    t2d = Tiler((0,), ((1,),), ((0,),), (1,))
    n = R * C
    model = builders.chain_model(
        [("t", "tile_copy", {"src": f"in float32 [{R},{C}]", "dst": f"out float32 [{C},{R}]"},
          {"src": t1s, "dst": t1d}, (R, C)),
         ("s", "tile_copy", {"src": f"in float32 [{n}]", "dst": f"out float32 [{n}]"},
          {"src": t2s, "dst": t2d}, (n,))],
        {"x": f"in float32 [{R},{C}]"}, {"y": f"out float32 [{n}]"},
        [("x", "t.src"), ("t.dst", "s.src"), ("s.dst", "y")])
    x = (np.random.default_rng(seed).permutation(n) + 1).astype(np.float32)
    ref = np.roll(x.reshape(R, C).T.ravel(), -5)
    return model, {"x": x}, "y", ref


def elementwise_chain_case(n=9001, seed=4):
    """copy -> scale -> axpy on identity tilers: every rank reads only what it wrote, so the
    plan exchanges nothing; the final output is gathered to the root once."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.model import (AllocationLink, AllocKind, Component, ComponentKind, Connector,
                                            Model, PartInstance, Shape)
    A = ComponentKind.APPLICATION
    p = builders.port
    comps = {
        "C": Component("C", A, ports=(p(f"src in float64 [{n}]"), p(f"dst out float64 [{n}]")),
                       repetition_space=Shape((n,)), elementary_op="copy"),
        "S": Component("S", A, ports=(p(f"y inout float64 [{n}]"), p("a in float64 [1]")),
                       repetition_space=Shape((n,)), elementary_op="scale"),
        "X": Component("X", A, ports=(p(f"y inout float64 [{n}]"), p(f"x in float64 [{n}]"), p("a in float64 [1]")),
                       repetition_space=Shape((n,)), elementary_op="axpy"),
    }
    comps["m"] = Component("m", A, ports=(p(f"i in float64 [{n}]"), p(f"v in float64 [{n}]"), p("s in float64 [1]"),
                                          p(f"o out float64 [{n}]")),
                           parts=(PartInstance("c", "C"), PartInstance("k", "S"), PartInstance("x", "X")),
                           connectors=tuple(Connector(a, b) for a, b in (
                               ("i", "c.src"), ("c.dst", "k.y"), ("s", "k.a"), ("k.y", "x.y"), ("v", "x.x"),
                               ("s", "x.a"), ("x.y", "o"))))
    allocs = [AllocationLink(AllocKind.DATA, d, "dev.gmem") for d in ("i", "v", "c.dst")]
    allocs += [AllocationLink(AllocKind.DATA, "s", "host.ram")]
    allocs += [AllocationLink(AllocKind.TASK, t, "dev.cu") for t in ("c", "k", "x")]
    model = Model(platform_components=builders.platform(), application_components=comps, platform_root="p",
                  application_root="m", allocations=tuple(allocs))
    rng = np.random.default_rng(seed)
    i, v, s = rng.standard_normal(n), rng.standard_normal(n), np.array([0.625])
    ref = i * 0.625
    ref = ref + 0.625 * v
    return model, {"i": i, "v": v, "s": s}, "o", ref


CASES = {"matmul": matmul_case, "stencil_chain": stencil_chain_case, "downscaler": downscaler_case,
         "transpose_chain": transpose_chain_case, "elementwise": elementwise_chain_case}


def fir_model(n=16384, taps=7, memory="dev.gmem"):
    """1-D FIR (tile_filter, rep [n], pattern [taps], torus origin) whose input array is allocated
    onto ``memory``: "dev.gmem" (deviceGlobal) or "dev.cu.lmem" (deviceLocal, 227 KB capacity)."""
    import dataclasses
    from paper_1105_4424_b200 import Tiler, builders
    tx = Tiler((n - taps // 2,), ((1,),), ((1,),), (taps,))
    ty = Tiler((0,), ((1,),), ((0,),), (1,))
    model = builders.single_task_model(
        "tile_filter", [f"x in float32 [{n}]", f"w in float32 [{taps}]", f"y out float32 [{n}]"],
        [f"p_x in float32 [{n}]", f"p_w in float32 [{taps}]", f"p_y out float32 [{n}]"],
        ["p_x -> t.x", "p_w -> t.w", "t.y -> p_y"],
        [f"allocate data p_x onto {memory}", "allocate data p_w onto dev.gmem",
         "allocate data t.y onto dev.gmem", "allocate task t onto dev.cu"],
        repeat=(n,), tilers={"x": tx, "y": ty})
    model = dataclasses.replace(model, platform_components=builders.platform(local_capacity=227 * 1024))
    rng = np.random.default_rng(taps)
    x = rng.random(n).astype(np.float32)
    w = (rng.integers(1, 8, taps) / 8).astype(np.float32)
    d = lambda t, arr: dict(array=arr, rep=(n,), pattern=tuple(t.pattern), origin=tuple(t.origin),  # noqa: E731
                            paving=tuple(map(tuple, t.paving)), fitting=tuple(map(tuple, t.fitting)))
    ref = np.zeros(n, np.float32)
    orc.tile_filter(x, w, ref, d(tx, (n,)), d(ty, (n,)), 0, n)
    return model, {"p_x": x, "p_w": w}, "p_y", ref
