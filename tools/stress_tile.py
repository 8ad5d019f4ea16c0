"""Random STRUCTURED tile tasks (the shapes the specialised plans take: dense / gapped /
overlapping / strided / row-stride copies, 2-D crops and toroidal shifts, K x K toroidal
stencils, row and column line filters, box pools, row / column sums), random sizes, origins,
shard counts D = 1..8 and dtypes, each compared bit for bit with the oracle.  Prints the plan
mix; exits non-zero on the first mismatch or error with the case printed.

    SEED=1 CASES=400 python tools/stress_tile.py"""
import collections
import os
import sys
import traceback
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from oracle import aol_oracle as orc  # noqa: E402
from paper_1105_4424_b200 import Tiler, _capi, builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor, execute_schedule  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
N_CASES = int(os.environ.get("CASES", "400"))


def spec(d, direction, dt):
    return f"{direction} {dt} [{','.join(str(x) for x in d['array'])}]"


def dense_out(rep, pat):
    R, P = int(np.prod(rep)), int(np.prod(pat))
    q = len(rep)
    return dict(array=(R * P,), rep=rep, pattern=pat, origin=(0,),
                paving=(tuple(int(np.prod(rep[j + 1:])) * P for j in range(q)),),
                fitting=(tuple(int(np.prod(pat[k + 1:])) for k in range(len(pat))),))


def t(d):
    return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"])


def case_copy(dt):
    kind = rng.choice(["dense", "gaps", "overlap", "strided", "rowstride", "crop", "shift"])
    m = int(rng.choice([1, 2, 3, 4, 8, 16, 32, 64]))
    T = int(rng.integers(1, 200000))
    if kind == "rowstride":
        src = dict(array=(m, T), rep=(T,), pattern=(m,), origin=(0, 0), paving=((0,), (1,)), fitting=((1,), (0,)))
    elif kind in ("crop", "shift"):
        H, W = int(rng.integers(2, 700)), int(rng.integers(2, 900))
        h, w = (int(rng.integers(1, H + 1)), int(rng.integers(1, W + 1))) if kind == "crop" else (H, W)
        oh, ow = int(rng.integers(0, H)), int(rng.integers(0, W))
        if kind == "crop":
            oh, ow = min(oh, H - h), min(ow, W - w)
        src = dict(array=(H, W), rep=(h, w), pattern=(1,), origin=(oh, ow), paving=((1, 0), (0, 1)),
                   fitting=((0,), (0,)))
        return "tile_copy", {"src": src, "dst": dense_out((h, w), (1,))}, None
    else:
        p = {"dense": m, "overlap": max(1, m // 2), "gaps": 2 * m, "strided": 2 * m}[kind]
        f = 2 if kind == "strided" else 1
        span = (T - 1) * p + (m - 1) * f + 1 + int(rng.integers(0, 5))
        src = dict(array=(span,), rep=(T,), pattern=(m,), origin=(int(rng.integers(0, 3)) if kind != "dense" else 0,),
                   paving=((p,),), fitting=((f,),))
    return "tile_copy", {"src": src, "dst": dense_out(src["rep"], src["pattern"])}, None


def case_stencil(dt):
    H, W = int(rng.integers(3, 600)), int(rng.integers(3, 900))
    k = int(rng.choice([3, 5, 7]))
    x = dict(array=(H, W), rep=(H, W), pattern=(k, k), origin=(H - k // 2, W - k // 2), paving=((1, 0), (0, 1)),
             fitting=((1, 0), (0, 1)))
    y = dict(array=(H, W), rep=(H, W), pattern=(1,), origin=(0, 0), paving=((1, 0), (0, 1)), fitting=((0,), (0,)))
    w = (rng.integers(1, 5, k * k) / 16.0)
    return "stencil", {"x": x, "y": y}, w


def case_line(dt):
    F, H = int(rng.integers(1, 4)), int(rng.integers(1, 120))
    taps, step, outs = rng.choice([(13, 8, 3), (14, 9, 4), (8, 4, 2), (16, 8, 1), (7, 3, 1)])
    along_rows = bool(rng.integers(0, 2))
    if along_rows:
        W = int(step) * int(rng.integers(1, 120))
        rep = (F, H, W // step)
        x = dict(array=(F, H, W), rep=rep, pattern=(int(taps),), origin=(0, 0, 0),
                 paving=((1, 0, 0), (0, 1, 0), (0, 0, int(step))), fitting=((0,), (0,), (1,)))
        y = dict(array=(F, H, (W // step) * int(outs)), rep=rep, pattern=(int(outs),), origin=(0, 0, 0),
                 paving=((1, 0, 0), (0, 1, 0), (0, 0, int(outs))), fitting=((0,), (0,), (1,)))
    else:
        Hh = int(step) * int(rng.integers(1, 60))
        W = int(rng.integers(1, 700))
        rep = (F, Hh // step, W)
        x = dict(array=(F, Hh, W), rep=rep, pattern=(int(taps),), origin=(0, 0, 0),
                 paving=((1, 0, 0), (0, int(step), 0), (0, 0, 1)), fitting=((0,), (1,), (0,)))
        y = dict(array=(F, (Hh // step) * int(outs), W), rep=rep, pattern=(int(outs),), origin=(0, 0, 0),
                 paving=((1, 0, 0), (0, int(outs), 0), (0, 0, 1)), fitting=((0,), (1,), (0,)))
    w = rng.integers(1, 9, int(taps) * int(outs)) / 32.0
    return "tile_filter", {"x": x, "y": y}, w


def case_pool(dt):
    kh, kw = int(rng.choice([2, 3, 4])), int(rng.choice([2, 3, 4]))
    H, W = kh * int(rng.integers(1, 300)), kw * int(rng.integers(1, 300))
    rep = (H // kh, W // kw)
    x = dict(array=(H, W), rep=rep, pattern=(kh, kw), origin=(0, 0), paving=((kh, 0), (0, kw)),
             fitting=((1, 0), (0, 1)))
    y = dense_out(rep, (1,))
    w = np.full(kh * kw, 1.0 / (kh * kw) if (kh * kw) & (kh * kw - 1) == 0 else 0.25)
    return "tile_filter", {"x": x, "y": y}, w


def case_sum(dt):
    H, W = int(rng.integers(1, 900)), int(rng.integers(1, 1500))
    if rng.integers(0, 2):
        x = dict(array=(H, W), rep=(H,), pattern=(W,), origin=(0, 0), paving=((1,), (0,)), fitting=((0,), (1,)))
    else:
        x = dict(array=(H, W), rep=(W,), pattern=(H,), origin=(0, 0), paving=((0,), (1,)), fitting=((1,), (0,)))
    return "tile_sum", {"x": x, "s": dense_out(x["rep"], (1,))}, None


FAMILIES = [case_copy, case_copy, case_stencil, case_line, case_pool, case_sum]
plans = collections.Counter()
for case in range(N_CASES):
    fam = FAMILIES[int(rng.integers(0, len(FAMILIES)))]
    dt = "float32" if rng.random() < 0.8 else "float64"
    npdt = np.float32 if dt == "float32" else np.float64
    op, tl, w = fam(dt)
    D = int(rng.integers(1, 9))
    names = {"tile_copy": ("src", "dst"), "stencil": ("x", "y"), "tile_filter": ("x", "y"), "tile_sum": ("x", "s")}[op]
    ti, to = tl[names[0]], tl[names[1]]
    R = int(np.prod(ti["rep"]))
    nx = int(np.prod(ti["array"]))
    x = (np.arange(nx) % 4093).astype(npdt) if op == "tile_copy" else rng.random(nx).astype(npdt)
    ports = {names[0]: spec(ti, "in", dt), names[1]: spec(to, "out", dt)}
    inputs = {names[0]: x}
    if w is not None:
        w = np.asarray(w, dtype=npdt)
        ports["w"] = f"in {dt} [{w.size}]"
        inputs["w"] = w
    model = builders.tile_task_model(op, ports, {k: t(v) for k, v in tl.items()}, ti["rep"])
    nout = int(np.prod(to["array"]))
    try:
        sched = build_schedule(model, D)
        ex = Executor(model, sched, {f"p_{k}": v for k, v in inputs.items()}, D)
        tk = ex.task(sched.device_steps()[0].task_path)
        l0 = sched.device_steps()[0].launches[0]
        ptrs = [ex.storage.array(tk.nodes[p]).data_ptr() for p in tk.port_order]
        plans[_capi.plan_name(tk.ctask, l0.range.offset, l0.range.count, ptrs)] += 1
        ex.run()
        got = ex.outputs()[f"p_{names[1]}"]
        oracle_op = "tile_filter" if op == "stencil" else op
        ref = orc.run_tile_task(oracle_op, tl, inputs, {names[1]: (nout, npdt)}, R, D)[names[1]]
        ok = np.array_equal(got.view(np.uint8), ref.view(np.uint8))
        if ok and rng.random() < 0.4:            # the streamed path (chunked H2D / launch / D2H)
            pipe = int(rng.integers(2, 10))
            res = execute_schedule(model, sched, {f"p_{k}": v for k, v in inputs.items()}, D, pipeline=pipe)
            ok = np.array_equal(res.outputs[f"p_{names[1]}"].view(np.uint8), ref.view(np.uint8))
            plans["(streamed)"] += 1
    except Exception:
        traceback.print_exc()
        ok = False
    if not ok:
        print(f"FAIL case {case}: op={op} D={D} dtype={dt} tilers={tl}", flush=True)
        sys.exit(1)
    if case % 50 == 49:
        print(f"{case + 1} cases ok", flush=True)
print("all ok; plans:", dict(plans))
