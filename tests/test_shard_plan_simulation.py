"""The exchange plan (paper_1105_4424_b200.distributed.ShardPlan) simulated on CPU: random
chains of tile filters with toroidal windows and dense / non-dense output tilers run with
every rank holding its own copy of every array.  Rank r runs the launches d with
d mod world == r (partition.py:105-121) through the oracle, then exactly the plan's transfers
are applied (dense ranges writer -> reader; non-dense writes read later: the packed-pattern
all-gather; root outputs: gathered to rank 0 at the end).  Rank 0's outputs must equal the
single-copy oracle run bit for bit -- i.e. the plan never leaves a reader with a stale element
and never needs more than it sends.  No GPU: this checks the host logic multi-GPU correctness
rests on at world sizes the box cannot run (up to 8)."""

import numpy as np
import pytest

from oracle import aol_oracle as orc


def _tiler(d):
    from paper_1105_4424_b200 import Tiler
    return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"])


def _random_chain(rng, n_steps):
    H, W = int(rng.integers(6, 20)), int(rng.integers(6, 20))
    arr = (H, W)
    stages, tilers = [], []
    for k in range(n_steps):
        kh, kw = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        oh, ow = int(rng.integers(-2, 3)) % H, int(rng.integers(-2, 3)) % W
        tx = dict(array=arr, rep=arr, pattern=(kh, kw), origin=(oh, ow), paving=((1, 0), (0, 1)),
                  fitting=((1, 0), (0, 1)))
        kind = rng.choice(["dense", "rowrev", "colrev"])
        if kind == "dense":
            ty = dict(array=arr, rep=arr, pattern=(1,), origin=(0, 0), paving=((1, 0), (0, 1)), fitting=((0,), (0,)))
        elif kind == "rowrev":      # each row written right to left: not a dense stream in rho order
            ty = dict(array=arr, rep=arr, pattern=(1,), origin=(0, W - 1), paving=((1, 0), (0, -1)),
                      fitting=((0,), (0,)))
        else:                       # rows in reverse order
            ty = dict(array=arr, rep=arr, pattern=(1,), origin=(H - 1, 0), paving=((-1, 0), (0, 1)),
                      fitting=((0,), (0,)))
        w = (rng.integers(1, 5, size=kh * kw) / 8.0).astype(np.float64)
        tilers.append((tx, ty, w))
        spec = f"float64 [{H},{W}]"
        stages.append((f"f{k}", "tile_filter", {"x": f"in {spec}", "w": f"in float64 [{kh * kw}]", "y": f"out {spec}"},
                       {"x": _tiler(tx), "y": _tiler(ty)}, arr))
    return arr, stages, tilers


def _model(arr, stages):
    from paper_1105_4424_b200 import builders
    H, W = arr
    spec = f"float64 [{H},{W}]"
    root_in = {"x": f"in {spec}"}
    links = [("x", "f0.x")]
    for k, st in enumerate(stages):
        root_in[f"w{k}"] = f"in float64 [{len(st[2]) and st[2]['w'].split('[')[1].rstrip(']')}]"
        links.append((f"w{k}", f"f{k}.w"))
        if k + 1 < len(stages):
            links.append((f"f{k}.y", f"f{k + 1}.x"))
    links.append((f"f{len(stages) - 1}.y", "y"))
    return builders.chain_model(stages, root_in, {"y": f"out {spec}"}, links)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_plan_transfers_suffice(seed, world):
    from paper_1105_4424_b200.distributed import ROOT_GATHER, PlanHost, ShardPlan, rank_of
    from paper_1105_4424_b200.partition import build_schedule
    rng = np.random.default_rng(1000 * world + seed)
    arr, stages, tilers = _random_chain(rng, int(rng.integers(2, 4)))
    model = _model(arr, stages)
    D = world + int(rng.integers(0, 3))           # more launches than ranks: d -> rank d mod world
    sched = build_schedule(model, D)
    host = PlanHost(model, sched)
    plan = ShardPlan(host, world)
    n = arr[0] * arr[1]
    x = rng.random(n)

    # single-copy oracle
    ref = x.copy()
    for tx, ty, w in tilers:
        y = np.zeros(n)
        orc.tile_filter(ref, w, y, tx, ty, 0, n)
        ref = y

    # per-rank copies; group of each task port -> the rank's array
    groups = host.storage.groups
    copies = [{} for _ in range(world)]

    def arr_of(r, node):
        g = groups[node]
        if g not in copies[r]:
            copies[r][g] = x.copy() if "x" in g else np.zeros(n)
        return copies[r][g]

    pending = []                                    # (written group, [(rank, first, count)], ty)
    for k, step in enumerate(sched.device_steps()):
        tx, ty, w = tilers[k]
        path = step.task_path
        for l in step.launches:
            r = rank_of(l.device_index, world)
            orc.tile_filter(arr_of(r, f"{path}.x"), w, arr_of(r, f"{path}.y"), tx, ty, l.range.offset, l.range.count)
        for name, g, tr, wr in plan.writes.get(path, []):
            if tr is None or tr == ROOT_GATHER:
                mine = [(rank_of(l.device_index, world), l.range.offset, l.range.count) for l in step.launches]
                if tr is None:                      # packed-pattern all-gather now
                    for w_, f, c in mine:
                        offs = orc.tiler_offsets(ty, f, c).ravel()
                        for r in range(world):
                            if r != w_:
                                arr_of(r, f"{path}.y")[offs] = arr_of(w_, f"{path}.y")[offs]
                else:
                    pending.append((f"{path}.y", mine, ty))
                continue
            for w_, r, lo, hi in tr:
                arr_of(r, f"{path}.y")[lo:hi] = arr_of(w_, f"{path}.y")[lo:hi]
            if path == sched.device_steps()[-1].task_path:      # dense root output: gather what others wrote
                for w_, lo, hi in wr:
                    if w_ != 0:
                        arr_of(0, f"{path}.y")[lo:hi] = arr_of(w_, f"{path}.y")[lo:hi]
    for node, mine, ty in pending:
        for w_, f, c in mine:
            if w_ != 0:
                offs = orc.tiler_offsets(ty, f, c).ravel()
                arr_of(0, node)[offs] = arr_of(w_, node)[offs]
    got = arr_of(0, f"{sched.device_steps()[-1].task_path}.y")
    assert np.array_equal(got, ref), (seed, world, D)
