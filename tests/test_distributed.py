"""Multi-rank path on CPU: world size 2 over gloo (127.0.0.1), the oracle standing in for the kernels.

Checks the host logic of paper_1105_4424_b200.distributed: contiguous shards
per rank, the packed output-pattern exchange that makes a sharded output
whole (unequal shard sizes included), the ascending-device-order dot combine,
and the input hull a shard needs resident.
"""

import os
import socket

import numpy as np
import pytest

from oracle import aol_oracle as orc


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tdict(bt):
    t = bt.tiler
    return dict(array=bt.array, rep=bt.rep, pattern=t.pattern, origin=t.origin, paving=t.paving,
                fitting=t.fitting)


def _oracle_pack(array, bt, first, count):
    import torch
    offs = orc.tiler_offsets(_tdict(bt), first, count).ravel()
    return array[torch.from_numpy(offs)].clone()


def _oracle_unpack(array, bt, first, count, stream):
    import torch
    offs = orc.tiler_offsets(_tdict(bt), first, count).ravel()
    array[torch.from_numpy(offs)] = stream


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_1105_4424_b200 import Tiler
    from paper_1105_4424_b200.distributed import Exchange, combine_partials, gather_output, input_hull, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = Exchange()
        results = {}

        def tiler(d):
            return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"])

        # 1) toroidal stencil 33x45 (odd repetition total -> shards differ by one)
        t = orc.stencil_tilers(33, 45)
        w = orc.stencil_weights()
        x = np.random.default_rng(1).random(33 * 45).astype(np.float32)
        R = 33 * 45
        sh = shard(R, rank, world)
        y = np.zeros(R, np.float32)
        orc.tile_filter(x, w, y, t["x"], t["y"], sh.mine.offset, sh.mine.count)     # this rank's launch
        yt = torch.from_numpy(y)
        gather_output(yt, tiler(t["y"]).bind(t["y"]["array"], t["y"]["rep"]), sh, ex, _oracle_pack, _oracle_unpack)
        ref = orc.run_tile_task("stencil", t, {"x": x, "w": w}, {"y": (R, np.float32)}, R, 1)["y"]
        results["stencil"] = bool(np.array_equal(yt.numpy(), ref))

        # 2) matmul with unaligned row shards and a 2-D output tiler
        g = orc.gemm_tilers(13, 7, 5)
        a = np.random.default_rng(2).standard_normal(13 * 5).astype(np.float32)
        b = np.random.default_rng(3).standard_normal(5 * 7).astype(np.float32)
        sh = shard(13 * 7, rank, world)
        c = np.zeros(13 * 7, np.float32)
        orc.matmul(a, b, c, g["a"], g["b"], g["c"], sh.mine.offset, sh.mine.count)
        ct = torch.from_numpy(c)
        gather_output(ct, tiler(g["c"]).bind(g["c"]["array"], g["c"]["rep"]), sh, ex, _oracle_pack, _oracle_unpack)
        ref = orc.run_tile_task("matmul", g, {"a": a, "b": b}, {"c": (91, np.float32)}, 91, 1)["c"]
        results["matmul"] = bool(np.array_equal(ct.numpy(), ref))

        # 3) downscaler H filter: a 3-element output pattern per repetition
        th = orc.hfilter_tilers(2, 3, 64)
        xh = np.random.default_rng(4).random(2 * 3 * 64).astype(np.float32)
        Rh = int(np.prod(th["x"]["rep"]))
        ny = int(np.prod(th["y"]["array"]))
        sh = shard(Rh, rank, world)
        yh = np.zeros(ny, np.float32)
        orc.tile_filter(xh, orc.hfilter_weights(), yh, th["x"], th["y"], sh.mine.offset, sh.mine.count)
        yht = torch.from_numpy(yh)
        gather_output(yht, tiler(th["y"]).bind(th["y"]["array"], th["y"]["rep"]), sh, ex, _oracle_pack,
                      _oracle_unpack)
        ref = orc.run_tile_task("hfilter", th, {"x": xh, "w": orc.hfilter_weights()}, {"y": (ny, np.float32)},
                                Rh, 1)["y"]
        results["hfilter"] = bool(np.array_equal(yht.numpy(), ref))

        # 4) dot combine in ascending device order == the reference's simulated-device combine
        va = np.random.default_rng(5).standard_normal(1001)
        vb = np.random.default_rng(6).standard_normal(1001)
        sh = shard(1001, rank, world)
        part = float(np.dot(va[sh.mine.offset:sh.mine.offset + sh.mine.count],
                            vb[sh.mine.offset:sh.mine.offset + sh.mine.count]))
        tot = combine_partials(ex, part)
        arrays = {"a": va, "b": vb, "s": np.zeros(1)}
        orc.run_identity_op("dot_partial", arrays, orc.partition_equally(1001, world))
        results["dot"] = tot == arrays["s"][0]

        # 5) input hull of a row shard of A in a GEMM covers exactly the rows it reads
        g = orc.gemm_tilers(64, 32, 16)
        bt = tiler(g["a"]).bind(g["a"]["array"], g["a"]["rep"])
        sh = shard(64 * 32, rank, world)
        lo, hi = input_hull(bt, sh.mine.offset, sh.mine.count)
        offs = orc.tiler_offsets(g["a"], sh.mine.offset, sh.mine.count)
        results["hull"] = (lo == int(offs.min()) and hi == int(offs.max()) + 1)
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_exchange():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        rank, res = q.get(timeout=240)
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        for k, v in out[rank].items():
            assert v, (rank, k)


def test_input_hull_matches_offsets_single_process():
    from paper_1105_4424_b200 import Tiler
    from paper_1105_4424_b200.distributed import input_hull, shard
    rng = np.random.default_rng(9)
    for _ in range(30):
        M, N, K = (int(v) for v in rng.integers(2, 40, 3))
        g = orc.gemm_tilers(M, N, K)
        for key in ("a", "b"):
            d = g[key]
            bt = Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"]).bind(d["array"], d["rep"])
            for D in (1, 3, 5):
                s = shard(M * N, 0, D)
                for r in s.ranges:
                    lo, hi = input_hull(bt, r.offset, r.count)
                    offs = orc.tiler_offsets(d, r.offset, r.count)
                    assert lo <= offs.min() and hi >= offs.max() + 1
                    if key == "a":   # rows of A: the hull is exact
                        assert lo == offs.min() and hi == offs.max() + 1


def test_input_ranges_cover_toroidal_offsets():
    """Seam-split ranges of wrapping tilers cover every offset the index function produces,
    and stay small (a stencil chunk needs its rows plus the wrapped halo row only)."""
    from paper_1105_4424_b200 import Tiler
    from paper_1105_4424_b200.distributed import add_range, input_ranges, missing_ranges
    rng = np.random.default_rng(17)
    H, W = 64, 48
    t = orc.stencil_tilers(H, W)
    d = t["x"]
    bt = Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"]).bind(d["array"], d["rep"])
    for first, count in ((0, 8 * W), (5 * W + 3, 17 * W), ((H - 4) * W, 4 * W), (0, H * W), (7, 1)):
        rs = input_ranges(bt, first, count)
        offs = orc.tiler_offsets(d, first, count)
        covered = np.zeros(H * W, bool)
        for lo, hi in rs:
            covered[lo:hi] = True
        assert covered[offs].all()
        if count == 8 * W and first == 0:
            assert rs == [(0, 9 * W), ((H - 1) * W, H * W)]
    # random wrapping tilers
    for _ in range(40):
        arr = tuple(int(v) for v in rng.integers(3, 20, 2))
        rep = tuple(int(v) for v in rng.integers(1, 9, 2))
        d = dict(array=arr, rep=rep, pattern=(int(rng.integers(1, 4)),),
                 origin=tuple(int(v) for v in rng.integers(-30, 30, 2)),
                 paving=tuple(tuple(int(v) for v in rng.integers(-3, 4, 2)) for _ in range(2)),
                 fitting=tuple(tuple(int(v) for v in rng.integers(-2, 3, 1)) for _ in range(2)))
        bt = Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"]).bind(d["array"], d["rep"])
        R = int(np.prod(rep))
        first = int(rng.integers(0, R))
        count = int(rng.integers(1, R - first + 1))
        covered = np.zeros(int(np.prod(arr)), bool)
        for lo, hi in input_ranges(bt, first, count):
            covered[lo:hi] = True
        assert covered[orc.tiler_offsets(d, first, count)].all()
    assert missing_ranges([(0, 4), (10, 12)], 2, 14) == [(4, 10), (12, 14)]
    assert add_range([(0, 4), (10, 12)], 4, 10) == [(0, 12)]
