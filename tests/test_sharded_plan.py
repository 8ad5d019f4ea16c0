"""Host logic of sharded execution on CPU: the exchange plan (what crosses shards) and the
torch.distributed transport (world size 2 over gloo, 127.0.0.1) that carries it.

The plan is derived from the model alone (paper_1105_4424_b200.distributed.ShardPlan):
launch d of a step runs on rank d mod world (partition.py:105-121 ranges), a written
dense-stream range travels only to ranks whose later reads intersect it, non-dense output
tilers fall back to the packed-pattern all-gather, and dot partials are reduced slot-wise.
"""

import os
import socket

import numpy as np
import pytest

from _sharded_cases import CASES


def _plan(case, D, world=None, **kw):
    from paper_1105_4424_b200.distributed import ShardPlan
    from paper_1105_4424_b200.partition import build_schedule
    model, bind, out, ref = CASES[case](**kw)
    sched = build_schedule(model, D)
    return ShardPlan.for_model(model, sched, world or D), sched


def test_elementwise_chain_exchanges_nothing():
    plan, sched = _plan("elementwise", 2)
    for path, entries in plan.writes.items():
        for name, g, tr, wr in entries:
            assert tr == [], (path, name)
            assert [w for w, _, _ in wr] == [0, 1]


def test_matmul_output_has_no_readers():
    plan, _ = _plan("matmul", 4)
    (entries,) = plan.writes.values()
    assert entries[0][2] == []


@pytest.mark.parametrize("D", [2, 3, 4])
def test_stencil_chain_exchanges_halo_rows_only(D):
    H, W = 48, 80
    plan, sched = _plan("stencil_chain", D, H=H, W=W)
    tr = plan.writes["s1"][0][2]
    rows = {}
    for w, r, lo, hi in tr:
        assert (hi - lo) % W == 0 and lo % W == 0
        rows.setdefault((w, r), []).extend(range(lo // W, hi // W))
    ranges = [l.range for l in sched.steps[0].launches]
    for r, rg in enumerate(ranges):
        first_row, last_row = rg.offset // W, (rg.offset + rg.count) // W - 1
        want = {(first_row - 1) % H, (last_row + 1) % H}
        got = {row for (w, rr), rs in rows.items() if rr == r for row in rs}
        assert got == want, (r, got, want)
    assert plan.writes["s2"][0][2] == []             # the final output is only gathered to the root


def test_transpose_output_falls_back_to_pack():
    plan, _ = _plan("transpose_chain", 2)
    assert plan.writes["t"][0][2] is None
    assert plan.writes["s"][0][2] == []


def test_cg_plan_all_gathers_p_only(golden):
    """CG (the paper's case study): spmv gathers p whole, so p travels to every other rank --
    after init_p and after axpy_p, but not after scale_p, whose shards axpy_p rewrites on the
    same ranks before anyone reads them; r, x, ap are read only on the writer's own range
    (refexec.py:488-514)."""
    from paper_1105_4424_b200.distributed import ShardPlan
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    data, meta = golden
    model = model_from_dict(meta["cg_k20"]["model"])
    n = 400
    for D in (2, 4):
        plan = ShardPlan.for_model(model, build_schedule(model, D), D)
        moved = {path: sum(hi - lo for name, g, tr, wr in entries for _, _, lo, hi in (tr or []))
                 for path, entries in plan.writes.items()}
        assert moved == {"init_r": 0, "init_p": (D - 1) * n, "loop.spmv": 0, "loop.axpy_x": 0, "loop.axpy_r": 0,
                         "loop.scale_p": 0, "loop.axpy_p": (D - 1) * n}, moved


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_1105_4424_b200.distributed import DistTransport, Replica
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import types
        tr = DistTransport()
        n = 100
        arr = torch.full((n,), float(-1 - rank))
        arr[rank * 50:(rank + 1) * 50] = torch.arange(rank * 50, (rank + 1) * 50, dtype=torch.float32)
        rep = Replica(rank, torch.device("cpu"), types.SimpleNamespace(arrays={"g": arr}))
        # several transfers between the same pair in one batch, both directions
        moves = [(0, 1, 10, 20), (1, 0, 50, 55), (0, 1, 40, 50), (1, 0, 90, 100)]
        tr.move({rank: rep}, "g", moves)
        ok = True
        for w, r, lo, hi in moves:
            if r == rank:
                ok &= bool(torch.equal(arr[lo:hi], torch.arange(lo, hi, dtype=torch.float32)))
        # dot partials: slot k owned by rank k % world, zero elsewhere -> exact slot values
        buf = torch.zeros(5, dtype=torch.float64)
        for k in range(5):
            if k % world == rank:
                buf[k] = -0.1 * (k + 1) if k != 3 else -0.0
        rep.pbuf["k"] = buf
        tr.reduce_partials({rank: rep}, "k")
        ok &= buf.tolist()[:3] == [-0.1, -0.2, -0.30000000000000004] and buf[4].item() == -0.5
        sent = tr.bytes_moved
        # variable-size streams to the root only (the packed gather of a non-dense output)
        local = torch.arange(3 + 4 * rank, dtype=torch.float32) + 100 * rank
        got = tr.gather_v({rank: rep}, local, [3, 7], 0)
        if rank == 0:
            ok &= set(got) == {1} and torch.equal(got[1], torch.arange(7, dtype=torch.float32) + 100)
        else:
            ok &= got == {}
        q.put((rank, ok, sent))
    finally:
        dist.destroy_process_group()


def test_dist_transport_world2_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, ok, moved = q.get(timeout=240)
        res[rank] = (ok, moved)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] and res[1][0]
    assert res[0][1] == 20 * 4 and res[1][1] == 15 * 4      # each rank counts the bytes it sent


@pytest.mark.parametrize("D", [2, 3])
def test_downscaler_root_output_is_gathered_not_exchanged(D):
    """The V filter writes 4 rows per repetition (not a dense stream) and nothing reads it
    after: it is packed to the root at output time only (ROOT_GATHER), never all-gathered.
    At D=2 the H and V shards cover the same frames, so the intermediate does not travel; at
    D=3 the V shards straddle H shards and only the rows they read cross."""
    from paper_1105_4424_b200.distributed import ROOT_GATHER
    plan, sched = _plan("downscaler", D)
    (h,) = plan.writes["h"]
    (v,) = plan.writes["v"]
    if D == 2:
        assert h[2] == []
    else:
        assert h[2] and all(w != r for w, r, _, _ in h[2])
    assert v[2] == ROOT_GATHER
    assert plan.exchanged_bytes("v", {}) == 0


def test_transpose_chain_pack_is_kept_when_read_later():
    """A non-dense write that a later step reads still takes the packed all-gather."""
    from paper_1105_4424_b200.distributed import ROOT_GATHER
    plan, _ = _plan("transpose_chain", 3)
    assert plan.writes["t"][0][2] is None and plan.writes["t"][0][2] != ROOT_GATHER


def test_cg_plan_with_bound_matrix_exchanges_halos_only(golden):
    """With the matrix bound (and never rewritten), spmv's x reads are the columns its rows
    name (refexec.py:111-121): on the 20x20 Poisson grid a launch of whole grid rows reads
    one grid row (20 elements) beyond each end, so p moves 20 elements each way across each
    shard boundary instead of being all-gathered."""
    from paper_1105_4424_b200.distributed import ShardPlan
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    data, meta = golden
    model = model_from_dict(meta["cg_k20"]["model"])
    bind = {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}
    for D in (2, 4):
        plan = ShardPlan.for_model(model, build_schedule(model, D), D, bindings=bind)
        moved = {path: sum(hi - lo for name, g, tr, wr in entries for _, _, lo, hi in (tr or []))
                 for path, entries in plan.writes.items()}
        halo = 2 * 20 * (D - 1)
        assert moved == {"init_r": 0, "init_p": halo, "loop.spmv": 0, "loop.axpy_x": 0, "loop.axpy_r": 0,
                         "loop.scale_p": 0, "loop.axpy_p": halo}, moved
        # each rank's input hull of the matrix is its own rows' entries only
        g = plan.groups["colidx"]
        rp = bind["rowptr"]
        for r, rng in enumerate(plan.reads_by_rank[g]):
            lo, hi = 100 * 4 // D * r, 100 * 4 // D * (r + 1)
            assert rng == [(int(rp[lo]), int(rp[hi]))], (D, r, rng)


def test_fused_gather_candidates(golden):
    """Root outputs that only device steps write and no step reads are stored into the root's
    array by their producers (fused gather): matmul's C, the stencil chain's and downscaler's
    final outputs; not CG's x, which the loop body reads and updates."""
    from paper_1105_4424_b200.distributed import PlanHost, ShardPlan, fused_gather_candidates
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    for case, port in (("matmul", "p_c"), ("stencil_chain", "y"), ("downscaler", "y"), ("transpose_chain", "y")):
        model, bind, out, ref = CASES[case]()
        host = PlanHost(model, build_schedule(model, 2))
        plan = ShardPlan(host, 2)
        assert fused_gather_candidates(host, plan) == [host.storage.groups[out]], case
    data, meta = golden
    model = model_from_dict(meta["cg_k20"]["model"])
    host = PlanHost(model, build_schedule(model, 2))
    assert fused_gather_candidates(host, ShardPlan(host, 2)) == []
