"""The paper's CG case study through the exchange plan, simulated on CPU with one array copy
per rank (launch d on rank d mod world): elementwise ops and spmv run per rank through the
oracle's restatement of refexec.py:111-121 / :488-514, dot partials are combined in ascending
launch order on every rank (refexec.py:478-487), host scalar ops run on every rank
(refexec.py:462-474), and after every device step exactly the plan's transfers are applied.
Inputs are uploaded only inside each rank's hull (ShardPlan.reads_by_rank, with the matrix
bound so spmv's reads are data-aware halos); everything outside a hull starts as NaN, so a
read the plan did not provide poisons the result.  Rank 0's x must equal the UNMODIFIED
reference executor's golden x at D launches bit for bit, with the same iteration count."""

import math

import numpy as np
import pytest

from oracle import aol_oracle as orc


def _simulate(model, sched, bind, world, plan, host):
    from paper_1105_4424_b200.distributed import ROOT_GATHER, rank_of
    from paper_1105_4424_b200.model import enum_value
    groups = host.storage.groups
    root = model.application_components[model.application_root]
    ports = {}
    for path, comp in __import__("paper_1105_4424_b200.model", fromlist=["iter_app_instances"]).iter_app_instances(model):
        for p in comp.ports:
            ports[f"{path}.{p.name}" if path else p.name] = p
    bound_groups = {groups[p.name]: p.name for p in root.ports if p.name in bind}
    copies = [{} for _ in range(world)]

    def arr(r, node):
        g = groups[node]
        if g not in copies[r]:
            p = ports[node]
            dt = np.dtype(enum_value(p.data_type))
            if g in bound_groups:
                src = np.asarray(bind[bound_groups[g]]).astype(dt).ravel()
                a = np.full(src.size, np.nan, dtype=dt) if dt.kind == "f" else np.full(src.size, -1, dtype=dt)
                for lo, hi in plan.reads_by_rank.get(g, [[] for _ in range(world)])[r]:
                    a[lo:hi] = src[lo:hi]
            else:
                a = np.zeros(p.shape.total, dtype=dt)
            copies[r][g] = a
        return copies[r][g]

    def task_arrays(r, t):
        return {name: arr(r, node) for name, node in t.nodes.items()}

    iterations = 0

    def run(steps):
        nonlocal iterations
        for step in steps:
            if hasattr(step, "body"):
                while True:
                    run(step.body)
                    iterations += 1
                    relres = float(arr(0, step.relres_port)[0])
                    if relres <= step.tolerance or iterations >= step.max_iterations:
                        return
                continue
            t = host.task(step.task_path)
            if not hasattr(step, "launches"):                 # host scalar op, on every rank
                for r in range(world):
                    a = task_arrays(r, t)
                    if step.op == "div":
                        a["q"][0] = a["num"][0] / a["den"][0]
                    elif step.op == "neg":
                        a["z"][0] = -a["a"][0]
                    else:
                        a["z"][0] = math.sqrt(float(a["num"][0])) / math.sqrt(float(a["den"][0]))
                continue
            if step.op == "dot_partial":
                parts = {}
                for l in step.launches:
                    a = task_arrays(rank_of(l.device_index, world), t)
                    lo, n = l.range.offset, l.range.count
                    parts[l.device_index] = float(np.dot(a["a"][lo:lo + n], a["b"][lo:lo + n]))
                total = 0.0
                for d in sorted(parts):
                    total += parts[d]
                for r in range(world):
                    task_arrays(r, t)["s"][0] = total
                continue
            for l in step.launches:
                r = rank_of(l.device_index, world)
                a = task_arrays(r, t)
                scal = float(a["a"][0]) if "a" in a and step.op in ("scale", "axpy") else None
                orc.run_identity_op(step.op, a, [(l.range.offset, l.range.count)], scal)
            for name, g, tr, wr in plan.writes.get(step.task_path, []):
                assert tr is not None and tr != ROOT_GATHER          # identity tilers write dense streams
                for w_, r, lo, hi in tr:
                    arr(r, t.nodes[name])[lo:hi] = arr(w_, t.nodes[name])[lo:hi]

    run(sched.steps)
    return copies, iterations


@pytest.mark.parametrize("world,D", [(2, 2), (4, 4), (3, 4), (2, 4), (8, 4)])
def test_cg_plan_simulation_equals_reference(golden, world, D):
    from paper_1105_4424_b200.distributed import PlanHost, ShardPlan, rank_of
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    data, meta = golden
    m = meta["cg_k20"]
    model = model_from_dict(m["model"])
    bind = {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}
    sched = build_schedule(model, D)
    host = PlanHost(model, sched, bindings=bind)
    plan = ShardPlan(host, world)
    copies, iters = _simulate(model, sched, bind, world, plan, host)
    assert iters == m["runs"][str(D)]["iterations"]
    # x: every rank holds its own rows; gather them to compare with the reference's result
    x_ref = data[f"cg_k20/x_d{D}"]
    x = np.full(x_ref.size, np.nan)
    xg = host.storage.groups["x"]
    for l in sched.device_steps()[0].launches:
        r = rank_of(l.device_index, world)
        lo, hi = l.range.offset, l.range.offset + l.range.count
        x[lo:hi] = copies[r][xg][lo:hi]
    assert np.array_equal(x, x_ref)
