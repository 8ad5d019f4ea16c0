"""Multi-GPU execution: one process per GPU, contiguous repetition shards, no data-path collective.

The reference simulates D devices in one process: launch d covers
``partition_equally(T, D)[d]`` (partition.py:105-121, refexec.py:488) and
devices share nothing except host-ordered dot reductions (refexec.py:5-7,
:478-487).  Here launch d runs on rank d mod world (``ShardedExecutor``):

  * ``ShardPlan`` lists, for every written port, exactly the ranges another
    rank reads before they are rewritten (writer, reader, lo, hi); only those
    travel, as one grouped batch of exact-size point-to-point transfers
    (NCCL over NVLink on GPUs, gloo host-staged on CPU);
  * output tilers that do not write a dense stream fall back to packed
    output-pattern streams: each rank gathers its patterns in rho order
    through the output tiler (a ``tile_copy`` into a dense [count, P]
    buffer), the streams are all-gathered and scattered back through the
    same tiler -- no indices travel, unequal shards need no padding;
  * dot_partial partials are reduced on the device and summed in ascending
    launch order by the partials_sum kernel, exactly the reference's combine;
  * the caller's outputs are gathered to the root only when asked for.

The exchange primitives (``gather_output``, ``combine_partials``) take injected
pack / unpack / launch callables, so the same logic runs on CPU (gloo, world
size 2, the oracle as the launcher) in tests/test_distributed.py.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from .partition import WorkRange, partition_equally
from .tiler import BoundTiler


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    ranges: tuple[WorkRange, ...]

    @property
    def mine(self) -> WorkRange | None:
        return self.ranges[self.rank] if self.rank < len(self.ranges) else None


def shard(total: int, rank: int, world: int) -> Shard:
    """Rank ``rank``'s contiguous block of a repetition space of ``total`` points."""
    return Shard(rank, world, tuple(partition_equally(total, world)))


def input_hull(bt: BoundTiler, first: int, count: int) -> tuple[int, int]:
    """[lo, hi) flat-offset range of the array that repetitions [first, first+count) read.

    Exact bounding range for non-wrapping tilers (each repetition row of the
    covered box is affine); the whole array for toroidal tilers.  A rank
    needs only this slice of the input resident.
    """
    if count <= 0:
        return (0, 0)
    aff = bt.affine
    if aff is None:
        return (0, bt.array_total)
    c0, rc, pc = aff
    # unravel first/last repetition; the covered set lies inside the box spanned by the
    # outermost differing coordinate (full extent for inner dims)
    import numpy as np
    r_lo = np.unravel_index(first, bt.rep)
    r_hi = np.unravel_index(first + count - 1, bt.rep)
    lo_box, hi_box = [], []
    differ = False
    for j, ext in enumerate(bt.rep):
        if differ:
            lo_box.append(0)
            hi_box.append(ext - 1)
        else:
            lo_box.append(int(r_lo[j]))
            hi_box.append(int(r_hi[j]))
            if r_lo[j] != r_hi[j]:
                differ = True
    lo = c0
    hi = c0
    for c, a, b in zip(rc, lo_box, hi_box):
        lo += min(c * a, c * b)
        hi += max(c * a, c * b)
    for c, ext in zip(pc, bt.tiler.pattern):
        lo += min(0, c * (ext - 1))
        hi += max(0, c * (ext - 1))
    return (int(lo), int(hi) + 1)


def input_ranges(bt: BoundTiler, first: int, count: int) -> list[tuple[int, int]]:
    """Disjoint [lo, hi) flat-offset ranges covering what repetitions [first, first+count) read.

    Affine (non-wrapping) tilers: the exact bounding range of :func:`input_hull`.
    Toroidal tilers: the unwrapped coordinate range of the outermost array axis over the
    repetition box and the full pattern, taken modulo its extent -- one range, or two when
    it crosses the wrap seam (e.g. a stencil chunk needs its rows plus the last row), with
    the inner axes whole.  Covers every offset the index function produces (tested).
    """
    if count <= 0:
        return []
    if bt.affine is not None:
        return [input_hull(bt, first, count)]
    import numpy as np
    r_lo = np.unravel_index(first, bt.rep)
    r_hi = np.unravel_index(first + count - 1, bt.rep)
    lo_box, hi_box, differ = [], [], False
    for j, ext in enumerate(bt.rep):
        if differ:
            lo_box.append(0)
            hi_box.append(ext - 1)
        else:
            lo_box.append(int(r_lo[j]))
            hi_box.append(int(r_hi[j]))
            differ = differ or r_lo[j] != r_hi[j]
    tl = bt.tiler
    mn = mx = int(tl.origin[0])
    for j in range(len(bt.rep)):
        p = int(tl.paving[0][j])
        mn += min(p * lo_box[j], p * hi_box[j])
        mx += max(p * lo_box[j], p * hi_box[j])
    for k, ext in enumerate(tl.pattern):
        f = int(tl.fitting[0][k])
        mn += min(0, f * (ext - 1))
        mx += max(0, f * (ext - 1))
    s0 = int(bt.array[0])
    stride0 = bt.array_total // s0
    if mx - mn + 1 >= s0:
        return [(0, bt.array_total)]
    a0 = mn % s0
    b0 = a0 + (mx - mn)
    ivs = [(a0, b0)] if b0 < s0 else [(0, b0 - s0), (a0, s0 - 1)]
    return [(a * stride0, (b + 1) * stride0) for a, b in ivs]


def missing_ranges(have: list[tuple[int, int]], lo: int, hi: int) -> list[tuple[int, int]]:
    """Parts of [lo, hi) not covered by the sorted disjoint ranges in `have`."""
    out, pos = [], lo
    for a, b in have:
        if b <= pos or a >= hi:
            continue
        if a > pos:
            out.append((pos, a))
        pos = max(pos, b)
        if pos >= hi:
            break
    if pos < hi:
        out.append((pos, hi))
    return out


def add_range(have: list[tuple[int, int]], lo: int, hi: int) -> list[tuple[int, int]]:
    """Union of sorted disjoint ranges with [lo, hi), merged and sorted."""
    out = []
    for a, b in sorted(have + [(lo, hi)]):
        if out and a <= out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], b))
        else:
            out.append((a, b))
    return out


class Exchange:
    """Variable-size all-gather of packed pattern streams over a torch.distributed group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_v(self, local, counts: list[int]):
        """``local`` is this rank's flat stream (counts[rank] elements); returns every rank's stream.

        One grouped batch of point-to-point sends/receives of the exact stream sizes
        (``batch_isend_irecv``: ncclGroupStart/End on NCCL), so the unequal shard sizes
        of partition_equally need no padding."""
        import torch
        dist = self.dist
        out = []
        ops = []
        for r in range(self.world):
            if r == self.rank:
                out.append(local)
                continue
            buf = torch.empty(counts[r], dtype=local.dtype, device=local.device)
            out.append(buf)
            if counts[r]:
                ops.append(dist.P2POp(dist.irecv, buf, self._peer(r), self.group))
            if counts[self.rank]:
                ops.append(dist.P2POp(dist.isend, local, self._peer(r), self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return out

    def _peer(self, r: int) -> int:
        """Global rank of group rank ``r`` (P2P ops address global ranks)."""
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def all_gather_scalars(self, value: float) -> list[float]:
        import torch
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([value], dtype=torch.float64, device=dev)
        out = [torch.empty(1, dtype=torch.float64, device=dev) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [float(o.item()) for o in out]


def gather_output(array, bt: BoundTiler, sh: Shard, ex: Exchange,
                  pack: Callable, unpack: Callable) -> None:
    """Make ``array`` (written by this rank on its shard) whole on every rank.

    ``pack(array, bt, first, count) -> flat stream`` and
    ``unpack(array, bt, first, count, stream)`` move patterns through the
    output tiler in rho order (tile_copy kernels on GPU, the oracle on CPU).
    """
    P = bt.pattern_total
    counts = [r.count * P for r in sh.ranges] + [0] * (sh.world - len(sh.ranges))
    mine = sh.mine
    local = pack(array, bt, mine.offset, mine.count) if mine else None
    if local is None:
        import torch
        local = torch.zeros(0, dtype=array.dtype, device=array.device)
    streams = ex.all_gather_v(local, counts)
    for r, rng in enumerate(sh.ranges):
        if r != sh.rank:
            unpack(array, bt, rng.offset, rng.count, streams[r])


def combine_partials(ex: Exchange, partial: float) -> float:
    """dot_partial combine: partials summed in ascending device order (refexec.py:483-486)."""
    total = 0.0
    for p in ex.all_gather_scalars(partial):
        total += p
    return total


# -- CUDA pack / unpack through libaolb200 tile_copy -----------------------------

def cuda_pack(array, bt: BoundTiler, first: int, count: int):
    """Gather this rank's output patterns (rho order) into a dense stream with one tile_copy launch."""
    import torch
    from . import _capi
    from .tiler import Tiler
    P = bt.pattern_total
    out = torch.empty(count * P, dtype=array.dtype, device=array.device)
    # dense side indexed by (rho - first): origin -first*P on a [count*P] array would wrap, so
    # address the dense buffer as a window [first*P, ...) of a virtual array of R*P elements
    R = bt.rep_total
    dense = Tiler((0,), (tuple(int(__import__("numpy").prod(bt.rep[j + 1:])) * P for j in range(len(bt.rep))),),
                  ((1,),), (P,)).bind((R * P,), bt.rep)
    task = _capi.make_task("tile_copy", str(array.dtype).replace("torch.", ""), [bt, dense])
    base = out.data_ptr() - first * P * out.element_size()
    _capi.launch(task, first, count, [array.data_ptr(), base], (),
                 int(torch.cuda.current_stream(array.device).cuda_stream))
    return out


def cuda_unpack(array, bt: BoundTiler, first: int, count: int, stream) -> None:
    """Scatter another rank's dense pattern stream back through the output tiler."""
    import numpy as np
    import torch
    from . import _capi
    from .tiler import Tiler
    P = bt.pattern_total
    R = bt.rep_total
    dense = Tiler((0,), (tuple(int(np.prod(bt.rep[j + 1:])) * P for j in range(len(bt.rep))),),
                  ((1,),), (P,)).bind((R * P,), bt.rep)
    task = _capi.make_task("tile_copy", str(array.dtype).replace("torch.", ""), [dense, bt])
    base = stream.data_ptr() - first * P * stream.element_size()
    _capi.launch(task, first, count, [base, array.data_ptr()], (),
                 int(torch.cuda.current_stream(array.device).cuda_stream))


# -- sharded execution: launch d on rank d mod world, exchange only what crosses shards ----

def rank_of(device_index: int, world: int) -> int:
    """Rank that runs launch ``device_index`` of a step (launch d -> rank d mod world)."""
    return device_index % world


def _walk(steps):
    for st in steps:
        if hasattr(st, "body"):
            yield from _walk(st.body)
        else:
            yield st


def _written_ports(task) -> list[str]:
    return [ps.name for ps in task.spec.ports if ps.direction in ("out", "inout") and task.comp.port(ps.name)]


def _read_ports(task) -> list[str]:
    return [ps.name for ps in task.spec.ports if ps.direction in ("in", "inout") and task.comp.port(ps.name)]


def _port_tiler(ex, task, name: str) -> BoundTiler:
    """Tiler of a port: the task's tiler for tile ops, the identity tiler for reference ops."""
    from .tiler import Tiler
    tl = dict(getattr(task.comp, "tilers", ()) or ())
    tl.update(ex.tilers.get(task.path, {}) or {})
    port = task.comp.port(name)
    rep = task.comp.repetition_space.dims if task.comp.repetition_space is not None else (1,)
    if name in tl:
        return tl[name].bind(port.shape.dims, rep)
    n = port.shape.total
    T = 1
    for d in rep:
        T *= int(d)
    if T == n:
        return Tiler((0,), ((1,),), ((0,),), (1,)).bind((n,), (T,))
    # repetition total 1 with a longer vector: only element 0 is touched (refexec probe)
    return Tiler((0,), ((0,),), ((0,),), (1,)).bind((n,), (T,))


def dense_stream(bt: BoundTiler) -> tuple[int, int] | None:
    """(c0, P) when repetition rho's pattern lands at [c0 + P*rho, c0 + P*rho + P) -- the
    tiler writes a dense stream in rho order, so a launch range writes one flat range --
    else None."""
    import numpy as np
    aff = bt.affine
    if aff is None:
        return None
    c0, rc, pc = aff
    P = bt.pattern_total
    pat = bt.tiler.pattern
    want_pc = tuple(int(np.prod(pat[k + 1:])) for k in range(len(pat)))
    want_rc = tuple(int(np.prod(bt.rep[j + 1:])) * P for j in range(len(bt.rep)))
    if tuple(int(p) if e > 1 else want_pc[k] for k, (p, e) in enumerate(zip(pc, pat))) != want_pc:
        return None
    if tuple(int(r) if e > 1 else want_rc[j] for j, (r, e) in enumerate(zip(rc, bt.rep))) != want_rc:
        return None
    return int(c0), P


def read_ranges(ex, task, name: str, first: int, count: int) -> list[tuple[int, int]]:
    """Flat ranges of port ``name`` that launch [first, first+count) of ``task`` reads.

    Tiled ports: :func:`input_ranges`.  spmv_csr (refexec.py:111-121): rowptr rows
    [first, first+count], x / colidx / values gathered anywhere (whole).  Filter weights,
    scalars: whole.  Identity ports of the reference ops: the launch range itself."""
    spec = task.spec
    n = task.comp.port(name).shape.total
    ps = spec.port_spec(name)
    if spec.tile:
        return input_ranges(_port_tiler(ex, task, name), first, count) if ps.tiled else [(0, n)]
    if spec.name == "spmv_csr":
        if name == "rowptr":
            return [(first, min(n, first + count + 1))]
        known = (getattr(ex, "gather_hulls", None) or {}).get((task.path, name, first, count))
        return known if known is not None else [(0, n)]
    if ps.scalar:
        return [(0, n)]
    return input_ranges(_port_tiler(ex, task, name), first, count)


def _set_owner(lst: list, lo: int, hi: int, owner) -> list:
    """Sorted disjoint (lo, hi, owner) intervals with [lo, hi) re-assigned to ``owner``
    (owner None removes it)."""
    out = []
    for a, b, o in lst:
        if b <= lo or a >= hi:
            out.append((a, b, o))
            continue
        if a < lo:
            out.append((a, lo, o))
        if b > hi:
            out.append((hi, b, o))
    if owner is not None and hi > lo:
        out.append((lo, hi, owner))
    return sorted(out)


def _bound_host_array(host, bindings: dict, node: str):
    """The caller's binding of the port group holding ``node`` as a flat numpy array, or None."""
    import numpy as np
    if not bindings:
        return None
    g = host.storage.groups.get(node)
    for name in sorted(g or ()):
        if name in bindings:
            v = bindings[name]
            if hasattr(v, "detach"):
                v = v.detach().cpu().numpy()
            return np.asarray(v).ravel()
    return None


def compute_gather_hulls(host, bindings: dict | None) -> dict:
    """Data-aware read ranges of spmv_csr launches (refexec.py:111-121): rows [first,
    first+count) read entries rowptr[first] .. rowptr[first+count] of colidx / values and
    the x elements colidx names there -- for a banded matrix a halo around the launch's own
    rows instead of all of x.  Only for matrices the caller bound and no step rewrites (the
    reference caches its spmv plans on the same immutability, refexec.py:404-409).
    Returns {(task path, port, first, count): [(lo, hi)]}."""
    hulls: dict = {}
    if not bindings:
        return hulls
    written = set()
    steps = list(_walk(host.schedule.steps))
    for step in steps:
        t = host.task(step.task_path)
        for name in _written_ports(t):
            written.add(host.storage.groups[t.nodes[name]])
    for step in steps:
        if getattr(step, "op", None) != "spmv_csr":
            continue
        t = host.task(step.task_path)
        if any(host.storage.groups[t.nodes[n]] in written for n in ("rowptr", "colidx")):
            continue
        rp = _bound_host_array(host, bindings, t.nodes["rowptr"])
        ci = _bound_host_array(host, bindings, t.nodes["colidx"])
        if rp is None or ci is None:
            continue
        for l in step.launches:
            first, count = l.range.offset, l.range.count
            if count <= 0:
                continue
            lo_e, hi_e = int(rp[first]), int(rp[first + count])
            hulls[(t.path, "colidx", first, count)] = [(lo_e, hi_e)] if hi_e > lo_e else []
            hulls[(t.path, "values", first, count)] = [(lo_e, hi_e)] if hi_e > lo_e else []
            if hi_e > lo_e:
                cols = ci[lo_e:hi_e]
                hulls[(t.path, "x", first, count)] = [(int(cols.min()), int(cols.max()) + 1)]
            else:
                hulls[(t.path, "x", first, count)] = []
    return hulls


class PlanHost:
    """What a :class:`ShardPlan` reads from an executor -- the model's port groups, validated
    tasks, the schedule and per-task tilers -- without any device storage (host-side use
    and CPU tests)."""

    def __init__(self, model, schedule, tilers: dict | None = None, precision: str = "default",
                 bindings: dict | None = None):
        import types
        from .model import connected_port_groups
        self.model, self.schedule, self.tilers, self.precision = model, schedule, tilers or {}, precision
        self.storage = types.SimpleNamespace(groups=connected_port_groups(model))
        self._tasks: dict = {}
        self.gather_hulls = compute_gather_hulls(self, bindings)

    def task(self, path: str):
        from .executor import _Task
        t = self._tasks.get(path)
        if t is None:
            t = self._tasks[path] = _Task(self.model, self.storage, path, self.tilers.get(path), self.precision)
        return t


def _continuations(steps) -> dict:
    """id(step) -> the execution sequences that can follow it (loops flattened).

    A top-level step continues with the rest of the schedule.  A step at position k of a
    LoopStep body continues either with body[k+1:] and whatever follows the loop (the loop
    exits), or with body[k+1:] + body[:k+1] (one more iteration up to and including itself,
    refexec.py:525-541).  Nested loops are walked the same way, innermost first."""
    conts: dict = {}

    def flat(seq):
        return list(_walk(seq))

    def visit(seq, after: list, looping: bool):
        for k, st in enumerate(seq):
            rest = flat(seq[k + 1:])
            outs = [rest + a for a in after]
            if looping:
                outs.append(rest + flat(seq[:k + 1]))
            if hasattr(st, "body"):
                visit(st.body, outs if outs else [[]], True)
            else:
                conts[id(st)] = outs
    visit(list(steps), [[]], False)
    return conts


ROOT_GATHER = "root-gather"      # ShardPlan marker: a non-dense write no later step reads


class ShardPlan:
    """Static exchange plan of a schedule whose launch d runs on rank d mod ``world``.

    For every device step and written port: if the output tiler writes a dense stream,
    each launch writes one flat range, and exactly the part of it that another rank reads
    before that part is overwritten again by its own writer travels to that rank -- a list
    of (writer, reader, lo, hi) ranges.  Readers are found along every execution path that
    can follow the step (:func:`_continuations`; loop bodies wrap), stopping at the first
    later step that rewrites the same ranges on the same ranks (CG's ``scale_p`` is followed
    by ``axpy_p`` on the same shards, so only ``axpy_p``'s p travels to the spmv).
    Non-dense output tilers fall back to the packed-pattern all-gather (``None``) when a later
    step reads the group, and to a packed gather to the root at output time (``ROOT_GATHER``)
    when none does.  Host
    scalar ops read on every rank; dot_partial results are combined by the partial
    reduction, not exchanged.  Nothing is exchanged for the caller's outputs until
    :meth:`ShardedExecutor.outputs` gathers them to the root (NCCL only
    where an output crosses shards)."""

    def __init__(self, ex, world: int):
        self.world = world
        st = ex.storage
        self.groups = st.groups
        reads: dict = {}        # id(step) -> {group: [ranges per rank]}
        writes: dict = {}       # id(step) -> {group: (dense, [(w, lo, hi)])}
        steps = list(_walk(ex.schedule.steps))
        for step in steps:
            t = ex.task(step.task_path)
            rd: dict = {}

            def add(g, r, lo, hi):
                if hi > lo:
                    lst = rd.setdefault(g, [[] for _ in range(world)])
                    lst[r] = add_range(lst[r], lo, hi)
            if not hasattr(step, "launches"):
                for n in _read_ports(t):
                    for r in range(world):
                        add(st.groups[t.nodes[n]], r, 0, t.comp.port(n).shape.total)
                reads[id(step)] = rd
                continue
            for l in step.launches:
                r = rank_of(l.device_index, world)
                for n in _read_ports(t):
                    for lo, hi in read_ranges(ex, t, n, l.range.offset, l.range.count):
                        add(st.groups[t.nodes[n]], r, lo, hi)
            reads[id(step)] = rd
            wr: dict = {}
            if step.op != "dot_partial":
                for name in _written_ports(t):
                    bt = _port_tiler(ex, t, name)
                    ds = dense_stream(bt)
                    ranges = []
                    if ds is not None:
                        c0, P = ds
                        for l in step.launches:
                            lo, hi = c0 + P * l.range.offset, c0 + P * (l.range.offset + l.range.count)
                            if hi > lo:
                                ranges.append((rank_of(l.device_index, world), lo, hi))
                    wr[st.groups[t.nodes[name]]] = (name, ds is not None, ranges)
            writes[id(step)] = wr
        # every range of every group each rank reads at some point (the input hulls)
        self.reads_by_rank: dict = {}
        for rd in reads.values():
            for g, per in rd.items():
                acc = self.reads_by_rank.setdefault(g, [[] for _ in range(world)])
                for r in range(world):
                    for a, b in per[r]:
                        acc[r] = add_range(acc[r], a, b)
        conts = _continuations(ex.schedule.steps)

        def kills(later: dict, g, ranges) -> bool:
            """The later step rewrites every range of this write on the same rank."""
            if g not in later or not later[g][1]:
                return False
            cover = later[g][2]
            return all(any(w2 == w and lo2 <= lo and hi2 >= hi for w2, lo2, hi2 in cover) for w, lo, hi in ranges)

        # task path -> [(port, group, dense transfers | None, [(writer, lo, hi)])]
        self.writes: dict[str, list] = {}
        self.need: dict = {}
        for step in steps:
            if not hasattr(step, "launches") or step.op == "dot_partial":
                continue
            entries = []
            for g, (name, dense, ranges) in writes[id(step)].items():
                if not dense:
                    # packed-pattern exchange only if some later step reads the group at all;
                    # otherwise (a root output) the patterns go to the root when it gathers
                    read_later = any(reads[id(nxt)].get(g) for seq in conts[id(step)] for nxt in seq)
                    entries.append((name, g, None if read_later else ROOT_GATHER, []))
                    continue
                need = [[] for _ in range(world)]
                for seq in conts[id(step)]:
                    for nxt in seq:
                        rd = reads[id(nxt)].get(g)
                        if rd:
                            for r in range(world):
                                for a, b in rd[r]:
                                    need[r] = add_range(need[r], a, b)
                        if kills(writes.get(id(nxt), {}), g, ranges):
                            break
                self.need[(step.task_path, g)] = need
                tr = []
                for w, lo, hi in ranges:
                    for r in range(world):
                        if r == w:
                            continue
                        for a, b in need[r]:
                            if min(hi, b) > max(lo, a):
                                tr.append((w, r, max(lo, a), min(hi, b)))
                entries.append((name, g, tr, ranges))
            self.writes[step.task_path] = entries

    @classmethod
    def for_model(cls, model, schedule, world: int, tilers: dict | None = None,
                  bindings: dict | None = None) -> "ShardPlan":
        return cls(PlanHost(model, schedule, tilers, bindings=bindings), world)

    def exchanged_bytes(self, task_path: str, esize: dict) -> int:
        """Bytes the dense transfers of one step move (for tests / reports)."""
        tot = 0
        for name, g, tr, _ in self.writes.get(task_path, []):
            if tr and tr != ROOT_GATHER:
                tot += sum(hi - lo for _, _, lo, hi in tr) * esize.get(g, 4)
        return tot


class Replica:
    """One rank's storage in this process: the rank, its CUDA device, its port arrays."""

    def __init__(self, rank: int, device, storage):
        self.rank, self.device, self.storage = rank, device, storage
        self.pbuf = {}


class DistTransport:
    """Exchange over a torch.distributed group: NCCL over NVLink on GPUs (device buffers
    straight into the NCCL send/recv), or host-staged over gloo (CPU ranks, or several
    ranks sharing one GPU in tests).  One grouped batch of exact-size point-to-point
    transfers per exchange (ncclGroupStart/End); every rank derives the same transfer
    list from the same plan, so the k-th send w->r matches the k-th receive on r."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.staged = dist.get_backend(group) != "nccl"
        self.bytes_moved = 0

    def _peer(self, r: int) -> int:
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def move(self, replicas: dict, g, transfers: list) -> None:
        dist = self.dist
        me = self.rank
        rep = replicas[me]
        arr = rep.storage.arrays[g]
        ops, back = [], []
        for w, r, lo, hi in transfers:
            if w == me:
                buf = arr[lo:hi].cpu() if self.staged else arr[lo:hi]
                ops.append(dist.P2POp(dist.isend, buf, self._peer(r), self.group))
                self.bytes_moved += (hi - lo) * arr.element_size()
            elif r == me:
                if self.staged:
                    import torch
                    buf = torch.empty(hi - lo, dtype=arr.dtype)
                    back.append((buf, lo, hi))
                else:
                    buf = arr[lo:hi]
                ops.append(dist.P2POp(dist.irecv, buf, self._peer(w), self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for buf, lo, hi in back:
            arr[lo:hi].copy_(buf)

    def reduce_partials(self, replicas: dict, key) -> None:
        """Every rank's dot partials (zeros in the slots it does not own) summed slot-wise:
        x + 0 is exact, so each slot ends up holding its launch's partial bit for bit."""
        buf = replicas[self.rank].pbuf[key]
        if self.staged:
            h = buf.cpu()
            self.dist.all_reduce(h, group=self.group)
            buf.copy_(h)
        else:
            self.dist.all_reduce(buf, group=self.group)

    def all_gather_v(self, replicas: dict, local, counts: list[int]):
        import torch
        if self.staged:
            ex = Exchange(self.group)
            streams = ex.all_gather_v(local.cpu(), counts)
            dev = replicas[self.rank].device
            return [s_.to(dev) if isinstance(s_, torch.Tensor) else s_ for s_ in streams]
        return Exchange(self.group).all_gather_v(local, counts)

    def gather_v(self, replicas: dict, local, counts: list[int], root: int) -> dict:
        """Variable-size streams to ``root`` only (one grouped batch of send/recv): the root
        gets {rank: stream} for every other rank with a non-empty stream, the others {}."""
        import torch
        dist, me = self.dist, self.rank
        ops, out = [], {}
        if me == root:
            for r in range(self.world):
                if r == root or counts[r] == 0:
                    continue
                buf = torch.empty(counts[r], dtype=local.dtype, device="cpu" if self.staged else local.device)
                out[r] = buf
                ops.append(dist.P2POp(dist.irecv, buf, self._peer(r), self.group))
        elif counts[me]:
            ops.append(dist.P2POp(dist.isend, local.cpu() if self.staged else local, self._peer(root), self.group))
            self.bytes_moved += local.numel() * local.element_size()
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        dev = replicas[me].device
        return {r: b.to(dev) for r, b in out.items()}

    def barrier(self):
        self.dist.barrier(group=self.group)


class LocalTransport:
    """Exchange between replicas in one process (``execute_schedule(device_count=D)`` with
    several visible GPUs): peer copies, which travel over NVLink between devices.  Two
    replicas may share a device (used by tests on one GPU); the copies are then local."""

    def __init__(self, world: int):
        self.world = world
        self.bytes_moved = 0

    def move(self, replicas: dict, g, transfers: list) -> None:
        import torch
        for w, r, lo, hi in transfers:
            src = replicas[w].storage.arrays[g]
            dst = replicas[r].storage.arrays[g]
            with torch.cuda.device(replicas[r].device):
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
            self.bytes_moved += (hi - lo) * src.element_size()

    def reduce_partials(self, replicas: dict, key) -> None:
        import torch
        bufs = {r: rep.pbuf[key] for r, rep in replicas.items()}
        n = next(iter(bufs.values())).numel()
        for k in range(n):
            w = k % self.world
            for r, b in bufs.items():
                if r != w:
                    with torch.cuda.device(replicas[r].device):
                        b[k:k + 1].copy_(bufs[w][k:k + 1], non_blocking=True)

    def all_gather_v(self, replicas: dict, local, counts):
        raise NotImplementedError

    def barrier(self):
        pass


def fused_gather_candidates(host, plan: "ShardPlan") -> list:
    """Root output groups that only device steps write and no step reads (any rank): their
    producing kernels may store straight into the root's array (fused gather).  Sorted, so
    every rank derives the same list."""
    root = host.model.application_components[host.model.application_root]
    outs = {host.storage.groups[p.name] for p in root.ports if getattr(p.direction, "value", p.direction) == "out"}
    device_written, host_written = set(), set()
    for step in _walk(host.schedule.steps):
        t = host.task(step.task_path)
        dst = device_written if hasattr(step, "launches") else host_written
        for name in _written_ports(t):
            dst.add(host.storage.groups[t.nodes[name]])
    return sorted((g for g in outs if g in device_written and g not in host_written and g not in plan.reads_by_rank),
                  key=lambda g: sorted(g))


class ShardedExecutor:
    """Mixin over :class:`executor.Executor`: launch d of every device step runs on rank
    d mod world; only what a later step of another rank reads is exchanged (ShardPlan);
    dot partials are reduced on the device and combined in ascending launch order by the
    partials_sum kernel (refexec.py:478-487) -- no host round trip per dot; host scalar ops
    run as device scalar kernels on every rank, so a CG iteration syncs the host once, for
    the loop test (refexec.py:525-541).  Outputs are gathered to the root (rank 0)."""

    _SKIP_COVERED_ZERO = False          # each replica writes only its launches' slice

    def _init_sharded(self, transport, replicas: list, world: int, bindings: dict | None = None,
                      fused_gather: bool | None = None):
        self.transport = transport
        self.world = world
        self.replicas = {rep.rank: rep for rep in replicas}
        self.gather_hulls = compute_gather_hulls(self, bindings)
        self.root = 0
        self.plan = ShardPlan(self, world)
        self.stale: dict = {}          # group -> [(lo, hi, owner)] ranges the root holds stale
        self.pending_pack: dict = {}   # group -> (step, task, port): non-dense write the root lacks
        self.exchanged_bytes = 0
        self._upload_hulls()
        self._setup_fused_gather(fused_gather)

    def _setup_fused_gather(self, enabled: bool | None = None) -> None:
        """Fused output gather: a root output that no step reads is written
        by every rank's kernels straight into the ROOT's array through a CUDA IPC peer mapping
        (NVLink between GPUs), so nothing is gathered afterwards.  Only over a
        torch.distributed transport (one process per GPU); ``fused_gather=False`` (or
        AOL_FUSED_GATHER=0) keeps outputs sharded until gather_to_root."""
        import os
        self.fused_out: dict = {}          # group -> this rank's output pointer (None on the root)
        self.fused_bytes = 0               # bytes this rank's launches store into the root per run()
        self._ipc_ptrs: list = []
        if enabled is None:
            enabled = os.environ.get("AOL_FUSED_GATHER", "1") != "0"
        if not isinstance(self.transport, DistTransport) or not enabled:
            return
        from . import _capi
        cand = fused_gather_candidates(self, self.plan)
        if not cand:
            return
        tr = self.transport
        me = tr.rank
        tokens = None
        if me == self.root:
            try:
                tokens = [_capi.ipc_export(self.replicas[me].storage.arrays[g].data_ptr()) for g in cand]
            except _capi.AolError:
                tokens = None           # not exportable (e.g. expandable segments): nobody fuses
        box = [tokens]
        tr.dist.broadcast_object_list(box, src=tr._peer(self.root), group=tr.group)
        if box[0] is None:
            return
        ok = True
        try:
            for g, tok in zip(cand, box[0]):
                if me == self.root:
                    self.fused_out[g] = None
                    continue
                ptr = _capi.ipc_import(tok)
                self._ipc_ptrs.append(ptr)
                self.fused_out[g] = ptr
        except _capi.AolError:
            ok = False          # e.g. the root's GPU is not visible to this process
        flags = [None] * tr.world
        tr.dist.all_gather_object(flags, ok, group=tr.group)
        if not all(flags):      # every rank must take the same path, or the exchanges diverge
            self.close()
            self.fused_out = {}
            return
        for step in self.schedule.device_steps():
            t = self.task(step.task_path)
            for name in _written_ports(t):
                g = self.storage.groups[t.nodes[name]]
                if g in self.fused_out and me != self.root:
                    P = _port_tiler(self, t, name).pattern_total
                    esz = self.replicas[me].storage.arrays[g].element_size()
                    self.fused_bytes += sum(l.range.count for l in self._mine(step, me)) * P * esz

    def _port_ptr(self, rep, t, name: str) -> int:
        """Device pointer a launch of this rank uses for port ``name``: the root's mapped
        array for a fused output, else the rank's own array."""
        g = rep.storage.groups[t.nodes[name]]
        p = self.fused_out.get(g) if self.fused_out else None
        return p if p is not None else rep.storage.array(t.nodes[name]).data_ptr()

    def close(self) -> None:
        """Unmap the root's arrays (fused gather)."""
        ptrs, self._ipc_ptrs = getattr(self, "_ipc_ptrs", []), []
        if not ptrs:
            return
        from . import _capi
        for p in ptrs:
            try:
                _capi.ipc_close(p)
            except Exception:  # noqa: BLE001 - teardown must not raise
                pass

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown: nothing left to unmap into
            pass

    def _upload_hulls(self) -> None:
        """Deferred host bindings: each rank uploads only the ranges it ever reads (its input
        hull); the root also uploads every root-output group whole, so
        elements no launch writes keep their bound (or zero) value there."""
        import torch
        root_groups = set()
        root = self.model.application_components[self.model.application_root]
        for port in root.ports:
            if getattr(port.direction, "value", port.direction) == "out":
                root_groups.add(self.storage.groups[port.name])
        self.h2d_bytes = 0
        for rep in self._each():
            st = rep.storage
            for g, h in list(st.host.items()):
                dev = st.arrays[g]
                if rep.rank == self.root and g in root_groups:
                    ranges = [(0, dev.numel())]
                else:
                    ranges = self.plan.reads_by_rank.get(g, [[]] * self.world)[rep.rank]
                for lo, hi in ranges:
                    dev[lo:hi].copy_(h[lo:hi], non_blocking=True)
                    self.h2d_bytes += (hi - lo) * dev.element_size()
                st.host.clear()
            torch.cuda.current_stream(rep.device).synchronize()

    # -- per-replica context -------------------------------------------------------
    def _enter(self, rep):
        self.storage, self.device = rep.storage, rep.device

    def _each(self):
        import torch
        home = (self.storage, self.device)
        try:
            for r in sorted(self.replicas):
                rep = self.replicas[r]
                self._enter(rep)
                with torch.cuda.device(rep.device):
                    yield rep
        finally:
            self.storage, self.device = home

    def _mine(self, step, rank):
        return [l for l in step.launches if rank_of(l.device_index, self.world) == rank]

    # -- steps ---------------------------------------------------------------------
    def run_host(self, step) -> None:
        t = self.task(step.task_path)
        dt = enum_value_dtype(t)
        for rep in self._each():
            self._scalar_seq([step], dt, self._stream_handle())

    def run_device(self, step) -> None:
        from . import _capi
        t = self.task(step.task_path)
        if step.op == "dot_partial":
            self._dot(step, t)
            return
        ctask, names = self._dev_task(step)
        for rep in self._each():
            mine = self._mine(step, rep.rank)
            if not mine:
                continue
            ptrs = [self._port_ptr(rep, t, n) for n in names]
            s = self._stream_handle()
            for l in mine:
                _capi.launch(ctask, l.range.offset, l.range.count, ptrs, (), s)
        self._after_write(step, t)

    def _dot(self, step, t) -> None:
        import torch
        from . import _capi
        from .executor import torch_dtype
        n = len(step.launches)
        key = (t.dtype, n)
        red = _capi.make_task("partials_sum", t.dtype)
        for rep in self._each():
            buf = rep.pbuf.get(key)
            if buf is None:
                buf = rep.pbuf[key] = torch.zeros(n, dtype=torch_dtype(t.dtype), device=rep.device)
            else:
                buf.zero_()
            a, b = rep.storage.array(t.nodes["a"]), rep.storage.array(t.nodes["b"])
            s = self._stream_handle()
            for l in self._mine(step, rep.rank):
                _capi.launch(t.ctask, l.range.offset, l.range.count,
                             [a.data_ptr(), b.data_ptr(), buf.data_ptr() + l.device_index * buf.element_size()],
                             (), s)
        self.transport.reduce_partials(self.replicas, key)
        for rep in self._each():
            _capi.launch(red, 0, n, [rep.pbuf[key].data_ptr(), rep.storage.array(t.nodes["s"]).data_ptr()], (),
                         self._stream_handle())

    def _after_write(self, step, t) -> None:
        for name, g, tr, wr in self.plan.writes.get(step.task_path, []):
            if g in self.fused_out:
                continue                    # already stored into the root's array by the kernels
            if g in self.pending_pack:
                # an older packed write of this group by ANOTHER step must reach the root before
                # this one lands (program order); the same step again (the next run(), a loop
                # iteration) rewrites exactly the same elements, so its older pack is dropped
                old = self.pending_pack.pop(g)
                if old[0] is not step:
                    self._pack_to_root(*old)
            if tr is None:
                self._pack_exchange(step, t, name)
                continue
            if tr == ROOT_GATHER:
                self.pending_pack[g] = (step, t, name)
                continue
            if tr:
                self.transport.move(self.replicas, g, tr)
                esz = next(iter(self.replicas.values())).storage.arrays[g].element_size()
                self.exchanged_bytes += sum(hi - lo for _, _, lo, hi in tr) * esz
            lst = self.stale.get(g, [])
            for w, lo, hi in wr:
                lst = _set_owner(lst, lo, hi, None if w == self.root else w)
            for w, r, lo, hi in tr:
                if r == self.root:
                    lst = _set_owner(lst, lo, hi, None)
            self.stale[g] = lst

    def _pack_exchange(self, step, t, name) -> None:
        """Non-dense output tiler: every rank packs its launches' patterns (rho order) through
        the output tiler, the packed streams are all-gathered, and each rank scatters the
        others' streams back through the same tiler."""
        import torch
        bt = _port_tiler(self, t, name)
        P = bt.pattern_total
        by_rank = {r: self._mine(step, r) for r in range(self.world)}
        counts = [sum(l.range.count for l in by_rank[r]) * P for r in range(self.world)]
        if isinstance(self.transport, LocalTransport):
            for rep in self._each():
                src = rep.storage.array(t.nodes[name])
                for w in range(self.world):
                    if w == rep.rank or not by_rank[w]:
                        continue
                    other = self.replicas[w].storage.array(t.nodes[name])
                    for l in by_rank[w]:
                        with torch.cuda.device(self.replicas[w].device):
                            packed = cuda_pack(other, bt, l.range.offset, l.range.count)
                        cuda_unpack(src, bt, l.range.offset, l.range.count, packed.to(rep.device))
            return
        rep = self.replicas[self.transport.rank]
        arr = rep.storage.array(t.nodes[name])
        with torch.cuda.device(rep.device):
            parts = [cuda_pack(arr, bt, l.range.offset, l.range.count) for l in by_rank[rep.rank]]
            local = torch.cat(parts) if parts else torch.zeros(0, dtype=arr.dtype, device=rep.device)
            streams = self.transport.all_gather_v(self.replicas, local, counts)
            for r in range(self.world):
                if r == rep.rank:
                    continue
                pos = 0
                for l in by_rank[r]:
                    k = l.range.count * P
                    cuda_unpack(arr, bt, l.range.offset, l.range.count, streams[r][pos:pos + k])
                    pos += k

    def _pack_to_root(self, step, t, name) -> int:
        """Non-dense output written by the ranks' launches: each rank other than the root packs
        its patterns in rho order through the output tiler, the streams travel to the root only,
        and the root scatters them back through the same tiler.  Returns bytes moved."""
        import torch
        bt = _port_tiler(self, t, name)
        P = bt.pattern_total
        by_rank = {r: self._mine(step, r) for r in range(self.world)}
        moved = 0
        if isinstance(self.transport, LocalTransport):
            root = self.replicas[self.root]
            dst = root.storage.array(t.nodes[name])
            for w in range(self.world):
                if w == self.root or not by_rank[w]:
                    continue
                src = self.replicas[w].storage.array(t.nodes[name])
                for l in by_rank[w]:
                    with torch.cuda.device(self.replicas[w].device):
                        packed = cuda_pack(src, bt, l.range.offset, l.range.count)
                    with torch.cuda.device(root.device):
                        cuda_unpack(dst, bt, l.range.offset, l.range.count, packed.to(root.device))
                    moved += packed.numel() * packed.element_size()
            return moved
        counts = [sum(l.range.count for l in by_rank[r]) * P for r in range(self.world)]
        rep = self.replicas[self.transport.rank]
        arr = rep.storage.array(t.nodes[name])
        with torch.cuda.device(rep.device):
            if rep.rank != self.root and by_rank[rep.rank]:
                local = torch.cat([cuda_pack(arr, bt, l.range.offset, l.range.count) for l in by_rank[rep.rank]])
            else:
                local = torch.zeros(0, dtype=arr.dtype, device=rep.device)
            streams = self.transport.gather_v(self.replicas, local, counts, self.root)
            for r, stream in streams.items():
                pos = 0
                for l in by_rank[r]:
                    k = l.range.count * P
                    cuda_unpack(arr, bt, l.range.offset, l.range.count, stream[pos:pos + k])
                    pos += k
        # every rank reports the same total (like move()), so callers may reduce over it
        return sum(c for r, c in enumerate(counts) if r != self.root) * arr.element_size()

    def _run_fused(self, s1, s2) -> bool:
        from . import _capi
        t1, t2 = self.task(s1.task_path), self.task(s2.task_path)
        first = True
        for rep in self._each():
            a1 = [self._port_ptr(rep, t1, n) for n in t1.port_order]
            a2 = [self._port_ptr(rep, t2, n) for n in t2.port_order]
            s = self._stream_handle()
            if first and not _capi.launch_fused2(t1.ctask, t2.ctask, 0, 0, a1, a2, s):
                self._fusable[(s1.task_path, s2.task_path)] = False
                return False
            first = False
            for l in self._mine(s2, rep.rank):
                if not _capi.launch_fused2(t1.ctask, t2.ctask, l.range.offset, l.range.count, a1, a2, s):
                    raise RuntimeError("fusion became unsupported mid-step")
                self.fused_launches += 1
        self._after_write(s2, t2)
        return True

    # -- results -------------------------------------------------------------------
    def gather_to_root(self) -> int:
        """Move every range of a root output the root holds stale to the root; returns bytes.
        Fused outputs need no move: every rank waits for its own kernels' remote stores, then
        all ranks meet at a barrier, after which the root's arrays are complete."""
        import torch
        root = self.model.application_components[self.model.application_root]
        moved = 0
        if self.fused_out:
            for rep in self._each():
                torch.cuda.current_stream(rep.device).synchronize()
            self.transport.barrier()
        for port in root.ports:
            if getattr(port.direction, "value", port.direction) != "out":
                continue
            g = self.storage.groups[port.name]
            tr = [(o, self.root, lo, hi) for lo, hi, o in self.stale.get(g, [])]
            if tr:
                self.transport.move(self.replicas, g, tr)
                moved += sum(hi - lo for _, _, lo, hi in tr) * self.replicas[next(iter(self.replicas))] \
                    .storage.arrays[g].element_size()
            self.stale[g] = []
        outs = {self.storage.groups[p.name] for p in root.ports
                if getattr(p.direction, "value", p.direction) == "out"}
        for g in list(self.pending_pack):
            pend = self.pending_pack.pop(g)
            if g in outs:                   # groups nobody reads and the caller never sees stay put
                moved += self._pack_to_root(*pend)
        return moved

    def outputs(self, on_device: bool = False, out: dict | None = None) -> dict:
        """Root outputs, flat row-major (refexec.py:545-547), after gathering the stale ranges to
        the root; other ranks take part in the gather and return {} (the root holds results)."""
        self.gather_to_root()
        if self.root not in self.replicas:
            res = {}
        else:
            self._enter(self.replicas[self.root])
            from .executor import Executor
            res = Executor.outputs(self, on_device=on_device, out=out)
        if self.fused_out:
            # the root has copied the fused arrays before any rank's next run() may store
            # into them again
            if not on_device:
                import torch
                torch.cuda.current_stream(self.device).synchronize()
            self.transport.barrier()
        return res


def enum_value_dtype(task) -> str:
    from .model import enum_value
    return enum_value(task.comp.ports[0].data_type)


def make_sharded_executor(model, schedule, bindings: dict, device_count: int, devices: list, **kw):
    """In-process sharding over ``devices`` (one replica per entry; launch d on replica
    d mod len(devices)).  The replicas hold full copies of the inputs; outputs gather to
    replica 0."""
    import torch
    from .executor import DeviceStorage, Executor

    if kw.get("stream") is not None and len({str(torch.device(d)) for d in devices}) > 1:
        raise ValueError("stream= names one device's stream; it cannot drive replicas on several devices")

    class LocalShardedExecutor(ShardedExecutor, Executor):
        def __init__(self):
            kw["graphs"] = False             # loop bodies need the per-step exchange
            kw["pipeline"] = 0
            Executor.__init__(self, model, schedule, bindings, device_count, device=devices[0], **kw)
            reps = [Replica(0, self.device, self.storage)]
            for r, dev in enumerate(devices[1:], start=1):
                d = torch.device(dev)
                with torch.cuda.device(d):
                    reps.append(Replica(r, d, DeviceStorage(model, bindings, d)))
            self._init_sharded(LocalTransport(len(devices)), reps, len(devices), bindings)

    return LocalShardedExecutor()


def make_distributed_executor(model, schedule, bindings: dict, *, group=None, fused_gather: bool | None = None,
                              **kw):
    """Executor for rank ``dist.get_rank(group)`` of a schedule whose launches are spread over
    the group's ranks (launch d on rank d mod world; build the schedule with device_count ==
    world size for one launch per rank, as the reference's D simulated devices).
    ``fused_gather``: root outputs no step reads are stored into the root's array by the
    producing kernels (default: on unless AOL_FUSED_GATHER=0)."""
    from .executor import Executor

    class DistributedExecutor(ShardedExecutor, Executor):
        def __init__(self):
            tr = DistTransport(group)
            kw["graphs"] = False             # loop bodies need the per-step exchange
            kw["pipeline"] = 0
            D = max((len(st.launches) for st in schedule.device_steps()), default=1)
            kw.setdefault("defer", True)      # host bindings: upload only this rank's input hull
            Executor.__init__(self, model, schedule, bindings, D, **kw)
            self.rank = tr.rank
            self._init_sharded(tr, [Replica(tr.rank, self.device, self.storage)], tr.world, bindings, fused_gather)

    return DistributedExecutor()
