"""B200 drop-in for ``gmodelc.refexec.execute_schedule`` (refexec.py:427-549).

Same signature, same return type (:class:`ExecutionResult`), same binding
checks (``MissingBinding``, refexec.py:390-396), same signature errors
(``UnknownIntrinsic`` / ``IntrinsicShapeMismatch`` incl. the
output-aliases-input check, :440-455), zero-initialised unwritten outputs
(:399-403), flat row-major outputs (:545-547) and the same LoopStep
semantics (:518-541).  What changes is where the arrays live and who runs
the launches:

  * storage: one CUDA tensor per connected-port group (``_Storage``
    :375-412) in HBM, allocated through PyTorch (tensor handoff only);
  * every ``KernelLaunch`` of a ``DeviceStep`` becomes one ``aol_launch``
    of libaolb200.so over the same ``[offset, offset+count)`` range
    (replacing the numpy body of refexec.py:488-514);
  * dot_partial keeps the reference's host combine: one partial per
    launch, summed on the host in ascending device order (:478-487).

Keyword-only additions: ``tilers`` (task path -> port -> Tiler, for
reference models whose Component has no tiler field), ``precision`` for
the matmul elementary task, ``device_outputs`` to keep results in HBM,
``out`` (caller-owned host buffers), ``pipeline`` (chunked H2D / compute /
D2H overlap for one-step schedules bound to host memory) and ``stream``.
There is no CPU fallback: a missing library raises.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._refcompat import ref_bases
from .intrinsics import (INTRINSICS, IntrinsicShapeMismatch, _ports_match_spec, check_task_signature,
                         check_tile_signature)
from .model import connected_port_groups, enum_value, iter_app_instances, task_component


class MissingBinding(*ref_bases("refexec", "MissingBinding", KeyError)):
    pass


def partition_equally_local(total: int, parts: int) -> list[tuple[int, int]]:
    """(offset, count) sub-chunks of [0, total) — the partition.py:105-121 rule, reused for pipelining."""
    from .partition import partition_equally
    return [(r.offset, r.count) for r in partition_equally(total, parts)] if total > 0 else []


@dataclass
class ExecutionResult:
    outputs: dict
    iterations: int
    final_relres: float | None
    converged: bool


_TORCH_DTYPES = None


def _torch():
    import torch
    return torch


def torch_dtype(name: str):
    global _TORCH_DTYPES
    torch = _torch()
    if _TORCH_DTYPES is None:
        _TORCH_DTYPES = {"float32": torch.float32, "float64": torch.float64,
                         "int32": torch.int32, "int64": torch.int64}
    return _TORCH_DTYPES[name]


class HostStager:
    """Pinned staging ring for uploads from pageable host memory (numpy bindings).

    A DMA from pageable memory is staged by the driver synchronously, piece by piece, so
    it neither overlaps the host nor runs at PCIe speed.  Here piece k of a copy is
    memcpy'd on the host into pinned slot k mod R (torch's multi-threaded CPU copy) while
    the DMAs of the previous pieces run asynchronously on the copy stream; a slot is reused
    only after its DMA's event completed.  Pinned sources bypass the ring."""

    def __init__(self, slot_bytes: int = 16 << 20, slots: int = 4):
        import threading
        torch = _torch()
        self.lock = threading.Lock()        # one ring per process: callers on several threads take turns
        self.slot_bytes = slot_bytes
        self.bufs = [torch.empty(slot_bytes, dtype=torch.uint8, pin_memory=True) for _ in range(slots)]
        self.events = [None] * slots
        self.k = 0

    def copy(self, dst, src, stream) -> None:
        """dst[:] = src (1-D, same dtype): dst on the device, src in host memory."""
        torch = _torch()
        if src.is_pinned():
            with torch.cuda.stream(stream):
                dst.copy_(src, non_blocking=True)
            return
        with self.lock:
            self._copy_staged(dst, src, stream)

    def copy2d(self, dst_ptr: int, dpitch: int, src, stream) -> None:
        """Device rows dst_ptr + r * dpitch (bytes) <- host 2-D view src [rows, width] (any
        strides; pageable or pinned): through the ring piece by piece (a piece = as many rows
        as fit a slot, gathered contiguous on the host), each piece one aol_memcpy2d."""
        torch = _torch()
        rows, width = src.shape
        wb = width * src.element_size()
        if rows == 0 or wb == 0:
            return
        per = max(1, self.slot_bytes // wb)
        with self.lock:
            for r0 in range(0, rows, per):
                m = min(per, rows - r0)
                i = self.k % len(self.bufs)
                self.k += 1
                if self.events[i] is not None:
                    self.events[i].synchronize()
                buf = self.bufs[i][:m * wb].view(src.dtype).view(m, width)
                buf.copy_(src[r0:r0 + m])
                _capi.memcpy2d(dst_ptr + r0 * dpitch, dpitch, buf.data_ptr(), wb, wb, m, stream.cuda_stream)
                ev = torch.cuda.Event()
                ev.record(stream)
                self.events[i] = ev

    def download(self, dst, src, stream) -> None:
        """dst[:] = src (1-D, same dtype): src on the device, dst in pageable host memory.
        Piece k is DMA'd into slot k mod R on ``stream`` (after everything already queued
        there) while the host copies piece k-1 out of its slot; returns when dst is complete."""
        torch = _torch()
        sb, db = src.view(torch.uint8), dst.view(torch.uint8)
        n = sb.numel()
        with self.lock:
            prev = None
            for off in range(0, n, self.slot_bytes):
                m = min(self.slot_bytes, n - off)
                i = self.k % len(self.bufs)
                self.k += 1
                if self.events[i] is not None:
                    self.events[i].synchronize()
                buf = self.bufs[i][:m]
                with torch.cuda.stream(stream):
                    buf.copy_(sb[off:off + m], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(stream)
                self.events[i] = ev
                if prev is not None:
                    prev[0].synchronize()
                    db[prev[2]:prev[2] + prev[1].numel()].copy_(prev[1])
                prev = (ev, buf, off)
            if prev is not None:
                prev[0].synchronize()
                db[prev[2]:prev[2] + prev[1].numel()].copy_(prev[1])

    def _copy_staged(self, dst, src, stream) -> None:
        torch = _torch()
        sb, db = src.view(torch.uint8), dst.view(torch.uint8)
        n = sb.numel()
        for off in range(0, n, self.slot_bytes):
            m = min(self.slot_bytes, n - off)
            i = self.k % len(self.bufs)
            self.k += 1
            if self.events[i] is not None:
                self.events[i].synchronize()
            buf = self.bufs[i][:m]
            buf.copy_(sb[off:off + m])
            with torch.cuda.stream(stream):
                db[off:off + m].copy_(buf, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            self.events[i] = ev


_SIDE_STREAMS: dict = {}


def side_streams(device):
    """Three streams per device (compute / upload / download) for the streamed paths, created
    once: a new stream per call measurably stalled some calls (cudaStreamCreate)."""
    torch = _torch()
    key = torch.device(device).index
    st = _SIDE_STREAMS.get(key)
    if st is None:
        st = _SIDE_STREAMS[key] = tuple(torch.cuda.Stream(torch.device("cuda", key)) for _ in range(3))
    return st


_STAGERS: dict = {}


def host_stager() -> HostStager:
    """One staging ring per process (64 MiB pinned, from torch's caching host allocator)."""
    st = _STAGERS.get("default")
    if st is None:
        mb = int(os.environ.get("AOL_STAGE_SLOT_MB", "16"))
        n = int(os.environ.get("AOL_STAGE_SLOTS", "4"))
        st = _STAGERS["default"] = HostStager(slot_bytes=max(1, mb) << 20, slots=max(2, n))
    return st


class StorageLayout:
    """What DeviceStorage derives from the model alone, computed once per model object
    (model_memo): port nodes, connected groups, the B200 placement of each group, the HBM
    arenas and each placed group's slice of its arena, and the size / dtype of every group."""

    def __init__(self, model):
        from .placement import hbm_arenas, placement_of_groups
        self.groups = connected_port_groups(model)
        self.ports = {}
        for path, comp in iter_app_instances(model):
            for port in comp.ports:
                self.ports[f"{path}.{port.name}" if path else port.name] = port
        self.placement = placement_of_groups(model)
        self.arenas = hbm_arenas(model)
        self.arena_views: dict = {}      # group -> (memory, lo, hi, torch dtype)
        self.zero_groups: dict = {}      # group -> (elements, torch dtype), first port seen wins
        for node, port in self.ports.items():
            g = self.groups[node]
            if g in self.zero_groups:
                continue
            tdt = torch_dtype(enum_value(port.data_type))
            self.zero_groups[g] = (port.shape.total, tdt)
            pl = self.placement.get(g)
            if pl is not None and pl.tier == "hbm" and pl.memory in self.arenas:
                self.arena_views[g] = (pl.memory, pl.b200_offset, pl.b200_offset + pl.size_bytes, tdt)


def storage_layout(model) -> StorageLayout:
    from .model import model_memo
    return model_memo(model, "storage_layout", StorageLayout)


def _covered_outputs(model) -> frozenset:
    """Port groups that no task reads and exactly one tile task writes, through an output tiler
    that is injective (checked at validation) with repetition x pattern == array elements: a
    bijection, so the schedule's launches (which cover the whole repetition space) write every
    element and the reference's zero-fill of the group (refexec.py:399-403) is dead work."""
    lay = storage_layout(model)
    writers: dict = {}
    readers: set = set()
    for path, comp in iter_app_instances(model):
        if not path or comp.elementary_op is None:
            continue
        for port in comp.ports:
            g = lay.groups.get(f"{path}.{port.name}")
            d = enum_value(port.direction)
            if d in ("in", "inout"):
                readers.add(g)
            if d in ("out", "inout"):
                writers.setdefault(g, []).append((path, comp, port))
    covered = set()
    for g, ws in writers.items():
        if g in readers or len(ws) != 1:
            continue
        path, comp, port = ws[0]
        spec = INTRINSICS.get(comp.elementary_op)
        if spec is None or not spec.tile:
            continue
        try:
            bound = check_tile_signature(path, comp, spec, None)
        except Exception:                      # invalid task: the run reports it, zero-fill stays
            continue
        b = bound.get(port.name)
        if b is not None and b.rep_total * b.pattern_total == b.array_total == port.shape.total:
            covered.add(g)
    return frozenset(covered)


def covered_outputs(model) -> frozenset:
    from .model import model_memo
    return model_memo(model, "covered_outputs", _covered_outputs)


class DeviceStorage:
    """Arrays per connected-port group, resident on one CUDA device (refexec.py:375-412)."""

    def __init__(self, model, bindings: dict, device, stream=None, defer: bool = False,
                 skip_zero: frozenset = frozenset()):
        """``defer``: allocate device arrays for host bindings but do not copy them; the
        streamed path uploads each chunk's input hull itself (``self.host`` keeps the sources).
        ``skip_zero``: placed groups the run writes completely (covered_outputs), not zero-filled."""
        torch = _torch()
        lay = storage_layout(model)
        self.host: dict = {}
        self.groups = lay.groups
        self.ports = lay.ports
        self.arrays: dict = {}
        self.h2d_bytes = 0
        # MARTE placement drives allocation: every deviceGlobal memory is ONE HBM arena and each
        # of its port groups lives at the plan's 256 B-aligned offset (placement.plan_placement);
        # groups without a data allocation, or placed on another tier, get their own buffers
        self.placement = lay.placement
        # uninitialised arena: bound inputs are overwritten by their upload, and every other
        # placed group is zero-filled below (refexec.py:399-403) -- zeroing the inputs too would
        # cost a memset of them and race with uploads issued on another stream
        self.arenas = {mem: torch.empty(nbytes, dtype=torch.uint8, device=device)
                       for mem, nbytes in lay.arenas.items()}
        for g, (mem, lo, hi, tdt) in lay.arena_views.items():
            self.arrays[g] = self.arenas[mem][lo:hi].view(tdt)
        self.device = device
        self._standalone_zero: set = set()
        self._fill(model, bindings, device, defer, skip_zero)

    def rebind(self, model, bindings: dict, skip_zero: frozenset = frozenset()) -> None:
        """Refill the same arrays for a new call (the prepared-executor cache): bound inputs are
        copied in, every other group is zeroed again exactly as a fresh storage would be."""
        self.host = {}
        self.h2d_bytes = 0
        self._fill(model, bindings, self.device, False, skip_zero)

    def _fill(self, model, bindings: dict, device, defer: bool, skip_zero: frozenset) -> None:
        torch = _torch()
        lay = storage_layout(model)
        bound: set = set()
        root = model.application_components[model.application_root]
        for port in root.ports:
            if enum_value(port.direction) not in ("in", "inout"):
                continue
            if port.name not in bindings:
                raise MissingBinding(f"no binding for input port '{port.name}'")
            data = bindings[port.name]
            dt = enum_value(port.data_type)
            if isinstance(data, torch.Tensor):
                flat = data.reshape(-1)
                if flat.numel() != port.shape.total:
                    raise MissingBinding(f"binding '{port.name}' has {flat.numel()} elements, "
                                         f"port expects {port.shape.total}")
                if flat.device.type != "cuda":
                    self.h2d_bytes += flat.numel() * flat.element_size()
                g = self.groups[port.name]
                if defer and flat.device.type != "cuda" and flat.dtype == torch_dtype(dt):
                    self.host[g] = flat
                    t = self.arrays.get(g)
                    if t is None:
                        t = torch.empty(flat.numel(), dtype=flat.dtype, device=device)
                elif g in self.arrays:
                    t = self.arrays[g]
                    t.copy_(flat, non_blocking=True)
                else:
                    t = flat.to(device=device, dtype=torch_dtype(dt), copy=True, non_blocking=True)
            else:
                arr = np.asarray(data).ravel()
                if arr.size != port.shape.total:
                    raise MissingBinding(f"binding '{port.name}' has {arr.size} elements, "
                                         f"port expects {port.shape.total}")
                arr = np.ascontiguousarray(arr.astype(dt, copy=False))
                self.h2d_bytes += arr.nbytes
                g = self.groups[port.name]
                if defer:
                    self.host[g] = torch.from_numpy(arr)
                    t = self.arrays.get(g)
                    if t is None:
                        t = torch.empty(arr.size, dtype=torch_dtype(dt), device=device)
                elif g in self.arrays:
                    t = self.arrays[g]
                    t.copy_(torch.from_numpy(arr))
                else:
                    t = torch.from_numpy(arr).to(device=device, copy=True)
            self.arrays[self.groups[port.name]] = t
            bound.add(self.groups[port.name])
        for g in lay.arena_views:
            if g not in bound and g not in skip_zero:
                self.arrays[g].zero_()
        for g, (n, tdt) in lay.zero_groups.items():
            if g not in self.arrays:
                self.arrays[g] = torch.zeros(n, dtype=tdt, device=device)
                self._standalone_zero.add(g)
            elif g in self._standalone_zero and g not in bound:
                self.arrays[g].zero_()

    def array(self, node: str):
        return self.arrays[self.groups[node]]


def _task_placement_flags(model, groups: dict, path: str, spec) -> int:
    """Kernel-staging flags the MARTE placement implies for a tile task: a tiled input placed
    in deviceLocal memory (tier "smem") asks for the shared-memory-staged kernel form."""
    pg = storage_layout(model).placement
    flags = 0
    for ps in spec.ports:
        if ps.tiled and enum_value(ps.direction) in ("in", "inout"):
            pl = pg.get(groups.get(f"{path}.{ps.name}"))
            if pl is not None and pl.tier == "smem":
                flags |= _capi.FLAG_STAGE_SMEM
    return flags


class _Task:
    """A validated leaf task: spec, bound tilers, C task struct and port nodes in spec order."""

    def __init__(self, model, storage: DeviceStorage, task_path: str, tilers: dict | None, precision: str):
        comp = task_component(model, task_path)
        spec = INTRINSICS.get(comp.elementary_op) if comp.elementary_op else None
        bound = None
        if spec is not None and spec.tile:
            _ports_match_spec(task_path, comp, spec)
            bound = check_tile_signature(task_path, comp, spec, tilers)
        else:
            spec = check_task_signature(task_path, comp, tilers)
        for port in comp.ports:
            if enum_value(port.direction) != "out":
                continue
            g = storage.groups[f"{task_path}.{port.name}"]
            for other in comp.ports:
                if enum_value(other.direction) == "in" and storage.groups[f"{task_path}.{other.name}"] is g:
                    raise IntrinsicShapeMismatch(
                        f"task '{task_path}': output port '{port.name}' aliases input port '{other.name}'")
        self.comp, self.spec, self.path = comp, spec, task_path
        self.nodes = {p.name: f"{task_path}.{p.name}" for p in comp.ports}
        self.flags = 0
        self.dtype = None
        self.ctask = None
        if spec.kind != "device":
            return
        if spec.tile:
            self.dtype = enum_value(comp.port(spec.ports[0].name).data_type)
            self.flags = _task_placement_flags(model, storage.groups, task_path, spec)
            self.ctask = _capi.make_task(spec.name, self.dtype,
                                         [bound[ps.name] for ps in spec.ports if ps.tiled],
                                         precision=precision, flags=self.flags)
            self.port_order = [ps.name for ps in spec.ports]
            self.scalar_ports = []
        else:
            val = "values" if spec.name == "spmv_csr" else next(
                ps.name for ps in spec.ports if not ps.integer and not ps.scalar)
            self.dtype = enum_value(comp.port(val).data_type)
            index_dtype = enum_value(comp.port("rowptr").data_type) if spec.name == "spmv_csr" else "int32"
            self.index_dtype = index_dtype
            self.scalar_ports = [ps.name for ps in spec.ports
                                 if ps.scalar and enum_value(ps.direction) == "in" and comp.port(ps.name)]
            self.port_order = [ps.name for ps in spec.ports
                               if not (ps.scalar and enum_value(ps.direction) == "in") and comp.port(ps.name)]
            self.ctask = _capi.make_task(spec.name, self.dtype, n_scalars=len(self.scalar_ports),
                                         index_dtype=index_dtype)


class Executor:
    """Prepared schedule: storage resident in HBM, tasks validated, ready to run repeatedly."""

    _STREAMABLE_REF_OPS = ("copy", "sub", "scale", "axpy")
    # single-device runs write a covered output whole; sharded replicas each write a slice
    _SKIP_COVERED_ZERO = True

    def __init__(self, model, schedule, bindings: dict, device_count: int, *, tilers: dict | None = None,
                 precision: str = "default", device=None, stream=None, pipeline: int = 0, fuse: bool = True,
                 graphs: bool = True, defer: bool = False):
        torch = _torch()
        _capi.load()
        if not torch.cuda.is_available():
            raise _capi.NativeLibraryError("no CUDA device: the B200 executor has no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.model, self.schedule = model, schedule
        # MARTE memory allocation -> B200 placement; CapacityExceeded before anything is launched
        from .model import model_memo
        from .placement import check_private_and_tmem, plan_placement
        self.placement = plan_placement(model)
        model_memo(model, "private_tmem_checked", lambda m: check_private_and_tmem(m, self.placement) or True)
        self.device_count = device_count
        self.tilers = tilers or {}
        self.precision = precision
        self.stream = stream
        steps = [st for st in schedule.steps]
        from .intrinsics import FILTER_OPS
        # streaming splits launch ranges into chunks: only ops whose chunks are independent
        # repetitions qualify (tile ops, identity elementwise ops); spmv_csr gathers whole
        # index/value arrays and dot_partial sums one partial per launch, so they run plainly
        single = (len(steps) == 1 and hasattr(steps[0], "launches") and steps[0].op in INTRINSICS
                  and (INTRINSICS[steps[0].op].tile or steps[0].op in self._STREAMABLE_REF_OPS))
        # a two-step filter chain the fusion pass runs as one kernel streams like one step
        pair = (fuse and len(steps) == 2 and all(hasattr(s_, "launches") for s_ in steps)
                and steps[0].op in FILTER_OPS and steps[1].op in FILTER_OPS)
        self.pipeline = pipeline if (pipeline > 1 and (single or pair)) else 0
        with self._device_ctx():
            skip = covered_outputs(model) if (self._SKIP_COVERED_ZERO and not self.tilers) else frozenset()
            self.storage = DeviceStorage(model, bindings, self.device, stream, defer=defer or bool(self.pipeline),
                                         skip_zero=skip)
        self._tasks: dict[str, _Task] = {}
        self.fuse = fuse
        self.graphs = graphs
        self._loops: dict[tuple, tuple] = {}
        self._gbufs: dict[str, object] = {}
        self._dev_tasks: dict[str, object] = {}
        self.device_loops = 0
        self.persistent_loops = 0
        self.persistent = os.environ.get("AOL_LOOP_PERSISTENT", "1") != "0"
        self._programs: dict[str, object] = {}
        self._fusable: dict[tuple, bool] = {}
        self.fused_launches = 0
        self._dot_buf = None
        self.iterations = 0
        self.final_relres = None
        self.converged = True

    def rebind(self, bindings: dict) -> None:
        """Prepare this executor for another call on new bindings (execute_schedule's prepared
        executor cache): same storage, inputs copied in, everything else reset as when fresh."""
        skip = covered_outputs(self.model) if (self._SKIP_COVERED_ZERO and not self.tilers) else frozenset()
        with self._device_ctx():
            self.storage.rebind(self.model, bindings, skip)
        self.iterations = 0
        self.final_relres = None
        self.converged = True

    def _device_ctx(self):
        """``self.device`` current and the caller's stream current; no context switch at all when
        both already hold (the common single-GPU call: saves the per-call context overhead)."""
        import contextlib
        torch = _torch()
        if self.stream is None and torch.cuda.current_device() == self.device.index:
            return contextlib.nullcontext()
        stack = contextlib.ExitStack()
        stack.enter_context(torch.cuda.device(self.device))
        stack.enter_context(self._on_stream())
        return stack

    def _on_stream(self):
        """Make the caller's ``stream`` torch's current stream, so uploads, zero-fills, scalar
        reads, kernels and downloads are all ordered on it (no cross-stream races)."""
        import contextlib
        torch = _torch()
        return torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext()

    def placement_report(self) -> str:
        """Placement of every data allocation plus the staging each device task's kernel uses."""
        from .placement import emit_placement_report, kernel_staging
        lines = [emit_placement_report(self.placement)]
        for step in self.schedule.device_steps():
            t = self.task(step.task_path)
            l = step.launches[0]
            ptrs = [self.storage.array(t.nodes[n]).data_ptr() for n in t.port_order]
            name = _capi.plan_name(t.ctask, l.range.offset, l.range.count, ptrs)
            lines.append(f"task {step.task_path} ({step.op}): kernel {name}: {kernel_staging(name)}\n")
        return "".join(lines)

    def task(self, path: str) -> _Task:
        t = self._tasks.get(path)
        if t is None:
            tl = self.tilers.get(path)
            if tl is None:
                # a validated task depends only on the (immutable) model, the path and the
                # precision: validate once per model, not once per execute_schedule call
                from .model import model_memo
                t = model_memo(self.model, f"task:{path}:{self.precision}",
                               lambda m: _Task(m, self.storage, path, None, self.precision))
            else:
                t = _Task(self.model, self.storage, path, tl, self.precision)
            self._tasks[path] = t
        return t

    def _stream_handle(self) -> int:
        torch = _torch()
        s = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        return int(s.cuda_stream)

    # -- steps -------------------------------------------------------------
    def run_host(self, step) -> None:
        t = self.task(step.task_path)
        a = lambda name: self.storage.array(t.nodes[name])   # noqa: E731
        if step.op == "div":
            a("q")[0] = float(a("num")[0].item()) / float(a("den")[0].item())
        elif step.op == "neg":
            a("z")[0] = -a("a")[0].item()
        elif step.op == "rel_residual":
            a("z")[0] = math.sqrt(float(a("num")[0].item())) / math.sqrt(float(a("den")[0].item()))
        else:
            raise IntrinsicShapeMismatch(f"intrinsic '{INTRINSICS[step.op].name}' cannot run as a host scalar op")

    def run_device(self, step) -> None:
        torch = _torch()
        t = self.task(step.task_path)
        s = self._stream_handle()
        arrays = {name: self.storage.array(node) for name, node in t.nodes.items()}
        scalars = [float(arrays[n][0].item()) for n in t.scalar_ports]
        if step.op == "dot_partial":
            n = len(step.launches)
            if self._dot_buf is None or self._dot_buf.numel() < n or self._dot_buf.dtype != arrays["a"].dtype:
                self._dot_buf = torch.zeros(max(n, 8), dtype=arrays["a"].dtype, device=self.device)
            for i, l in enumerate(step.launches):
                ptrs = [arrays["a"].data_ptr(), arrays["b"].data_ptr(),
                        self._dot_buf.data_ptr() + i * self._dot_buf.element_size()]
                _capi.launch(t.ctask, l.range.offset, l.range.count, ptrs, (), s)
            partials = self._dot_buf[:n].double().cpu().tolist()
            total = 0.0
            for p in partials:                      # ascending device order (refexec.py:483-486)
                total += p
            arrays["s"][0] = total
            return
        ptrs = [arrays[name].data_ptr() for name in t.port_order]
        for l in step.launches:
            _capi.launch(t.ctask, l.range.offset, l.range.count, ptrs, scalars, s)

    # -- streamed execution from host memory -----------------------------------
    def _port_bound(self, t: _Task, name: str):
        from .distributed import _port_tiler
        return _port_tiler(self, t, name)

    def _run_streamed_gemm2d(self, step, t, out: dict | None) -> dict | None:
        """C = A B streamed from PINNED host memory in an R x S grid of C blocks.

        Row streaming (run_streamed) cannot compute any C row before all of B is resident, so
        the download of C starts only after ~half of the upload.  Here B goes up in column
        blocks (2-D copies, aol_memcpy2d) interleaved with the first row block of A, and block
        C[i, j] = A[i, :] B[:, j] is launched as soon as its operands landed -- a derived task
        over the same arrays whose tilers have the block's origin and repetition space (every
        repetition is independent, so a sub-space is a valid launch; the TF32 kernel sees an
        ordinary GEMM with offsets and leading dimensions) -- and downloaded with a 2-D copy
        while the next blocks upload.  Canonical row-major GEMM tilers, pinned torch host
        (or pageable, through the staging ring) host tensors on a single device only; returns
        None (nothing done) otherwise."""
        from .builders import gemm_tilers
        from .tiler import Tiler
        torch = _torch()
        st = self.storage
        ta, tb, tc = (self._port_bound(t, n) for n in ("a", "b", "c"))
        if len(tc.rep) != 2:
            return None
        M, N = (int(d) for d in tc.rep)
        K = int(ta.tiler.pattern[-1])
        canon = gemm_tilers(M, N, K)
        if (ta.tiler, tb.tiler, tc.tiler) != (canon["a"], canon["b"], canon["c"]):
            return None
        if (tuple(ta.array), tuple(tb.array), tuple(tc.array)) != ((M, K), (K, N), (M, N)) or K % 4 or N % 4:
            return None
        if sum(l.range.count for l in step.launches) != M * N or M < 512 or N < 512:
            return None
        ga, gb = st.groups[t.nodes["a"]], st.groups[t.nodes["b"]]
        if ga not in st.host or gb not in st.host:
            return None
        ha, hb = st.host[ga], st.host[gb]
        if ha.dtype != torch.float32 or hb.dtype != torch.float32:
            return None
        # pageable sources (numpy bindings, the reference's call) go through the pinned staging
        # ring: A rows as contiguous pieces, B column blocks gathered piece by piece
        stager = None if (ha.is_pinned() and hb.is_pinned()) else host_stager()
        root = self.model.application_components[self.model.application_root]
        yname = next((p.name for p in root.ports if enum_value(p.direction) == "out"), None)
        if yname is None or st.groups[t.nodes["c"]] is not st.groups[yname]:
            return None
        if out is not None and yname in out:
            hc = out[yname]
            hc = torch.from_numpy(hc) if isinstance(hc, np.ndarray) else hc.view(-1)
            if not hc.is_pinned() or hc.numel() != M * N or hc.dtype != torch.float32:
                return None
        else:
            hc = torch.empty(M * N, dtype=torch.float32, pin_memory=True)

        def up_rows(i0, mi):
            if stager is None:
                with torch.cuda.stream(cin):
                    A[i0 * K:(i0 + mi) * K].copy_(ha[i0 * K:(i0 + mi) * K], non_blocking=True)
            else:
                stager.copy(A[i0 * K:(i0 + mi) * K], ha[i0 * K:(i0 + mi) * K], cin)

        def up_cols(j0, nj):
            if stager is None:
                _capi.memcpy2d(pb + j0 * esz, N * esz, hb.data_ptr() + j0 * esz, N * esz, nj * esz, K, cin.cuda_stream)
            else:
                stager.copy2d(pb + j0 * esz, N * esz, hb.view(K, N)[:, j0:j0 + nj], cin)

        def cuts(n, parts):                  # block starts at multiples of 256 (whole tiles)
            step_ = max(256, -(-n // parts) // 256 * 256)
            return [(lo, min(step_, n - lo)) for lo in range(0, n, step_)]
        # The first row block of C goes block by block as B's column blocks arrive (2-D copies);
        # after that B is resident and the remaining rows go in full-width row chunks, so their
        # uploads and downloads are contiguous; the last chunk is small, because everything
        # downloaded after the last upload is pure tail.  Measured timelines
        # (tools/probe_e2e_timeline.py, C2): four equal 2-D row blocks 11.7 ms; A/B blocks
        # alternating with every C block 2-D 11.8 ms; this order 11.3 ms (row streaming: 11.5-11.8)
        rows0, cols = cuts(M, 4)[0], cuts(N, 4)
        r0 = int(os.environ.get("AOL_GEMM2D_ROWS0", "0"))          # diagnostic: first row block height
        if r0 > 0:
            rows0 = (0, min(M, max(256, r0 // 256 * 256)))
        rest = []
        lo = rows0[1]
        while lo < M:
            left = M - lo
            n = min(left, 1024) if left > 1536 else (left if left <= 512 else left - 512)
            rest.append((lo, n))
            lo += n
        if len(cols) < 2:
            return None
        A, B, Cd = st.arrays[ga], st.arrays[gb], st.array(yname)
        pa, pb, pc = A.data_ptr(), B.data_ptr(), Cd.data_ptr()
        caller = torch.cuda.current_stream(self.device) if self.stream is None else self.stream
        comp, cin, cout = side_streams(self.device)
        comp.wait_stream(caller)
        cin.wait_stream(caller)              # uploads land after the storage's zero-fills
        tl = [] if os.environ.get("AOL_E2E_TIMELINE") == "1" else None

        def mark(tag, stream):
            if tl is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                tl.append((tag, e))

        def block(i0, mi, j0, nj, tag):
            ev = torch.cuda.Event()
            ev.record(cin)
            comp.wait_event(ev)
            task = _capi.make_task("matmul", "float32", [
                Tiler((i0, 0), ((1, 0), (0, 0)), ((0,), (1,)), (K,)).bind((M, K), (mi, nj)),
                Tiler((0, j0), ((0, 0), (0, 1)), ((1,), (0,)), (K,)).bind((K, N), (mi, nj)),
                Tiler((i0, j0), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((M, N), (mi, nj))],
                precision=self.precision)
            _capi.launch(task, 0, mi * nj, [pa, pb, pc], (), int(comp.cuda_stream))
            mark(f"gemm {tag}", comp)
            ev_done = torch.cuda.Event()
            ev_done.record(comp)
            cout.wait_event(ev_done)
            if nj == N:
                with torch.cuda.stream(cout):
                    hc[i0 * N:(i0 + mi) * N].copy_(Cd[i0 * N:(i0 + mi) * N], non_blocking=True)
            else:
                _capi.memcpy2d(hc.data_ptr() + (i0 * N + j0) * esz, N * esz, pc + (i0 * N + j0) * esz, N * esz,
                               nj * esz, mi, cout.cuda_stream)
            mark(f"d2h {tag}", cout)
        mark("start", cin)
        esz = 4
        i0, mi = rows0
        up_rows(i0, mi)
        mark("h2d A0", cin)
        for bj, (j0, nj) in enumerate(cols):
            up_cols(j0, nj)
            mark(f"h2d B{bj}", cin)
            block(i0, mi, j0, nj, f"C0{bj}")
        for bi, (i0, mi) in enumerate(rest, start=1):
            up_rows(i0, mi)
            mark(f"h2d A{bi}", cin)
            block(i0, mi, 0, N, f"C{bi}")
        cout.synchronize()
        comp.synchronize()
        caller.wait_stream(comp)
        if tl is not None:
            self.timeline = [(tag, tl[0][1].elapsed_time(e)) for tag, e in tl]
        if out is not None and yname in out:
            return {yname: out[yname]}
        return {yname: hc.numpy()}

    def _upload_deferred(self) -> None:
        """Copy every deferred host binding to its device array (streaming fell through)."""
        st = self.storage
        for g, h in st.host.items():
            st.arrays[g].copy_(h, non_blocking=True)

    def _dense_stream_rep(self, bt):
        from .distributed import dense_stream
        return dense_stream(bt)

    def _run_streamed_pair(self, s1, s2, out: dict | None) -> dict | None:
        """Stream a fusable producer -> consumer filter chain: consumer chunks in order; each
        chunk's producer-input ranges (consumer input ranges on the intermediate, mapped to
        producer repetitions through its dense output stream, then the producer's input
        ranges) go up on one stream, the fused kernel runs on another, the chunk's output
        comes down on a third.  Returns None (nothing run) when the pair is not streamable."""
        from .distributed import add_range, input_hull, input_ranges, missing_ranges
        torch = _torch()
        if not self._fusion_candidate(s1, s2) or len(s2.launches) != 1:
            return None
        t1, t2 = self.task(s1.task_path), self.task(s2.task_path)
        bx, bm_out, bm_in, by = (self._port_bound(t1, "x"), self._port_bound(t1, "y"),
                                 self._port_bound(t2, "x"), self._port_bound(t2, "y"))
        ds = self._dense_stream_rep(bm_out)
        if ds is None:
            return None
        c0, P1 = ds
        st = self.storage
        xg = st.groups[t1.nodes["x"]]
        if xg not in st.host:
            return None
        a1 = [st.array(t1.nodes[n]).data_ptr() for n in t1.port_order]
        a2 = [st.array(t2.nodes[n]).data_ptr() for n in t2.port_order]
        # an empty launch is the library's fusability query: nothing runs, EUNSUPPORTED -> False
        if not _capi.launch_fused2(t1.ctask, t2.ctask, 0, 0, a1, a2, self._stream_handle()):
            self._fusable[(s1.task_path, s2.task_path)] = False
            return None
        comp = torch.cuda.current_stream(self.device) if self.stream is None else self.stream
        _, cin, cout = side_streams(self.device)
        cin.wait_stream(comp)            # uploads land after the storage's zero-fills
        # whole-array inputs (filter weights) first
        with torch.cuda.stream(cin):
            for t in (t1, t2):
                g = st.groups[t.nodes["w"]]
                if g in st.host:
                    st.arrays[g].copy_(st.host[g], non_blocking=True)
        comp.wait_stream(cin)
        xdev, xhost = st.arrays[xg], st.host[xg]
        stager = host_stager()
        root = self.model.application_components[self.model.application_root]
        yname = next(p.name for p in root.ports if enum_value(p.direction) == "out")
        ydev = st.array(yname)
        if st.groups[t2.nodes["y"]] is not st.groups[yname]:
            return None
        if out is not None and yname in out:
            h = out[yname]
            yhost = torch.from_numpy(h) if isinstance(h, np.ndarray) else h.view(-1)
        else:
            yhost = torch.empty(ydev.numel(), dtype=ydev.dtype, pin_memory=True)
        l = s2.launches[0]
        uploaded: list = []
        covered: list = []
        for off, cnt in partition_equally_local(l.range.count, self.pipeline):
            first = l.range.offset + off
            with torch.cuda.stream(cin):
                for lo, hi in input_ranges(bm_in, first, cnt):
                    r_lo = max(0, (lo - c0) // P1)
                    r_hi = min(bx.rep_total, -(-(hi - c0) // P1))
                    if r_hi <= r_lo:
                        continue
                    for xlo, xhi in input_ranges(bx, r_lo, r_hi - r_lo):
                        for a, b in missing_ranges(uploaded, xlo, xhi):
                            stager.copy(xdev[a:b], xhost[a:b], cin)
                            uploaded = add_range(uploaded, a, b)
                ev_in = torch.cuda.Event()
                ev_in.record(cin)
            comp.wait_event(ev_in)
            if not _capi.launch_fused2(t1.ctask, t2.ctask, first, cnt, a1, a2, int(comp.cuda_stream)):
                raise RuntimeError("fused pair became unsupported mid-stream")
            self.fused_launches += 1
            ev_done = torch.cuda.Event()
            ev_done.record(comp)
            cout.wait_event(ev_done)
            with torch.cuda.stream(cout):
                lo, hi = input_hull(by, first, cnt)
                yhost[lo:hi].copy_(ydev[lo:hi], non_blocking=True)
                covered.append((lo, hi))
        with torch.cuda.stream(cout):            # never-written elements keep the zero init
            pos = 0
            for lo, hi in sorted(covered) + [(ydev.numel(), ydev.numel())]:
                if lo > pos:
                    yhost[pos:lo].copy_(ydev[pos:lo], non_blocking=True)
                pos = max(pos, hi)
        cout.synchronize()
        comp.synchronize()
        return {yname: (out[yname] if out is not None and yname in out else yhost.numpy())}

    def run_streamed(self, out: dict | None = None) -> dict:
        """Run a one-step schedule chunk by chunk straight from host memory.

        Each launch range is split into ``pipeline`` contiguous chunks.  For
        chunk c: the part of every input's ranges (distributed.input_ranges) not
        yet resident is copied H2D on a copy stream; the chunk launches on the
        compute stream once its inputs landed; its output hull is copied D2H
        on a third stream.  PCIe upload, tensor-core compute and download of
        consecutive chunks overlap.  Returns the root outputs (host).
        """
        from .distributed import add_range, input_hull, input_ranges, missing_ranges
        torch = _torch()
        steps = list(self.schedule.steps)
        if len(steps) == 2:
            res = self._run_streamed_pair(steps[0], steps[1], out)
            if res is not None:
                return res
            self._upload_deferred()               # not streamable: plain run on the uploaded inputs
            self.run()
            return self.outputs(out=out)
        step = steps[0]
        t = self.task(step.task_path)
        if step.op == "matmul":
            res = self._run_streamed_gemm2d(step, t, out)
            if res is not None:
                return res
        comp = torch.cuda.current_stream(self.device) if self.stream is None else self.stream
        _, cin, cout = side_streams(self.device)
        cin.wait_stream(comp)            # uploads land after the storage's zero-fills
        st = self.storage
        arrays = {name: st.array(node) for name, node in t.nodes.items()}
        in_ports = [ps.name for ps in t.spec.ports if enum_value(ps.direction) in ("in", "inout")
                    and t.comp.port(ps.name) and st.groups[t.nodes[ps.name]] in st.host]
        out_ports = [ps.name for ps in t.spec.ports if enum_value(ps.direction) in ("out", "inout")
                     and t.comp.port(ps.name)]
        # whole-array inputs (filter coefficients, scalars) go up first; tiled / identity
        # vector inputs stream chunk by chunk through their hulls
        whole = [n for n in in_ports if (t.spec.tile and not t.spec.port_spec(n).tiled)
                 or t.spec.port_spec(n).scalar]
        in_ports = [n for n in in_ports if n not in whole]
        bound = {n: self._port_bound(t, n) for n in in_ports + out_ports}
        uploaded: dict[str, list] = {n: [] for n in in_ports}
        root = self.model.application_components[self.model.application_root]
        root_out = {p.name: st.array(p.name) for p in root.ports if enum_value(p.direction) == "out"}
        hosts = {}
        for name, dev in root_out.items():
            if out is not None and name in out:
                h = out[name]
                hosts[name] = torch.from_numpy(h) if isinstance(h, np.ndarray) else h.view(-1)
            else:
                hosts[name] = torch.empty(dev.numel(), dtype=dev.dtype, pin_memory=True)
        out_group = {n: st.groups[t.nodes[n]] for n in out_ports}
        root_of = {st.groups[n]: n for n in root_out}
        covered = {n: [] for n in out_ports}
        ptrs = [arrays[name].data_ptr() for name in t.port_order]
        with torch.cuda.stream(cin):
            for n in whole:
                arrays[n].copy_(st.host[st.groups[t.nodes[n]]], non_blocking=True)
        comp.wait_stream(cin)
        scal = []
        for n in t.scalar_ports:
            g = st.groups[t.nodes[n]]
            scal.append(float(st.host[g][0]) if g in st.host else float(arrays[n][0].item()))
        chunks = []
        for l in step.launches:
            for r in partition_equally_local(l.range.count, self.pipeline):
                chunks.append((l.range.offset + r[0], r[1]))

        stager = host_stager()

        def upload(name, lo, hi):
            g = st.groups[t.nodes[name]]
            if hi > lo:
                stager.copy(arrays[name][lo:hi], st.host[g][lo:hi], cin)

        for first, count in chunks:
            with torch.cuda.stream(cin):
                for n in in_ports:
                    need = input_ranges(bound[n], first, count) if n in bound else [(0, arrays[n].numel())]
                    for lo, hi in need:
                        for a, b in missing_ranges(uploaded[n], lo, hi):
                            upload(n, a, b)
                            uploaded[n] = add_range(uploaded[n], a, b)
                ev_in = torch.cuda.Event()
                ev_in.record(cin)
            comp.wait_event(ev_in)
            _capi.launch(t.ctask, first, count, ptrs, scal, int(comp.cuda_stream))
            ev_done = torch.cuda.Event()
            ev_done.record(comp)
            cout.wait_event(ev_done)
            with torch.cuda.stream(cout):
                for n in out_ports:
                    rn = root_of.get(out_group[n])
                    if rn is None:
                        continue
                    lo, hi = input_hull(bound[n], first, count)
                    hosts[rn][lo:hi].copy_(root_out[rn][lo:hi], non_blocking=True)
                    covered[n].append((lo, hi))
        # elements no chunk wrote keep the zero initialisation (refexec.py:399-403) -- or, for an
        # inout group the caller bound, its bound values, which were uploaded only where a chunk
        # read them: take those from the host source
        with torch.cuda.stream(cout):
            for n in out_ports:
                rn = root_of.get(out_group[n])
                if rn is None:
                    continue
                bound_src = st.host.get(out_group[n])
                pos = 0
                for lo, hi in sorted(covered[n]) + [(root_out[rn].numel(), root_out[rn].numel())]:
                    if lo > pos:
                        if bound_src is not None:
                            hosts[rn][pos:lo].copy_(bound_src[pos:lo])
                        else:
                            hosts[rn][pos:lo].copy_(root_out[rn][pos:lo], non_blocking=True)
                    pos = max(pos, hi)
        cout.synchronize()
        comp.synchronize()
        return {n: (out[n] if out is not None and n in out else h.numpy()) for n, h in hosts.items()}

    # -- CUDA-graph loop bodies -----------------------------------------------------
    _GRAPH_HOST_OPS = ("div", "neg", "rel_residual")

    def _graphable(self, body) -> bool:
        for st in body:
            if hasattr(st, "body"):
                return False
            if not hasattr(st, "launches") and st.op not in self._GRAPH_HOST_OPS:
                return False
        return True

    def _dev_task(self, step):
        """Device-resident variant of a step's task: host scalar ops as kernels, scalar inputs by pointer."""
        d = self._dev_tasks.get(step.task_path)
        if d is None:
            t = self.task(step.task_path)
            if not hasattr(step, "launches"):
                dt = enum_value(t.comp.ports[0].data_type)
                d = (_capi.make_task(step.op, dt), [ps.name for ps in t.spec.ports])
            elif step.op in ("scale", "axpy") and t.scalar_ports:
                d = (_capi.make_task(step.op, t.dtype, n_scalars=len(t.scalar_ports),
                                     flags=_capi.FLAG_DEVICE_SCALARS), t.port_order + t.scalar_ports)
            else:
                d = (t.ctask, t.port_order)
            self._dev_tasks[step.task_path] = d
        return d

    def _run_body_device(self, body) -> None:
        """Enqueue one loop iteration with no host round trip (capturable).

        Consecutive host scalar ops of one dtype go out as ONE scalar_seq launch; a dot
        with a single launch writes its result straight into `s` (the kernel stores
        0.0 + partial, which is the reference's combine of one partial)."""
        s = self._stream_handle()
        i = 0
        while i < len(body):
            step = body[i]
            t = self.task(step.task_path)
            arrays = {name: self.storage.array(node) for name, node in t.nodes.items()}
            if not hasattr(step, "launches"):
                j = i
                dt = enum_value(t.comp.ports[0].data_type)
                while (j < len(body) and j - i < 8 and not hasattr(body[j], "launches")
                       and enum_value(self.task(body[j].task_path).comp.ports[0].data_type) == dt):
                    j += 1
                self._scalar_seq(body[i:j], dt, s)
                i = j
                continue
            i += 1
            if step.op == "dot_partial":
                if len(step.launches) == 1:
                    l = step.launches[0]
                    _capi.launch(t.ctask, l.range.offset, l.range.count,
                                 [arrays["a"].data_ptr(), arrays["b"].data_ptr(), arrays["s"].data_ptr()], (), s)
                    continue
                buf = self._gbufs[step.task_path]
                for k, l in enumerate(step.launches):
                    _capi.launch(t.ctask, l.range.offset, l.range.count,
                                 [arrays["a"].data_ptr(), arrays["b"].data_ptr(),
                                  buf.data_ptr() + k * buf.element_size()], (), s)
                ctask = _capi.make_task("partials_sum", t.dtype)
                _capi.launch(ctask, 0, len(step.launches), [buf.data_ptr(), arrays["s"].data_ptr()], (), s)
                continue
            ctask, names = self._dev_task(step)
            ptrs = [arrays[n].data_ptr() for n in names]
            for l in step.launches:
                _capi.launch(ctask, l.range.offset, l.range.count, ptrs, (), s)

    def _scalar_seq(self, ops, dtype: str, stream) -> None:
        """Host scalar ops (refexec.py:462-474) as one device launch, in program order."""
        ptrs: list[int] = []
        index: dict[int, int] = {}

        def slot(ptr: int) -> int:
            if ptr not in index:
                index[ptr] = len(ptrs)
                ptrs.append(ptr)
            return index[ptr]
        prog: list[float] = []
        for op in ops:
            t = self.task(op.task_path)
            names = [ps.name for ps in t.spec.ports]
            p = [self.storage.array(t.nodes[n]).data_ptr() for n in names]
            if op.op == "neg":
                prog += [_capi.OP["neg"], slot(p[0]), -1, slot(p[1])]
            else:
                prog += [_capi.OP[op.op], slot(p[0]), slot(p[1]), slot(p[2])]
        _capi.launch(_capi.make_task("scalar_seq", dtype), 0, len(ops), ptrs, prog, stream)

    _PERSISTENT_OPS = ("copy", "sub", "scale", "axpy", "spmv_csr", "dot_partial")

    def _persistent_program(self, step):
        """The LoopStep body as an aol_loop_persistent program: (ops, ports, dtype, index dtype,
        relres slot), or None when it has ops outside the interpreter's set."""
        ptrs: list[int] = []
        slots: dict[int, int] = {}

        def slot(arr) -> int:
            p = arr.data_ptr()
            if p not in slots:
                slots[p] = len(ptrs)
                ptrs.append(p)
            return slots[p]
        ops, dtypes, index = [], set(), set()
        for st in step.body:
            if hasattr(st, "body"):
                return None
            t = self.task(st.task_path)
            arr = {n: self.storage.array(node) for n, node in t.nodes.items()}
            if not hasattr(st, "launches"):
                if st.op not in self._GRAPH_HOST_OPS:
                    return None
                dtypes.add(enum_value(t.comp.ports[0].data_type))
                ops.append(_capi.loop_op(st.op, [slot(arr[ps.name]) for ps in t.spec.ports]))
                continue
            if st.op not in self._PERSISTENT_OPS:
                return None
            dtypes.add(t.dtype)
            if st.op == "spmv_csr":
                index.add(t.index_dtype)
            ports = [slot(arr[n]) for n in t.port_order + t.scalar_ports]
            for k, l in enumerate(st.launches):
                ops.append(_capi.loop_op(st.op, ports, l.range.offset, l.range.count,
                                         n_scalars=len(t.scalar_ports), part=k, n_parts=len(st.launches)))
        if len(dtypes) != 1 or len(index) > 1:
            return None
        relres = slot(self.storage.array(step.relres_port))
        return ops, ptrs, dtypes.pop(), index.pop() if index else "int32", relres

    def _loop_device(self, step, tol: float, max_iter: int):
        """Run a LoopStep on the device with no host round trip per iteration.

        First choice: ONE persistent cooperative kernel interpreting the body
        (aol_loop_persistent).  Otherwise: one CUDA graph with a conditional WHILE node
        (aol_loop_begin/end/run).  Both are bit-identical to the eager interpreter."""
        torch = _torch()
        if self.persistent:
            prog = self._programs.get(step.task_path, False)
            if prog is False:
                prog = self._programs[step.task_path] = self._persistent_program(step)
            if prog is not None:
                ops, ptrs, dt, idt, rr = prog
                res = _capi.loop_persistent(ops, ptrs, dt, idt, rr, tol, max(1, int(max_iter)),
                                            self._stream_handle())
                if res is not None:
                    self.device_loops += 1
                    self.persistent_loops += 1
                    return res
                self._programs[step.task_path] = None
        key = (step.task_path, tol, max_iter)
        entry = self._loops.get(key)
        if entry is None:
            for st in step.body:                   # everything allocated before capture
                if getattr(st, "op", None) == "dot_partial":
                    t = self.task(st.task_path)
                    self._gbufs[st.task_path] = torch.zeros(max(8, len(st.launches)),
                                                            dtype=torch_dtype(t.dtype), device=self.device)
                else:
                    self._dev_task(st)
            stream = torch.cuda.Stream(self.device)          # captures need a non-default stream
            relres = self.storage.array(step.relres_port)
            torch.cuda.synchronize(self.device)
            handle = None
            # the body's launches go to the capture stream, also when the caller passed stream=:
            # launched on the caller's stream they would run once, eagerly, outside the graph
            caller_stream, self.stream = self.stream, stream
            try:
                with torch.cuda.stream(stream):
                    handle = _capi.loop_begin(stream.cuda_stream, relres.data_ptr(),
                                              str(relres.dtype).replace("torch.", ""), tol, max(1, int(max_iter)))
                    try:
                        self._run_body_device(step.body)
                    finally:
                        try:
                            _capi.loop_end(handle)
                        except Exception:
                            _capi.loop_destroy(handle)
                            raise
            finally:
                self.stream = caller_stream
            entry = (handle, stream)
            self._loops[key] = entry
        handle, stream = entry
        stream.wait_stream(torch.cuda.current_stream(self.device))
        self.device_loops += 1
        return _capi.loop_run(handle, stream.cuda_stream)

    def __del__(self):
        for handle, _ in getattr(self, "_loops", {}).values():
            try:
                _capi.loop_destroy(handle)
            except Exception:
                pass

    # -- task fusion ---------------------------------------------------------------
    def _fusion_candidate(self, s1, s2) -> bool:
        """s1's filter output feeds s2's filter input through a group nobody else touches."""
        from .intrinsics import FILTER_OPS
        key = (s1.task_path, s2.task_path)
        if key in self._fusable:
            return self._fusable[key]
        ok = False
        if self.fuse and s1.op in FILTER_OPS and s2.op in FILTER_OPS:
            st = self.storage
            g = st.groups.get(f"{s1.task_path}.y")
            ok = g is not None and g is st.groups.get(f"{s2.task_path}.x") and \
                set(g) == {f"{s1.task_path}.y", f"{s2.task_path}.x"}
        self._fusable[key] = ok
        return ok

    def _run_fused(self, s1, s2) -> bool:
        t1, t2 = self.task(s1.task_path), self.task(s2.task_path)
        a1 = [self.storage.array(t1.nodes[n]).data_ptr() for n in t1.port_order]
        a2 = [self.storage.array(t2.nodes[n]).data_ptr() for n in t2.port_order]
        st = self._stream_handle()
        for i, l in enumerate(s2.launches):
            if not _capi.launch_fused2(t1.ctask, t2.ctask, l.range.offset, l.range.count, a1, a2, st):
                if i == 0:
                    self._fusable[(s1.task_path, s2.task_path)] = False
                    return False
                raise RuntimeError("fusion became unsupported mid-step")
            self.fused_launches += 1
        return True

    def run_steps(self, steps, tol=None, max_iter=None) -> None:
        steps = list(steps)
        i = 0
        while i < len(steps):
            step = steps[i]
            nxt = steps[i + 1] if i + 1 < len(steps) else None
            if (hasattr(step, "launches") and nxt is not None and hasattr(nxt, "launches")
                    and self._fusion_candidate(step, nxt) and self._run_fused(step, nxt)):
                i += 2
                continue
            i += 1
            if hasattr(step, "launches"):
                self.run_device(step)
            elif hasattr(step, "body"):
                loop_tol = tol if tol is not None else step.tolerance
                loop_max = max_iter if max_iter is not None else step.max_iterations
                done = False
                n = 0
                if self.graphs and self._graphable(step.body):
                    n, relres, done = self._loop_device(step, loop_tol, loop_max)
                    self.iterations += n
                    self.final_relres = relres
                    self.converged = self.converged and done
                    continue
                while True:
                    self.run_steps(step.body, tol, max_iter)
                    n += 1
                    self.iterations += 1
                    relres = float(self.storage.array(step.relres_port)[0].item())
                    self.final_relres = relres
                    if relres <= loop_tol:
                        done = True
                        break
                    if n >= loop_max:
                        break
                self.converged = self.converged and done
            else:
                self.run_host(step)

    def run(self, tol=None, max_iter=None) -> None:
        torch = _torch()
        with self._device_ctx():
            self.run_steps(self.schedule.steps, tol, max_iter)

    # numpy outputs up to this size come back in pinned blocks (the caller keeps them: a cap on
    # how much page-locked memory results can pin); larger ones go through the staging ring
    PINNED_OUTPUT_BYTES = 8 << 20

    def outputs(self, on_device: bool = False, out: dict | None = None) -> dict:
        """Root out-port arrays, flat row-major (refexec.py:545-547).

        ``out`` maps port name -> caller-owned host buffer (numpy array or
        pinned torch tensor) that receives the result instead of a fresh array.
        """
        torch = _torch()
        with self._device_ctx():
            return self._outputs(on_device, out)

    def _outputs(self, on_device: bool, out: dict | None) -> dict:
        torch = _torch()
        root = self.model.application_components[self.model.application_root]
        res = {}
        pending = False
        for port in root.ports:
            if enum_value(port.direction) != "out":
                continue
            t = self.storage.array(port.name)
            if out is not None and port.name in out:
                dst = out[port.name]
                host = torch.from_numpy(dst) if isinstance(dst, np.ndarray) else dst
                if host.numel() != t.numel():
                    raise MissingBinding(f"output buffer '{port.name}' has {host.numel()} elements, "
                                         f"port has {t.numel()}")
                host.view(-1).copy_(t, non_blocking=True)
                pending = True
                res[port.name] = dst
            elif on_device:
                res[port.name] = t.clone()
            elif t.numel() * t.element_size() <= self.PINNED_OUTPUT_BYTES:
                # a DMA from the device into pageable memory is staged by the driver piece by
                # piece (~2x slower than into pinned memory at 0.25-4 MB,
                # tools/probe_small_copies.py); small outputs land in a block of torch's
                # caching pinned allocator, handed to the caller as the numpy array's base
                host = torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
                host.copy_(t, non_blocking=True)
                pending = True
                res[port.name] = host.numpy()
            else:
                host = torch.empty(t.numel(), dtype=t.dtype)
                host_stager().download(host, t.reshape(-1), torch.cuda.current_stream(self.device))
                res[port.name] = host.numpy()
        if pending:
            torch.cuda.current_stream(self.device).synchronize()
        return res


# Prepared-executor cache: repeated small calls on the same (model, schedule) -- the C1 regime,
# where building the storage and validating tasks costs more than the kernels -- reuse one
# Executor: its HBM arena is refilled (inputs copied, other groups zeroed as when fresh) and the
# outputs are always copied out (clone / host copy), so no call sees another's data.  Only
# schedules of device steps, arenas up to AOL_PREPARED_ARENA_MB (default 64), at most
# AOL_PREPARED_MAX entries (default 8, 0 disables); a busy entry (another thread) is bypassed.
_PREPARED: dict = {}
_PREPARED_LOCK = __import__("threading").Lock()   # guards the dict; each entry has its own lock
_PREPARED_MAX = int(os.environ.get("AOL_PREPARED_MAX", "8"))
_PREPARED_ARENA = int(os.environ.get("AOL_PREPARED_ARENA_MB", "64")) << 20


def _prepared_executor(model, schedule, bindings, device_count, precision, device, fuse, graphs):
    """(executor rebound to ``bindings``, its held lock), or None (not cacheable / busy)."""
    import threading
    import weakref
    torch = _torch()
    if not torch.cuda.is_available():
        return None
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if sum(storage_layout(model).arenas.values()) > _PREPARED_ARENA:
        return None
    key = (id(model), id(schedule), device_count, precision, str(dev), fuse, graphs)
    with _PREPARED_LOCK:
        ent = _PREPARED.get(key)
        if ent is not None and (ent[0]() is not model or ent[1]() is not schedule):
            _PREPARED.pop(key, None)             # ids reused by new objects
            ent = None
        if ent is not None:
            _, _, ex, lock = ent
            if not lock.acquire(blocking=False):
                return None                      # busy (another thread): build a fresh executor
            _PREPARED[key] = _PREPARED.pop(key)  # most recently used last
    if ent is None:
        try:
            mref, sref = weakref.ref(model), weakref.ref(schedule)
        except TypeError:
            return None
        ex = Executor(model, schedule, bindings, device_count, precision=precision, device=dev, fuse=fuse,
                      graphs=graphs)
        lock = threading.Lock()
        lock.acquire()
        with _PREPARED_LOCK:
            if key in _PREPARED:                 # another thread cached one meanwhile: ours runs once
                return ex, lock
            while len(_PREPARED) >= _PREPARED_MAX:
                _PREPARED.pop(next(iter(_PREPARED)))
            _PREPARED[key] = (mref, sref, ex, lock)
        return ex, lock
    try:
        ex.rebind(bindings)
    except BaseException:
        lock.release()
        raise
    return ex, lock


def clear_prepared() -> None:
    """Drop every cached prepared executor (frees their HBM arenas)."""
    with _PREPARED_LOCK:
        _PREPARED.clear()


def _default_devices(device_count: int, device, pipeline: int):
    """Launch d of a step goes to cuda:(d mod P) when P > 1 GPUs are visible (P = min(D, visible));
    None keeps every launch on one device (one GPU, an explicit ``device``, the streamed path,
    or AOL_MULTI_DEVICE=0)."""
    if device is not None or device_count < 2 or pipeline > 1 or os.environ.get("AOL_MULTI_DEVICE", "1") == "0":
        return None
    torch = _torch()
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        return None
    return [torch.device("cuda", i) for i in range(min(device_count, n))]


def execute_schedule(model, schedule, bindings: dict, device_count: int, tol: float | None = None,
                     max_iter: int | None = None, *, tilers: dict | None = None, precision: str = "default",
                     device_outputs: bool = False, out: dict | None = None, device=None,
                     stream=None, pipeline: int = 0, fuse: bool = True, graphs: bool = True,
                     devices: list | None = None) -> ExecutionResult:
    """Interpret ``schedule`` on the B200 with ``device_count`` launch shards per device step.

    ``graphs`` (default on): a LoopStep runs on the device -- the persistent interpreter, else
    one CUDA graph with a WHILE node -- bit-identical to host-driven iterations (graphs=False).
    ``devices``: run launch d on ``devices[d mod len(devices)]`` (one replica of the storage per
    entry; only what crosses shards is exchanged, outputs gather to ``devices[0]``).  By default
    the D launches spread over min(D, visible GPUs) devices."""
    if devices is None:
        devices = _default_devices(device_count, device, pipeline)
    if devices is not None and len(devices) > 1:
        from .distributed import make_sharded_executor
        ex = make_sharded_executor(model, schedule, bindings, device_count, list(devices), tilers=tilers,
                                   precision=precision, stream=stream, fuse=fuse)
        ex.run(tol, max_iter)
        outs = ex.outputs(on_device=device_outputs, out=out)
        return ExecutionResult(outputs=outs, iterations=ex.iterations, final_relres=ex.final_relres,
                               converged=ex.converged)
    prepared = None
    if (stream is None and tilers is None and not pipeline and _PREPARED_MAX > 0
            and all(hasattr(st, "launches") for st in schedule.steps)):
        prepared = _prepared_executor(model, schedule, bindings, device_count, precision, device, fuse, graphs)
    if prepared is not None:
        ex, lock = prepared
        try:
            ex.run(tol, max_iter)
            outs = ex.outputs(on_device=device_outputs, out=out)
        finally:
            lock.release()
        return ExecutionResult(outputs=outs, iterations=ex.iterations, final_relres=ex.final_relres,
                               converged=ex.converged)
    ex = Executor(model, schedule, bindings, device_count, tilers=tilers, precision=precision,
                  device=device, stream=stream, pipeline=0 if device_outputs else pipeline, fuse=fuse,
                  graphs=graphs)
    if ex.pipeline:
        torch = _torch()
        with torch.cuda.device(ex.device), ex._on_stream():
            outs = ex.run_streamed(out)
    else:
        ex.run(tol, max_iter)
        outs = ex.outputs(on_device=device_outputs, out=out)
    return ExecutionResult(outputs=outs, iterations=ex.iterations, final_relres=ex.final_relres,
                           converged=ex.converged)
