"""Programmatic single-task models — the reference test harness, without its DSL.

Builds the model that the reference suite writes as text in
``SINGLE_TASK`` / ``_single_task_model`` (pkg/tests/test_refexec.py:250-293):
a host (cpu + hostRam), one device processor ``dev.cu`` of 4 compute units
x 8 processing elements, and a ``dev.gmem`` global memory; one repetitive
task ``t`` of type ``T`` deployed on ``dev.cu`` inside root ``m``.  Port and
allocation specs use the same strings as that harness
(``"src in float32 [64]"``, ``"allocate data i onto dev.gmem"``), so the
GPU tests read like the reference's own.
"""

from __future__ import annotations

import re

from .model import (AllocationLink, AllocKind, Component, ComponentKind, Connector, DataType, Direction,
                    FlowPort, HwStereotype, MemoryRole, Model, PartInstance, Shape, StereotypeKind)
from .tiler import Tiler

_PORT = re.compile(r"^\s*(\w+)\s+(in|out|inout)\s+(float32|float64|int32|int64)\s+\[([\d,\s]+)\]\s*$")
_ALLOC = re.compile(r"^\s*allocate\s+(data|task)\s+([\w.]+)\s+onto\s+([\w.]+)\s*$")


def port(spec: str) -> FlowPort:
    m = _PORT.match(spec)
    if not m:
        raise ValueError(f"bad port spec {spec!r}")
    dims = tuple(int(d) for d in m.group(4).split(","))
    return FlowPort(m.group(1), Direction(m.group(2)), Shape(dims), DataType(m.group(3)))


def platform(cus: int = 4, pes: int = 8, local_capacity: int | None = None) -> dict:
    P = ComponentKind.PLATFORM
    comps = {
        "Host": Component("Host", P, parts=(PartInstance("cpu", "Cpu"), PartInstance("ram", "Ram"))),
        "Cpu": Component("Cpu", P, stereotype=HwStereotype(StereotypeKind.PROCESSOR)),
        "Ram": Component("Ram", P, stereotype=HwStereotype(StereotypeKind.MEMORY, MemoryRole.HOST_RAM)),
        "Pe": Component("Pe", P, stereotype=HwStereotype(StereotypeKind.PROCESSOR)),
        "Cu": Component("Cu", P, parts=(PartInstance("pe", "Pe", Shape((pes,))),)
                        + ((PartInstance("lmem", "Lmem"),) if local_capacity else ()),
                        stereotype=HwStereotype(StereotypeKind.PROCESSOR)),
        "Gmem": Component("Gmem", P, stereotype=HwStereotype(StereotypeKind.MEMORY, MemoryRole.DEVICE_GLOBAL)),
        "Cmem": Component("Cmem", P, stereotype=HwStereotype(StereotypeKind.MEMORY, MemoryRole.DEVICE_CONSTANT)),
        "Dev": Component("Dev", P, parts=(PartInstance("cu", "Cu", Shape((cus,))), PartInstance("gmem", "Gmem"),
                                          PartInstance("cmem", "Cmem"))),
        "p": Component("p", P, parts=(PartInstance("host", "Host"), PartInstance("dev", "Dev"))),
    }
    if local_capacity:
        comps["Lmem"] = Component("Lmem", P, stereotype=HwStereotype(
            StereotypeKind.MEMORY, MemoryRole.DEVICE_LOCAL, capacity_bytes=local_capacity))
    return comps


def allocation(spec: str) -> AllocationLink:
    m = _ALLOC.match(spec)
    if not m:
        raise ValueError(f"bad allocation spec {spec!r}")
    return AllocationLink(AllocKind(m.group(1)), m.group(2), m.group(3))


def single_task_model(op: str, ports, root_ports, conns, allocs, n=None, *, repeat=None,
                      tilers: dict[str, Tiler] | None = None) -> Model:
    """The reference harness's one-task model; ``repeat`` (dims) overrides ``[n]``."""
    A = ComponentKind.APPLICATION
    rep = Shape(tuple(repeat)) if repeat is not None else (Shape((n,)) if n is not None else None)
    task = Component("T", A, ports=tuple(port(p) for p in ports), repetition_space=rep, elementary_op=op,
                     tilers=tuple(sorted((tilers or {}).items())))
    conn = []
    for c in conns:
        src, dst = (s.strip() for s in c.split("->"))
        conn.append(Connector(src, dst))
    root = Component("m", A, ports=tuple(port(p) for p in root_ports), parts=(PartInstance("t", "T"),),
                     connectors=tuple(conn))
    return Model(platform_components=platform(), application_components={"T": task, "m": root},
                 platform_root="p", application_root="m",
                 allocations=tuple(allocation(a) for a in allocs))


def tile_task_model(op: str, ports: dict[str, str], tilers: dict[str, Tiler], repeat) -> Model:
    """Single tile-intrinsic task whose root ports mirror the task ports one to one.

    ``ports`` maps task port name -> "<dir> <dtype> [dims]"; root port names
    are the task port names prefixed with ``p_``.
    """
    tp, rp, conns, allocs = [], [], [], []
    for name, spec in ports.items():
        tp.append(f"{name} {spec}")
        rp.append(f"p_{name} {spec}")
        d = spec.split()[0]
        if d == "out":
            conns.append(f"t.{name} -> p_{name}")
            allocs.append(f"allocate data t.{name} onto dev.gmem")
        else:
            conns.append(f"p_{name} -> t.{name}")
            allocs.append(f"allocate data p_{name} onto dev.gmem")
    allocs.append("allocate task t onto dev.cu")
    return single_task_model(op, tp, rp, conns, allocs, repeat=repeat, tilers=tilers)


def chain_model(stages: list[tuple[str, str, dict[str, str], dict[str, Tiler], tuple]], root_in: dict[str, str],
                root_out: dict[str, str], links: list[tuple[str, str]]) -> Model:
    """Several repetitive tasks wired by connectors (one storage group per connected port set).

    ``stages``: (part name, op, {port: "<dir> <dtype> [dims]"}, tilers, repeat);
    ``root_in`` / ``root_out``: root port name -> spec; ``links``: (source, target)
    endpoints in the reference connector syntax ("x", "h.x", "h.y" ...).  Every
    root input and every task output is allocated onto dev.gmem and every task
    onto dev.cu (the device-processor geometry of the reference harness).
    """
    A = ComponentKind.APPLICATION
    comps = {}
    parts = []
    allocs = []
    for part, op, ports, tilers, rep in stages:
        tname = part.capitalize() + "T"
        comps[tname] = Component(tname, A, ports=tuple(port(f"{n} {s}") for n, s in ports.items()),
                                 repetition_space=Shape(tuple(rep)), elementary_op=op,
                                 tilers=tuple(sorted(tilers.items())))
        parts.append(PartInstance(part, tname))
        for n, s in ports.items():
            if s.split()[0] == "out":
                allocs.append(AllocationLink(AllocKind.DATA, f"{part}.{n}", "dev.gmem"))
        allocs.append(AllocationLink(AllocKind.TASK, part, "dev.cu"))
    rports = tuple(port(f"{n} {s}") for n, s in {**root_in, **root_out}.items())
    for n in root_in:
        allocs.insert(0, AllocationLink(AllocKind.DATA, n, "dev.gmem"))
    comps["m"] = Component("m", A, ports=rports, parts=tuple(parts),
                           connectors=tuple(Connector(a, b) for a, b in links))
    return Model(platform_components=platform(), application_components=comps, platform_root="p",
                 application_root="m", allocations=tuple(allocs))


def b200_platform(n_sm: int = 148, lanes: int = 128, smem_bytes: int = 227 * 1024,
                  hbm_bytes: int = 183_359 * 1024 * 1024, cmem_bytes: int = 64 * 1024) -> dict:
    """A MARTE platform model of one B200, in the reference's vocabulary.

    host (cpu + hostRam) | gpu.sm : Sm shaped [148] with lane : Lane shaped [128] (the PE
    multiplicity that derive_launch_config reads as the work-group size, partition.py:124-154),
    a deviceLocal shared memory of 227 KB per SM and a devicePrivate register file; gpu.hbm
    (deviceGlobal, 180 GB) and gpu.cmem (deviceConstant, 64 KB).
    """
    P = ComponentKind.PLATFORM
    return {
        "Host": Component("Host", P, parts=(PartInstance("cpu", "Cpu"), PartInstance("ram", "Ram"))),
        "Cpu": Component("Cpu", P, stereotype=HwStereotype(StereotypeKind.PROCESSOR)),
        "Ram": Component("Ram", P, stereotype=HwStereotype(StereotypeKind.MEMORY, MemoryRole.HOST_RAM)),
        "Lane": Component("Lane", P, stereotype=HwStereotype(StereotypeKind.PROCESSOR)),
        "Smem": Component("Smem", P, stereotype=HwStereotype(StereotypeKind.MEMORY, MemoryRole.DEVICE_LOCAL,
                                                              capacity_bytes=smem_bytes)),
        "Rf": Component("Rf", P, stereotype=HwStereotype(StereotypeKind.MEMORY, MemoryRole.DEVICE_PRIVATE,
                                                          capacity_bytes=256 * 1024)),
        "Sm": Component("Sm", P, parts=(PartInstance("lane", "Lane", Shape((lanes,))), PartInstance("smem", "Smem"),
                                        PartInstance("rf", "Rf")),
                        stereotype=HwStereotype(StereotypeKind.PROCESSOR, frequency_mhz=1965)),
        "Hbm": Component("Hbm", P, stereotype=HwStereotype(StereotypeKind.MEMORY, MemoryRole.DEVICE_GLOBAL,
                                                            capacity_bytes=hbm_bytes)),
        "Cmem": Component("Cmem", P, stereotype=HwStereotype(StereotypeKind.MEMORY, MemoryRole.DEVICE_CONSTANT,
                                                              capacity_bytes=cmem_bytes)),
        "B200": Component("B200", P, parts=(PartInstance("sm", "Sm", Shape((n_sm,))), PartInstance("hbm", "Hbm"),
                                            PartInstance("cmem", "Cmem"))),
        "p": Component("p", P, parts=(PartInstance("host", "Host"), PartInstance("gpu", "B200"))),
    }


# -- the BASELINE.json configs as models (SURVEY.md §8(d), Appendix A canonical tilers) -----

def _bound(origin, paving, fitting, pattern, array, rep) -> tuple[Tiler, tuple, tuple]:
    return Tiler(origin, paving, fitting, pattern), tuple(array), tuple(rep)


def gemm_tilers(M: int, N: int, K: int) -> dict[str, Tiler]:
    """C[i, j] = sum_k A[i, k] B[k, j] as a repetitive task over rep [M, N] (Appendix A):
    A row i (pattern [K] along axis 1), B column j (pattern [K] along axis 0), C element."""
    return {"a": Tiler((0, 0), ((1, 0), (0, 0)), ((0,), (1,)), (K,)),
            "b": Tiler((0, 0), ((0, 0), (0, 1)), ((1,), (0,)), (K,)),
            "c": Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,))}


def matmul_model(M: int, N: int, K: int) -> Model:
    """Configs C1/C2: the paper's MatMul repetitive task, fp32 in / fp32 out."""
    return tile_task_model("matmul", {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]",
                                      "c": f"out float32 [{M},{N}]"}, gemm_tilers(M, N, K), (M, N))


def stencil_tilers(H: int, W: int) -> dict[str, Tiler]:
    """3x3 window centred on each point of an H x W torus: origin (-1, -1) written mod the
    shape as (H-1, W-1) (DSL numbers are unsigned), identity paving and fitting."""
    return {"x": Tiler((H - 1, W - 1), ((1, 0), (0, 1)), ((1, 0), (0, 1)), (3, 3)),
            "y": Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,))}


def stencil_weights():
    """[1,2,1]^T [1,2,1] / 16: powers of two, so products are exact."""
    import numpy as np
    v = np.array([1.0, 2.0, 1.0])
    return (np.outer(v, v) / 16.0).astype(np.float32).ravel()


def stencil_model(H: int, W: int) -> Model:
    """Config C4: toroidal 3x3 stencil on an H x W fp32 array."""
    return tile_task_model("stencil", {"x": f"in float32 [{H},{W}]", "w": "in float32 [9]",
                                       "y": f"out float32 [{H},{W}]"}, stencil_tilers(H, W), (H, W))


def line_filter_tilers(F: int, H: int, W: int, axis: int, taps: int, step: int, outs: int):
    """1-D window of `taps` along `axis` (1 = rows / vertical, 2 = columns / horizontal) paved by
    `step`, `outs` outputs per repetition paved by `outs`: the Array-OL downscaler stage."""
    rep = [F, H, W]
    rep[axis] //= step
    arr_out = [F, H, W]
    arr_out[axis] = rep[axis] * outs
    pav_x = [[1, 0, 0], [0, 1, 0], [0, 0, 1]]
    pav_y = [[1, 0, 0], [0, 1, 0], [0, 0, 1]]
    pav_x[axis][axis] = step
    pav_y[axis][axis] = outs
    fit = tuple((1,) if d == axis else (0,) for d in range(3))
    x = Tiler((0, 0, 0), tuple(map(tuple, pav_x)), fit, (taps,))
    y = Tiler((0, 0, 0), tuple(map(tuple, pav_y)), fit, (outs,))
    return {"x": x, "y": y}, tuple(rep), tuple(arr_out)


def downscaler_weights(taps: int, outs: int):
    """Frozen downscaler weights: output j is a normalised triangle of half-width 3 centred at
    (taps-1)(j+1/2)/outs (the spec decision the oracle also freezes)."""
    import numpy as np
    w = np.zeros((outs, taps))
    for j in range(outs):
        c = (taps - 1) * (j + 0.5) / outs
        for i in range(taps):
            w[j, i] = max(0.0, 3.0 - abs(i - c))
        w[j] /= w[j].sum()
    return w.astype(np.float32).ravel()


def downscaler_model(F: int, H: int, W: int) -> Model:
    """Config C3: hfilter (13 taps, paving 8 -> 3 outputs) then vfilter (14 taps, paving 9 ->
    4 outputs) on F frames of H x W, chained through an intermediate array."""
    th, rep_h, arr_h = line_filter_tilers(F, H, W, 2, 13, 8, 3)
    Wo = arr_h[2]
    tv, rep_v, arr_v = line_filter_tilers(F, H, Wo, 1, 14, 9, 4)

    def dims(a):
        return ",".join(str(d) for d in a)
    return chain_model(
        [("h", "hfilter", {"x": f"in float32 [{F},{H},{W}]", "w": "in float32 [39]",
                           "y": f"out float32 [{dims(arr_h)}]"}, th, rep_h),
         ("v", "vfilter", {"x": f"in float32 [{dims(arr_h)}]", "w": "in float32 [56]",
                           "y": f"out float32 [{dims(arr_v)}]"}, tv, rep_v)],
        {"x": f"in float32 [{F},{H},{W}]", "wh": "in float32 [39]", "wv": "in float32 [56]"},
        {"y": f"out float32 [{dims(arr_v)}]"},
        [("x", "h.x"), ("wh", "h.w"), ("h.y", "v.x"), ("wv", "v.w"), ("v.y", "y")])
