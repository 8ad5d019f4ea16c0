"""Operator registry (the reference's plugin API) extended with Array-OL tile intrinsics.

Mirrors /root/reference/pkg/src/gmodelc/intrinsics.py:
  * ``PortSpec`` / ``IntrinsicSpec``           :27-46
  * ``INTRINSICS`` (device: spmv_csr, dot_partial, axpy, scale, copy, sub;
    host: div, neg, rel_residual)               :51-102
  * ``check_task_signature``                    :105-156 (same checks, same messages)

Additive tile intrinsics.  Their
vector ports are whole arrays reached through tilers, so the reference's
extent rule (vector extent == repetition total, :138-146) is replaced for
them by tiler checks (:func:`check_tile_signature`):

  ``tile_copy``  src --tiler--> pattern --tiler--> dst (bit moves)
  ``matmul``     c[r] = sum_k a_pat(r)[k] * b_pat(r)[k]        (pattern dot)
  ``tile_filter`` / ``hfilter`` / ``vfilter`` / ``stencil``
                 y_pat(r)[j] = sum_i w[j, i] * x_pat(r)[i]    (pattern linear map)
  ``tile_sum``   s[r] = sum_i x_pat(r)[i]                      (pattern reduction)

Accumulation order is the pattern order with every product and every
sum rounded to the port dtype (no FMA contraction) — the order the
unmodified ``spmv_csr`` executor uses (refexec.py:111-121), which is how
the oracle is pinned (tests/golden/make_golden.py).
"""

from __future__ import annotations

from dataclasses import dataclass

from ._refcompat import ref_bases
from .model import enum_value
from .tiler import BoundTiler, Tiler, TilerError


class UnknownIntrinsic(*ref_bases("intrinsics", "UnknownIntrinsic", ValueError)):
    def __init__(self, task_path: str, op_name: str):
        ValueError.__init__(self, f"task '{task_path}' deploys unknown intrinsic '{op_name}'")
        self.task_path = task_path
        self.op_name = op_name


class IntrinsicShapeMismatch(*ref_bases("intrinsics", "IntrinsicShapeMismatch", ValueError)):
    pass


@dataclass(frozen=True)
class PortSpec:
    name: str
    direction: str            # "in" | "out" | "inout"
    scalar: bool = False      # shape total must be exactly 1
    integer: bool = False     # int32/int64 instead of float
    optional: bool = False
    tiled: bool = False       # reached through a tiler (tile intrinsics)


@dataclass(frozen=True)
class IntrinsicSpec:
    name: str
    kind: str                 # "device" | "host"
    ports: tuple[PortSpec, ...]
    tile: bool = False        # Array-OL tile intrinsic (tilers, no extent rule)
    float_only: bool = False  # tiled ports must be float32/float64

    def port_spec(self, name: str) -> PortSpec | None:
        for s in self.ports:
            if s.name == name:
                return s
        return None


_IN, _OUT, _INOUT = "in", "out", "inout"

_REFERENCE_OPS = (
    IntrinsicSpec("spmv_csr", "device", (
        PortSpec("rowptr", _IN, integer=True), PortSpec("colidx", _IN, integer=True),
        PortSpec("values", _IN), PortSpec("x", _IN), PortSpec("y", _OUT))),
    IntrinsicSpec("dot_partial", "device", (
        PortSpec("a", _IN), PortSpec("b", _IN), PortSpec("s", _OUT, scalar=True))),
    IntrinsicSpec("axpy", "device", (
        PortSpec("y", _INOUT), PortSpec("x", _IN),
        PortSpec("a", _IN, scalar=True, optional=True))),
    IntrinsicSpec("scale", "device", (PortSpec("y", _INOUT), PortSpec("a", _IN, scalar=True))),
    IntrinsicSpec("copy", "device", (PortSpec("src", _IN), PortSpec("dst", _OUT))),
    IntrinsicSpec("sub", "device", (PortSpec("x", _IN), PortSpec("y", _IN), PortSpec("z", _OUT))),
    IntrinsicSpec("div", "host", (
        PortSpec("num", _IN, scalar=True), PortSpec("den", _IN, scalar=True),
        PortSpec("q", _OUT, scalar=True))),
    IntrinsicSpec("neg", "host", (PortSpec("a", _IN, scalar=True), PortSpec("z", _OUT, scalar=True))),
    IntrinsicSpec("rel_residual", "host", (
        PortSpec("num", _IN, scalar=True), PortSpec("den", _IN, scalar=True),
        PortSpec("z", _OUT, scalar=True))),
)


def _filter_spec(name: str) -> IntrinsicSpec:
    return IntrinsicSpec(name, "device", (
        PortSpec("x", _IN, tiled=True), PortSpec("w", _IN), PortSpec("y", _OUT, tiled=True)),
        tile=True, float_only=True)


_TILE_OPS = (
    IntrinsicSpec("tile_copy", "device", (
        PortSpec("src", _IN, tiled=True), PortSpec("dst", _OUT, tiled=True)), tile=True),
    IntrinsicSpec("matmul", "device", (
        PortSpec("a", _IN, tiled=True), PortSpec("b", _IN, tiled=True),
        PortSpec("c", _OUT, tiled=True)), tile=True, float_only=True),
    _filter_spec("tile_filter"),
    _filter_spec("hfilter"),
    _filter_spec("vfilter"),
    _filter_spec("stencil"),
    IntrinsicSpec("tile_sum", "device", (
        PortSpec("x", _IN, tiled=True), PortSpec("s", _OUT, tiled=True)),
        tile=True, float_only=True),
)

INTRINSICS: dict[str, IntrinsicSpec] = {s.name: s for s in _REFERENCE_OPS + _TILE_OPS}
TILE_INTRINSICS = frozenset(s.name for s in _TILE_OPS)
FILTER_OPS = frozenset(("tile_filter", "hfilter", "vfilter", "stencil"))


def _is_float(port) -> bool:
    return enum_value(port.data_type) in ("float32", "float64")


def _ports_match_spec(task_path: str, comp, spec: IntrinsicSpec) -> None:
    declared = {p.name for p in comp.ports}
    expected = {s.name for s in spec.ports}
    required = {s.name for s in spec.ports if not s.optional}
    if not required <= declared or not declared <= expected:
        raise IntrinsicShapeMismatch(
            f"task '{task_path}': intrinsic '{spec.name}' expects ports "
            f"{sorted(expected)} (optional: {sorted(expected - required)}), got {sorted(declared)}")
    for port in comp.ports:
        ps = spec.port_spec(port.name)
        if enum_value(port.direction) != ps.direction:
            raise IntrinsicShapeMismatch(f"task '{task_path}': port '{port.name}' must be {ps.direction}")
        if ps.integer != (not _is_float(port)):
            kind = "an integer" if ps.integer else "a floating-point"
            raise IntrinsicShapeMismatch(f"task '{task_path}': port '{port.name}' must have {kind} type")
        if ps.scalar and port.shape.total != 1:
            raise IntrinsicShapeMismatch(f"task '{task_path}': port '{port.name}' must be scalar")


def check_task_signature(task_path: str, comp, tilers: dict | None = None):
    """Validate a leaf task against its intrinsic; returns the spec (intrinsics.py:105-156).

    Reference intrinsics keep the reference's extent rule; tile intrinsics
    are checked by :func:`check_tile_signature` (``tilers`` maps port name
    to :class:`Tiler`, falling back to ``comp.tilers``).
    """
    op = comp.elementary_op
    if op is None or op not in INTRINSICS:
        raise UnknownIntrinsic(task_path, op or "<none>")
    spec = INTRINSICS[op]
    _ports_match_spec(task_path, comp, spec)
    if spec.tile:
        check_tile_signature(task_path, comp, spec, tilers)
        return spec
    extents: set[int] = set()
    for port in comp.ports:
        ps = spec.port_spec(port.name)
        if not ps.scalar and port.name not in ("rowptr", "colidx", "values"):
            extents.add(port.shape.total)
    if spec.kind == "device":
        if len(extents) > 1:
            raise IntrinsicShapeMismatch(
                f"task '{task_path}': vector ports disagree on extent: {sorted(extents)}")
        repeat = comp.repetition_space.total if comp.repetition_space else 1
        if extents and repeat not in (1, next(iter(extents))):
            raise IntrinsicShapeMismatch(
                f"task '{task_path}': repetition space {repeat} does not match "
                f"vector extent {next(iter(extents))}")
        if op == "spmv_csr":
            n = comp.port("y").shape.total
            if comp.port("rowptr").shape.total != n + 1:
                raise IntrinsicShapeMismatch(f"task '{task_path}': rowptr extent must be row count + 1")
            if comp.port("colidx").shape.total != comp.port("values").shape.total:
                raise IntrinsicShapeMismatch(f"task '{task_path}': colidx and values extents differ")
    return spec


def task_tilers(comp, tilers: dict | None) -> dict[str, Tiler]:
    out = dict(getattr(comp, "tilers", ()) or ())
    if tilers:
        out.update(tilers)
    return out


def bind_tilers(task_path: str, comp, spec: IntrinsicSpec, tilers: dict | None) -> dict[str, BoundTiler]:
    """Bind every tiled port's tiler to (port shape, repetition shape); raise on a missing tiler."""
    tl = task_tilers(comp, tilers)
    rep = comp.repetition_space.dims if comp.repetition_space is not None else (1,)
    bound: dict[str, BoundTiler] = {}
    for ps in spec.ports:
        if not ps.tiled:
            continue
        port = comp.port(ps.name)
        t = tl.get(ps.name)
        if t is None:
            raise IntrinsicShapeMismatch(f"task '{task_path}': tiled port '{ps.name}' has no tiler")
        try:
            bound[ps.name] = t.bind(port.shape.dims, rep)
        except TilerError as e:
            raise IntrinsicShapeMismatch(f"task '{task_path}': port '{ps.name}': {e}") from None
    return bound


def check_tile_signature(task_path: str, comp, spec: IntrinsicSpec, tilers: dict | None) -> dict:
    """Tiler rules for tile intrinsics; returns the bound tilers."""
    bound = bind_tilers(task_path, comp, spec, tilers)
    for ps in spec.ports:
        port = comp.port(ps.name)
        if spec.float_only and ps.tiled and not _is_float(port):
            raise IntrinsicShapeMismatch(
                f"task '{task_path}': port '{port.name}' must have a floating-point type")
    dtypes = {enum_value(comp.port(ps.name).data_type) for ps in spec.ports}
    if len(dtypes) > 1:
        raise IntrinsicShapeMismatch(f"task '{task_path}': ports disagree on data type: {sorted(dtypes)}")
    P = {name: b.pattern_total for name, b in bound.items()}
    op = spec.name
    if op == "tile_copy" and P["src"] != P["dst"]:
        raise IntrinsicShapeMismatch(
            f"task '{task_path}': src pattern has {P['src']} elements, dst pattern {P['dst']}")
    if op == "matmul":
        if P["a"] != P["b"]:
            raise IntrinsicShapeMismatch(
                f"task '{task_path}': a and b patterns differ in length ({P['a']} vs {P['b']})")
        if P["c"] != 1:
            raise IntrinsicShapeMismatch(f"task '{task_path}': c pattern must be a single element")
    if op in FILTER_OPS:
        w = comp.port("w")
        if w.shape.total != P["y"] * P["x"]:
            raise IntrinsicShapeMismatch(
                f"task '{task_path}': coefficient port 'w' must hold {P['y']}x{P['x']} values, "
                f"has {w.shape.total}")
    if op == "tile_sum" and P["s"] != 1:
        raise IntrinsicShapeMismatch(f"task '{task_path}': s pattern must be a single element")
    for ps in spec.ports:
        if ps.tiled and ps.direction == _OUT:
            try:
                bound[ps.name].check_injective()
            except TilerError as e:
                raise IntrinsicShapeMismatch(f"task '{task_path}': port '{ps.name}': {e}") from None
    return bound


def register_into(registry: dict) -> None:
    """Additively register the tile intrinsics into a reference ``gmodelc.intrinsics.INTRINSICS``.

    Only names the registry does not already define are added; reference
    entries are never replaced (keeps the reference suite and goldens intact).
    """
    for name in TILE_INTRINSICS:
        registry.setdefault(name, INTRINSICS[name])
