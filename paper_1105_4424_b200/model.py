"""Host-side mirror of the reference metamodel types the repetitive-task path consumes.

The GPU path is a drop-in for ``gmodelc.refexec.execute_schedule``
(/root/reference/pkg/src/gmodelc/refexec.py:427-549).  That function reads
a ``Model`` / ``Schedule`` built by the reference front-end.  This module
restates only the slice of the metamodel that the executor touches
(/root/reference/pkg/src/gmodelc/metamodel.py:14-194, :272-376) so the
package runs on a GPU box where the reference is not installed.

Field names and enum *values* are identical to the reference, and every
consumer in this package reads them by value (``Direction.IN.value ==
"in"``), so a real ``gmodelc.Model`` and the mirror are interchangeable
inputs to :func:`paper_1105_4424_b200.executor.execute_schedule`.

The one additive field is ``Component.tilers`` (port name -> Tiler),
which carries the Array-OL tilers the reference metamodel lacks
(SURVEY.md Appendix A).  For reference models, tilers are supplied to the
executor with its ``tilers=`` keyword instead.
"""

from __future__ import annotations

import enum
import weakref
from dataclasses import dataclass, field
from typing import Any, Iterator


class Direction(str, enum.Enum):
    IN = "in"
    OUT = "out"
    INOUT = "inout"


class DataType(str, enum.Enum):
    FLOAT32 = "float32"
    FLOAT64 = "float64"
    INT32 = "int32"
    INT64 = "int64"

    @property
    def size_bytes(self) -> int:
        return 4 if self.value in ("float32", "int32") else 8

    @property
    def is_float(self) -> bool:
        return self.value in ("float32", "float64")


class AddressSpace(str, enum.Enum):
    GLOBAL = "global"
    CONSTANT = "constant"
    LOCAL = "local"
    PRIVATE = "private"


class StereotypeKind(str, enum.Enum):
    PROCESSOR = "hwProcessor"
    MEMORY = "hwMemory"
    BUS = "hwBus"


class MemoryRole(str, enum.Enum):
    HOST_RAM = "hostRam"
    DEVICE_GLOBAL = "deviceGlobal"
    DEVICE_CONSTANT = "deviceConstant"
    DEVICE_LOCAL = "deviceLocal"
    DEVICE_PRIVATE = "devicePrivate"


# metamodel.py:59-65: one address-space qualifier per memory role.
QUALIFIER_FOR_ROLE = {
    MemoryRole.HOST_RAM: AddressSpace.GLOBAL,
    MemoryRole.DEVICE_GLOBAL: AddressSpace.GLOBAL,
    MemoryRole.DEVICE_CONSTANT: AddressSpace.CONSTANT,
    MemoryRole.DEVICE_LOCAL: AddressSpace.LOCAL,
    MemoryRole.DEVICE_PRIVATE: AddressSpace.PRIVATE,
}


class ComponentKind(str, enum.Enum):
    PLATFORM = "platform"
    APPLICATION = "application"


class AllocKind(str, enum.Enum):
    DATA = "data"
    TASK = "task"


def enum_value(x: Any) -> Any:
    """Value of a (possibly foreign) str-enum, so mirror and reference enums compare equal."""
    return getattr(x, "value", x)


@dataclass(frozen=True)
class Shape:
    dims: tuple[int, ...]

    @property
    def total(self) -> int:
        t = 1
        for d in self.dims:
            t *= int(d)
        return t

    def __str__(self) -> str:
        return "[" + ",".join(str(d) for d in self.dims) + "]"


@dataclass(frozen=True)
class FlowPort:
    name: str
    direction: Direction
    shape: Shape
    data_type: DataType


@dataclass(frozen=True)
class HwStereotype:
    kind: StereotypeKind
    memory_role: MemoryRole | None = None
    capacity_bytes: int | None = None
    frequency_mhz: int | None = None


@dataclass(frozen=True)
class PartInstance:
    name: str
    type_ref: str
    shaped: Shape | None = None


@dataclass(frozen=True)
class Connector:
    source: str
    target: str


@dataclass(frozen=True)
class UntilCondition:
    port: str
    tolerance: float


@dataclass(frozen=True)
class Component:
    name: str
    kind: ComponentKind
    ports: tuple[FlowPort, ...] = ()
    parts: tuple[PartInstance, ...] = ()
    connectors: tuple[Connector, ...] = ()
    stereotype: HwStereotype | None = None
    repetition_space: Shape | None = None
    elementary_op: str | None = None
    until: UntilCondition | None = None
    # additive: Array-OL tilers of a repetitive task, keyed by port name
    tilers: tuple = field(default=(), compare=False)

    def port(self, name: str) -> FlowPort | None:
        for p in self.ports:
            if p.name == name:
                return p
        return None

    def part(self, name: str) -> PartInstance | None:
        for p in self.parts:
            if p.name == name:
                return p
        return None

    @property
    def is_leaf_task(self) -> bool:
        return self.elementary_op is not None

    def tiler(self, port_name: str):
        for name, t in self.tilers:
            if name == port_name:
                return t
        return None


@dataclass(frozen=True)
class AllocationLink:
    kind: AllocKind
    source_path: str
    target_path: str


@dataclass(frozen=True)
class Model:
    platform_components: dict[str, Component]
    application_components: dict[str, Component]
    platform_root: str
    application_root: str
    allocations: tuple[AllocationLink, ...] = ()

    def component(self, kind, name: str) -> Component | None:
        comps = (self.platform_components if enum_value(kind) == "platform"
                 else self.application_components)
        return comps.get(name)

    def root(self, kind) -> Component | None:
        name = self.platform_root if enum_value(kind) == "platform" else self.application_root
        return self.component(kind, name)


# -- model-walking helpers (duck-typed: accept reference models too) ----------


def _side(model, kind: str) -> dict:
    return model.platform_components if kind == "platform" else model.application_components


def _root(model, kind: str):
    name = model.platform_root if kind == "platform" else model.application_root
    return _side(model, kind).get(name)


def iter_app_instances(model) -> Iterator[tuple[str, Any]]:
    """(instance_path, component) for the application root ("") and every nested part.

    Same depth-first, declaration-order walk as metamodel.py:272-289.
    """
    comps = model.application_components
    root = comps.get(model.application_root)
    if root is None:
        return
    stack = [("", root)]
    while stack:
        path, comp = stack.pop()
        yield path, comp
        for part in reversed(comp.parts):
            sub = comps.get(part.type_ref)
            if sub is not None:
                stack.append((f"{path}.{part.name}" if path else part.name, sub))


def _node(path: str, port: str) -> str:
    return f"{path}.{port}" if path else port


_MODEL_MEMO: dict[int, dict] = {}


def model_memo(model, key: str, fn):
    """``fn(model)`` computed once per model object.  Models are treated as immutable once
    built (the executor never mutates them); an entry is dropped when its model is
    garbage-collected.  Objects that take no weak reference are not cached."""
    mid = id(model)
    slot = _MODEL_MEMO.get(mid)
    if slot is None:
        try:
            weakref.finalize(model, _MODEL_MEMO.pop, mid, None)
        except TypeError:
            return fn(model)
        slot = _MODEL_MEMO[mid] = {}
    if key not in slot:
        slot[key] = fn(model)
    return slot[key]


def connected_port_groups(model) -> dict[str, frozenset[str]]:
    """Cached :func:`port_groups` (read-only result)."""
    return model_memo(model, "port_groups", port_groups)


def port_groups(model) -> dict[str, frozenset[str]]:
    """Port nodes grouped by connector reachability: one group = one storage array.

    Restates metamodel.py:315-349 (union-find over connectors of every
    instance; dangling endpoints ignored).
    """
    parent: dict[str, str] = {}

    def find(x: str) -> str:
        parent.setdefault(x, x)
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    comps = model.application_components
    nodes: list[str] = []
    for path, comp in iter_app_instances(model):
        for port in comp.ports:
            n = _node(path, port.name)
            find(n)
            nodes.append(n)
        for conn in comp.connectors:
            ends = []
            for ep in (conn.source, conn.target):
                segs = ep.split(".")
                if len(segs) == 1 and comp.port(segs[0]) is not None:
                    ends.append(_node(path, segs[0]))
                elif len(segs) == 2:
                    part = comp.part(segs[0])
                    sub = comps.get(part.type_ref) if part else None
                    if sub is not None and sub.port(segs[1]) is not None:
                        ends.append(_node(_node(path, segs[0]), segs[1]))
            if len(ends) == 2:
                a, b = find(ends[0]), find(ends[1])
                if a != b:
                    parent[max(a, b)] = min(a, b)
    groups: dict[str, set[str]] = {}
    for n in nodes:
        groups.setdefault(find(n), set()).add(n)
    out: dict[str, frozenset[str]] = {}
    for members in groups.values():
        fz = frozenset(members)
        for n in members:
            out[n] = fz
    return out


def platform_part(model, path: str):
    """PartInstance at a dotted platform path, or None (metamodel.py:261-267)."""
    comps = model.platform_components
    comp = comps.get(model.platform_root)
    segs = path.split(".") if path else []
    if comp is None or not segs or any(not s for s in segs):
        return None
    part = None
    for i, seg in enumerate(segs):
        part = comp.part(seg)
        if part is None:
            return None
        if i < len(segs) - 1:
            comp = comps.get(part.type_ref)
            if comp is None:
                return None
    return part


def is_host_processor(model, target_path: str) -> bool:
    """A processor is host-side when a sibling memory has the hostRam role (metamodel.py:358-376)."""
    comps = model.platform_components
    owner = comps.get(model.platform_root)
    for seg in target_path.split(".")[:-1]:
        part = owner.part(seg) if owner else None
        owner = comps.get(part.type_ref) if part else None
    if owner is None:
        return False
    for sib in owner.parts:
        sub = comps.get(sib.type_ref)
        st = sub.stereotype if sub else None
        if st is not None and enum_value(st.kind) == "hwMemory" \
                and enum_value(st.memory_role) == "hostRam":
            return True
    return False


def memory_role_of(model, target_path: str) -> str | None:
    """Memory-role value of the platform part at target_path (metamodel.py:379-386)."""
    part = platform_part(model, target_path)
    if part is None:
        return None
    comp = model.platform_components.get(part.type_ref)
    if comp is None or comp.stereotype is None:
        return None
    return enum_value(comp.stereotype.memory_role)


def task_component(model, task_path: str):
    """Application component type instantiated at a dotted task path."""
    comps = model.application_components
    comp = comps[model.application_root]
    for seg in task_path.split("."):
        part = comp.part(seg)
        comp = comps[part.type_ref]
    return comp


# -- JSON round trip (lets models built by the reference front-end travel without the DSL) ----

def model_to_dict(model) -> dict:
    """Plain-data form of a (mirror or reference) Model; inverse of :func:`model_from_dict`."""
    def shape(s):
        return None if s is None else [int(d) for d in s.dims]

    def comp(c):
        st = c.stereotype
        return {
            "name": c.name, "kind": enum_value(c.kind),
            "ports": [[p.name, enum_value(p.direction), shape(p.shape), enum_value(p.data_type)] for p in c.ports],
            "parts": [[p.name, p.type_ref, shape(p.shaped)] for p in c.parts],
            "connectors": [[k.source, k.target] for k in c.connectors],
            "stereotype": None if st is None else [enum_value(st.kind), enum_value(st.memory_role),
                                                   st.capacity_bytes, st.frequency_mhz],
            "repetition_space": shape(c.repetition_space),
            "elementary_op": c.elementary_op,
            "until": None if c.until is None else [c.until.port, c.until.tolerance],
        }
    return {
        "platform_components": [comp(c) for c in model.platform_components.values()],
        "application_components": [comp(c) for c in model.application_components.values()],
        "platform_root": model.platform_root, "application_root": model.application_root,
        "allocations": [[enum_value(a.kind), a.source_path, a.target_path] for a in model.allocations],
    }


def model_from_dict(d: dict) -> Model:
    def shape(v):
        return None if v is None else Shape(tuple(int(x) for x in v))

    def comp(c):
        st = c["stereotype"]
        return Component(
            name=c["name"], kind=ComponentKind(c["kind"]),
            ports=tuple(FlowPort(n, Direction(di), shape(s), DataType(t)) for n, di, s, t in c["ports"]),
            parts=tuple(PartInstance(n, t, shape(s)) for n, t, s in c["parts"]),
            connectors=tuple(Connector(a, b) for a, b in c["connectors"]),
            stereotype=None if st is None else HwStereotype(StereotypeKind(st[0]),
                                                            None if st[1] is None else MemoryRole(st[1]),
                                                            st[2], st[3]),
            repetition_space=shape(c["repetition_space"]), elementary_op=c["elementary_op"],
            until=None if c["until"] is None else UntilCondition(c["until"][0], float(c["until"][1])))
    return Model(
        platform_components={c["name"]: comp(c) for c in d["platform_components"]},
        application_components={c["name"]: comp(c) for c in d["application_components"]},
        platform_root=d["platform_root"], application_root=d["application_root"],
        allocations=tuple(AllocationLink(AllocKind(k), s, t) for k, s, t in d["allocations"]))
