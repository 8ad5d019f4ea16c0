"""MARTE GPU-model memory allocation -> concrete B200 placement.

Restates the reference's memory-mapping transformation
(/root/reference/pkg/src/gmodelc/memmap.py):

  * ``DataAllocate`` / ``MemoryMap`` ................... memmap.py:28-53
  * ``build_memory_maps``: one map per memory, first-fit in link order,
    bases rounded up to the element size, connected ports share one record,
    ``CapacityExceeded`` on overflow ..................... memmap.py:65-133
  * ``emit_memory_map_report`` (byte-identical text) ... memmap.py:136-148

and turns each record into a B200 placement through the memory role's
address-space qualifier (metamodel.py:59-65, the same mapping the
reference's code generator uses for kernel parameters, codegen.py:85-102):

  deviceGlobal   -> HBM: its own 256 B-aligned allocation (TMA needs 16 B
                    bases/pitches; the reference packs bases element-aligned
                    only, memmap.py:104-106, which TMA cannot use)
  deviceConstant -> read-only path: <= 64 KB, broadcast / staged in shared
                    memory by the kernels (filter coefficients)
  deviceLocal    -> shared memory staged by TMA / cp.async, capacity checked
                    against the 227 KB per-CTA limit (and the model's own)
  devicePrivate  -> registers
  hostRam        -> by-value kernel arguments (scalars only)

Kernel-level staging (which operand tiles go to the TMA ring, TMEM or
registers) is fixed per kernel and reported with :func:`kernel_staging`.
"""

from __future__ import annotations

from dataclasses import dataclass

from .model import (QUALIFIER_FOR_ROLE, AddressSpace, DataType, MemoryRole, Shape, connected_port_groups, enum_value,
                    memory_role_of, platform_part)

B200_SMEM_PER_CTA = 227 * 1024
B200_CONSTANT_BYTES = 64 * 1024
B200_HBM_BYTES = 183_359 * 1024 * 1024      # nvidia-smi total on the pool's B200s
B200_TMEM_BYTES_PER_SM = 256 * 1024
HBM_ALIGN = 256


class CapacityExceeded(ValueError):
    def __init__(self, owner_path: str, needed_bytes: int, capacity_bytes: int):
        super().__init__(f"memory '{owner_path}' needs {needed_bytes} bytes but has capacity {capacity_bytes}")
        self.owner_path = owner_path
        self.needed_bytes = needed_bytes
        self.capacity_bytes = capacity_bytes


@dataclass(frozen=True)
class DataAllocate:
    name: str
    space_address: AddressSpace
    base_address: int
    dim_allocation: Shape
    type_allocation: DataType
    associated_parts: tuple[str, ...]

    @property
    def size_bytes(self) -> int:
        return self.dim_allocation.total * DataType(enum_value(self.type_allocation)).size_bytes


@dataclass(frozen=True)
class MemoryMap:
    owner_path: str
    capacity_bytes: int | None
    data_allocations: tuple[DataAllocate, ...]

    @property
    def used_bytes(self) -> int:
        if not self.data_allocations:
            return 0
        last = self.data_allocations[-1]
        return last.base_address + last.size_bytes


def app_port_at(model, node: str):
    """FlowPort at an instance-path-qualified application node ("loop.spmv.y"), or None."""
    comps = model.application_components
    comp = comps.get(model.application_root)
    segs = node.split(".")
    for seg in segs[:-1]:
        part = comp.part(seg) if comp else None
        comp = comps.get(part.type_ref) if part else None
    return comp.port(segs[-1]) if comp else None


def build_memory_maps(model) -> list[MemoryMap]:
    """memmap.py:65-133 restated: first-fit packing per memory in allocation-link order."""
    groups = connected_port_groups(model)
    memories: list[str] = []
    per_memory: dict[str, list[str]] = {}
    for link in model.allocations:
        if enum_value(link.kind) != "data":
            continue
        if link.target_path not in per_memory:
            per_memory[link.target_path] = []
            memories.append(link.target_path)
        per_memory[link.target_path].append(link.source_path)
    maps = []
    for owner in memories:
        role = memory_role_of(model, owner)
        space = QUALIFIER_FOR_ROLE[MemoryRole(role)]
        comp = model.platform_components[platform_part(model, owner).type_ref]
        capacity = comp.stereotype.capacity_bytes
        cursor = 0
        allocs: list[DataAllocate] = []
        index: dict[frozenset, int] = {}
        linked: dict[frozenset, list[str]] = {}
        for path in per_memory[owner]:
            g = groups.get(path, frozenset({path}))
            if g in index:
                linked[g].append(path)
                continue
            port = app_port_at(model, path)
            align = DataType(enum_value(port.data_type)).size_bytes
            base = (cursor + align - 1) // align * align
            cursor = base + port.shape.total * align
            index[g] = len(allocs)
            linked[g] = [path]
            allocs.append(DataAllocate(path.replace(".", "_"), space, base, Shape(tuple(port.shape.dims)),
                                       DataType(enum_value(port.data_type)), ()))
        if capacity is not None and cursor > capacity:
            raise CapacityExceeded(owner, cursor, capacity)
        done = []
        for g, i in index.items():
            explicit = linked[g]
            rest = sorted(set(g) - set(explicit))
            a = allocs[i]
            done.append((i, DataAllocate(a.name, a.space_address, a.base_address, a.dim_allocation,
                                         a.type_allocation, tuple(explicit + rest))))
        done.sort(key=lambda p: p[0])
        maps.append(MemoryMap(owner, capacity, tuple(a for _, a in done)))
    return maps


def emit_memory_map_report(maps: list[MemoryMap]) -> str:
    """memmap.py:136-148 restated (the same text, so it can be compared byte for byte)."""
    lines = []
    for mm in maps:
        cap = str(mm.capacity_bytes) if mm.capacity_bytes is not None else "-"
        lines.append(f"map {mm.owner_path} used={mm.used_bytes} capacity={cap}")
        for a in mm.data_allocations:
            lines.append(f"  {a.name} space={enum_value(a.space_address)} base={a.base_address} "
                         f"dim={a.dim_allocation} type={enum_value(a.type_allocation)} size={a.size_bytes} "
                         f"parts={','.join(a.associated_parts)}")
    return "".join(line + "\n" for line in lines)


# -- B200 placement ---------------------------------------------------------------

TIER_FOR_ROLE = {
    "deviceGlobal": "hbm",
    "deviceConstant": "readonly_broadcast",
    "deviceLocal": "smem",
    "devicePrivate": "registers",
    "hostRam": "by_value",
}


@dataclass(frozen=True)
class Placement:
    name: str                 # the DataAllocate name (first linked port)
    memory: str               # platform memory path
    role: str                 # MARTE memory role
    qualifier: str            # address-space qualifier (metamodel.py:59-65)
    tier: str                 # B200 placement
    size_bytes: int
    b200_offset: int          # offset in the B200 layout (256 B-aligned for HBM)
    ports: tuple[str, ...]


def plan_placement(model, maps: list[MemoryMap] | None = None) -> list[Placement]:
    """Concrete B200 placement of every data allocation; raises CapacityExceeded on B200 limits.
    Computed once per model object when ``maps`` is not given (model_memo)."""
    if maps is None:
        from .model import model_memo
        return model_memo(model, "placement", lambda m: plan_placement(m, build_memory_maps(m)))
    out = []
    for mm in maps:
        role = memory_role_of(model, mm.owner_path)
        tier = TIER_FOR_ROLE[role]
        cursor = 0
        for a in mm.data_allocations:
            size = a.size_bytes
            if tier == "hbm":
                off = (cursor + HBM_ALIGN - 1) // HBM_ALIGN * HBM_ALIGN
                cursor = off + size
            else:
                off = a.base_address
            if tier == "readonly_broadcast" and size > B200_CONSTANT_BYTES:
                tier_a = "hbm_readonly"      # too big to broadcast: stays in HBM, read via ld.global.nc
            else:
                tier_a = tier
            if tier == "by_value" and a.dim_allocation.total != 1:
                tier_a = "host_staging"      # host-resident arrays are copied in by the executor
            out.append(Placement(a.name, mm.owner_path, role, enum_value(a.space_address), tier_a, size, off,
                                 a.associated_parts))
        if tier == "smem" and mm.used_bytes > B200_SMEM_PER_CTA:
            raise CapacityExceeded(mm.owner_path, mm.used_bytes, B200_SMEM_PER_CTA)
        if tier == "hbm" and cursor > B200_HBM_BYTES:
            raise CapacityExceeded(mm.owner_path, cursor, B200_HBM_BYTES)
    return out


# B200 register file per thread: 255 x 32-bit registers (ptxas' limit); a devicePrivate
# (work-item private) allocation has to fit there next to the kernel's own state
B200_PRIVATE_BYTES_PER_THREAD = 255 * 4
# TMEM per SM (512 columns x 128 lanes x 4 B); the tcgen05 matmul allocates all 512 columns
TMEM_COLS_PER_SM = 512


def check_private_and_tmem(model, plan: list[Placement]) -> None:
    """Capacity checks of the on-chip tiers the reference's memmap cannot see:
    devicePrivate data must fit a thread's register file; every matmul task's accumulators
    (2 x 256 fp32 TMEM columns for the TF32 kernel, 3 x 128 for the fp32-faithful one)
    must fit the SM's 512 TMEM columns (raises CapacityExceeded)."""
    for p in plan:
        if p.tier == "registers" and p.size_bytes > B200_PRIVATE_BYTES_PER_THREAD:
            raise CapacityExceeded(p.memory, p.size_bytes, B200_PRIVATE_BYTES_PER_THREAD)
    from .model import iter_app_instances
    for _, comp in iter_app_instances(model):
        if comp.elementary_op == "matmul":
            need = max(2 * 256, 3 * 128)
            if need > TMEM_COLS_PER_SM:
                raise CapacityExceeded("tmem", need * 128 * 4, TMEM_COLS_PER_SM * 128 * 4)


def placement_of_groups(model, plan: list[Placement] | None = None) -> dict:
    """Connected-port group -> its Placement (groups without a data allocation are absent)."""
    plan = plan_placement(model) if plan is None else plan
    groups = connected_port_groups(model)
    out = {}
    for p in plan:
        for node in p.ports:
            g = groups.get(node)
            if g is not None:
                out[g] = p
    return out


def hbm_arenas(model, plan: list[Placement] | None = None) -> dict:
    """deviceGlobal memory path -> arena bytes: the span of its placements at their 256 B offsets."""
    plan = plan_placement(model) if plan is None else plan
    out: dict = {}
    for p in plan:
        if p.tier in ("hbm",):
            end = p.b200_offset + p.size_bytes
            out[p.memory] = max(out.get(p.memory, 0), (end + HBM_ALIGN - 1) // HBM_ALIGN * HBM_ALIGN)
    return out


KERNEL_STAGING = {
    "matmul.tcgen05_tf32": "A,B k-blocks: HBM -> TMA (128B swizzle; MN-major tf32: 128B/32B-atom) -> 4 x 48 KB smem "
                           "ring; accumulators: TMEM 2 x (128 lanes x 256 cols fp32); C: TMEM -> registers -> "
                           "st.global.v4",
    "matmul.generic_exact": "patterns gathered from HBM to registers; pattern offset tables in smem",
    "matmul.exact_tiled": "64x16 A and 16x64 B slabs in smem; 4x4 outputs per thread in registers (k-ascending, no FMA)",
    "tile_copy.stream16": "HBM -> registers (16 B vectors, streaming hints) -> HBM",
    "tile_copy.tma_stream": "HBM -> TMA 256 B-row boxes -> shared-memory ring (4 x 8 KB, 2 CTAs/SM) -> TMA store -> HBM",
    "tile_copy.tma_transpose": "HBM -> TMA {32 reps, m} boxes (128B swizzle) -> smem transpose -> TMA store -> HBM",
    "tile_copy.seam_boxes": "split at the wrap seams into affine boxes, each on its own plan (rows_shift / tma_plane / stream / affine2d)",
    "tile_copy.interleave": "HBM -> one float4 per pattern row (m = 2 / 4) -> register transpose -> m float4 stores -> HBM",
    "tile_copy.tma_plane": "HBM -> TMA {256 B x 32 rows} boxes -> 4-stage smem ring -> TMA store -> HBM",
    "tile_copy.rows_shift": "HBM -> two aligned float4 loads (L1) -> funnel shift in registers -> aligned float4 store -> HBM",
    "tile_copy.affine2d": "HBM -> registers (V-element vectors along the inner pattern row) -> HBM",
    "tile_copy.stride2": "HBM -> registers (two 16 B source vectors per 4 repetitions) -> HBM (16 B stores)",
    "tile_filter.box_pool": "HBM -> registers (KH rows x 4*KW floats as float4) -> HBM (float4 stores)",
    "tile_filter.line_stream": "HBM -> cp.async.bulk whole rows (+32 B wrap halo) -> 8-stage smem ring -> 16-float window per repetition -> registers -> HBM",
    "tile_filter.line_tiled": "HBM -> coalesced window per tile of <= 8192 repetitions -> padded smem -> registers -> HBM",
    "tile_sum.rows": "HBM -> cp.async 32x32 tiles (coalesced rows) -> smem ring (4 chunks) -> one ordered add chain per lane",
    "tile_sum.batched": "the batched filter kernel with unit weights: int32 pattern tables in smem, 8 repetitions per lane, window in registers",
    "tile_sum.columns": "HBM -> TMA {32 columns x 8 KB} boxes -> 4-stage smem ring -> one ordered add chain per lane",
    "tile_sum.direct": "HBM -> registers (64 loads in flight per repetition) -> ordered add chain",
    "tile_copy.window": "HBM -> one bulk copy per tile of the overlapping source window -> smem ring -> registers (16 B stores) -> HBM",
    "tile_copy.tma_box": "HBM -> TMA pattern-row boxes -> shared-memory ring (32-64 KB in flight/SM) -> TMA store -> HBM",
    "tile_copy.vec": "HBM -> registers (V-element vectors) -> HBM",
    "tile_copy.vec_store": "HBM -> registers (strided scalars) -> HBM (V-element vector stores)",
    "tile_copy.affine": "HBM -> registers -> HBM (4-way unrolled scalars)",
    "tile_copy.generic": "HBM -> registers -> HBM (full index function; 32-bit compile-time-rank form, 4 in flight, when it fits)",
    "tile_filter.stencil_box": "coefficients: smem broadcast; (4+KH-1) x 6 input window: registers; outputs float4",
    "tile_filter.line_13x3_stream": "x rows: HBM -> cp.async.bulk -> 8-stage smem ring (mbarriers); 16-float window: "
                                    "ld.shared.v4 -> registers; outputs HBM",
    "tile_filter.line_14x4_stream": "input rows: HBM -> cp.async.bulk -> 8-stage smem ring; 3 columns per thread; "
                                    "2 x 12 consumer accumulators in registers; outputs HBM",
    "tile_filter.fused_stream": "x rows: HBM -> cp.async.bulk -> 8-stage smem ring; producer outputs in registers "
                                "folded into 2 x 12 consumer accumulators; intermediate never stored",
    "tile_filter.line_13x3": "coefficients: smem broadcast; 13-tap window: registers (float4 loads); outputs HBM",
    "tile_filter.line_14x4": "coefficients: smem broadcast; 14-tap window: registers (coalesced row taps)",
    "tile_filter.line_14x4_vstrip": "coefficients: smem broadcast; 4 overlapping 14-tap windows (41 rows): registers "
                                    "(coalesced row taps)",
    "tile_filter.line": "coefficients: smem broadcast; window: registers",
    "tile_filter.batched": "coefficients + int32 pattern tables: smem; 8-16 repetitions per lane, window: registers",
    "tile_filter.window_vec": "coefficients + pattern tables: smem; window: registers",
    "tile_filter.generic": "coefficients + pattern tables: smem; window: registers",
    "tile_sum.generic": "pattern table: smem; accumulation: registers",
    "identity": "element rho of every port: HBM -> registers -> HBM; host scalars by value",
}


def kernel_staging(plan_name: str) -> str:
    return KERNEL_STAGING.get(plan_name, "registers")


def emit_placement_report(plan: list[Placement]) -> str:
    lines = ["placement (B200): name memory role qualifier -> tier size offset ports"]
    for p in plan:
        lines.append(f"  {p.name} {p.memory} {p.role} {p.qualifier} -> {p.tier} size={p.size_bytes} "
                     f"offset={p.b200_offset} ports={','.join(p.ports)}")
    return "\n".join(lines) + "\n"
