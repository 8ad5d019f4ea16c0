"""MARTE memory allocation (memmap.py restated) and the B200 placement plan — no GPU needed."""

import pytest

from paper_1105_4424_b200 import builders, build_schedule
from paper_1105_4424_b200.model import (AllocationLink, AllocKind, Component, ComponentKind, Model, model_from_dict)
from paper_1105_4424_b200.placement import (B200_SMEM_PER_CTA, CapacityExceeded, build_memory_maps,
                                            emit_memory_map_report, emit_placement_report, kernel_staging,
                                            plan_placement)


@pytest.mark.parametrize("key", ["cg_bundled", "cg_k20"])
def test_memmap_report_equals_reference(golden, key):
    """build_memory_maps + emit_memory_map_report reproduce the reference's report byte for byte."""
    _, meta = golden
    model = model_from_dict(meta[key]["model"])
    assert emit_memory_map_report(build_memory_maps(model)) == meta[key]["memmap_report"]


def _model_on(platform, ports, allocs, op="copy", n=64):
    A = ComponentKind.APPLICATION
    task = Component("T", A, ports=tuple(builders.port(p) for p in ports),
                     repetition_space=builders.Shape((n,)), elementary_op=op)
    root = Component("m", A, ports=tuple(builders.port(p.replace("src", "i").replace("dst", "o"))
                                         for p in ports),
                     parts=(builders.PartInstance("t", "T"),),
                     connectors=(builders.Connector("i", "t.src"), builders.Connector("t.dst", "o")))
    return Model(platform, {"T": task, "m": root}, "p", "m",
                 tuple(builders.allocation(a) for a in allocs))


def test_capacity_exceeded_like_the_reference():
    """A 16K local memory overflows exactly as memmap.py:117-118 reports it (test_memmap.py:103-119 style)."""
    plat = builders.platform(local_capacity=16 * 1024)
    plat["Dev"] = plat["Dev"]   # Cu carries lmem
    m = _model_on(plat, ["src in float64 [2048]", "dst out float64 [2048]"],
                  ["allocate data i onto dev.cu.lmem", "allocate data t.dst onto dev.cu.lmem",
                   "allocate task t onto dev.cu"], n=2048)
    with pytest.raises(CapacityExceeded) as e:
        build_memory_maps(m)
    assert e.value.needed_bytes == 2 * 2048 * 8 and e.value.capacity_bytes == 16 * 1024


def test_b200_placement_tiers_and_alignment():
    plat = builders.b200_platform()
    m = _model_on(plat, ["src in float32 [33]", "dst out float32 [33]"],
                  ["allocate data i onto gpu.hbm", "allocate data t.dst onto gpu.hbm",
                   "allocate task t onto gpu.sm"], n=33)
    maps = build_memory_maps(m)
    assert [a.base_address for a in maps[0].data_allocations] == [0, 132]     # reference: element-aligned
    plan = plan_placement(m, maps)
    assert [p.tier for p in plan] == ["hbm", "hbm"]
    assert [p.b200_offset for p in plan] == [0, 256]                          # B200: 256 B aligned for TMA
    s = build_schedule(m, 2)
    assert s.steps[0].launches[0].local_size == 128                         # lane multiplicity per SM
    assert "hbm" in emit_placement_report(plan)


def test_b200_smem_limit_enforced():
    plat = builders.b200_platform(smem_bytes=10 ** 9)        # model claims more than the chip has
    n = B200_SMEM_PER_CTA // 4
    m = _model_on(plat, [f"src in float32 [{n}]", f"dst out float32 [{n}]"],
                  ["allocate data i onto gpu.sm.smem", "allocate data t.dst onto gpu.hbm",
                   "allocate task t onto gpu.sm"], n=n)
    plan_placement(m)                                        # exactly 227 KB fits
    m2 = _model_on(plat, [f"src in float32 [{n + 1}]", f"dst out float32 [{n + 1}]"],
                   ["allocate data i onto gpu.sm.smem", "allocate data t.dst onto gpu.hbm",
                    "allocate task t onto gpu.sm"], n=n + 1)
    with pytest.raises(CapacityExceeded):
        plan_placement(m2)


def test_constant_and_host_tiers():
    plat = builders.b200_platform(cmem_bytes=10 ** 9)
    big = 32 * 1024
    m = _model_on(plat, [f"src in float32 [{big}]", f"dst out float32 [{big}]"],
                  ["allocate data i onto gpu.cmem", "allocate data t.dst onto gpu.hbm",
                   "allocate task t onto gpu.sm"], n=big)
    tiers = {p.name: p.tier for p in plan_placement(m)}
    assert tiers["i"] == "hbm_readonly"                      # 128 KB > 64 KB broadcast limit
    assert kernel_staging("matmul.tcgen05_tf32").startswith("A,B k-blocks")


def test_placement_drives_arena_offsets_and_staging_flags():
    """Row a9/f3: the plan decides where groups live (one HBM arena per deviceGlobal memory at
    256 B offsets) and which staging a kernel uses (deviceLocal input -> AOL_FLAG_STAGE_SMEM)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from _sharded_cases import fir_model
    from paper_1105_4424_b200 import _capi
    from paper_1105_4424_b200.executor import _task_placement_flags
    from paper_1105_4424_b200.intrinsics import INTRINSICS
    from paper_1105_4424_b200.model import connected_port_groups
    from paper_1105_4424_b200.placement import hbm_arenas, placement_of_groups
    flags = {}
    for mem in ("dev.gmem", "dev.cu.lmem"):
        model, _, _, _ = fir_model(memory=mem)
        groups = connected_port_groups(model)
        flags[mem] = _task_placement_flags(model, groups, "t", INTRINSICS["tile_filter"])
        pg = placement_of_groups(model)
        arenas = hbm_arenas(model)
        assert list(arenas) == ["dev.gmem"]
        offs = sorted(p.b200_offset for p in pg.values() if p.tier == "hbm")
        assert all(o % 256 == 0 for o in offs) and len(set(offs)) == len(offs)
        assert arenas["dev.gmem"] >= max(p.b200_offset + p.size_bytes for p in pg.values() if p.tier == "hbm")
    assert flags == {"dev.gmem": 0, "dev.cu.lmem": _capi.FLAG_STAGE_SMEM}


def test_private_register_budget_enforced():
    from paper_1105_4424_b200.placement import B200_PRIVATE_BYTES_PER_THREAD, check_private_and_tmem
    plat = builders.b200_platform()
    n = B200_PRIVATE_BYTES_PER_THREAD // 4 + 1
    m = _model_on(plat, [f"src in float32 [{n}]", f"dst out float32 [{n}]"],
                  ["allocate data i onto gpu.sm.rf", "allocate data t.dst onto gpu.hbm",
                   "allocate task t onto gpu.sm"], n=n)
    with pytest.raises(CapacityExceeded):
        check_private_and_tmem(m, plan_placement(m))
    m_ok = _model_on(plat, [f"src in float32 [{n - 1}]", f"dst out float32 [{n - 1}]"],
                     ["allocate data i onto gpu.sm.rf", "allocate data t.dst onto gpu.hbm",
                      "allocate task t onto gpu.sm"], n=n - 1)
    check_private_and_tmem(m_ok, plan_placement(m_ok))
