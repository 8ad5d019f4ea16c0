"""Host logic of the storage layout: which output groups the run writes completely (their
zero-fill is skipped on one device) and which keep the reference's zero-fill."""

from paper_1105_4424_b200 import builders
from paper_1105_4424_b200.executor import covered_outputs, storage_layout


def _group_of(model, node):
    return storage_layout(model).groups[node]


def test_matmul_output_is_covered():
    m = builders.matmul_model(64, 48, 32)
    cov = covered_outputs(m)
    assert _group_of(m, "p_c") in cov
    assert _group_of(m, "p_a") not in cov and _group_of(m, "p_b") not in cov


def test_stencil_output_is_covered():
    m = builders.stencil_model(32, 48)
    root = m.application_components[m.application_root]
    out = [p.name for p in root.ports if getattr(p.direction, "value", p.direction) == "out"]
    assert out and all(_group_of(m, n) in covered_outputs(m) for n in out)


def test_downscaler_chain_intermediate_keeps_zero_fill():
    """The H->V intermediate (h.y = v.x) is read by the V stage: zero-filled as the reference
    does; the V output is written whole through a bijective tiler: skipped."""
    m = builders.downscaler_model(2, 48, 64)
    cov = covered_outputs(m)
    assert _group_of(m, "h.y") is _group_of(m, "v.x") and _group_of(m, "h.y") not in cov
    assert _group_of(m, "y") in cov
    assert _group_of(m, "x") not in cov


def test_axpy_inout_is_not_covered():
    m = builders.single_task_model(
        "axpy", ["y inout float64 [16]", "x in float64 [16]", "a in float64 [1]"],
        ["i in float64 [16]", "v in float64 [16]", "s in float64 [1]", "o out float64 [16]"],
        ["i -> t.y", "v -> t.x", "s -> t.a", "t.y -> o"],
        ["allocate data i onto dev.gmem", "allocate data v onto dev.gmem", "allocate data s onto host.ram",
         "allocate task t onto dev.cu"], None)
    assert not covered_outputs(m)
