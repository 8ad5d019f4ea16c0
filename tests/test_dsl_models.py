"""Row f2 end to end: models AUTHORED in .gmodel text with `tiler` lines (tests/golden/dsl/),
parsed by the unmodified reference front-end into tests/golden/dsl_models.json
(tests/golden/make_dsl_models.py), run through the drop-in's kernels and compared with the
oracle -- bit-exact for the stencil, the downscaler chain and the exact-order matmul, inside
the stated TF32 bound for the tensor-core matmul."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import aol_oracle as orc
from paper_1105_4424_b200 import build_schedule, check_task_signature
from paper_1105_4424_b200.model import enum_value, model_from_dict
from paper_1105_4424_b200.tiler_dsl import extract_tilers, tilers_by_task

GOLD = Path(__file__).resolve().parent / "golden"


def _load(name):
    text = (GOLD / "dsl" / f"{name}.gmodel").read_text()
    stripped, per_type = extract_tilers(text)
    fx = json.loads((GOLD / "dsl_models.json").read_text())[name]
    assert hashlib.sha256(stripped.encode()).hexdigest() == fx["sha256"], "fixture is stale: rerun make_dsl_models.py"
    model = model_from_dict(fx["model"])
    return model, tilers_by_task(model, per_type)


def _task(model, path):
    root = model.application_components[model.application_root]
    part = next(p for p in root.parts if p.name == path)
    return model.application_components[part.type_ref]


def _oracle_tilers(model, path, tilers):
    """Oracle-form tiler dicts (array = the task port's shape, rep = the repetition space)."""
    comp = _task(model, path)
    rep = tuple(comp.repetition_space.dims)
    shapes = {p.name: tuple(p.shape.dims) for p in comp.ports}
    return {port: dict(array=shapes[port], rep=rep, pattern=t.pattern, origin=t.origin, paving=t.paving,
                       fitting=t.fitting) for port, t in tilers[path].items()}


NAMES = ["matmul_c1", "stencil_torus", "downscaler_chain"]


@pytest.mark.parametrize("name", NAMES)
def test_dsl_fixture_is_current_and_valid(name):
    model, tilers = _load(name)
    for path, tl in tilers.items():
        assert check_task_signature(path, _task(model, path), tl) is not None
    sched = build_schedule(model, 3)
    assert sched.device_steps()


def test_negative_origin_equals_wrapped_origin():
    """`origin [-1,-1]` in the text is the oracle's (H-1, W-1) modulo the array shape."""
    model, tilers = _load("stencil_torus")
    t = _oracle_tilers(model, "st", tilers)
    canon = orc.stencil_tilers(96, 160)
    for port in ("x", "y"):
        a = orc.tiler_offsets(t[port], 0, 96 * 160)
        b = orc.tiler_offsets(canon[port], 0, 96 * 160)
        assert np.array_equal(a, b)


def _inputs(name, rng):
    if name == "matmul_c1":
        return {"pa": rng.standard_normal(256 * 256).astype(np.float32),
                "pb": rng.standard_normal(256 * 256).astype(np.float32)}
    if name == "stencil_torus":
        return {"px": rng.random(96 * 160).astype(np.float32), "pw": orc.stencil_weights()}
    return {"frames": rng.random(2 * 36 * 64).astype(np.float32), "wh": orc.hfilter_weights(),
            "wv": orc.vfilter_weights()}


def _oracle(name, model, tilers, bind, D):
    if name == "matmul_c1":
        t = _oracle_tilers(model, "mm", tilers)
        return {"pc": orc.run_tile_task("matmul", t, {"a": bind["pa"], "b": bind["pb"]},
                                        {"c": (256 * 256, np.float32)}, 256 * 256, D)["c"]}
    if name == "stencil_torus":
        t = _oracle_tilers(model, "st", tilers)
        return {"py": orc.run_tile_task("stencil", t, {"x": bind["px"], "w": bind["pw"]},
                                        {"y": (96 * 160, np.float32)}, 96 * 160, D)["y"]}
    th, tv = _oracle_tilers(model, "h", tilers), _oracle_tilers(model, "v", tilers)
    mid = orc.run_tile_task("hfilter", th, {"x": bind["frames"], "w": bind["wh"]},
                            {"y": (2 * 36 * 24, np.float32)}, 2 * 36 * 8, D)["y"]
    return {"out": orc.run_tile_task("vfilter", tv, {"x": mid, "w": bind["wv"]},
                                     {"y": (2 * 16 * 24, np.float32)}, 2 * 4 * 24, D)["y"]}


@pytest.mark.gpu
@pytest.mark.parametrize("D", [1, 3, 8])
@pytest.mark.parametrize("name", NAMES)
def test_dsl_authored_models_on_gpu_vs_oracle(name, D):
    from paper_1105_4424_b200.executor import execute_schedule
    model, tilers = _load(name)
    bind = _inputs(name, np.random.default_rng(11 + D))
    want = _oracle(name, model, tilers, bind, D)
    sched = build_schedule(model, D)
    exact = execute_schedule(model, sched, bind, D, tilers=tilers, precision="exact")
    for port, ref in want.items():
        assert np.array_equal(exact.outputs[port], ref), (name, port)
    if name == "matmul_c1":
        got = execute_schedule(model, sched, bind, D, tilers=tilers).outputs["pc"].reshape(256, 256)
        a64 = bind["pa"].reshape(256, 256).astype(np.float64)
        b64 = bind["pb"].reshape(256, 256).astype(np.float64)
        bound = (2.0 ** -9 + 256 * 2.0 ** -23) * (np.abs(a64) @ np.abs(b64))
        assert np.all(np.abs(got - a64 @ b64) <= bound)
    else:
        fused = execute_schedule(model, sched, bind, D, tilers=tilers)
        for port, ref in want.items():
            assert np.array_equal(fused.outputs[port], ref), (name, port)
