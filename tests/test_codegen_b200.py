"""Row f4: generated B200 programs -- host C++ over the C ABI, and standalone CUDA text (kernels
generated from the model) -- compile here, run on the B200."""

import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import aol_oracle as orc

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_1105_4424_b200" / "_lib"
CUDA = Path("/usr/local/cuda")


def _compile(src: str, out: Path) -> Path:
    cpp = out.with_suffix(".cpp")
    cpp.write_text(src)
    r = subprocess.run(["g++", "-std=c++17", "-O2", str(cpp), "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
                        "-L", str(LIB), "-laolb200", "-L", str(CUDA / "lib64"), "-lcudart",
                        f"-Wl,-rpath,{LIB}", "-o", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def _tiler(d):
    from paper_1105_4424_b200 import Tiler
    return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"])


def _cases(golden):
    """(name, model, schedule, bindings) for a CG loop, a TF32 matmul, a stencil and a 2-task chain."""
    from paper_1105_4424_b200 import builders
    from paper_1105_4424_b200.model import model_from_dict
    from paper_1105_4424_b200.partition import build_schedule
    data, meta = golden
    out = []
    cg = model_from_dict(meta["cg_k20"]["model"])
    out.append(("cg", cg, build_schedule(cg, 2), {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}))
    M, N, K = 300, 264, 96
    g = orc.gemm_tilers(M, N, K)
    mm = builders.tile_task_model("matmul", {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]",
                                             "c": f"out float32 [{M},{N}]"}, {k: _tiler(v) for k, v in g.items()},
                                  (M, N))
    rng = np.random.default_rng(3)
    out.append(("matmul", mm, build_schedule(mm, 3), {"p_a": rng.standard_normal(M * K).astype(np.float32),
                                                     "p_b": rng.standard_normal(K * N).astype(np.float32)}))
    t = orc.stencil_tilers(64, 96)
    st = builders.tile_task_model("stencil", {"x": "in float32 [64,96]", "w": "in float32 [9]",
                                              "y": "out float32 [64,96]"}, {k: _tiler(v) for k, v in t.items()},
                                  (64, 96))
    out.append(("stencil", st, build_schedule(st, 2), {"p_x": rng.random(64 * 96).astype(np.float32),
                                                      "p_w": orc.stencil_weights()}))
    return out


def _check_vs_oracle(golden, name, sched, bind, outputs, stdout, exact):
    """Pin a generated program's outputs to the oracle / the reference golden, not only the drop-in:
    CG -> the reference executor's iteration count and x within 1e-10 (tests/test_refexec.py:237-247);
    stencil -> bit-exact oracle; matmul -> bit-exact oracle for the exact order, else the TF32 bound."""
    data, meta = golden
    D = len(sched.device_steps()[0].launches)
    if name == "cg":
        ref = meta["cg_k20"]["runs"][str(D)]
        assert f"iterations={ref['iterations']} " in stdout, stdout
        x_ref = data[f"cg_k20/x_d{D}"]
        assert np.max(np.abs(outputs["x"] - x_ref)) / np.max(np.abs(x_ref)) <= 1e-10
    elif name == "stencil":
        t = orc.stencil_tilers(64, 96)
        want = orc.run_tile_task("stencil", t, {"x": bind["p_x"], "w": bind["p_w"]},
                                 {"y": (64 * 96, np.float32)}, 64 * 96, D)["y"]
        assert np.array_equal(outputs["p_y"], want)
    elif name == "matmul":
        M, N, K = 300, 264, 96
        if exact:
            want = orc.run_tile_task("matmul", orc.gemm_tilers(M, N, K), {"a": bind["p_a"], "b": bind["p_b"]},
                                     {"c": (M * N, np.float32)}, M * N, D)["c"]
            assert np.array_equal(outputs["p_c"], want)
        else:
            a64 = bind["p_a"].reshape(M, K).astype(np.float64)
            b64 = bind["p_b"].reshape(K, N).astype(np.float64)
            bound = (2.0 ** -9 + K * 2.0 ** -23) * (np.abs(a64) @ np.abs(b64))
            assert np.all(np.abs(outputs["p_c"].reshape(M, N) - a64 @ b64) <= bound)


def test_generated_programs_compile(golden):
    from paper_1105_4424_b200.codegen_b200 import generate_host_cpp
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        for name, model, sched, _ in _cases(golden):
            src = generate_host_cpp(model, sched)
            assert "aol_launch(&task" in src
            _compile(src, Path(d) / name)


@pytest.mark.gpu
def test_generated_programs_match_the_drop_in(golden, tmp_path):
    """The compiled host programs produce bit-identical outputs to execute_schedule on the same inputs,
    and those outputs match the oracle / the reference golden (_check_vs_oracle)."""
    from paper_1105_4424_b200.codegen_b200 import generate_host_cpp
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.model import enum_value
    for name, model, sched, bind in _cases(golden):
        exe = _compile(generate_host_cpp(model, sched), tmp_path / name)
        work = tmp_path / f"{name}_io"
        work.mkdir()
        root = model.application_components[model.application_root]
        for p in root.ports:
            if enum_value(p.direction) in ("in", "inout"):
                np.ascontiguousarray(np.asarray(bind[p.name]).astype(enum_value(p.data_type))).tofile(
                    work / f"{p.name}.bin")
        r = subprocess.run([str(exe), str(work)], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stderr
        ref = execute_schedule(model, sched, bind, len(sched.device_steps()[0].launches))
        got_all = {}
        for p in root.ports:
            if enum_value(p.direction) == "out":
                got = np.fromfile(work / f"{p.name}.out.bin", dtype=enum_value(p.data_type))
                assert np.array_equal(got, ref.outputs[p.name]), (name, p.name)
                got_all[p.name] = got
        if name == "cg":
            assert f"iterations={ref.iterations} " in r.stdout
        _check_vs_oracle(golden, name, sched, bind, got_all, r.stdout, exact=False)


def _nvcc(src: str, out: Path, link: bool) -> Path:
    cu = out.with_suffix(".cu")
    cu.write_text(src)
    cmd = ["nvcc", "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a", str(cu), "-o", str(out)]
    r = subprocess.run(cmd if link else cmd[:-2] + ["-c", "-o", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "warning" not in r.stderr, r.stderr
    return out


def test_generated_cuda_programs_compile(golden, tmp_path):
    """backend="cuda": the kernels are CUDA text generated from the model (the analog of the
    reference's OpenCL templates); the programs cross-compile for sm_100a without warnings."""
    from paper_1105_4424_b200.codegen_b200 import generate_host_cpp, generate_kernels_cu
    for name, model, sched, _ in _cases(golden):
        src = generate_host_cpp(model, sched, backend="cuda")
        assert "aol_launch" not in src and "__global__ void k_" in src
        assert generate_kernels_cu(model, sched) in src
        _nvcc(src, tmp_path / f"{name}.o", link=False)


@pytest.mark.gpu
def test_generated_cuda_programs_match_the_drop_in(golden, tmp_path):
    """The generated CUDA programs are bit-identical to execute_schedule: CG (same iteration count,
    the same deterministic dot tree), the exact-order matmul (precision="exact") and the stencil."""
    from paper_1105_4424_b200.codegen_b200 import generate_host_cpp
    from paper_1105_4424_b200.executor import execute_schedule
    from paper_1105_4424_b200.model import enum_value
    for name, model, sched, bind in _cases(golden):
        exe = _nvcc(generate_host_cpp(model, sched, backend="cuda"), tmp_path / name, link=True)
        work = tmp_path / f"{name}_io"
        work.mkdir()
        root = model.application_components[model.application_root]
        for p in root.ports:
            if enum_value(p.direction) in ("in", "inout"):
                np.ascontiguousarray(np.asarray(bind[p.name]).astype(enum_value(p.data_type))).tofile(
                    work / f"{p.name}.bin")
        r = subprocess.run([str(exe), str(work)], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stderr
        kw = {"precision": "exact"} if name == "matmul" else {}
        ref = execute_schedule(model, sched, bind, len(sched.device_steps()[0].launches), **kw)
        got_all = {}
        for p in root.ports:
            if enum_value(p.direction) == "out":
                got = np.fromfile(work / f"{p.name}.out.bin", dtype=enum_value(p.data_type))
                assert np.array_equal(got, ref.outputs[p.name]), (name, p.name)
                got_all[p.name] = got
        if name == "cg":
            assert f"iterations={ref.iterations} " in r.stdout
        _check_vs_oracle(golden, name, sched, bind, got_all, r.stdout, exact=(name == "matmul"))
