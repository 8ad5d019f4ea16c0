"""execute_schedule under random combinations of its keyword arguments (pipeline, device_outputs,
out= (numpy / pinned torch), stream=, devices=, fuse=, graphs=, precision=) on the sharded
test cases and CG: every combination must return exactly the plain call's outputs.

    SEED=1 CASES=120 python tools/stress_api.py"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from _sharded_cases import CASES  # noqa: E402
from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.model import enum_value, model_from_dict  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
meta = json.loads((ROOT / "tests" / "golden" / "reference_golden.json").read_text())
data = np.load(ROOT / "tests" / "golden" / "reference_golden.npz")


def cg_case():
    model = model_from_dict(meta["cg_k20"]["model"])
    return model, {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}, "x", None


def ref_op_case(op):
    """A reference elementwise op (refexec.py:504-514) on n elements: y inout for axpy / scale,
    a host-resident scalar `a` where the op takes one."""
    from paper_1105_4424_b200 import builders
    n = 4999 if op == "axpy" else 6007             # fixed per op: the plain results are cached per name
    r = np.random.default_rng(n)
    if op == "axpy":
        tp = ["y inout float64 [%d]" % n, "x in float64 [%d]" % n, "a in float64 [1]"]
        rp = ["i in float64 [%d]" % n, "v in float64 [%d]" % n, "s in float64 [1]", "o out float64 [%d]" % n]
        cn = ["i -> t.y", "v -> t.x", "s -> t.a", "t.y -> o"]
        al = ["allocate data i onto dev.gmem", "allocate data v onto dev.gmem", "allocate data s onto host.ram",
              "allocate task t onto dev.cu"]
        bind = {"i": r.standard_normal(n), "v": r.standard_normal(n), "s": np.array([0.75])}
    else:                                          # sub: z = x - y
        tp = ["x in float64 [%d]" % n, "y in float64 [%d]" % n, "z out float64 [%d]" % n]
        rp = ["p in float64 [%d]" % n, "q in float64 [%d]" % n, "o out float64 [%d]" % n]
        cn = ["p -> t.x", "q -> t.y", "t.z -> o"]
        al = ["allocate data p onto dev.gmem", "allocate data q onto dev.gmem", "allocate data t.z onto dev.gmem",
              "allocate task t onto dev.cu"]
        bind = {"p": r.standard_normal(n), "q": r.standard_normal(n)}
    model = builders.single_task_model(op, tp, rp, cn, al, n)
    return model, bind, "o", None


cases = dict(CASES)
cases["cg"] = cg_case
cases["axpy"] = lambda: ref_op_case("axpy")
cases["sub"] = lambda: ref_op_case("sub")
names = sorted(cases)
plain_cache = {}
for case in range(int(os.environ.get("CASES", "120"))):
    name = names[int(rng.integers(0, len(names)))]
    model, bind, out_port, _ = cases[name]()
    D = int(rng.integers(1, 9))
    sched = build_schedule(model, D)
    prec = str(rng.choice(["exact", "default", "3xtf32"])) if name == "matmul" else "default"
    loop_kw = {}
    if name == "cg" and rng.random() < 0.3:
        loop_kw = {"tol": float(rng.choice([1e-4, 1e-8])), "max_iter": int(rng.integers(3, 60))}
    key = (name, D, prec, tuple(sorted(loop_kw.items())))
    if key not in plain_cache:
        plain_cache[key] = execute_schedule(model, sched, bind, D, precision=prec, **loop_kw).outputs
    plain = plain_cache[key]
    kw = {"precision": prec, **loop_kw}
    combo = [f"prec={prec}"] + [f"{k}={v}" for k, v in loop_kw.items()]
    if rng.random() < 0.4:
        kw["pipeline"] = int(rng.integers(2, 9))
        combo.append(f"pipeline={kw['pipeline']}")
    if rng.random() < 0.3 and "pipeline" not in kw:
        kw["devices"] = [0] * int(rng.integers(2, 5))
        combo.append(f"devices={len(kw['devices'])}")
    if rng.random() < 0.3:
        kw["stream"] = torch.cuda.Stream()
        combo.append("stream")
        if "devices" in kw:
            kw.pop("devices")
            combo.remove(combo[-2])
    if rng.random() < 0.3:
        kw["fuse"] = False
        combo.append("fuse=False")
    if rng.random() < 0.3:
        kw["graphs"] = False
        combo.append("graphs=False")
    out_kind = rng.choice(["none", "numpy", "pinned", "device"])
    root = model.application_components[model.application_root]
    outs = {p.name: p for p in root.ports if enum_value(p.direction) == "out"}
    if out_kind == "numpy":
        kw["out"] = {n: np.empty(p.shape.total, dtype=enum_value(p.data_type)) for n, p in outs.items()}
    elif out_kind == "pinned":
        kw["out"] = {n: torch.empty(p.shape.total, dtype=getattr(torch, enum_value(p.data_type))).pin_memory()
                     for n, p in outs.items()}
    elif out_kind == "device" and "devices" not in kw:
        kw["device_outputs"] = True
    combo.append(f"out={out_kind}")
    if rng.random() < 0.3:                         # pinned torch bindings instead of numpy
        bind = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in bind.items()}
        combo.append("pinned-in")
    try:
        res = execute_schedule(model, sched, bind, D, **kw).outputs
        torch.cuda.synchronize()
        ok = True
        for n, v in plain.items():
            g = res[n]
            g = g.detach().cpu().numpy() if isinstance(g, torch.Tensor) else np.asarray(g)
            ok &= np.array_equal(g.ravel(), np.asarray(v).ravel())
    except Exception as e:  # noqa: BLE001
        print(f"ERROR case {case} {name} D={D} {combo}: {type(e).__name__}: {str(e)[:200]}", flush=True)
        ok = False
    if not ok:
        print(f"FAIL case {case}: {name} D={D} {combo}", flush=True)
        sys.exit(1)
    if case % 20 == 19:
        print(f"{case + 1} cases ok", flush=True)
print("all ok")
