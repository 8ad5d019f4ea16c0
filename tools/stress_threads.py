"""execute_schedule from several host threads at once (a server's usage): each thread draws
random cases (sharded test cases, CG, matmul in three precisions) and checks every result
against the single-threaded plain call.  THREADS=4 CASES=100 python tools/stress_threads.py"""
import os
import sys
import threading
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from _sharded_cases import CASES  # noqa: E402
from paper_1105_4424_b200 import builders  # noqa: E402
from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.model import model_from_dict  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

meta = json.loads((ROOT / "tests" / "golden" / "reference_golden.json").read_text())
data = np.load(ROOT / "tests" / "golden" / "reference_golden.npz")
torch.zeros(1, device="cuda")


def cg_case():
    model = model_from_dict(meta["cg_k20"]["model"])
    return model, {k: data[f"cg_k20/{k}"] for k in ("rowptr", "colidx", "values", "b")}, "x", None


def mm_case():
    rng = np.random.default_rng(9)
    model = builders.matmul_model(320, 288, 96)
    return model, {"p_a": rng.standard_normal(320 * 96, dtype=np.float32),
                   "p_b": rng.standard_normal(96 * 288, dtype=np.float32)}, "p_c", None


cases = dict(CASES)
cases["cg"] = cg_case
cases["matmul"] = mm_case
# one model / schedule object per (case, D), shared by every thread (the cache's regime)
built = {}
for name, fn in cases.items():
    model, bind, out, _ = fn()
    for D in (1, 3, 5):
        sched = build_schedule(model, D)
        for prec in (("default", "exact", "3xtf32") if name == "matmul" else ("default",)):
            want = execute_schedule(model, sched, bind, D, precision=prec).outputs[out]
            built[(name, D, prec)] = (model, sched, bind, out, want)
keys = sorted(built)
errors = []


def worker(tid):
    rng = np.random.default_rng(1000 + tid)
    stream = torch.cuda.Stream() if tid % 2 else None
    for c in range(int(os.environ.get("CASES", "100"))):
        k = keys[int(rng.integers(0, len(keys)))]
        model, sched, bind, out, want = built[k]
        kw = {"precision": k[2]}
        if stream is not None:
            kw["stream"] = stream
        if rng.random() < 0.3:
            kw["pipeline"] = int(rng.integers(2, 6))    # streamed paths: shared side streams + staging ring
        try:
            got = execute_schedule(model, sched, bind, k[1], **kw).outputs[out]
            if not np.array_equal(np.asarray(got), np.asarray(want)):
                errors.append(f"thread {tid} case {c} {k}: mismatch")
        except Exception as e:  # noqa: BLE001
            errors.append(f"thread {tid} case {c} {k}: {type(e).__name__}: {str(e)[:160]}")
        if errors:
            return


threads = [threading.Thread(target=worker, args=(t,)) for t in range(int(os.environ.get("THREADS", "4")))]
for t in threads:
    t.start()
for t in threads:
    t.join()
torch.cuda.synchronize()
if errors:
    print("\n".join(errors[:10]))
    sys.exit(1)
print(f"all ok: {len(threads)} threads x {os.environ.get('CASES', '100')} calls")
