"""Random filter chains (toroidal windows, dense and non-dense output tilers; the generator of
tests/test_shard_plan_simulation.py) through execute_schedule(devices=[0] * W): W replicas on one
GPU exchanging exactly what the plan says (LocalTransport, cuda_pack / cuda_unpack for non-dense
outputs, the root gather at the end), D = W..W+2 launches, compared bit for bit with the oracle.

    SEED=1 CASES=200 python tools/stress_sharded.py"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

from oracle import aol_oracle as orc  # noqa: E402
from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402
from test_shard_plan_simulation import _model, _random_chain  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
for case in range(int(os.environ.get("CASES", "200"))):
    W = int(rng.integers(2, 9))
    arr, stages, tilers = _random_chain(rng, int(rng.integers(2, 4)))
    model = _model(arr, stages)
    D = W + int(rng.integers(0, 3))
    n = arr[0] * arr[1]
    x = rng.random(n)
    ref = x.copy()
    for tx, ty, w in tilers:
        y = np.zeros(n)
        orc.tile_filter(ref, w, y, tx, ty, 0, n)
        ref = y
    bind = {"x": x, **{f"w{k}": tl[2] for k, tl in enumerate(tilers)}}
    got = execute_schedule(model, build_schedule(model, D), bind, D, devices=[0] * W).outputs["y"]
    if not np.array_equal(got, ref):
        print(f"FAIL case {case}: W={W} D={D} arr={arr} tilers={tilers}", flush=True)
        sys.exit(1)
    if case % 50 == 49:
        print(f"{case + 1} cases ok", flush=True)
print("all ok")
