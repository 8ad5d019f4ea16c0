"""Random filter chains through make_distributed_executor with one process per rank (launch with
torchrun; gloo, ranks may share one GPU): the plan's exchanges over torch.distributed, packed
non-dense outputs, the fused output gather through CUDA IPC, D = world..world+2 launches; rank 0
compares with the oracle bit for bit.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/stress_dist.py"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import aol_oracle as orc  # noqa: E402
from paper_1105_4424_b200.distributed import make_distributed_executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402
from test_shard_plan_simulation import _model, _random_chain  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
dist.init_process_group("gloo")
rng = np.random.default_rng(int(os.environ.get("SEED", "1")))           # same stream on every rank
bad = 0
cases = int(os.environ.get("CASES", "60"))
for case in range(cases):
    arr, stages, tilers = _random_chain(rng, int(rng.integers(2, 4)))
    model = _model(arr, stages)
    D = world + int(rng.integers(0, 3))
    fused = bool(rng.integers(0, 2))
    n = arr[0] * arr[1]
    x = rng.random(n)
    bind = {"x": x, **{f"w{k}": tl[2] for k, tl in enumerate(tilers)}}
    ex = make_distributed_executor(model, build_schedule(model, D), bind, fused_gather=fused)
    ex.run()
    out = ex.outputs()
    ex.close()
    if rank == 0:
        ref = x.copy()
        for tx, ty, w in tilers:
            y = np.zeros(n)
            orc.tile_filter(ref, w, y, tx, ty, 0, n)
            ref = y
        if not np.array_equal(out["y"], ref):
            print(f"FAIL case {case}: D={D} fused={fused} arr={arr} tilers={tilers}", flush=True)
            bad += 1
    elif out:
        print(f"FAIL case {case}: rank {rank} got outputs", flush=True)
        bad += 1
flag = torch.tensor([bad], dtype=torch.int64)
dist.all_reduce(flag)
if rank == 0:
    print("all ok" if flag.item() == 0 else f"{flag.item()} failures", flush=True)
dist.destroy_process_group()
sys.exit(1 if flag.item() else 0)
