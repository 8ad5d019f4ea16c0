"""Run one tile_copy sweep point (for ncu): python tools/sweep_point.py m kind T [reps]."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench

m, kind, T = int(sys.argv[1]), sys.argv[2], int(float(sys.argv[3]))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
sw = bench.SweepWorkload.__new__(bench.SweepWorkload)
sw.torch, sw.device = torch, torch.device("cuda", 0)
t = sw._make(m, kind, T)
from paper_1105_4424_b200 import _capi
for _ in range(reps):
    _capi.launch(t["task"], 0, T, t["ptrs"], (), int(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print(t["plan"], t["bytes"])
