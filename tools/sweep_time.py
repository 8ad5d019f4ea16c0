"""Time tile_copy sweep points: python tools/sweep_time.py "m:kind:T" ... -> GB/s per point (CUDA events)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1105_4424_b200 import _capi  # noqa: E402

sw = bench.SweepWorkload.__new__(bench.SweepWorkload)
sw.torch, sw.device = torch, torch.device("cuda", 0)
for spec in sys.argv[1:]:
    m, kind, T = spec.split(":")
    m, T = int(m), int(float(T))
    t = sw._make(m, kind, T)
    st = int(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        _capi.launch(t["task"], 0, T, t["ptrs"], (), st)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    s.record()
    for _ in range(reps):
        _capi.launch(t["task"], 0, T, t["ptrs"], (), st)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"{spec:22s} {t['plan']:22s} {ms:8.3f} ms {t['bytes'] / ms / 1e6:8.0f} GB/s")
    del t
    torch.cuda.empty_cache()
