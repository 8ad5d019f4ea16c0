"""Probe sweep points under different L2 states and L2 fetch-granularity limits.

python tools/sweep_probe.py [--gran N] "m:kind:T" ...
  flush modes per point: none (back to back), write (256 MiB fill before each launch: leaves
  L2 full of DIRTY lines the timed kernel must write back), write+read (fill, then read a
  separate 256 MiB buffer: L2 left holding clean lines), plus torch's own copy of the same
  byte count as a yardstick.
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1105_4424_b200 import _capi  # noqa: E402

args = sys.argv[1:]
gran = None
if args and args[0] == "--gran":
    gran = int(args[1])
    args = args[2:]
torch.zeros(1, device="cuda")
if gran is not None:
    cu = ctypes.CDLL("libcuda.so.1")
    rc = cu.cuCtxSetLimit(ctypes.c_int(5), ctypes.c_size_t(gran))      # CU_LIMIT_MAX_L2_FETCH_GRANULARITY
    v = ctypes.c_size_t(0)
    cu.cuCtxGetLimit(ctypes.byref(v), ctypes.c_int(5))
    print(f"cuCtxSetLimit(MAX_L2_FETCH_GRANULARITY, {gran}) rc={rc} -> {v.value}")
sw = bench.SweepWorkload.__new__(bench.SweepWorkload)
sw.torch, sw.device = torch, torch.device("cuda", 0)
scrub = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
rd = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
acc = torch.zeros(1, device="cuda")


def timed(fn, mode, reps=20):
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for _ in range(3):
        fn()
    if mode == "none":
        ev[0][0].record()
        for _ in range(reps):
            fn()
        ev[0][1].record()
        torch.cuda.synchronize()
        return ev[0][0].elapsed_time(ev[0][1]) / reps
    for i, (a, b) in enumerate(ev):
        scrub.fill_(float(i))
        if mode == "write+read":
            acc.copy_(rd.sum())
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]


for spec in args:
    m, kind, T = spec.split(":")
    m, T = int(m), int(float(T))
    t = sw._make(m, kind, T)
    st = int(torch.cuda.current_stream().cuda_stream)

    def run():
        _capi.launch(t["task"], 0, T, t["ptrs"], (), st)
    res = {mode: timed(run, mode) for mode in ("none", "write", "write+read")}
    a = torch.empty(t["bytes"] // 8, device="cuda")        # copy_ of n floats moves 8n bytes
    b = torch.empty_like(a)
    ref = timed(lambda: b.copy_(a), "write+read")
    line = " ".join(f"{k}={v * 1e3:7.1f}us/{t['bytes'] / v / 1e6:6.0f}GB/s" for k, v in res.items())
    print(f"{spec:18s} {t['plan']:22s} {line}  torch.copy_ same bytes (w+r) {ref * 1e3:7.1f}us/"
          f"{t['bytes'] / ref / 1e6:6.0f}GB/s", flush=True)
    del t, a, b
    torch.cuda.empty_cache()
