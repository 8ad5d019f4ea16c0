"""H2D / D2H bandwidth alone and concurrently (pinned host memory, 1 GiB each way)."""
import json
import time
import torch

n = 1 << 28
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.ones(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


gb = n * 4 / 1e9
t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_GBps": gb / t1, "d2h_GBps": gb / t2, "duplex_total_GBps": 2 * gb / t3,
                  "duplex_ms": t3 * 1e3, "serial_ms": (t1 + t2) * 1e3}))
