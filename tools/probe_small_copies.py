"""Small host<->device copies (C1-sized, 64 KB - 4 MB): torch's pageable copy_ against staging
through a pinned buffer (host memcpy + async DMA), both directions, wall time per copy."""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
pin = torch.empty(8 << 20, dtype=torch.uint8).pin_memory()
pnp = pin.numpy()
d = torch.empty(8 << 20, dtype=torch.uint8, device=dev)
for kb in (64, 256, 1024, 4096):
    n = kb << 10
    src = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
    dst = np.empty(n, dtype=np.uint8)
    st = torch.from_numpy(src)
    res = {}
    for name in ("pageable", "staged"):
        for _ in range(20):
            pass
        ts = []
        for it in range(60):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if name == "pageable":
                d[:n].copy_(st)
            else:
                np.copyto(pnp[:n], src)
                d[:n].copy_(pin[:n], non_blocking=True)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        res["h2d_" + name] = sorted(ts)[30] * 1e6
        ts = []
        for it in range(60):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if name == "pageable":
                dst[:] = d[:n].cpu().numpy()
            else:
                pin[:n].copy_(d[:n], non_blocking=True)
                torch.cuda.current_stream().synchronize()
                np.copyto(dst, pnp[:n])
            ts.append(time.perf_counter() - t0)
        res["d2h_" + name] = sorted(ts)[30] * 1e6
    print(f"{kb:5d} KB  " + "  ".join(f"{k}={v:7.1f}us" for k, v in res.items()), flush=True)
