"""H2D of a 8192 x 8192 fp32 matrix from pinned memory: one contiguous copy vs 4 column-block
2-D copies (aol_memcpy2d, 8 KB rows) vs 4 row-block copies; and the 2-D D2H of C blocks."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1105_4424_b200 import _capi  # noqa: E402

K = N = 8192
h = torch.randn(K * N).pin_memory()
d = torch.empty(K * N, device="cuda")
s = torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        s.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def contig():
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)


def cols(nb):
    w = N // nb

    def f():
        for j in range(nb):
            _capi.memcpy2d(d.data_ptr() + j * w * 4, N * 4, h.data_ptr() + j * w * 4, N * 4, w * 4, K, s.cuda_stream)
    return f


def d2h_cols(nb):
    w = N // nb

    def f():
        for j in range(nb):
            _capi.memcpy2d(h.data_ptr() + j * w * 4, N * 4, d.data_ptr() + j * w * 4, N * 4, w * 4, K, s.cuda_stream)
    return f


gb = K * N * 4 / 1e9
for name, fn in [("contiguous H2D", contig), ("2-D H2D 4 col blocks", cols(4)), ("2-D H2D 8 col blocks", cols(8)),
                 ("2-D H2D 16 col blocks", cols(16)), ("2-D D2H 4 col blocks", d2h_cols(4))]:
    t = timed(fn)
    print(f"{name:24s} {t * 1e3:7.2f} ms  {gb / t:6.1f} GB/s", flush=True)
