"""Wide vs narrow 3xTF32 forms on one 1024 x 1024 x K product: normwise error against fp64 per
form and K-chunk, bit differences between chunk sizes, and where the wide form's error sits
(row quarter / column half of the CTA tile)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if len(sys.argv) > 1:
    sys.path.insert(0, str(ROOT))
    import torch
    from oracle import aol_oracle as orc
    from paper_1105_4424_b200 import Tiler, _capi
    M = N = 1024
    K = int(sys.argv[1])
    rng = np.random.default_rng(K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    g = orc.gemm_tilers(M, N, K)
    bt = [Tiler(g[k]["origin"], g[k]["paving"], g[k]["fitting"], g[k]["pattern"]).bind(g[k]["array"], (M, N))
          for k in "abc"]
    da, db = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dc = torch.zeros(M, N, device="cuda")
    _capi.launch(_capi.make_task("matmul", "float32", bt, precision="3xtf32"), 0, M * N,
                 [da.data_ptr(), db.data_ptr(), dc.data_ptr()])
    torch.cuda.synchronize()
    np.save(sys.argv[2], dc.cpu().numpy())
    sys.exit(0)

for K in (64, 256, 2048):
    rng = np.random.default_rng(K)
    A = rng.standard_normal((1024, K)).astype(np.float32)
    B = rng.standard_normal((K, 1024)).astype(np.float32)
    c64 = A.astype(np.float64) @ B.astype(np.float64)
    res = {}
    for name, env in (("narrow64", {"AOL_3XTF32_WIDE": "0"}), ("wide32", {"AOL_3XTF32_CHUNK": "32"}),
                      ("wide64", {"AOL_3XTF32_CHUNK": "64"}), ("wide128", {"AOL_3XTF32_CHUNK": "128"}),
                      ("wide_all", {"AOL_3XTF32_CHUNK": str(K)})):
        out = f"/tmp/c_{name}_{K}.npy"
        subprocess.run([sys.executable, __file__, str(K), out], env={**os.environ, **env}, check=True)
        c = np.load(out)
        res[name] = c
        err = np.abs(c - c64)
        nw = np.linalg.norm(c - c64) / np.linalg.norm(c64)
        q = [float(np.linalg.norm(err.reshape(4, 256, 1024)[:, 32 * i:32 * i + 32]) ) for i in range(4)]
        h = [float(np.linalg.norm(err.reshape(1024, 4, 256)[:, :, 128 * j:128 * j + 128])) for j in range(2)]
        print(f"K={K:5d} {name:9s} normwise {nw:.3e}  row-lane-quarter err {['%.2e' % x for x in q]}  "
              f"col-half err {['%.2e' % x for x in h]}", flush=True)
    print(f"K={K:5d} wide64 == wide128 bits: {np.array_equal(res['wide64'], res['wide128'])}; "
          f"wide64 == narrow64: {np.array_equal(res['wide64'], res['narrow64'])}", flush=True)
