"""Normwise error of tf32 vs 3xtf32 vs K, printed."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from oracle import aol_oracle as orc
from paper_1105_4424_b200 import Tiler, _capi
for K in (256, 2048, 8192):
    M = N = 1024
    rng = np.random.default_rng(K)
    A = rng.standard_normal((M, K)).astype(np.float32); B = rng.standard_normal((K, N)).astype(np.float32)
    c64 = A.astype(np.float64) @ B.astype(np.float64)
    g = orc.gemm_tilers(M, N, K)
    bt = [Tiler(g[k]["origin"], g[k]["paving"], g[k]["fitting"], g[k]["pattern"]).bind(g[k]["array"], (M, N)) for k in "abc"]
    da, db = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for prec in ("tf32", "3xtf32"):
        dc = torch.zeros(M, N, device="cuda")
        _capi.launch(_capi.make_task("matmul", "float32", bt, precision=prec), 0, M * N, [da.data_ptr(), db.data_ptr(), dc.data_ptr()])
        torch.cuda.synchronize()
        c = dc.cpu().numpy()
        print(K, prec, np.linalg.norm(c - c64) / np.linalg.norm(c64), np.max(np.abs(c - c64) / (np.abs(A) @ np.abs(B))))
    c32 = (torch.from_numpy(A).cuda().double() @ torch.from_numpy(B).cuda().double()).float().cpu().numpy()
    torch.backends.cuda.matmul.allow_tf32 = False
    cf = (da @ db).cpu().numpy()
    print(K, "cublas-fp32", np.linalg.norm(cf - c64) / np.linalg.norm(c64))
