"""Diagnostic: tcgen05 GEMM under the 4 operand-majorness layouts."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_1105_4424_b200 import Tiler, _capi

M, N, K = 128, 256, 64
rng = np.random.default_rng(0)
A = rng.standard_normal((M, K)).astype(np.float32)
B = rng.standard_normal((K, N)).astype(np.float32)
C64 = A.astype(np.float64) @ B
tc = Tiler((0, 0), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((M, N), (M, N))
for a_k in (True, False):
    for b_k in (True, False):
        if a_k:
            ta = Tiler((0, 0), ((1, 0), (0, 0)), ((0,), (1,)), (K,)).bind((M, K), (M, N)); a = A
        else:
            ta = Tiler((0, 0), ((0, 0), (1, 0)), ((1,), (0,)), (K,)).bind((K, M), (M, N)); a = A.T.copy()
        if b_k:
            tb = Tiler((0, 0), ((0, 1), (0, 0)), ((0,), (1,)), (K,)).bind((N, K), (M, N)); b = B.T.copy()
        else:
            tb = Tiler((0, 0), ((0, 0), (0, 1)), ((1,), (0,)), (K,)).bind((K, N), (M, N)); b = B
        task = _capi.make_task("matmul", "float32", [ta, tb, tc])
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        dc = torch.full((M, N), -7.0, device="cuda")
        ptrs = [da.data_ptr(), db.data_ptr(), dc.data_ptr()]
        name = _capi.plan_name(task, 0, M * N, ptrs)
        _capi.launch(task, 0, M * N, ptrs)
        torch.cuda.synchronize()
        c = dc.cpu().numpy()
        print(f"a_kmajor={a_k} b_kmajor={b_k} {name}: maxerr={np.abs(c - C64).max():.4g} "
              f"nz={np.count_nonzero(c)} c[0,:3]={c[0,:3]} ref={C64[0,:3]}")
