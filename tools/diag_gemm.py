"""Diagnostic: run the tcgen05 GEMM on structured inputs and save C (gpurun_out/diag_gemm.npz)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from oracle import aol_oracle as orc
from paper_1105_4424_b200 import Tiler, _capi


def run(A, B, precision="default"):
    M, K = A.shape
    N = B.shape[1]
    g = orc.gemm_tilers(M, N, K)
    bt = [Tiler(g[k]["origin"], g[k]["paving"], g[k]["fitting"], g[k]["pattern"]).bind(g[k]["array"], (M, N)) for k in "abc"]
    task = _capi.make_task("matmul", "float32", bt, precision=precision)
    a = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    b = torch.from_numpy(np.ascontiguousarray(B)).cuda()
    c = torch.full((M, N), -7.0, device="cuda")
    ptrs = [a.data_ptr(), b.data_ptr(), c.data_ptr()]
    print(_capi.plan_name(task, 0, M * N, ptrs))
    _capi.launch(task, 0, M * N, ptrs)
    torch.cuda.synchronize()
    return c.cpu().numpy()


out = {}
M, N, K = 128, 256, 32
m = np.arange(M)[:, None]; k = np.arange(K)[None, :]
A1 = (k == (m % 32)).astype(np.float32)
kk = np.arange(K)[:, None]; n = np.arange(N)[None, :]
B1 = (kk * 64 + (n % 64)).astype(np.float32)
out["c1"] = run(A1, B1)
A2 = (m * 16 + (k % 16)).astype(np.float32)
B2 = (kk == (n % 32)).astype(np.float32)
out["c2"] = run(A2, B2)
rng = np.random.default_rng(0)
A3 = rng.standard_normal((M, K)).astype(np.float32); B3 = rng.standard_normal((K, N)).astype(np.float32)
out["a3"], out["b3"], out["c3"] = A3, B3, run(A3, B3)
np.savez("gpurun_out/diag_gemm.npz", **out)
print("saved")

