"""Build libaolb200.so in-tree for sm_100a (nvcc, no JIT cache) — used by __graft_entry__.build()."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib" / "libaolb200.so"
SOURCES = ["aol_capi.cu", "aol_tile.cu", "aol_ident.cu", "aol_gemm.cu", "aol_stencil.cu", "aol_linefilter.cu", "aol_loop.cu", "aol_loopk.cu", "aol_ipc.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "aol_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    objs = []
    jobs = []
    for src in SOURCES:
        obj = OUT.parent / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
               "-I", str(PKG.parent / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        jobs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
        objs.append(obj)
    errs = []
    for src, j in zip(SOURCES, jobs):
        out, _ = j.communicate()
        if j.returncode != 0:
            errs.append(f"--- {src}\n{out}")
        elif verbose and out:
            print(f"--- {src}\n{out}")
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
    tmp = OUT.with_suffix(".so.tmp")
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart_static", "-ldl",
                    "-lpthread", "-lrt"], check=True)
    os.replace(tmp, OUT)
    for o in objs:
        o.unlink(missing_ok=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
