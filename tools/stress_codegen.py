"""Row f4 beyond the three test models: the generated B200 programs (host C++ over the C ABI,
and the standalone CUDA-text backend) for every sharded test case (matmul, stencil chain,
downscaler chain, transpose chain, elementwise chain) at D = 1..5, compiled here, run, and
compared bit for bit with execute_schedule on the same inputs (CUDA text: precision "exact"
for matmul, the order the generated kernels use).  python tools/stress_codegen.py"""
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

from _sharded_cases import CASES  # noqa: E402
from paper_1105_4424_b200.codegen_b200 import generate_host_cpp  # noqa: E402
from paper_1105_4424_b200.executor import execute_schedule  # noqa: E402
from paper_1105_4424_b200.model import enum_value  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402

LIB = ROOT / "paper_1105_4424_b200" / "_lib"
CUDA = Path("/usr/local/cuda")
fails = 0
with tempfile.TemporaryDirectory() as tmp:
    tmp = Path(tmp)
    for name, fn in sorted(CASES.items()):
        model, bind, out, _ = fn()
        root = model.application_components[model.application_root]
        for D in (1, 3, 5):
            sched = build_schedule(model, D)
            for backend in ("capi", "cuda"):
                exe = tmp / f"{name}_{D}_{backend}"
                if backend == "capi":
                    src = exe.with_suffix(".cpp")
                    src.write_text(generate_host_cpp(model, sched))
                    cmd = ["g++", "-std=c++17", "-O2", str(src), "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
                           "-L", str(LIB), "-laolb200", "-L", str(CUDA / "lib64"), "-lcudart", f"-Wl,-rpath,{LIB}",
                           "-o", str(exe)]
                else:
                    src = exe.with_suffix(".cu")
                    src.write_text(generate_host_cpp(model, sched, backend="cuda"))
                    cmd = ["nvcc", "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a", str(src), "-o", str(exe)]
                r = subprocess.run(cmd, capture_output=True, text=True)
                if r.returncode:
                    print(f"COMPILE FAIL {name} D={D} {backend}: {r.stderr[-400:]}", flush=True)
                    fails += 1
                    continue
                work = tmp / f"{name}_{D}_{backend}_io"
                work.mkdir()
                for p in root.ports:
                    if enum_value(p.direction) in ("in", "inout"):
                        np.ascontiguousarray(np.asarray(bind[p.name]).astype(enum_value(p.data_type))).tofile(
                            work / f"{p.name}.bin")
                r = subprocess.run([str(exe), str(work)], capture_output=True, text=True, timeout=300)
                if r.returncode:
                    print(f"RUN FAIL {name} D={D} {backend}: {r.stderr[-400:]}", flush=True)
                    fails += 1
                    continue
                kw = {"precision": "exact"} if (backend == "cuda" and name == "matmul") else {}
                ref = execute_schedule(model, sched, bind, D, **kw).outputs
                ok = True
                for p in root.ports:
                    if enum_value(p.direction) == "out":
                        got = np.fromfile(work / f"{p.name}.out.bin", dtype=enum_value(p.data_type))
                        ok = ok and np.array_equal(got, np.asarray(ref[p.name]).ravel())
                print(f"{name} D={D} {backend}: {'ok' if ok else 'MISMATCH'}", flush=True)
                fails += 0 if ok else 1
print("all ok" if not fails else f"{fails} failures")
sys.exit(1 if fails else 0)
