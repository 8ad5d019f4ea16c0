"""Per-chunk event timeline of the streamed matmul e2e (H2D / compute / D2H streams)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1105_4424_b200.executor as exmod  # noqa: E402
from paper_1105_4424_b200 import _capi  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "matmul"](torch, torch.device("cuda:0"), 0, 1)
w.e2e_setup()
marks = []
orig_launch = _capi.launch


def traced_launch(task, first, count, ports, scalars=(), stream=0):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
    e0.record(s)
    orig_launch(task, first, count, ports, scalars, stream)
    e1.record(s)
    marks.append((e0, e1))


_capi.launch = traced_launch
for rep in range(3):
    marks.clear()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    t0 = time.perf_counter()
    ex = exmod.Executor(w.model, w.schedule, w.hin, 1, pipeline=w.pipeline)
    ex.run_streamed(out=w.hout)
    end = torch.cuda.Event(enable_timing=True)
    end.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    print(f"rep {rep}: wall {wall:.2f} ms, device {start.elapsed_time(end):.2f} ms; launches (start..end ms): " +
          " ".join(f"{start.elapsed_time(a):.2f}..{start.elapsed_time(b):.2f}" for a, b in marks))
