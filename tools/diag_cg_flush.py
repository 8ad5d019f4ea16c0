import sys, time
from pathlib import Path
sys.path.insert(0, "/root/repo")
import torch, bench
from paper_1105_4424_b200.executor import Executor
w = bench.CGWorkload(torch, torch.device("cuda:0"), 0, 1)
scrub = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for flush in (False, True, False, True):
    ts = []
    for _ in range(6):
        if flush:
            scrub.fill_(1.0)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); s.record()
        ex = Executor(w.model, w.schedule, w.bind, 1, graphs=True)
        t1 = time.perf_counter()
        ex.run()
        e.record(); torch.cuda.synchronize(); t2 = time.perf_counter()
        ts.append((s.elapsed_time(e), 1e3 * (t1 - t0), 1e3 * (t2 - t1)))
    print("flush" if flush else "plain", " ".join(f"{a:.1f}({b:.1f}+{c:.1f})" for a, b, c in ts))
