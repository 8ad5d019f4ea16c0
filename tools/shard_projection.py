"""Per-rank shard times of the strong-scaling configs at N = 1, 2, 4, 8 (a PROJECTION).

gpurun has one GPU, so N > 1 over NVLink cannot be measured here.  This times, on one B200,
exactly the launch each rank would run (the schedule built with device_count = N; launch r =
partition_equally(T, N)[r], partition.py:105-121), one shard at a time, every shard of the
step, and reports the slowest shard per N as the concurrent per-rank phase,
and total work / that time as the projected whole-job throughput.  Not included: the gather
to the root (NVLink), inter-GPU clock/power differences.  Prints one JSON document."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1105_4424_b200 import _capi, builders  # noqa: E402
from paper_1105_4424_b200.executor import Executor  # noqa: E402
from paper_1105_4424_b200.partition import build_schedule  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


def shards(name, model, bind, units, unit, reps):
    """N = 1 is measured between every other N (1, 2, 1, 4, 1, 8, 1) and its median used, so
    the baseline sees the same thermal / power-cap state as the shards."""
    out = {"workload": name, "unit": unit, "per_n": {}}
    base_runs = []
    for n in (1, 2, 1, 4, 1, 8, 1):
        sched = build_schedule(model, n)
        ex = Executor(model, sched, bind, n)
        st = int(torch.cuda.current_stream().cuda_stream)
        steps = sched.device_steps()
        times = []
        if len(steps) == 2:                      # the fused H -> V pair, shards of V's range
            t1, t2 = ex.task(steps[0].task_path), ex.task(steps[1].task_path)
            a1 = [ex.storage.array(t1.nodes[p]).data_ptr() for p in t1.port_order]
            a2 = [ex.storage.array(t2.nodes[p]).data_ptr() for p in t2.port_order]
            for l in steps[1].launches:
                times.append(timed(lambda: _capi.launch_fused2(t1.ctask, t2.ctask, l.range.offset, l.range.count,
                                                               a1, a2, st), reps))
        else:
            t = ex.task(steps[0].task_path)
            ptrs = [ex.storage.array(t.nodes[p]).data_ptr() for p in t.port_order]
            for l in steps[0].launches:
                times.append(timed(lambda: _capi.launch(t.ctask, l.range.offset, l.range.count, ptrs, (), st), reps))
        slow = max(times)
        del ex
        torch.cuda.empty_cache()
        if n == 1:
            base_runs.append(slow)
            continue
        out["per_n"][n] = {"shard_ms": times, "slowest_ms": slow, "median_ms": statistics.median(times),
                           "projected_value": units / (slow * 1e-3)}
    b1 = statistics.median(base_runs)
    out["per_n"][1] = {"shard_ms": base_runs, "slowest_ms": b1, "median_ms": b1, "projected_value": units / (b1 * 1e-3),
                       "note": "the whole step on one GPU, measured 4 times between the shard runs (median)"}
    out["per_n"] = {k: out["per_n"][k] for k in (1, 2, 4, 8)}
    base = out["per_n"][1]["projected_value"]
    for n, d in out["per_n"].items():
        d["projected_speedup"] = d["projected_value"] / base
    return out


res = {"note": __doc__.split("\n\n")[1].replace("\n", " "), "configs": []}
M = N = K = 8192
a = torch.randn(M * K, device="cuda")
b = torch.randn(K * N, device="cuda")
res["configs"].append(shards("C2 matmul 8192^3 TF32", builders.matmul_model(M, N, K), {"p_a": a, "p_b": b},
                             2.0 * M * N * K / 1e12, "TFLOP/s", 20))
del a, b
n = 16384
x = torch.randn(n * n, device="cuda")
w = torch.from_numpy(builders.stencil_weights()).cuda()
res["configs"].append(shards("C4 stencil 16384^2", builders.stencil_model(n, n), {"p_x": x, "p_w": w},
                             2.0 * n * n * 4 / 1e9, "GB/s", 20))
del x
F, H, W = 256, 2160, 3840
x = torch.rand(F * H * W, device="cuda")
wh = torch.from_numpy(builders.downscaler_weights(13, 3)).cuda()
wv = torch.from_numpy(builders.downscaler_weights(14, 4)).cuda()
res["configs"].append(shards("C3 downscaler 256x2160x3840 (fused H->V)", builders.downscaler_model(F, H, W),
                             {"x": x, "wh": wh, "wv": wv}, (F * H * W + F * (H // 9 * 4) * (W // 8 * 3)) * 4 / 1e9,
                             "GB/s", 10))
print(json.dumps(res, indent=1))
