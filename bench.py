"""Benchmark of the Array-OL repetitive-task path on B200 (contract: one JSON line from rank 0).

Default workload (BASELINE.json configs[1]): the MatMul repetitive task
8192x8192x8192 fp32 (TF32 tensor cores) — repetition space [M, N] with the
canonical GEMM tilers, sharded over ranks by contiguous blocks of the
linearised repetition space (partition.py:105-121).  Weak scaling: every
rank owns 8192 rows of C (its shard of an [8192*N, 8192] repetition space),
its A row block and all of B — no data-path collective.

  value : TFLOP/s of the whole job with inputs resident in HBM (device-timed,
          CUDA events on the launching stream, max over ranks)
  e2e   : the same metric through the public API ``execute_schedule`` with
          pinned host bindings: H2D of A and B, the launch, D2H of C, every step
  roofline : the GEMM kernel's achieved TFLOP/s vs the measured TF32 peak
  cpu_baseline : the oracle's C restatement (oracle/aol_oracle.c) on the host
          cores, on a bounded sample of rows of the same workload

``--impl reference`` times the reference's CPU algorithm (the oracle port)
on the same workload and prints the reference arm's line.
``--workload stencil|downscaler|sweep`` runs the tiler-bound configs.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Repetitive-task GB/s & MatMul TFLOP/s at 1/2/4/8 B200, % roofline vs CPU ref"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- helpers --

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        deadline = time.time() + 8.0            # wait for the first sample before timing
        while time.time() < deadline and Path(self.path).stat().st_size == 0:
            time.sleep(0.05)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if r[3].replace(".", "").isdigit()), default=None)}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            pass
    return {}


def profile_traffic(key: str):
    """dram bytes per launch of the dominant kernel from the committed ncu summary, if any."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(key)
        except ValueError:
            return None
    return None


def tf32_peak(torch, device, sustain_s: float = 4.0):
    """cuBLAS TF32 8192^3 TFLOP/s: best of 10 (burst) and back to back for ``sustain_s`` seconds
    (sustained, under the power cap) — the recipe MEASURED_PEAKS.json uses for bf16."""
    try:
        torch.backends.cuda.matmul.allow_tf32 = True
        n = 8192
        a = torch.randn(n, n, device=device)
        b = torch.randn(n, n, device=device)
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch.matmul(a, b)
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        burst = 2 * n ** 3 / (best * 1e-3) / 1e12
        sustained = None
        if sustain_s > 0:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(1, int(sustain_s / (best * 1e-3)))
            s.record()
            for _ in range(reps):
                torch.matmul(a, b)
            e.record()
            e.synchronize()
            sustained = 2 * n ** 3 * reps / (s.elapsed_time(e) * 1e-3) / 1e12
        del a, b
        torch.cuda.empty_cache()
        return burst, sustained
    finally:
        torch.backends.cuda.matmul.allow_tf32 = False


# --------------------------------------------------------------- workloads --

class MatmulWorkload:
    name = "matmul"
    unit = "TFLOP/s"
    bound = "tensor"

    def __init__(self, torch, device, rank, world, M=8192, N=8192, K=8192):
        from oracle import aol_oracle as orc
        from paper_1105_4424_b200 import Tiler, builders
        from paper_1105_4424_b200.executor import Executor
        from paper_1105_4424_b200.partition import build_schedule, partition_equally
        self.torch, self.device = torch, device
        self.M, self.N, self.K = M, N, K
        # weak scaling: the job's repetition space is [M*world, N]; this rank's contiguous
        # shard is M whole rows, executed as a local task over its input hull.
        shard = partition_equally(M * world * N, world)[rank]
        assert shard.count == M * N and shard.offset == rank * M * N
        g = orc.gemm_tilers(M, N, K)
        self.tilers = {k: Tiler(v["origin"], v["paving"], v["fitting"], v["pattern"]) for k, v in g.items()}
        self.model = builders.tile_task_model(
            "matmul", {"a": f"in float32 [{M},{K}]", "b": f"in float32 [{K},{N}]", "c": f"out float32 [{M},{N}]"},
            self.tilers, (M, N))
        self.schedule = build_schedule(self.model, 1)
        gen = torch.Generator(device=device).manual_seed(2 + rank)
        a = torch.randn(M * K, device=device, generator=gen)
        b = torch.randn(K * N, device=device, generator=torch.Generator(device=device).manual_seed(3))
        self.ex = Executor(self.model, self.schedule, {"p_a": a, "p_b": b}, 1)
        del a, b
        self.units_per_step = 2.0 * M * N * K / 1e12          # TFLOP
        self.algorithmic = {"flop_per_launch": 2 * M * N * K, "per_unit": "2 FLOP per (m, n, k)"}
        self.workload = f"matmul {M}x{N}x{K} fp32 (TF32 tcgen05), rep space [{M}x{world},{N}] sharded by rows"

    def step(self):
        self.ex.run()

    # e2e through the public API with pinned host bindings
    def e2e_setup(self):
        torch = self.torch
        gen = torch.Generator().manual_seed(7)
        self.ha = torch.randn(self.M * self.K, generator=gen).pin_memory()
        self.hb = torch.randn(self.K * self.N, generator=gen).pin_memory()
        self.hc = torch.empty(self.M * self.N).pin_memory()
        self.e2e_bytes = (self.ha.numel() * 4 + self.hb.numel() * 4, self.M * self.N * 4)

    def e2e_step(self):
        from paper_1105_4424_b200.executor import execute_schedule
        res = execute_schedule(self.model, self.schedule, {"p_a": self.ha, "p_b": self.hb}, 1,
                               out={"p_c": self.hc})
        return res.outputs["p_c"]

    def e2e_free(self):
        del self.ha, self.hb, self.hc

    # CPU oracle on a bounded sample of rows
    def cpu_sample(self, seconds: float = 8.0):
        from oracle import c_oracle as co
        M, N, K = self.M, self.N, self.K
        rng = np.random.default_rng(0)
        A = rng.standard_normal(M * K, dtype=np.float32)
        B = rng.standard_normal(K * N, dtype=np.float32)
        Cm = np.zeros(M * N, np.float32)
        thr = co.threads()
        rows = max(1, thr)
        t0 = time.perf_counter()
        co.gemm_rows(A, B, Cm, N, K, 0, rows)
        dt = time.perf_counter() - t0
        target = int(rows * seconds / max(dt, 1e-3))
        rows2 = max(rows, min(M, (target // thr) * thr))
        t0 = time.perf_counter()
        co.gemm_rows(A, B, Cm, N, K, 0, rows2)
        dt = time.perf_counter() - t0
        flops = 2.0 * rows2 * N * K
        return {"value": flops / dt / 1e12, "unit": self.unit, "cores": thr, "kind": "port",
                "sample": f"{rows2} of {M} rows of C ({flops / 1e9:.1f} GFLOP), oracle/aol_oracle.c "
                          f"k-ascending fp32, OpenMP {thr} threads, {dt:.2f} s"}


WORKLOADS = {"matmul": MatmulWorkload}


# ---------------------------------------------------------------- the arms --

def time_steps(torch, fn, steps, warmup, stream, barrier):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for s, e in ev:
        s.record(stream)
        fn()
        e.record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    total_ms = t0.elapsed_time(t1)
    per = [s.elapsed_time(e) for s, e in ev]
    return total_ms, per


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_1105_4424_b200 import _capi

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    _capi.load()
    wl = WORKLOADS[args.workload](torch, device, rank, world)
    stream = torch.cuda.current_stream(device)

    clocks = Clocks(local)
    launches0 = _capi.launch_counter()
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    warm_launches = _capi.launch_counter() - launches0
    clocks.start()
    total_ms, per = time_steps(torch, wl.step, args.steps, 0, stream, barrier)
    clk = clocks.stop()
    launches = (_capi.launch_counter() - launches0 - warm_launches)
    total_ms = allmax(total_ms)
    ms_per_step = total_ms / args.steps
    value = wl.units_per_step * world * args.steps / (total_ms * 1e-3)
    kernel_ms = allmax(statistics.mean(per))

    # end to end through the public API (H2D + launch + D2H every step)
    e2e = None
    if not args.no_e2e:
        wl.e2e_setup()
        for _ in range(3):
            wl.e2e_step()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            wl.e2e_step()
        torch.cuda.synchronize()
        el = allmax(time.perf_counter() - t0)
        wl.e2e_free()
        e2e = {"value": wl.units_per_step * world * args.e2e_steps / el, "unit": wl.unit,
               "h2d_bytes_per_step": wl.e2e_bytes[0] * world, "d2h_bytes_per_step": wl.e2e_bytes[1] * world,
               "ms_per_step": el * 1e3 / args.e2e_steps, "steps": args.e2e_steps,
               "path": "paper_1105_4424_b200.executor.execute_schedule, pinned host bindings and pinned out= buffers"}

    peaks = measured_peaks()
    out = None
    if rank == 0:
        achieved = wl.units_per_step / (kernel_ms * 1e-3)
        if wl.bound == "tensor":
            burst, sustained = (None, None) if args.no_peak else tf32_peak(torch, device)
            long_region = total_ms > 250.0
            if sustained and long_region:
                peak, peak_src = sustained, ("cuBLAS TF32 8192^3 back to back for 4 s (sustained, power-capped), "
                                             "measured in this run; the timed region is a long step")
            elif burst:
                peak, peak_src = burst, "cuBLAS TF32 8192^3 best of 10 (burst), measured in this run"
            else:
                peak, peak_src = peaks.get("bf16_tflops", 1590.0) / 2, "half of MEASURED_PEAKS bf16_tflops"
            roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": profile_traffic(wl.name), "peak_source": peak_src,
                    "tf32_cublas_burst": burst, "tf32_cublas_sustained": sustained,
                    "frac_of_burst": achieved / burst if burst else None,
                    "bf16_peak_measured": peaks.get("bf16_tflops"),
                    "frac_of_bf16_peak": achieved / peaks["bf16_tflops"] if peaks.get("bf16_tflops") else None,
                    "kernel_ms": kernel_ms, "algorithmic": wl.algorithmic}
        else:
            peak = peaks.get("hbm_gbs", 6650.0)
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": profile_traffic(wl.name),
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650",
                    "kernel_ms": kernel_ms, "algorithmic": wl.algorithmic}
        cpu = None if args.no_cpu else wl.cpu_sample(args.cpu_seconds)
        out = {
            "metric": METRIC, "value": value, "unit": wl.unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if wl.bound == "hbm" else "tf32 (fp32 in/out)",
            "data": "synthetic (torch.randn, seeded)",
            "config": {"workload": wl.workload, "l2": "inputs (768 MiB/rank) exceed the 126 MB L2",
                       "parallelism": f"repetition space sharded by contiguous blocks over {world} rank(s)"},
            "e2e": e2e, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "clocks": clk,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_reference(args):
    """The reference arm: the reference's CPU algorithm (oracle port) on the host cores, rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT))
    from oracle import c_oracle as co
    M = N = K = 8192
    rng = np.random.default_rng(0)
    A = rng.standard_normal(M * K, dtype=np.float32)
    B = rng.standard_normal(K * N, dtype=np.float32)
    Cm = np.zeros(M * N, np.float32)
    thr = co.threads()
    rows = max(thr, 8)
    for _ in range(args.warmup):
        co.gemm_rows(A, B, Cm, N, K, 0, thr)
    t = []
    for i in range(args.steps):
        lo = (i * rows) % (M - rows)
        t0 = time.perf_counter()
        co.gemm_rows(A, B, Cm, N, K, lo, lo + rows)
        t.append(time.perf_counter() - t0)
    el = sum(t)
    flops = 2.0 * rows * N * K * args.steps
    value = flops / el / 1e12
    out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (numpy default_rng)",
           "impl": "reference",
           "config": {"workload": f"matmul {M}x{N}x{K} fp32, bounded sample of {rows} rows of C per step"},
           "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": thr, "kind": "port",
                            "sample": f"{rows} rows x {N} cols x {K} k per step (oracle/aol_oracle.c, "
                                      f"k-ascending fp32, OpenMP {thr} threads)"},
           "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="matmul", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-peak", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("note: warmup < 3 is below the timing rules; using 3")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
