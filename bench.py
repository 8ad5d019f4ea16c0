"""Benchmark of the Array-OL repetitive-task path on B200 (contract: one JSON line from rank 0).

Default workload (BASELINE.json configs[1]): the MatMul repetitive task
8192x8192x8192 fp32 (TF32 tensor cores) — repetition space [M, N] with the
canonical GEMM tilers.  At N ranks the SAME repetition space is sharded by
contiguous blocks (partition.py:105-121): launch d of the schedule built with
device_count = N runs on rank d through the drop-in's distributed executor
(strong scaling; 1024 rows of C per rank at N = 8), with no data-path
collective; the output gather to rank 0 is timed separately.

  value : TFLOP/s of the whole job with inputs resident in HBM (device-timed,
          CUDA events on the launching stream, max over ranks)
  e2e   : the same metric through the public API ``execute_schedule`` with
          pinned host bindings: H2D of A and B, the launch, D2H of C, every step
          (plus ``e2e_numpy``: numpy in, numpy out, exactly the reference call)
  roofline : the GEMM kernel's achieved TFLOP/s vs the measured TF32 peak
  cpu_baseline : numpy.matmul fp32 (OpenBLAS sgemm, every host core) on the
          same A and B, with its accuracy next to ours

``--impl reference`` times the reference's CPU path for the workload on the host
cores and prints the reference arm's line.
``--workload stencil|downscaler|sweep|cg|cg27|c1`` runs the other configs.
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

def bind_host_to_gpu_numa(torch, device_index: int) -> dict:
    """Restrict this process to the CPUs of the GPU's NUMA node (sysfs local_cpulist), so the
    pinned host buffers of the e2e path are first-touched on the node whose PCIe root the
    GPU hangs off; a remote node adds a socket hop to every DMA.  Returns what was done."""
    try:
        pr = torch.cuda.get_device_properties(device_index)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        base = Path("/sys/bus/pci/devices") / bus
        cpus = (base / "local_cpulist").read_text().strip()
        node = (base / "numa_node").read_text().strip()
        sel = set()
        for part in cpus.split(","):
            lo, _, hi = part.partition("-")
            sel.update(range(int(lo), int(hi or lo) + 1))
        sel &= os.sched_getaffinity(0)
        if sel:
            os.sched_setaffinity(0, sel)
        return {"pci": bus, "numa_node": int(node), "cpus": len(sel)}
    except (OSError, ValueError, AttributeError) as e:
        return {"unavailable": str(e)[:80]}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """SM clock / throttle-reason sampler running during the timed region: an NVML thread at a
    2 ms period (so a 30 ms region still gets ~15 samples), nvidia-smi -lms 100 as a fallback."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits (nvml.h: nvmlClocksEventReason*)
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}
    PERIOD_S = 0.002

    def __init__(self, gpu_index: int, pci_bus_id: str | None = None):
        self.gpu = gpu_index
        self.pci = pci_bus_id
        self.proc = None
        self.path = None
        self.thread = None
        self.rows = []
        self.nvml = None
        self.handle = None

    def _nvml_handle(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            if self.pci:
                try:
                    h = pynvml.nvmlDeviceGetHandleByPciBusId(self.pci.encode() if isinstance(self.pci, str)
                                                             else self.pci)
                except Exception:
                    h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nvml = pynvml
            return h
        except Exception:
            return None

    def _sample_loop(self):
        nv, h = self.nvml, self.handle
        try:
            reasons_fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
        except AttributeError:
            reasons_fn = None
        k, pw = 0, None
        while not self.stop_flag.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = reasons_fn(h) if reasons_fn else 0
                if k % 16 == 0:                     # the power query is slow; the clock is the point
                    pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.rows.append((float(sm), pw, int(rs)))
            except Exception:
                pass
            k += 1
            self.stop_flag.wait(self.PERIOD_S)

    def start(self):
        import threading
        self.handle = self._nvml_handle()
        if self.handle is not None:
            self.rows = []
            self.stop_flag = threading.Event()
            self.thread = threading.Thread(target=self._sample_loop, daemon=True)
            self.thread.start()
            return
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
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join(timeout=2)
            rows, nv = self.rows, self.nvml
            try:
                mx = float(nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM))
            except Exception:
                mx = None
            if not rows:
                return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["no samples"], "source": "nvml"}
            sm = [r[0] for r in rows]
            reasons = sorted({n for r in rows for n, b in self.BITS.items() if r[2] & b})
            counts = {n: sum(1 for r in rows if r[2] & b) for n, b in self.BITS.items() if any(r[2] & b for r in rows)}
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "sm_mhz_min": min(sm),
                    "sm_mhz_max": max(sm), "reasons": reasons, "reason_samples": counts,
                    "samples": len(rows), "period_ms": self.PERIOD_S * 1e3, "source": "nvml",
                    "power_w_max": max((r[1] for r in rows if r[1] is not None), default=None),
                    "power_w_median": statistics.median([r[1] for r in rows if r[1] is not None] or [0.0])}
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
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi",
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

def _tiler(d):
    from paper_1105_4424_b200 import Tiler
    return Tiler(d["origin"], d["paving"], d["fitting"], d["pattern"])


def _spec(d, direction):
    return f"{direction} float32 [{','.join(str(x) for x in d['array'])}]"


def _x3_form() -> str:
    """The 3xTF32 kernel form the library picks (aol_gemm.cu gemm_core_3x)."""
    f = os.environ.get("AOL_3XTF32_FORM")
    if f in ("narrow", "wide", "regs"):
        return f
    return "narrow" if os.environ.get("AOL_3XTF32_WIDE") == "0" else "regs"


class Workload:
    """One repetitive-task schedule prepared in HBM; step() = one pass over one batch.

    ``scaling = "strong"``: the configured problem is the whole job at every N; at N > 1 the
    schedule is built with device_count = N and rank r runs launch r through the drop-in's
    distributed executor (make_distributed_executor).  ``"weak"``: every rank runs its own
    copy of the problem."""

    name = "?"
    unit = "GB/s"
    bound = "hbm"
    scaling = "strong"

    fuse = True

    def _prepare(self, torch, device, model, dev_bindings: dict, host_specs: dict, outputs: dict,
                 rank: int = 0, world: int = 1):
        from paper_1105_4424_b200.executor import Executor
        from paper_1105_4424_b200.partition import build_schedule
        self.torch, self.device = torch, device
        self.model, self.rank, self.world = model, rank, world
        if world > 1 and self.scaling == "strong":
            from paper_1105_4424_b200.distributed import make_distributed_executor
            self.schedule = build_schedule(model, world)
            # the timed phase keeps outputs sharded (scaling is measured on the
            # concurrent per-rank phase); the fused gather is timed separately (run_gpu)
            self.ex = make_distributed_executor(model, self.schedule, dev_bindings, fuse=Workload.fuse,
                                                fused_gather=False)
            self.dev_bindings = dev_bindings
            steps = self.schedule.device_steps()
            mine = sum(l.range.count for st in steps for l in st.launches if l.device_index == rank)
            self.rank_fraction = mine / max(1, sum(st.total_work for st in steps))
        else:
            self.schedule = build_schedule(model, 1)
            self.ex = Executor(model, self.schedule, dev_bindings, 1, fuse=Workload.fuse)
            self.rank_fraction = 1.0
        self.host_specs, self.out_sizes = host_specs, outputs

    def step(self):
        self.ex.run()

    def fused_step(self, time_steps, stream, barrier, steps: int):
        """N > 1, strong scaling: time ``steps`` steps of an executor whose root outputs are
        stored into rank 0's array by the producing kernels (fused gather), each step closed by
        gather_to_root's wait; returns (bytes this rank stores into the root per step, ms)."""
        if self.world < 2 or self.scaling != "strong" or not hasattr(self, "dev_bindings"):
            return None
        from paper_1105_4424_b200.distributed import make_distributed_executor
        ex = make_distributed_executor(self.model, self.schedule, self.dev_bindings, fuse=Workload.fuse,
                                       fused_gather=True)

        def step():
            ex.run()
            ex.gather_to_root()
        total_ms, _ = time_steps(self.torch, step, steps, 3, stream, barrier)
        fb = ex.fused_bytes
        ex.close()
        del ex
        return fb, total_ms / steps

    def gather(self):
        """N > 1: move every output range the root does not hold to rank 0 (the distributed
        executor's gather, NCCL send/recv of exact ranges); returns bytes moved to the root."""
        gt = getattr(self.ex, "gather_to_root", None)
        return gt() if gt is not None else None

    def e2e_setup(self):
        torch = self.torch
        gen = torch.Generator().manual_seed(7)
        self.hin = {k: (torch.rand(n, generator=gen) if isinstance(kind, str) else torch.from_numpy(kind)).pin_memory()
                    for k, (n, kind) in self.host_specs.items()}
        self.hout = {k: torch.empty(n).pin_memory() for k, n in self.out_sizes.items()}
        self.e2e_bytes = (sum(t.numel() * 4 for t in self.hin.values()),
                          sum(t.numel() * 4 for t in self.hout.values()))

    pipeline = int(os.environ.get("AOL_E2E_PIPELINE", "8"))

    def e2e_step(self):
        from paper_1105_4424_b200.executor import execute_schedule
        if self.world > 1 and self.scaling == "strong":
            # every rank uploads its input hull from the pinned host arrays, runs its launch,
            # the output ranges gather to rank 0, rank 0 copies the whole result down
            from paper_1105_4424_b200.distributed import make_distributed_executor
            ex = make_distributed_executor(self.model, self.schedule, self.hin, fuse=Workload.fuse)
            ex.run()
            self.e2e_h2d = ex.h2d_bytes
            return ex.outputs(out=self.hout if self.rank == 0 else None)
        return execute_schedule(self.model, build_schedule_1(self.model), self.hin, 1, out=self.hout,
                                pipeline=self.pipeline).outputs

    def e2e_numpy_setup(self):
        """The reference-call form: pageable numpy arrays in, fresh numpy arrays out."""
        self.nin = {k: t.numpy().copy() for k, t in self.hin.items()}

    def e2e_numpy_step(self):
        from paper_1105_4424_b200.executor import execute_schedule
        return execute_schedule(self.model, build_schedule_1(self.model), self.nin, 1,
                                pipeline=self.pipeline).outputs

    def e2e_free(self):
        del self.hin, self.hout
        self.__dict__.pop("nin", None)


_SCHED_CACHE: dict = {}


def build_schedule_1(model):
    from paper_1105_4424_b200.partition import build_schedule
    s = _SCHED_CACHE.get(id(model))
    if s is None:
        s = _SCHED_CACHE[id(model)] = build_schedule(model, 1)
    return s


def openblas_info() -> dict:
    """numpy / BLAS threading facts for the CPU baseline line."""
    info = {"cpu_count": os.cpu_count(), "numpy": np.__version__}
    try:
        from threadpoolctl import threadpool_info
        blas = [d for d in threadpool_info() if d.get("user_api") == "blas"]
        if blas:
            info.update(blas=blas[0].get("internal_api"), blas_version=blas[0].get("version"),
                        blas_threads=blas[0].get("num_threads"))
    except Exception as e:  # noqa: BLE001 - informational only
        info["blas"] = f"unknown ({type(e).__name__})"
    return info


def normwise(c, ref) -> float:
    """||C - C_ref||_F / ||C_ref||_F over the sampled rows."""
    c, ref = np.asarray(c, np.float64), np.asarray(ref, np.float64)
    return float(np.linalg.norm(c - ref) / np.linalg.norm(ref))


class MatmulWorkload(Workload):
    name = "matmul"
    unit = "TFLOP/s"
    bound = "tensor"

    def __init__(self, torch, device, rank, world, M=8192, N=8192, K=8192):
        from paper_1105_4424_b200 import builders
        self.M, self.N, self.K = M, N, K
        model = builders.matmul_model(M, N, K)
        # every rank holds the same A and B (seeded); at N > 1 rank r runs launch r of the
        # schedule built with device_count = N: rows [r*M/N, (r+1)*M/N) of C
        a = torch.randn(M * K, device=device, generator=torch.Generator(device=device).manual_seed(2))
        b = torch.randn(K * N, device=device, generator=torch.Generator(device=device).manual_seed(3))
        self._prepare(torch, device, model, {"p_a": a, "p_b": b}, {}, {"p_c": M * N}, rank, world)
        del a, b
        self.units_per_step = 2.0 * M * N * K / 1e12          # TFLOP of the whole job
        self.algorithmic = {"flop_per_launch": int(2 * M * N * K * self.rank_fraction),
                            "per_unit": "2 FLOP per (m, n, k)"}
        self.workload = (f"matmul {M}x{N}x{K} fp32 (TF32 tcgen05), rep space [{M},{N}] sharded by contiguous "
                         f"row blocks over {world} rank(s)")
        self.l2 = "inputs (768 MiB) exceed the 126 MB L2"

    def e2e_setup(self):
        torch = self.torch
        gen = torch.Generator().manual_seed(7)
        self.hin = {"p_a": torch.randn(self.M * self.K, generator=gen).pin_memory(),
                    "p_b": torch.randn(self.K * self.N, generator=gen).pin_memory()}
        self.hout = {"p_c": torch.empty(self.M * self.N).pin_memory()}
        self.e2e_bytes = ((self.M * self.K + self.K * self.N) * 4, self.M * self.N * 4)

    def fp32_faithful(self, reps: int = 10) -> dict:
        """Secondary line: the same task in precision='3xtf32' (the fused tcgen05 hi/lo kernel
        with K-chunked accumulation), device-timed like `value`, and its normwise error on 64
        sampled rows against an fp64 product, next to the TF32 default and cuBLAS SIMT fp32
        (torch.matmul, allow_tf32=False) on the same A and B."""
        from paper_1105_4424_b200.executor import Executor
        torch, M, N, K = self.torch, self.M, self.N, self.K
        st = self.ex.storage
        a, b = st.array("p_a"), st.array("p_b")
        rows = torch.randperm(M, generator=torch.Generator().manual_seed(1))[:64].to(self.device)
        A, B = a.view(M, K), b.view(K, N)
        ref = A[rows].double() @ B.double()

        def err(c):
            return float(torch.linalg.norm(c.view(M, N)[rows].double() - ref) / torch.linalg.norm(ref))

        def timed(fn):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            e1.synchronize()
            return e0.elapsed_time(e1) / reps
        ex3 = Executor(self.model, self.schedule, {"p_a": a, "p_b": b}, 1, precision="3xtf32")
        ms3 = timed(ex3.run)
        err3 = err(ex3.outputs(on_device=True)["p_c"])
        # the same kernel with 32-deep K chunks (a fold every k-block: tighter error, slower)
        os.environ["AOL_3XTF32_CHUNK"] = "32"
        try:
            ms3_32 = timed(ex3.run)
            err3_32 = err(ex3.outputs(on_device=True)["p_c"])
        finally:
            os.environ.pop("AOL_3XTF32_CHUNK", None)
        del ex3
        err_tf32 = err(self.ex.outputs(on_device=True)["p_c"])
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            ms_simt = timed(lambda: A @ B)
            err_simt = err(A @ B)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        torch.cuda.empty_cache()
        flop = 2.0 * M * N * K
        return {"precision": "3xtf32", "value": flop / (ms3 * 1e-3) / 1e12, "unit": "TFLOP/s", "ms": ms3,
                "normwise_vs_fp64": err3, "normwise_tf32_default": err_tf32,
                "kernel": {"narrow": "k_gemm_3xtf32_pair (256x128 pair tiles, running sum in TMEM",
                           "wide": "k_gemm_3xtf32_wide (256x256 pair tiles, one accumulator, running sum in TMEM",
                           "regs": "k_gemm_3xtf32_regs (256x256 pair tiles, two TMEM accumulators, running sum in "
                                   "registers"}[_x3_form()] +
                          "; hi/lo split in shared memory, 3 tcgen05 products per k-slice, 64-deep K chunks "
                          "summed with round-to-nearest adds)",
                "chunk32": {"value": flop / (ms3_32 * 1e-3) / 1e12, "ms": ms3_32, "normwise_vs_fp64": err3_32,
                            "switch": "AOL_3XTF32_CHUNK=32"},
                "cublas_fp32_simt": {"value": flop / (ms_simt * 1e-3) / 1e12, "ms": ms_simt,
                                     "normwise_vs_fp64": err_simt}}

    def cpu_sample(self, seconds: float = 8.0):
        """SURVEY.md §8(d) C2 baseline: numpy.matmul fp32 (OpenBLAS sgemm on every host core) on
        the same A and B the GPU multiplied, the whole 8192^3 product, best of 2; plus the
        normwise error of both results against an fp64 product on 64 sampled rows, and the
        oracle's k-ascending C port (the reference's order) on a few rows as a secondary."""
        from oracle import c_oracle as co
        M, N, K = self.M, self.N, self.K
        st = self.ex.storage
        A = st.array("p_a").cpu().numpy().reshape(M, K)
        B = st.array("p_b").cpu().numpy().reshape(K, N)
        ours = self.ex.outputs(on_device=True)["p_c"].view(M, N)
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            C = np.matmul(A, B)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
            if best * 2 > seconds * 2:
                break
        rows = np.random.default_rng(1).choice(M, 64, replace=False)
        ref64 = A[rows].astype(np.float64) @ B.astype(np.float64)
        err_blas = normwise(C[rows], ref64)
        err_ours = normwise(ours[rows].cpu().numpy(), ref64)
        del C
        # secondary: the oracle's order-pinned C port on a bounded block of rows
        thr = co.threads()
        Cm = np.zeros(M * N, np.float32)
        r2 = max(thr, 8)
        t0 = time.perf_counter()
        co.gemm_rows(A.ravel(), B.ravel(), Cm, N, K, 0, r2)
        dt2 = time.perf_counter() - t0
        flops = 2.0 * M * N * K
        return {"value": flops / best / 1e12, "unit": self.unit, "cores": os.cpu_count(), "kind": "port",
                "impl": "numpy.matmul fp32 (OpenBLAS sgemm)",
                "sample": f"the whole {M}x{N}x{K} product on the GPU's A and B, best of 2: {best:.2f} s",
                "blas": openblas_info(),
                "accuracy": {"normwise_vs_fp64_64_rows": {"openblas_fp32": err_blas, "ours": err_ours}},
                "secondary": {"value": 2.0 * r2 * N * K / dt2 / 1e12, "unit": self.unit, "cores": thr,
                              "kind": "port", "sample": f"{r2} rows of C with oracle/aol_oracle.c "
                                                        f"(k-ascending fp32, the reference's order), {dt2:.2f} s"}}


class StencilWorkload(Workload):
    """Config C4: 3x3 toroidal stencil on a 16384^2 fp32 torus (at N ranks: 16384/N rows each)."""

    name = "stencil"

    def __init__(self, torch, device, rank, world, n=16384):
        from paper_1105_4424_b200 import builders
        self.n = n
        w = builders.stencil_weights()
        x = torch.randn(n * n, device=device, generator=torch.Generator(device=device).manual_seed(5))
        self._prepare(torch, device, builders.stencil_model(n, n), {"p_x": x, "p_w": torch.from_numpy(w).to(device)},
                      {"p_x": (n * n, "rand"), "p_w": (9, w)}, {"p_y": n * n}, rank, world)
        del x
        self.units_per_step = 2.0 * n * n * 4 / 1e9            # GB (read x once, write y once)
        self.algorithmic = {"bytes_per_launch": int(2 * n * n * 4 * self.rank_fraction),
                            "per_unit": "4 B read + 4 B written per element"}
        self.workload = (f"toroidal 3x3 stencil {n}x{n} fp32, origin (-1,-1), weights [1,2,1]^T[1,2,1]/16, "
                         f"rows sharded over {world} rank(s)")
        self.l2 = "inputs (1 GiB) exceed the 126 MB L2"

    def cpu_sample(self, seconds: float = 8.0):
        from oracle import c_oracle as co
        n = self.n
        x = np.random.default_rng(5).standard_normal(n * n, dtype=np.float32)
        y = np.zeros_like(x)
        w = __import__("oracle.aol_oracle", fromlist=["x"]).stencil_weights()
        t0 = time.perf_counter()
        co.stencil_rows(x, w, y, n, n, 0, 256)
        dt = time.perf_counter() - t0
        rows = int(min(n, max(256, 256 * seconds / max(dt, 1e-3))))
        t0 = time.perf_counter()
        co.stencil_rows(x, w, y, n, n, 0, rows)
        dt = time.perf_counter() - t0
        return {"value": 2.0 * rows * n * 4 / dt / 1e9, "unit": "GB/s", "cores": co.threads(), "kind": "port",
                "sample": f"{rows} of {n} rows, oracle/aol_oracle.c stencil, {dt:.2f} s"}


class DownscalerWorkload(Workload):
    """Config C3: H filter (13 taps, paving 8 -> 3 outputs) then V filter (14 taps, paving 9 -> 4 outputs)."""

    name = "downscaler"

    def __init__(self, torch, device, rank, world, frames=256, H=2160, W=3840):
        from paper_1105_4424_b200 import builders
        model = builders.downscaler_model(frames, H, W)
        Wo = W // 8 * 3
        Ho = H // 9 * 4
        wh, wv = builders.downscaler_weights(13, 3), builders.downscaler_weights(14, 4)
        nx = frames * H * W
        x = torch.rand(nx, device=device, generator=torch.Generator(device=device).manual_seed(4))
        self._prepare(torch, device, model,
                      {"x": x, "wh": torch.from_numpy(wh).to(device), "wv": torch.from_numpy(wv).to(device)},
                      {"x": (nx, "rand"), "wh": (wh.size, wh), "wv": (wv.size, wv)}, {"y": frames * Ho * Wo},
                      rank, world)
        del x
        hbytes = (nx + frames * H * Wo) * 4
        vbytes = (frames * H * Wo + frames * Ho * Wo) * 4
        # probe whether the executor fuses the chain (H output kept on chip): the algorithmic
        # bytes are then x read once + y written once
        self.ex.run()
        torch.cuda.synchronize()
        fused = self.ex.fused_launches > 0
        step_bytes = (nx + frames * Ho * Wo) * 4 if fused else hbytes + vbytes
        self.units_per_step = step_bytes / 1e9
        self.algorithmic = {"bytes_per_step": int(step_bytes * self.rank_fraction), "fused": fused,
                            "unfused_h_bytes": hbytes, "unfused_v_bytes": vbytes,
                            "per_unit": "each array element read once / written once "
                                        + ("(fused: x and y only)" if fused else "per filter")}
        self.workload = (f"downscaler {frames}x{H}x{W} fp32: hfilter 13->3 paving 8 -> vfilter 14->4 paving 9, "
                         + ("fused into one streaming kernel (intermediate never leaves registers)" if fused
                            else "two tasks") + f", frames sharded over {world} rank(s)")
        self.l2 = "inputs (8.5 GB) exceed the 126 MB L2"
        self.dims = (frames, H, W, Wo, Ho)

    def cpu_sample(self, seconds: float = 8.0):
        from oracle import aol_oracle as orc
        from oracle import c_oracle as co
        _, H, W, Wo, Ho = self.dims
        f = 2
        th, tv = orc.hfilter_tilers(f, H, W), orc.vfilter_tilers(f, H, Wo)
        x = np.random.default_rng(4).random(f * H * W, dtype=np.float32)
        mid = np.zeros(f * H * Wo, np.float32)
        y = np.zeros(f * Ho * Wo, np.float32)
        t0 = time.perf_counter()
        co.tile_filter(x, orc.hfilter_weights(), mid, th["x"], th["y"], 0, int(np.prod(th["x"]["rep"])))
        co.tile_filter(mid, orc.vfilter_weights(), y, tv["x"], tv["y"], 0, int(np.prod(tv["x"]["rep"])))
        dt = time.perf_counter() - t0
        b = ((f * H * W + f * H * Wo) + (f * H * Wo + f * Ho * Wo)) * 4
        return {"value": b / dt / 1e9, "unit": "GB/s", "cores": co.threads(), "kind": "port",
                "sample": f"{f} frames through both filters, oracle/aol_oracle.c, {dt:.2f} s"}


class SweepWorkload(Workload):
    """Config C5: tile_copy sweep over pattern m, paving (dense / overlap / gaps), fitting and T.

    step() runs the largest point; the per-point table is measured separately (measure_points)."""

    name = "sweep"
    scaling = "weak"

    POINTS_M = (1, 2, 4, 8, 16, 32, 64)

    # per-point HBM footprint cap (input span + output): <= ~150 GB of the 180 GB
    MAX_FOOTPRINT = 120e9
    # the step()/e2e point stays resident while the table is measured
    MAIN_MAX_OUT = 8 << 30

    @staticmethod
    def _geometry(m, kind, T):
        """(input span, distinct input elements) of one sweep point."""
        if kind == "rowstride":
            return m * T, m * T
        p = {"dense": m, "overlap": max(1, m // 2), "gaps": 2 * m, "strided": m * 2}[kind]
        f = 2 if kind == "strided" else 1
        span = (T - 1) * p + (m - 1) * f + 1
        return span, (span if kind == "overlap" else T * m)

    def __init__(self, torch, device, rank, world):
        self.torch, self.device = torch, device
        self.rank, self.world, self.rank_fraction = rank, world, 1.0
        self.points = []
        for m in self.POINTS_M:
            for kind in ("dense", "overlap", "gaps", "strided", "rowstride"):
                if kind in ("overlap", "strided", "rowstride") and m == 1:
                    continue
                for T in (10 ** 3, 10 ** 5, 10 ** 7, 10 ** 8, 10 ** 9):
                    if (self._geometry(m, kind, T)[0] + T * m) * 4 > self.MAX_FOOTPRINT:
                        continue
                    self.points.append((m, kind, T))
        big = [p for p in self.points if p[2] >= 10 ** 7 and p[2] * p[0] * 4 <= self.MAIN_MAX_OUT]
        self.main = max(big, key=lambda p: p[2] * p[0])
        self.task = self._make(*self.main)
        self.units_per_step = self.task["bytes"] / 1e9
        self.algorithmic = {"bytes_per_launch": self.task["bytes"],
                            "per_unit": "distinct input elements read + output elements written, x 4 B"}
        self.workload = f"tile_copy sweep; step = pattern {self.main[0]} {self.main[1]} T={self.main[2]:.0e}"
        self.l2 = ("step point exceeds the L2; table points below 3x the L2 are timed with a 256 MiB "
                   "L2 flush before each launch (l2_flushed)")

    def _make(self, m, kind, T):
        from paper_1105_4424_b200 import Tiler, _capi
        torch = self.torch
        span, distinct = self._geometry(m, kind, T)
        if kind == "rowstride":
            # array [m, T] row-major: repetition r walks a row, pattern i walks down a column
            src = Tiler((0, 0), ((0,), (1,)), ((1,), (0,)), (m,)).bind((m, T), (T,))
        else:
            p = {"dense": m, "overlap": max(1, m // 2), "gaps": 2 * m, "strided": m * 2}[kind]
            f = 2 if kind == "strided" else 1
            src = Tiler((0,), ((p,),), ((f,),), (m,)).bind((span,), (T,))
        dst = Tiler((0,), ((m,),), ((1,),), (m,)).bind((T * m,), (T,))
        x = torch.empty(span, device=self.device).uniform_()
        y = torch.empty(T * m, device=self.device)
        task = _capi.make_task("tile_copy", "float32", [src, dst])
        ptrs = [x.data_ptr(), y.data_ptr()]
        return {"x": x, "y": y, "task": task, "ptrs": ptrs, "T": T, "bytes": (distinct + T * m) * 4,
                "plan": _capi.plan_name(task, 0, T, ptrs)}

    def step(self):
        from paper_1105_4424_b200 import _capi
        t = self.task
        _capi.launch(t["task"], 0, t["T"], t["ptrs"], (), int(self.torch.cuda.current_stream().cuda_stream))

    L2_BYTES = 126 << 20

    LINE = 128          # HBM fetch unit measured for these streams (profiles/r2_sweep_dram.json)

    def line_floor_bytes(self, m, kind, T):
        """DRAM-level floor of one point: distinct 128 B lines of the source touched + the output.

        ncu shows whole 128 B lines fetched for 32/64 B runs (m = 8/16 gaps read the full span,
        cudaLimitMaxL2FetchGranularity 32/64 changes nothing: profiles/r2_sweep_dram.json), so
        this -- not the 32 B sector count -- is what the kernel must move."""
        if kind == "rowstride":
            return 2 * m * T * 4
        p = {"dense": m, "overlap": max(1, m // 2), "gaps": 2 * m, "strided": m * 2}[kind]
        f = 2 if kind == "strided" else 1
        Ts = int(min(T, 1 << 15))
        Ts -= Ts % max(1, self.LINE // 4)
        Ts = max(Ts, min(T, 1))
        offs = (np.arange(Ts, dtype=np.int64)[:, None] * p + np.arange(m, dtype=np.int64)[None, :] * f) * 4
        lines = np.unique(offs // self.LINE).size * (T / Ts)
        span_lines = -(-(self._geometry(m, kind, T)[0] * 4) // self.LINE)
        return int(min(lines, span_lines) * self.LINE) + T * m * 4

    def _flush(self, i):
        # write a buffer larger than L2, then READ another one: the L2 is left holding clean
        # lines, so the timed launch pays neither for its inputs being cached nor for the
        # flush's own dirty write-backs (tools/sweep_probe.py: the write-only flush added
        # 4-8 us of write-back to 15-30 us launches)
        self.scrub.fill_(float(i))
        self.acc.copy_(self.rd.sum())

    def _time(self, fn, flush, steps, warmup):
        torch = self.torch
        for _ in range(warmup):
            fn()
        if flush:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for i, (a, b) in enumerate(ev):
                self._flush(i)
                a.record()
                fn()
                b.record()
            torch.cuda.synchronize()
            return statistics.median(a.elapsed_time(b) for a, b in ev)
        # back to back, one event pair per launch (>= 0.1 ms launches: the pairs cost nothing),
        # median -- a transient power-cap dip in one launch does not move the row
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ev[0].record()
        for i in range(steps):
            fn()
            ev[i + 1].record()
        ev[-1].synchronize()
        return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(steps))

    def measure_points(self, steps=10, warmup=3):
        """Per-point table.  Points whose footprint is below 3x the L2 are timed launch by
        launch with an L2 flush before each launch (outside its event pair, median of the
        launches); larger points are timed back to back (median of per-launch event pairs).  Each row carries its DRAM line floor
        (floor_frac = floor bytes / time / peak), a device-to-device copy of the same floor
        bytes timed the same way (the achievable rate at that size: frac_of_copy), and the ncu
        DRAM bytes of the same point from profiles/r2_sweep_dram.json when it was captured."""
        torch = self.torch
        from paper_1105_4424_b200 import _capi
        self.scrub = torch.empty(64 << 20, dtype=torch.float32, device=self.device)
        self.rd = torch.ones(64 << 20, dtype=torch.float32, device=self.device)
        self.acc = torch.zeros(1, device=self.device)
        peak = measured_peaks().get("hbm_gbs", 6650.0)
        ncu = {}
        pf = ROOT / "profiles" / "r2_sweep_dram.json"
        if pf.exists():
            try:
                ncu = {(r["m"], r["paving"], r["T"]): r for r in json.loads(pf.read_text())["points"]}
            except (ValueError, KeyError):
                ncu = {}
        # smallest footprint first: points measured after the 10-120 GB ones sometimes ran slow
        # in a full table (rows of a fresh allocation placed badly after the big frees; the same
        # point re-measured in a fresh process is at its floor, tools/probe_rowstride.py)
        order = sorted(self.points, key=lambda q: self._geometry(*q)[0] + q[2] * q[0])
        by_key = {}
        for m, kind, T in order:
            t = self._make(m, kind, T)
            st = int(torch.cuda.current_stream().cuda_stream)
            flush = (t["x"].numel() + t["y"].numel()) * 4 < 3 * self.L2_BYTES
            ms = self._time(lambda: _capi.launch(t["task"], 0, T, t["ptrs"], (), st), flush, steps, warmup)
            floor = self.line_floor_bytes(m, kind, T)
            row = {"m": m, "paving": kind, "T": T, "plan": t["plan"], "ms": ms,
                   "GBps": t["bytes"] / (ms * 1e-3) / 1e9, "frac": t["bytes"] / (ms * 1e-3) / 1e9 / peak,
                   "floor_bytes": floor, "floor_frac": floor / (ms * 1e-3) / 1e9 / peak, "l2_flushed": flush}
            if T <= 10 ** 8 and floor // 8 >= 1:
                n = floor // 8                                   # copy_ of n floats moves 8n bytes
                ca = torch.empty(n, device=self.device)
                cb = torch.empty_like(ca)
                cms = self._time(lambda: cb.copy_(ca), flush, steps, warmup)
                row["copy_ms"] = cms
                row["frac_of_copy"] = cms / ms
                del ca, cb
            k = ncu.get((m, kind, T))
            if k:
                row["ncu_dram_bytes"] = k["dram_bytes"]
                row["ncu_dram_over_floor"] = k["dram_bytes"] / floor
            by_key[(m, kind, T)] = row
            del t
            torch.cuda.empty_cache()
        del self.scrub, self.rd
        return [by_key[p] for p in self.points]

    def e2e_setup(self):
        # the main point as a one-task model through the public API: execute_schedule streams it
        # in `pipeline` chunks (H2D of each chunk's source range, launch, D2H of its output range
        # on three streams), so uploads and downloads overlap on PCIe
        from paper_1105_4424_b200 import Tiler, builders
        from paper_1105_4424_b200.partition import build_schedule
        torch = self.torch
        m, kind, T = self.main
        t = self.task
        span, _ = self._geometry(m, kind, T)
        if kind == "rowstride":
            src_t, src_arr = Tiler((0, 0), ((0,), (1,)), ((1,), (0,)), (m,)), (m, T)
        else:
            p = {"dense": m, "overlap": max(1, m // 2), "gaps": 2 * m, "strided": m * 2}[kind]
            src_t, src_arr = Tiler((0,), ((p,),), ((2 if kind == "strided" else 1,),), (m,)), (span,)
        dst_t = Tiler((0,), ((m,),), ((1,),), (m,))
        self.e2e_model = builders.tile_task_model(
            "tile_copy", {"src": f"in float32 [{','.join(map(str, src_arr))}]", "dst": f"out float32 [{T * m}]"},
            {"src": src_t, "dst": dst_t}, (T,))
        self.e2e_schedule = build_schedule(self.e2e_model, 1)
        self.hx = torch.empty(t["x"].numel()).uniform_().pin_memory()
        self.hy = torch.empty(t["y"].numel()).pin_memory()
        del self.task, t
        torch.cuda.empty_cache()
        self.e2e_bytes = (self.hx.numel() * 4, self.hy.numel() * 4)

    def e2e_step(self):
        from paper_1105_4424_b200.executor import execute_schedule
        return execute_schedule(self.e2e_model, self.e2e_schedule, {"p_src": self.hx}, 1, out={"p_dst": self.hy},
                                pipeline=self.pipeline).outputs

    def e2e_free(self):
        del self.hx, self.hy

    def cpu_sample(self, seconds: float = 8.0):
        from oracle import c_oracle as co
        m, kind, T = self.main
        p = {"dense": m, "overlap": max(1, m // 2), "gaps": 2 * m, "strided": m * 2}[kind]
        f = 2 if kind == "strided" else 1
        Ts = min(T, 2_000_000)
        span = (Ts - 1) * p + (m - 1) * f + 1
        ts = dict(array=(span,), rep=(Ts,), pattern=(m,), origin=(0,), paving=((p,),), fitting=((f,),))
        td = dict(array=(Ts * m,), rep=(Ts,), pattern=(m,), origin=(0,), paving=((m,),), fitting=((1,),))
        x = np.random.default_rng(0).random(span, dtype=np.float32)
        y = np.zeros(Ts * m, np.float32)
        t0 = time.perf_counter()
        co.tile_copy(x, y, ts, td, 0, Ts)
        dt = time.perf_counter() - t0
        distinct = span if kind == "overlap" else Ts * m
        return {"value": (distinct + Ts * m) * 4 / dt / 1e9, "unit": "GB/s", "cores": co.threads(), "kind": "port",
                "sample": f"T={Ts} repetitions of the main point, oracle/aol_oracle.c tile_copy, {dt:.2f} s"}


def _poisson_2d(k: int):
    """Five-point Poisson CSR (rows sorted), the reference's generator restated (refexec.py:330-347)."""
    n = k * k
    idx = np.arange(n, dtype=np.int64)
    gi, gj = idx // k, idx % k
    rows, cols, vals = [idx], [idx], [np.full(n, 4.0)]
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ok = (gi + di >= 0) & (gi + di < k) & (gj + dj >= 0) & (gj + dj < k)
        rows.append(idx[ok])
        cols.append((gi[ok] + di) * k + gj[ok] + dj)
        vals.append(np.full(int(ok.sum()), -1.0))
    r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rowptr = np.zeros(n + 1, np.int32)
    np.cumsum(np.bincount(r, minlength=n), out=rowptr[1:])
    return n, rowptr, c.astype(np.int32), v


def _poisson_3d27(k: int = 51, diag: float = 26.0):
    """27-point 3-D operator on a k^3 grid (diag 26, off-diagonals -1), CSR with sorted rows.
    k = 51 gives exactly the paper's matrix shape: N = 132,651, NNZ = (3k-2)^3 = 3,442,951
    (PAPER.md:289).  The paper does not give its values; this one is the standard SPD
    27-point operator (85 CG iterations to 1e-10 from b = 1, the paper reports 116)."""
    n = k ** 3
    idx = np.arange(n, dtype=np.int64).reshape(k, k, k)
    rows, cols = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                z0, z1 = max(0, -dz), k - max(0, dz)
                y0, y1 = max(0, -dy), k - max(0, dy)
                x0, x1 = max(0, -dx), k - max(0, dx)
                rows.append(idx[z0:z1, y0:y1, x0:x1].ravel())
                cols.append(idx[z0 + dz:z1 + dz, y0 + dy:y1 + dy, x0 + dx:x1 + dx].ravel())
    r, c = np.concatenate(rows), np.concatenate(cols)
    order = np.lexsort((c, r))
    r, c = r[order], c[order]
    v = np.where(r == c, diag, -1.0)
    rowptr = np.zeros(n + 1, np.int32)
    np.cumsum(np.bincount(r, minlength=n), out=rowptr[1:])
    return n, rowptr, c.astype(np.int32), v


def _resize_model_dict(d: dict, n_old: int, nnz_old: int, n: int, nnz: int) -> dict:
    """instantiate_for_matrix (refexec.py:552-596) restated on the plain-data model."""
    import copy
    d = copy.deepcopy(d)

    def m(x):
        return nnz if x == nnz_old else n if x == n_old else n + 1 if x == n_old + 1 else x
    for c in d["application_components"]:
        for p in c["ports"]:
            if p[2] is not None:
                p[2] = [m(v) for v in p[2]]
        if c["repetition_space"] is not None:
            c["repetition_space"] = [m(v) for v in c["repetition_space"]]
    return d


class CGWorkload(Workload):
    """Row f1 / the paper's case study: CG (cg.gmodel, resized) on a 2-D Poisson matrix, n ~ 132k.

    One step = one full solve to relres <= 1e-10 through execute_schedule's interpreter
    (LoopStep, host scalar ops, dot partials combined in device order).  Reported like
    the paper's Table 1: GFLOP/s over the solve."""

    name = "cg"
    unit = "GFLOP/s"
    dtype = "f64"

    matrix = "poisson_2d(364)"

    def _matrix(self):
        return _poisson_2d(364)

    def __init__(self, torch, device, rank, world):
        from paper_1105_4424_b200.executor import Executor
        from paper_1105_4424_b200.model import model_from_dict
        from paper_1105_4424_b200.partition import build_schedule
        meta = json.loads((ROOT / "tests" / "golden" / "reference_golden.json").read_text())
        base = meta["cg_k20"]["model"]
        n, rowptr, colidx, vals = self._matrix()
        self.n, self.nnz = n, int(rowptr[-1])
        self.model = model_from_dict(_resize_model_dict(base, 400, 1920, n, self.nnz))
        self.rank, self.world = rank, world
        # at N ranks: D = N launches per step, launch r on rank r (the distributed executor:
        # p all-gathered after each update, dot partials reduced on the device)
        self.schedule = build_schedule(self.model, world)
        self.rank_fraction = 1.0 / world
        self.bind = {"rowptr": rowptr, "colidx": colidx, "values": vals, "b": np.ones(n)}
        # `value` is measured with the inputs already resident in HBM (the executor's storage is
        # filled by device-to-device copies); e2e_step binds the host arrays instead
        self.dbind = {k: torch.from_numpy(np.ascontiguousarray(v)).to(device) for k, v in self.bind.items()}
        self.torch, self.device = torch, device
        ex = self._executor(self.bind)
        ex.run()
        torch.cuda.synchronize()
        self.iters = ex.iterations
        self.flop = self.iters * (2 * self.nnz + 12 * n) + 2 * n
        self.units_per_step = self.flop / 1e9
        # roofline bytes: per iteration the loop body's distinct HBM-level traffic -- spmv values
        # (8 B) + colidx (4 B) per nnz, rowptr 4 B and x read / y written 8 B each per row, then
        # dot(p,Ap) 16n, axpy x 24n, axpy r 24n, dot(r,r) 16n, scale p 16n, axpy p 24n
        self.roof_bytes = self.iters * (12 * self.nnz + 4 * (n + 1) + 16 * n + 120 * n)
        self.algorithmic = {"flop_per_solve": self.flop, "iterations": self.iters,
                            "per_unit": "per iteration 2*nnz (spmv) + 3 dots + 3 vector updates (12n)",
                            "roof_bytes_per_solve": self.roof_bytes,
                            "roof_bytes_per_unit": "per iteration 12*nnz + 4*(n+1) + 136*n (spmv + dots + updates)",
                            "note": "the ~12 MB working set stays in L2 across iterations; the solve is bound by "
                                    "the per-phase grid barriers (latency), so the HBM fraction is a floor"}
        how = ("the whole LoopStep as ONE persistent cooperative kernel interpreting the loop body" if world == 1
               else f"rows sharded over {world} ranks, p exchanged after each update, dots reduced on the device")
        self.workload = (f"CG (bundled cg.gmodel resized) {self.matrix}: n={n}, nnz={self.nnz}, {self.iters} "
                         f"iterations; {how} (Executor setup timed, inputs resident in HBM)")
        self.l2 = "working set (~12 MB) fits in L2: L2 flushed (256 MiB write + 256 MiB read) before every timed step"
        self.ex = None

    graphs = True
    l2_flush = True

    def _executor(self, bind):
        if self.world > 1:
            from paper_1105_4424_b200.distributed import make_distributed_executor
            return make_distributed_executor(self.model, self.schedule, bind)
        from paper_1105_4424_b200.executor import Executor
        return Executor(self.model, self.schedule, bind, 1, graphs=self.graphs)

    def step(self):
        self._executor(self.dbind).run()

    def gather(self):
        return None

    e2e_path = ("execute_schedule(model, schedule, pinned host bindings, 1, out={x: pinned buffer}): H2D of the "
                "CSR matrix and b from pinned memory, the whole solve as one persistent kernel, x back to the host")

    def e2e_setup(self):
        self.e2e_bytes = (sum(v.nbytes for v in self.bind.values()), self.n * 8)
        torch = self.torch
        self.pinned = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in self.bind.items()}
        self.hout = {"x": torch.empty(self.n, dtype=torch.float64).pin_memory()}

    def e2e_step(self):
        from paper_1105_4424_b200.executor import execute_schedule
        if self.world > 1:
            ex = self._executor(self.pinned)
            ex.run()
            return ex.outputs()
        return execute_schedule(self.model, self.schedule, self.pinned, 1, graphs=self.graphs, out=self.hout).outputs

    def e2e_numpy_setup(self):
        pass

    def e2e_numpy_step(self):
        from paper_1105_4424_b200.executor import execute_schedule
        if self.world > 1:
            ex = self._executor(self.bind)
            ex.run()
            return ex.outputs()
        return execute_schedule(self.model, self.schedule, self.bind, 1, graphs=self.graphs).outputs

    def e2e_free(self):
        pass

    def cpu_sample(self, seconds: float = 8.0):
        from oracle import aol_oracle as orc
        n = self.n
        rp, ci, va = self.bind["rowptr"], self.bind["colidx"], self.bind["values"]
        x = np.zeros(n)
        r = np.ones(n)
        p = r.copy()
        rr = float(np.dot(r, r))
        t0 = time.perf_counter()
        it = 0
        while it < 10:
            ap = np.zeros(n)
            orc.spmv_rows(rp, ci, va, p, ap, 0, n)
            alpha = rr / float(np.dot(p, ap))
            x += alpha * p
            r += (-alpha) * ap
            rrn = float(np.dot(r, r))
            p *= rrn / rr
            p += r
            rr = rrn
            it += 1
        dt = (time.perf_counter() - t0) / it
        return {"value": (2 * self.nnz + 12 * n) / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
                "sample": f"10 CG iterations with the oracle's level-synchronous spmv (numpy), {dt * 1e3:.1f} ms/iter"}


class CG27Workload(CGWorkload):
    """The paper's CG matrix shape (N = 132,651, NNZ = 3,442,951): a 27-point
    operator on a 51^3 grid.  Paper, Tesla T10: 116 iterations in 0.659 s, 1.45 GFLOP/s."""

    name = "cg27"
    matrix = "27-point 3-D operator on 51^3 (the paper's N and NNZ)"

    def _matrix(self):
        return _poisson_3d27(51)


class C1Workload(Workload):
    """Config C1: the paper-case-study MatMul 256x256 fp32 repetitive task, one full
    execute_schedule call per step (host numpy bindings -> numpy outputs, like the reference
    executor is called).  Launch/overhead-bound: reported, not a roofline target."""

    name = "c1"
    unit = "TFLOP/s"
    bound = "tensor"

    scaling = "weak"

    def __init__(self, torch, device, rank, world, n=256):
        from paper_1105_4424_b200 import builders
        from paper_1105_4424_b200.partition import build_schedule
        self.torch, self.device, self.n = torch, device, n
        self.rank, self.world, self.rank_fraction = rank, world, 1.0
        self.model = builders.matmul_model(n, n, n)
        self.schedule = build_schedule(self.model, 1)
        rng = np.random.default_rng(0)
        self.bind = {"p_a": rng.standard_normal(n * n, dtype=np.float32),
                     "p_b": rng.standard_normal(n * n, dtype=np.float32)}
        self.dbind = {k: torch.from_numpy(v).to(device) for k, v in self.bind.items()}
        self.units_per_step = 2.0 * n ** 3 / 1e12
        self.algorithmic = {"flop_per_launch": 2 * n ** 3, "per_unit": "2 FLOP per (m, n, k)"}
        self.workload = (f"C1 matmul {n}x{n}x{n} fp32 via execute_schedule (TF32 tcgen05): value with HBM-resident "
                         f"bindings and device outputs, e2e with host numpy in/out")
        self.l2 = ("small (768 KB): L2 flushed (256 MiB write + 256 MiB read) before every timed step; launch- and "
                   "API-overhead-bound")

    l2_flush = True

    def step(self):
        # inputs resident in HBM, result left in HBM (device_outputs): the API call itself
        from paper_1105_4424_b200.executor import execute_schedule
        execute_schedule(self.model, self.schedule, self.dbind, 1, device_outputs=True)

    e2e_path = ("execute_schedule(model, schedule, pinned host bindings, 1, out={p_c: pinned buffer}): H2D of "
                "A and B from pinned memory, the GEMM, C back into the caller's pinned buffer (steps back to back, "
                "no L2 flush between them, unlike `value`: hence e2e can exceed value at this size)")

    def e2e_setup(self):
        self.e2e_bytes = (2 * self.n * self.n * 4, self.n * self.n * 4)
        torch = self.torch
        self.pinned = {k: torch.from_numpy(v).pin_memory() for k, v in self.bind.items()}
        self.hout = {"p_c": torch.empty(self.n * self.n, dtype=torch.float32).pin_memory()}

    def e2e_step(self):
        from paper_1105_4424_b200.executor import execute_schedule
        execute_schedule(self.model, self.schedule, self.pinned, 1, out=self.hout)

    def e2e_numpy_setup(self):
        pass

    def e2e_numpy_step(self):
        # host numpy in, host numpy out, exactly like the reference executor is called
        from paper_1105_4424_b200.executor import execute_schedule
        execute_schedule(self.model, self.schedule, self.bind, 1)

    def e2e_free(self):
        pass

    def cpu_sample(self, seconds: float = 8.0):
        from oracle import c_oracle as co
        n = self.n
        c = np.zeros(n * n, np.float32)
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < min(seconds, 2.0):
            co.gemm_rows(self.bind["p_a"], self.bind["p_b"], c, n, n, 0, n)
            reps += 1
        dt = (time.perf_counter() - t0) / reps
        out = {"value": 2.0 * n ** 3 / dt / 1e12, "unit": "TFLOP/s", "cores": co.threads(), "kind": "port",
               "sample": f"full 256^3 product, oracle/aol_oracle.c, {dt * 1e3:.2f} ms per product"}
        # the UNMODIFIED reference executor cannot run here (the reference is absent on the GPU
        # box); its C1 timing in the build container is committed by tools/time_reference_executor.py
        ref = ROOT / "profiles" / "r2_reference_executor_c1.json"
        if ref.exists():
            try:
                d = json.loads(ref.read_text())
                out["reference_executor"] = {
                    "value_D1": d["runs"]["1"]["TFLOP/s"], "value_D8": d["runs"]["8"]["TFLOP/s"],
                    "e2e_s_D1": d["runs"]["1"]["e2e_s"], "e2e_s_D8": d["runs"]["8"]["e2e_s"],
                    "op_only_s": d["op_only"]["s"], "unit": "TFLOP/s", "cores": d["host"]["cpu_count"],
                    "kind": "reference", "where": d["host"]["where"], "source": "profiles/r2_reference_executor_c1.json",
                    "sample": d["workload"]}
            except (ValueError, KeyError):
                pass
        return out


WORKLOADS = {"matmul": MatmulWorkload, "stencil": StencilWorkload, "downscaler": DownscalerWorkload,
             "sweep": SweepWorkload, "cg": CGWorkload, "cg27": CG27Workload, "c1": C1Workload}


# ---------------------------------------------------------------- the arms --

def time_steps(torch, fn, steps, warmup, stream, barrier, flush=None):
    """K steps bracketed by barrier + synchronize.  With `flush` (workloads whose working set
    fits in the 126 MB L2) a 256 MiB buffer is written between steps, outside each step's
    event pair; the step time is then the sum of the per-step event times."""
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
        if flush is not None:
            flush()
        s.record(stream)
        fn()
        e.record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    per = [s.elapsed_time(e) for s, e in ev]
    total_ms = sum(per) if flush is not None else t0.elapsed_time(t1)
    return total_ms, per


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_1105_4424_b200 import _capi

    rank, world, local = dist_env()
    # AOL_BENCH_BACKEND=gloo: test mode for the multi-rank logic on a 1-GPU box (ranks share
    # cuda:0; their kernels never wait on each other, only the host barriers do).  Numbers
    # from this mode are not scaling results.
    backend = os.environ.get("AOL_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    red_dev = device if backend == "nccl" else torch.device("cpu")

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    _capi.load()
    all_cpus = os.sched_getaffinity(0)
    numa = bind_host_to_gpu_numa(torch, local)
    if world > 1:
        # torchrun exports OMP_NUM_THREADS=1; give each rank its share of the host cores for the
        # host-side copies of the e2e forms (pinned staging of numpy inputs)
        lws = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
        torch.set_num_threads(max(1, min(len(os.sched_getaffinity(0)), len(all_cpus) // lws)))
    t_start = time.perf_counter()

    def phase(name):
        log(f"[bench rank {rank}/{world}] {name} at {time.perf_counter() - t_start:.1f} s")
    wl = WORKLOADS[args.workload](torch, device, rank, world)
    phase("workload prepared")
    stream = torch.cuda.current_stream(device)

    _pp = torch.cuda.get_device_properties(device)
    clocks = Clocks(local, f"{_pp.pci_domain_id:08X}:{_pp.pci_bus_id:02X}:{_pp.pci_device_id:02X}.0")
    launches0 = _capi.launch_counter()
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    warm_launches = _capi.launch_counter() - launches0
    flush = None
    if getattr(wl, "l2_flush", False):
        scrub = torch.empty(64 << 20, dtype=torch.float32, device=device)      # 256 MiB > 126 MB L2
        rd = torch.ones(64 << 20, dtype=torch.float32, device=device)
        acc = torch.zeros(1, device=device)

        def flush():
            # write 256 MiB, then read another 256 MiB: the L2 is left holding clean lines, so the
            # timed step neither finds its inputs cached nor pays for the flush's write-backs.
            # Synchronised: the step's start event then fires when the step itself is enqueued,
            # so host-bound steps (C1) are not hidden behind the flush's GPU time
            scrub.fill_(1.0)
            acc.copy_(rd.sum())
            torch.cuda.synchronize()
    phase("warm")
    clocks.start()
    total_ms, per = time_steps(torch, wl.step, args.steps, 0, stream, barrier, flush)
    clk = clocks.stop()
    launches = (_capi.launch_counter() - launches0 - warm_launches)
    total_ms = allmax(total_ms)
    ms_per_step = total_ms / args.steps
    # whole-job units per step: the configured problem (strong) or one copy per rank (weak)
    job_units = wl.units_per_step * (world if wl.scaling == "weak" else 1)
    value = job_units * args.steps / (total_ms * 1e-3)
    kernel_ms = allmax(statistics.mean(per))

    def timed_e2e(step_fn, setup_fn, steps):
        setup_fn()
        for _ in range(2):
            step_fn()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            step_fn()
        torch.cuda.synchronize()
        return allmax(time.perf_counter() - t0)

    # end to end through the public API (H2D + launch + D2H every step)
    e2e = None
    e2e_np = None
    phase("timed region done")
    if not args.no_e2e:
        el = timed_e2e(wl.e2e_step, wl.e2e_setup, args.e2e_steps)
        h2d = wl.e2e_bytes[0] * (world if wl.scaling == "weak" else 1)
        if world > 1 and wl.scaling == "strong" and hasattr(wl, "e2e_h2d"):
            h2d = int(allsum(float(wl.e2e_h2d)))
        e2e = {"value": job_units * args.e2e_steps / el, "unit": wl.unit,
               "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": wl.e2e_bytes[1] * (world if wl.scaling == "weak" else 1),
               "ms_per_step": el * 1e3 / args.e2e_steps, "steps": args.e2e_steps,
               "path": (getattr(wl, "e2e_path", None) or
                        "paper_1105_4424_b200.executor.execute_schedule(pipeline=%d): pinned host bindings and "
                        "out= buffers; chunked H2D / launch / D2H overlap" % getattr(wl, "pipeline", 0))
               if world == 1 or wl.scaling == "weak" else
               ("make_distributed_executor on pinned host bindings: each rank uploads its input hull, runs "
                "its launch; output ranges gather to rank 0 (NCCL send/recv), rank 0 copies the result down"),
               "host_numa": numa}
        if not args.no_e2e_numpy and hasattr(wl, "e2e_numpy_setup") and wl.name not in ("downscaler", "sweep") \
                and (world == 1 or wl.scaling == "weak"):
            el = timed_e2e(wl.e2e_numpy_step, wl.e2e_numpy_setup, max(3, args.e2e_steps // 2))
            n = max(3, args.e2e_steps // 2)
            e2e_np = {"value": job_units * n / el, "unit": wl.unit, "ms_per_step": el * 1e3 / n, "steps": n,
                      "h2d_bytes_per_step": e2e["h2d_bytes_per_step"], "d2h_bytes_per_step": e2e["d2h_bytes_per_step"],
                      "path": "execute_schedule(model, schedule, {port: numpy array}, D) -> numpy outputs: the "
                              "reference's call (refexec.py:427), pageable host memory both ways"}
        wl.e2e_free()
        phase("e2e done")
    os.sched_setaffinity(0, all_cpus)            # the CPU baseline gets every host core again

    # N > 1: the output ranges gathered to rank 0, timed separately from the concurrent
    # per-rank phase (north_star: "NCCL output gather reported separately")
    gather = None
    if world > 1 and not args.no_gather and wl.scaling == "strong" and getattr(wl, "ex", None) is not None:
        times, nbytes = [], 0
        for _ in range(3):
            wl.step()
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            moved = wl.gather()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            nbytes = moved or 0
        # collectives on every rank (a rank that moved nothing still takes part)
        g = allmax(min(times))
        nb = int(allmax(float(nbytes)))
        if nb:
            gather = {"ms": g * 1e3, "bytes_to_root": nb, "GBps": nb / g / 1e9, "backend": backend,
                      "op": "ShardedExecutor.gather_to_root after the timed phase: each rank's written output "
                            "ranges to rank 0 (batched send/recv of exact ranges)"}
        # the same step with the fused output gather: the producing kernels store their output
        # ranges straight into rank 0's array (CUDA IPC peer mappings, NVLink), so a step ends
        # with the whole result at the root
        fstep = getattr(wl, "fused_step", None)
        if fstep is not None:
            fb, fms = fstep(time_steps, stream, barrier, min(args.steps, 20))
            fms = allmax(fms)
            fb = int(allsum(float(fb)))
            if fb:
                gather = {**(gather or {}), "fused": {
                    "step_ms": fms, "value": job_units / (fms * 1e-3), "unit": wl.unit,
                    "bytes_to_root_per_step": fb,
                    "op": "every rank's kernels store their output ranges into rank 0's array through CUDA IPC "
                          "peer mappings (NVLink); the step ends when all ranks' stores are done (barrier)"}}

    peaks = measured_peaks()
    out = None
    if rank == 0:
        achieved = wl.units_per_step * wl.rank_fraction / (kernel_ms * 1e-3)
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
            if getattr(wl, "roof_bytes", None):        # metric is not bytes (CG: GFLOP/s): roofline on bytes
                achieved = wl.roof_bytes * wl.rank_fraction / (kernel_ms * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": profile_traffic(wl.name),
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650",
                    "kernel_ms": kernel_ms, "algorithmic": wl.algorithmic}
        phase("gather done")
        cpu = None if (args.no_cpu or world > 1) else wl.cpu_sample(args.cpu_seconds)
        extra = {}
        if hasattr(wl, "fp32_faithful") and world == 1 and not args.no_peak:
            extra["fp32_faithful"] = wl.fp32_faithful()
        if wl.name == "sweep" and not args.no_points:
            extra["sweep_points"] = wl.measure_points()
        out = {
            "metric": METRIC, "value": value, "unit": wl.unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": wl.scaling,
            "vs_baseline": None, "dtype": getattr(wl, "dtype", "f32" if wl.bound == "hbm" else "tf32 (fp32 in/out)"),
            "data": "synthetic (torch.randn, seeded)",
            "config": {"workload": wl.workload, "l2": wl.l2,
                       "parallelism": f"repetition space sharded by contiguous blocks over {world} rank(s)"},
            "e2e": e2e, **({"e2e_numpy": e2e_np} if e2e_np else {}),
            "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "clocks": clk,
            **({"gather": gather} if gather else {}),
            **({"test_mode": "AOL_BENCH_BACKEND=gloo: ranks share one GPU; not a scaling result"}
               if backend != "nccl" and world > 1 else {}),
            **extra,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def _reference_arm(workload: str):
    """(setup-free step function, unit, sample text, cores) of the reference's CPU algorithm for one
    workload: the oracle's C restatement (oracle/aol_oracle.c, OpenMP) or its numpy interpreter
    (CG), each step a bounded sample of the same workload.  Returns step(i) -> units done."""
    from oracle import aol_oracle as orc
    from oracle import c_oracle as co
    thr = co.threads()
    rng = np.random.default_rng(0)
    if workload == "matmul":
        # the C2 CPU baseline is numpy.matmul fp32 (OpenBLAS sgemm, every
        # host core) -- the whole 8192^3 product every step, same config as the GPU arm
        M = N = K = 8192
        A = rng.standard_normal((M, K), dtype=np.float32)
        B = rng.standard_normal((K, N), dtype=np.float32)

        def step(i):
            np.matmul(A, B)
            return 2.0 * M * N * K / 1e12
        info = openblas_info()
        return step, "TFLOP/s", (f"matmul {M}x{N}x{K} fp32, the whole product per step: numpy.matmul "
                                 f"(OpenBLAS sgemm, {info.get('blas_threads')} threads)"), os.cpu_count()
    if workload == "c1":
        # the reference executor's route for the paper's MatMul: ONE spmv_csr
        # repetitive task over the Kronecker matrix I (x) A, rows left to right with product and
        # sum rounded separately -- refexec.py:111-121 restated by the oracle (numpy, 1 core)
        n = 256
        A = rng.standard_normal((n, n), dtype=np.float32)
        B = rng.standard_normal(n * n, dtype=np.float32)
        rows = np.repeat(np.arange(n * n), n)
        i, j = rows // n, rows % n          # output (i, j) of C = A B as row i*n+j of kron(A, I) . vec(B)
        k = np.tile(np.arange(n), n * n)
        colidx = (k * n + j).astype(np.int32)
        values = A[i, k].astype(np.float32)
        rowptr = (np.arange(n * n + 1) * n).astype(np.int32)

        y = np.zeros(n * n, np.float32)
        part = (n * n) // 8

        def step(i_):
            # a bounded sample: one eighth of the rows per step, cycling (the whole product took
            # 1.4 s per step, 9 min for the default 400 steps)
            lo = (i_ % 8) * part
            orc.spmv_rows(rowptr, colidx, values, B, y, lo, lo + part)
            return 2.0 * n ** 3 / 8 / 1e12
        return step, "TFLOP/s", ("matmul 256^3 fp32 as the reference executes it: one spmv_csr over the "
                                 "Kronecker CSR (16.8 M nnz), refexec.py:111-121 restated (oracle, numpy); "
                                 "one eighth of the rows per step, cycling"), 1
    if workload == "stencil":
        n = 16384
        x = rng.standard_normal(n * n, dtype=np.float32)
        y = np.zeros_like(x)
        w = orc.stencil_weights()
        rows = 256

        def step(i):
            lo = (i * rows) % (n - rows)
            co.stencil_rows(x, w, y, n, n, lo, lo + rows)
            return 2.0 * rows * n * 4 / 1e9
        return step, "GB/s", f"toroidal 3x3 stencil {n}x{n} fp32, {rows} rows per step (oracle/aol_oracle.c)", thr
    if workload == "downscaler":
        H, W = 2160, 3840
        th = orc.hfilter_tilers(1, H, W)
        Wo = th["y"]["array"][2]
        tv = orc.vfilter_tilers(1, H, Wo)
        Ho = tv["y"]["array"][1]
        x = rng.random(H * W, dtype=np.float32)
        mid = np.zeros(H * Wo, np.float32)
        y = np.zeros(Ho * Wo, np.float32)
        rh, rv = int(np.prod(th["x"]["rep"])), int(np.prod(tv["x"]["rep"]))
        wh, wv = orc.hfilter_weights(), orc.vfilter_weights()

        def step(i):
            co.tile_filter(x, wh, mid, th["x"], th["y"], 0, rh)
            co.tile_filter(mid, wv, y, tv["x"], tv["y"], 0, rv)
            return ((H * W + H * Wo) + (H * Wo + Ho * Wo)) * 4 / 1e9
        return step, "GB/s", (f"downscaler, one {H}x{W} frame per step through hfilter then vfilter "
                              f"(two tasks, as the reference schedules them; oracle/aol_oracle.c)"), thr
    if workload == "sweep":
        m, Ts = 2, 2_000_000
        span = Ts * m
        ts = dict(array=(span,), rep=(Ts,), pattern=(m,), origin=(0,), paving=((m,),), fitting=((1,),))
        x = rng.random(span, dtype=np.float32)
        y = np.zeros(Ts * m, np.float32)

        def step(i):
            co.tile_copy(x, y, ts, ts, 0, Ts)
            return 2.0 * Ts * m * 4 / 1e9
        return step, "GB/s", f"tile_copy sweep main point (pattern 2 dense), T={Ts} per step (oracle/aol_oracle.c)", thr
    if workload in ("cg", "cg27"):
        n, rp, ci, va = (_poisson_2d(364) if workload == "cg" else _poisson_3d27(51))
        nnz = int(rp[-1])
        st = {"x": np.zeros(n), "r": np.ones(n), "p": np.ones(n)}
        st["rr"] = float(np.dot(st["r"], st["r"]))

        def step(i):
            ap = np.zeros(n)
            orc.spmv_rows(rp, ci, va, st["p"], ap, 0, n)
            alpha = st["rr"] / float(np.dot(st["p"], ap))
            st["x"] += alpha * st["p"]
            st["r"] += (-alpha) * ap
            rrn = float(np.dot(st["r"], st["r"]))
            st["p"] *= rrn / st["rr"]
            st["p"] += st["r"]
            st["rr"] = rrn
            return (2 * nnz + 12 * n) / 1e9
        return step, "GFLOP/s", (f"one CG iteration per step (n={n}, nnz={nnz}) with the oracle's "
                                 f"level-synchronous spmv (refexec.py:111-121 restated, numpy)"), 1
    raise ValueError(f"no reference arm for workload '{workload}'")


def run_reference(args):
    """The reference arm: the reference's CPU algorithm (oracle port) on the host cores, rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # every host thread this process may use: torchrun exports OMP_NUM_THREADS=1 to each rank,
    # which would leave numpy's OpenBLAS and the OpenMP C port on one core at N > 1
    n_cpu = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(n_cpu)          # read when the C port's OpenMP starts
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=n_cpu)                  # BLAS / OpenMP pools already loaded
    except Exception:                                    # noqa: BLE001 -- env var still applies
        pass
    sys.path.insert(0, str(ROOT))
    step, unit, sample, cores = _reference_arm(args.workload)
    for i in range(args.warmup):
        step(i)
    t, units = [], 0.0
    for i in range(args.steps):
        t0 = time.perf_counter()
        units += step(i)
        t.append(time.perf_counter() - t0)
    el = sum(t)
    value = units / el
    out = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
           "scaling": WORKLOADS[args.workload].scaling, "vs_baseline": None,
           "dtype": "f64" if args.workload.startswith("cg") else "f32",
           "data": "synthetic (numpy default_rng)", "impl": "reference",
           "config": {"workload": f"{args.workload}: {sample}"},
           "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "port", "sample": sample,
                            **({"blas": openblas_info()} if args.workload == "matmul" else {})},
           "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="matmul", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-peak", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-points", action="store_true")
    ap.add_argument("--no-gather", action="store_true", help="N>1: skip the output-gather measurement")
    ap.add_argument("--no-e2e-numpy", action="store_true", help="skip the numpy-in / numpy-out e2e form")
    ap.add_argument("--no-fuse", action="store_true", help="disable task fusion (downscaler H->V as two kernels)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("note: warmup < 3 is below the timing rules; using 3")
        args.warmup = 3
    Workload.fuse = not args.no_fuse
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
