"""Benchmark: MDS points embedded / second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                    [--impl ours|reference]

Workloads (BASELINE.json configs; default = config 2, the metric's config):
  dc2      divide-and-conquer  n=1e6   p=100 fp64  l=1000 c=20 r=10
  fast3    fast MDS            n=1e6   p=100 fp64  l=1000 s=20 r=10
  interp4  interpolation       n=1e7   p=100 fp32  l=2000      r=10
  interp1  interpolation       n=1e4   p=10  fp64  l=500       r=2
  img5dc / img5fast / img5interp   config 5 (n=814,255, p=784 fp32, r=10)

A step = one full algorithm call over the whole (device-resident) input with
the plan passed explicitly (planning is host work done before timing); it
ends with the n x r configuration on the device in input row order.
Inputs are larger than L2 (126 MB) for every full-size workload, so no
separate flush is needed.  `e2e` repeats the measurement through the public
API from pinned HOST memory: H2D of the input, the plan's index upload, the
kernels, and the D2H of the n x r result and the fit figures, every step.

Multi-GPU (torchrun, one process per GPU): weak scaling.  Every algorithm
runs ONE global problem of N x the config's rows through
paper_2007_11919_b200.distributed (input replicated on every GPU outside the
timed region; each rank solves its contiguous share of subsets / rows /
level-1 subtrees; only per-segment sums and fit figures are exchanged —
all-gathers over NCCL).  The timed region is
bracketed by barriers and the max over ranks is reported; the n x r result
stays sharded on the devices (gathering it is not part of the metric).

--impl reference: the CPU oracle port of the reference algorithm (this repo's
oracle/, a restatement of /root/reference's numpy path) on the host cores,
rank 0 only, each step a bounded sample of the workload.
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

METRIC = "MDS points embedded/sec"
UNIT = "points/s"

WORKLOADS = {
    "dc2": dict(algo="divide", n=1_000_000, p=100, h=10, l=1000, c=20, s=None, r=10,
                dtype="f64", data="gaussian"),
    "fast3": dict(algo="fast", n=1_000_000, p=100, h=10, l=1000, c=None, s=20, r=10,
                  dtype="f64", data="gaussian"),
    "interp4": dict(algo="interpolate", n=10_000_000, p=100, h=10, l=2000, c=None, s=None, r=10,
                    dtype="f32", data="gaussian"),
    "interp1": dict(algo="interpolate", n=10_000, p=10, h=2, l=500, c=None, s=None, r=2,
                    dtype="f64", data="gaussian"),
    "img5dc": dict(algo="divide", n=814_255, p=784, h=0, l=1000, c=20, s=None, r=10,
                   dtype="f32", data="image"),
    "img5fast": dict(algo="fast", n=814_255, p=784, h=0, l=1000, c=None, s=20, r=10,
                     dtype="f32", data="image"),
    "img5interp": dict(algo="interpolate", n=814_255, p=784, h=0, l=1000, c=None, s=None, r=10,
                       dtype="f32", data="image"),
}


# dram__bytes_read.sum + dram__bytes_write.sum per launch from `ncu --set full`
# captures committed under profiles/ (same workload, same kernel build).
TRAFFIC = {
    ("dc2", "lanczos_smem_kernel"): {"bytes": (500.035 + 68.574) * 1e6,
                                     "src": "profiles/r01g_ncu_full_dc2.txt"},
    ("dc2", "gram_piece_kernel"): {"bytes": (439.716 + 27.652) * 1e6,
                                   "src": "profiles/r01g_ncu_full_dc2.txt"},
    ("interp4", "gower_bulk_kernel"): {"bytes": (4000.516 + 784.652) * 1e6,
                                       "src": "profiles/r01e_ncu_full_interp4.txt"},
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def measured_peaks(dev) -> dict:
    import torch
    peaks = {}
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        j = json.loads(mp.read_text())
        peaks["hbm_gbs"] = float(j["hbm_gbs"])
        peaks["hbm_src"] = "MEASURED_PEAKS.json"
    else:
        peaks["hbm_gbs"] = 6650.0
        peaks["hbm_src"] = "fallback (B200_PROFILING.md)"
    # fp64 peak: cuBLAS DGEMM 8192^3, best of 5, measured in this run
    a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    for _ in range(2):
        torch.matmul(a, b)
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    peaks["fp64_tflops"] = 2 * 8192 ** 3 / best / 1e12
    peaks["fp64_src"] = "cuBLAS DGEMM 8192^3 best of 5, this run"
    del a, b
    torch.cuda.empty_cache()
    return peaks


# ------------------------------------------------------------------ data
def make_data(w: dict, dev, seed: int):
    import torch
    n, p = w["n"], w["p"]
    if w["data"] == "image":
        from paper_2007_11919_b200.synthetic import image_like_device
        return image_like_device(n, seed=seed, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    dt = torch.float32 if w["dtype"] == "f32" else torch.float64
    x = torch.randn(n, p, generator=g, dtype=dt, device=dev)
    x[:, :w["h"]] *= 15.0 ** 0.5
    return x


def make_plan(w: dict, seed: int):
    from paper_2007_11919_b200 import plans
    if w["algo"] == "divide":
        return plans.plan_divide_conquer(w["n"], w["l"], w["c"], seed)
    if w["algo"] == "fast":
        return plans.plan_fast(w["n"], w["l"], w["s"], seed)
    return plans.interpolation_sample(w["n"], w["l"], seed)


class ShardedRun:
    """bench adapter for distributed.sharded_* (N>1, weak scaling)."""

    def __init__(self, w, x, plan, dev):
        from paper_2007_11919_b200 import AlgorithmParams
        from paper_2007_11919_b200 import distributed as dd
        self.dd, self.w = dd, w
        self.be = dd.GpuBackend(x, reuse=True)     # per-plan setup once, like the 1-GPU runners
        self.comm = dd.Comm(device=dev)
        self.plan = plan
        self.prm = AlgorithmParams(r=w["r"], l=w["l"], c=w["c"], s=w["s"], seed=0)
        self.res = None

    def launch(self):
        if self.w["algo"] == "divide":
            self.res = self.dd.sharded_divide_and_conquer(self.be, self.w["n"], self.prm, self.comm,
                                                          plan=self.plan)
        elif self.w["algo"] == "fast":
            self.res = self.dd.sharded_fast(self.be, self.w["n"], self.prm, self.comm, plan=self.plan)
        else:
            self.res = self.dd.sharded_interpolation(self.be, self.w["n"], self.prm, self.comm,
                                                     sample=self.plan)

    def finish(self, return_device=True):
        from paper_2007_11919_b200 import MdsConfiguration
        r = self.res
        return MdsConfiguration(r.out, r.estimates, r.gof_g1, r.gof_g2)


def make_run(w: dict, x, plan):
    from paper_2007_11919_b200 import DivideRun, FastRun, InterpolationRun
    if w["algo"] == "divide":
        return DivideRun(x, plan, w["r"], w["c"])
    if w["algo"] == "fast":
        return FastRun(x, plan, w["r"])
    return InterpolationRun(x, plan, w["r"])


# ------------------------------------------------------------------ work models
def piece_sizes(w: dict, plan) -> list:
    if w["algo"] == "divide":
        return [len(q) for q in plan.subsets]
    if w["algo"] == "fast":
        from paper_2007_11919_b200.plans import flatten_fast
        return list(np.diff(flatten_fast(plan).piece_off))
    return [w["l"]]


def fused_points(w: dict) -> bool:
    """The piece pipeline computes points inside the Lanczos kernel (mdsx_api.cu
    run_classical): form-0 pieces with k <= 104, r <= 10, aligned rows."""
    return (w["algo"] in ("divide", "fast") and w["p"] <= 104 and w["r"] <= 10
            and not os.environ.get("MDSX_NO_FUSE"))


def kernel_work(w: dict, plan, kernel: str, krylov_dims=None) -> dict | None:
    """Work of ONE launch of `kernel` in one step (DESIGN.md §3 work models):
    flops for compute-bound kernels (fp64), bytes for streaming ones."""
    p, r = w["p"], w["r"]
    esize = 4 if w["dtype"] == "f32" else 8
    sizes = piece_sizes(w, plan)
    if kernel in ("gram_dmma_kernel", "gram_piece_kernel", "gram_kernel"):
        fl = 0.0
        for m in sizes:
            if (p < m) == (kernel != "gram_kernel"):
                k, K = (p, m) if p < m else (m, p)
                fl += K * k * (k + 1)          # symmetric rank-K update of a k x k Gram
        return {"bound": "tensor", "flops": fl, "model": "SYRK m*p*(p+1) per piece"}
    if kernel == "lanczos_smem_kernel" and krylov_dims is not None:
        fl = 0.0
        for m, steps in zip(sizes, krylov_dims):
            k = min(m, p)
            if steps > 0:
                j = np.arange(int(steps))
                fl += float(np.sum(2.0 * k * k + 4.0 * k * (j + 1) + 6.0 * k))
        krylov_model = ("sum over Krylov steps of 2k^2 (matvec) + 4k(j+1) (one CGS pass) "
                        "+ 6k (three-term part)")
        if fused_points(w):
            # the piece pipeline's Lanczos kernel also streams every piece's rows
            # for its points (points_stream.cuh): its algorithmic traffic
            tot = sum(sizes)
            by = tot * p * esize + tot * r * 8 + sum(min(m, p) ** 2 * 8 for m in sizes)
            return {"bound": "hbm", "bytes": by, "flops": fl,
                    "model": "rows*p*sizeof(in) (points stream) + rows*r*8 (points) + k^2*8 "
                             "per piece (Gram read); Krylov phase: " + krylov_model}
        return {"bound": "tensor", "flops": fl, "model": krylov_model}
    if kernel in ("gower_affine_kernel", "gower_stream_kernel", "gower_bulk_kernel"):
        n = w["n"]
        return {"bound": "hbm", "bytes": n * p * esize + n * r * 8,
                "model": "n*p*sizeof(in) + n*r*8"}
    if kernel == "subtract_mean_kernel":
        n = w["n"]
        return {"bound": "hbm", "bytes": 2 * n * r * 8, "model": "read + write of the n x r output"}
    if kernel in ("points_kernel", "points_rows_kernel", "points_piece_kernel"):
        tot = sum(sizes)
        return {"bound": "hbm", "bytes": tot * p * esize + tot * r * 8,
                "model": "rows*p*sizeof(in) + rows*r*8"}
    return None


# ------------------------------------------------------------------ CPU oracle sample
def oracle_sample(w: dict, x_host: np.ndarray, budget_s: float, cores: int):
    """Time the oracle (oracle/mds_oracle.py, the reference's numpy path) on a
    bounded prefix of the workload's rows with the same p, l, c/s, r, using a
    pool of `cores` threads and single-threaded BLAS (the reference's tuned
    setting).  Returns (points/s, sample description)."""
    from threadpoolctl import threadpool_limits

    from oracle import mds_oracle as orc

    algo = w["algo"]
    kw = dict(l=w["l"])
    if algo == "divide":
        kw["c"] = w["c"]
    if algo == "fast":
        kw["s"] = w["s"]
    if algo == "fast":
        n_s = min(w["n"], (w["l"] // w["s"]) * 400)   # one level-1 subtree: 50 leaves + alignment
    elif algo == "divide":
        n_s = min(w["n"], max(4 * w["l"], 8 * cores * (w["l"] - w["c"])))
    else:
        n_s = min(w["n"], max(4 * w["l"], 100_000))
    with threadpool_limits(1):
        t0 = time.perf_counter()
        orc.run(algo, x_host[:n_s], w["r"], seed=0, threads=cores, **kw)
        dt = time.perf_counter() - t0
        if dt < budget_s * 0.5 and n_s < w["n"] and algo != "fast":
            n_s = int(min(w["n"], n_s * max(1.0, budget_s / max(dt, 1e-3))))
            t0 = time.perf_counter()
            orc.run(algo, x_host[:n_s], w["r"], seed=0, threads=cores, **kw)
            dt = time.perf_counter() - t0
    desc = (f"oracle {algo} on the first {n_s} rows (same p,l,c/s,r; seed 0), "
            f"{cores}-thread pool, BLAS 1 thread")
    return n_s / dt, desc, n_s


def host_copy(x) -> np.ndarray:
    return x.cpu().numpy()


# ------------------------------------------------------------------ arms
def run_reference(args, w):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import torch
    cores = os.cpu_count() or 1
    if w["data"] == "image":
        from paper_2007_11919_b200.synthetic import image_like
        xh = image_like(min(w["n"], 200_000), seed=0)
    else:
        from paper_2007_11919_b200.synthetic import scenario
        nh = min(w["n"], 300_000)
        xh = scenario(nh, w["p"], w["h"], seed=0)
        if w["dtype"] == "f32":
            xh = xh.astype(np.float32)
    w2 = dict(w, n=xh.shape[0])
    # size the per-step sample on one calibration run (~6 s per step)
    rate, desc, n_s = oracle_sample(w2, xh, 6.0, cores)
    from threadpoolctl import threadpool_limits

    from oracle import mds_oracle as orc
    kw = dict(l=w["l"])
    if w["algo"] == "divide":
        kw["c"] = w["c"]
    if w["algo"] == "fast":
        kw["s"] = w["s"]
    times = []
    with threadpool_limits(1):
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            orc.run(w["algo"], xh[:n_s], w["r"], seed=0, threads=cores, **kw)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = n_s / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, w, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name, w, gpus):
    cfg = {"workload": f"{name}: {w['algo']} n={w['n']} p={w['p']} {w['dtype']} l={w['l']}"
                       + (f" c={w['c']}" if w['c'] else "") + (f" s={w['s']}" if w['s'] else "")
                       + f" r={w['r']}",
           "algorithm": w["algo"], "n_per_gpu": w["n"], "p": w["p"], "l": w["l"], "r": w["r"],
           "input_dtype": w["dtype"], "parallelism": f"dp{gpus} (rows/partitions sharded)",
           "l2_flush": "inputs larger than L2 (126 MB)",
           "compute_precision": "fp64 throughout (fp32 inputs widened in-kernel)"}
    if w["c"]:
        cfg["c"] = w["c"]
    if w["s"]:
        cfg["s"] = w["s"]
    return cfg


def run_ours(args, w):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    force = os.environ.get("MDSX_BENCH_SHARDED") == "1"   # exercise the N>1 path on one GPU
    if ws > 1 or force:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2007_11919_b200 import _lib, divide_and_conquer_mds, fast_mds, interpolation_mds
    from paper_2007_11919_b200 import AlgorithmParams, InterpPlan
    from paper_2007_11919_b200 import _device as D

    peaks = measured_peaks(dev)
    sharded = ws > 1 or force
    if sharded:
        # one global problem of ws x n rows, replicated input, same seed everywhere
        w = dict(w, n=w["n"] * ws)
        seed = 0
    else:
        seed = 0
    x = make_data(w, dev, seed)
    plan = make_plan(w, seed)
    if sharded:
        run = ShardedRun(w, x, plan, dev)
    else:
        run = make_run(w, x, plan)
    h = D.handle(dev)
    log(f"[rank {rank}] data {tuple(x.shape)} {x.dtype}; warmup {args.warmup}")
    for _ in range(args.warmup):
        run.launch()
    torch.cuda.synchronize()
    run.finish(return_device=True)          # statuses OK (raises otherwise)

    stream = torch.cuda.current_stream(dev)
    h.timing_report()
    h.timing(True)
    l0 = h.launches()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    smi_idx = int(vis.split(",")[local]) if vis and vis.split(",")[local].isdigit() else local
    with ClockSampler(smi_idx) as clk:
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            run.launch()
        t1.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
    h.timing(False)
    launches = h.launches() - l0
    ms = t0.elapsed_time(t1) / args.steps
    kernels = h.timing_report()
    if ws > 1:
        tm = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms = float(tm.item())
    cfg_out = run.finish(return_device=True)
    value = (w["n"] if sharded else w["n"] * ws) / (ms / 1e3)
    try:       # Krylov dimension per piece (solver diagnostics in the status records)
        st = D.decode_status(run.status)
        krylov = [float(v) for v in st["value"]]
    except AttributeError:
        krylov = None

    # roofline of the dominant kernel (average launch duration over the timed region)
    total_k = sum(v[0] for v in kernels.values())
    dom = max(kernels, key=lambda k: kernels[k][0]) if kernels else None
    roof = None
    if dom:
        ms_k, cnt = kernels[dom]
        per_launch_ms = ms_k / cnt
        work = kernel_work(w, plan, dom, krylov)
        launches_per_step = cnt / args.steps
        if work and work["bound"] == "hbm":
            ach = work["bytes"] / launches_per_step / (per_launch_ms / 1e3) / 1e9
            peak = peaks["hbm_gbs"]
            roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": ach / peak, "traffic": None, "peak_src": peaks["hbm_src"],
                    "work_model": work["model"]}
        elif work:
            ach = work["flops"] / launches_per_step / (per_launch_ms / 1e3) / 1e12
            peak = peaks["fp64_tflops"]
            roof = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": peak,
                    "unit": "TFLOP/s", "frac": ach / peak, "traffic": None,
                    "precision": "fp64", "peak_src": peaks["fp64_src"],
                    "work_model": work["model"]}
        if roof is not None:
            roof["share_of_kernel_time"] = ms_k / total_k
            if w["algo"] in ("divide", "fast"):
                roof["note"] = ("two-stream piece pipeline: launch durations include time "
                                "shared with the other stream's kernels")
            roof["avg_launch_ms"] = per_launch_ms
            traffic = TRAFFIC.get((args.workload, dom))
            if traffic:
                roof["traffic"] = traffic["bytes"]
                roof["traffic_src"] = traffic["src"]
    per_kernel = {}
    for kname, (ms_k, cnt) in kernels.items():
        wk = kernel_work(w, plan, kname, krylov)
        if not wk:
            continue
        t = ms_k / cnt / 1e3
        lps = cnt / args.steps
        if wk["bound"] == "hbm":
            per_kernel[kname] = {"GB/s": wk["bytes"] / lps / t / 1e9,
                                 "frac_hbm": wk["bytes"] / lps / t / 1e9 / peaks["hbm_gbs"]}
            if "flops" in wk:
                per_kernel[kname]["TFLOP/s"] = wk["flops"] / lps / t / 1e12
                per_kernel[kname]["frac_fp64"] = wk["flops"] / lps / t / 1e12 / peaks["fp64_tflops"]
        else:
            per_kernel[kname] = {"TFLOP/s": wk["flops"] / lps / t / 1e12,
                                 "frac_fp64": wk["flops"] / lps / t / 1e12 / peaks["fp64_tflops"]}

    # e2e through the public API from pinned host memory
    if sharded:                 # per-rank kernel times cover 1/ws of the plan: no roofline
        roof, per_kernel = None, {}
    e2e = None
    if not args.no_e2e and sharded:
        # public distributed API from pinned host memory: H2D of the (replicated)
        # input on every rank, the sharded run, and the gather of n x r to rank 0
        host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        host.copy_(x)
        k_e2e = max(1, min(args.steps, 3))
        from paper_2007_11919_b200 import distributed as dd
        dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(k_e2e):
            x.copy_(host, non_blocking=True)
            run.launch()
            dd.gather_points(run.res, w["n"], w["r"], run.comm)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t) / k_e2e
        tm = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        e2e_s = float(tm.item())
        e2e = {"value": w["n"] / e2e_s, "unit": UNIT, "ms_per_step": e2e_s * 1e3,
               "h2d_bytes_per_step": int(x.numel() * x.element_size() * ws),
               "d2h_bytes_per_step": int(w["n"] * w["r"] * 8), "steps": k_e2e,
               "path": "paper_2007_11919_b200.distributed (pinned host input on every rank, "
                       "gather to rank 0)"}
    if not args.no_e2e and not sharded:
        host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        host.copy_(x)
        del run
        torch.cuda.empty_cache()
        prm = AlgorithmParams(r=w["r"], l=w["l"], c=w["c"], s=w["s"], seed=seed)
        fn = {"divide": divide_and_conquer_mds, "fast": fast_mds,
              "interpolate": interpolation_mds}[w["algo"]]
        kw = dict(plan=plan if w["algo"] != "interpolate" else InterpPlan([plan], w["n"], w["l"], seed),
                  device=dev)
        k_e2e = max(1, min(args.steps, 5))
        res = None
        for _ in range(2):        # steady state: one result alive while the next call runs
            res = fn(host, prm, **kw)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(k_e2e):
            res = fn(host, prm, **kw)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t) / k_e2e
        if ws > 1:
            tm = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            e2e_s = float(tm.item())
        n_idx = len(plan) if w["algo"] == "interpolate" else (
            sum(len(q) for q in plan.subsets) if w["algo"] == "divide" else 2 * w["n"])
        e2e = {"value": w["n"] * ws / e2e_s, "unit": UNIT, "ms_per_step": e2e_s * 1e3,
               "h2d_bytes_per_step": int(x.numel() * x.element_size() + 8 * n_idx),
               "d2h_bytes_per_step": int(w["n"] * w["r"] * 8), "steps": k_e2e,
               "path": f"paper_2007_11919_b200.{fn.__name__}(pinned host tensor, plan=...)"}
        del host

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        xh = host_copy(x[:min(w["n"], 300_000)])
        rate, desc, _ = oracle_sample(dict(w, n=xh.shape[0]), xh, 8.0, os.cpu_count() or 1)
        cpu = {"value": rate, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
               "sample": desc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.workload, w, ws),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
            "gpu_launches": launches,
            "kernels_ms_per_step": {k: v[0] / args.steps for k, v in sorted(kernels.items())},
            "kernel_rooflines": per_kernel,
            "peaks": peaks,
            "fit": {"g1": cfg_out.gof_g1, "estimates": [float(v) for v in cfg_out.eigenvalue_estimates]},
        }
        print(json.dumps(line), flush=True)
    if ws > 1 or force:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="dc2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)
    return run_ours(args, w)


if __name__ == "__main__":
    sys.exit(main())
