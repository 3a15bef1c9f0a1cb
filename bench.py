"""Benchmark: MDS points embedded / second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                    [--impl ours|reference] [--scaling auto|weak|strong]

Workloads (BASELINE.json configs; default = config 2, the metric's config):
  dc2      divide-and-conquer  n=1e6   p=100 fp64  l=1000 c=20 r=10
  fast3    fast MDS            n=1e6   p=100 fp64  l=1000 s=20 r=10
  interp4  interpolation       n=1e7   p=100 fp32  l=2000      r=10
  interp1  interpolation       n=1e4   p=10  fp64  l=500       r=2
  img5dc / img5fast / img5interp   config 5 (n=814,255, p=784 fp32, r=10)

Input: the reference's own scenario stream (simulation.py:68-80, bit-exact,
generated on the host by parallel PCG64 sub-streams; config 4 cast to
float32) or the config-5 image-like stand-in, so the result can be checked
against the fixtures produced by running the reference itself
(tests/golden/full_*.npz): the line's ``parity`` block.

A step = one full algorithm call over the device-resident input with the plan
passed explicitly (planning is host work, reported as ``planner_ms``); it
ends with the n x r configuration on the device in input row order.  Every
full-size input is larger than L2 (126 MB), so no flush is needed.  ``e2e``
repeats the call through the public API from a page-locked host tensor: H2D
of the input and of the plan indices, the kernels, and the D2H of the n x r
result into numpy; ``e2e.numpy_input`` is the same with the input as a
PAGEABLE numpy array (what a scalemds user passes; staged by mdsx_h2d).

Multi-GPU: ``--gpus N`` without torchrun starts N ranks itself (torch's
launcher on 127.0.0.1); under torchrun one process per GPU.  Scaling: weak
for D&C / fast (N x the config's rows, one global plan), strong for config 4
("rows sharded across 1/2/4/8 GPUs", fixed n = 1e7).  Each rank holds only
the rows its share needs (distributed.local_rows); the step exchanges only
small record tensors over NCCL; max over ranks.

--impl reference: the reference algorithm's CPU restatement (oracle/, the
reference's own numpy code path) on the host cores, rank 0 only, each step a
bounded sample of the workload.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "MDS points embedded/sec"
UNIT = "points/s"

WORKLOADS = {
    "dc2": dict(algo="divide", n=1_000_000, p=100, h=10, l=1000, c=20, s=None, r=10,
                dtype="f64", data="gaussian"),
    "fast3": dict(algo="fast", n=1_000_000, p=100, h=10, l=1000, c=None, s=20, r=10,
                  dtype="f64", data="gaussian"),
    "interp4": dict(algo="interpolate", n=10_000_000, p=100, h=10, l=2000, c=None, s=None, r=10,
                    dtype="f32", data="gaussian", strong=True),
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
    ("dc2", "lanczos_smem_kernel"): {"bytes": (40.936 + 0.223) * 1e6,
                                     "src": "profiles/r02j_ncu_dram_dc2.csv"},
    ("dc2", "gram_piece_kernel"): {"bytes": (439.722 + 29.207) * 1e6,
                                   "src": "profiles/r02j_ncu_dram_dc2.csv"},
    ("interp4", "gower_bulk_kernel"): {"bytes": (4000.050 + 786.500) * 1e6,
                                       "src": "profiles/r02j_ncu_dram_interp4.csv"},
    ("img5dc", "gram_tile_async_kernel"): {"bytes": (1726.715 + 1647.288) * 1e6,
                                           "src": "profiles/r02j_ncu_dram_img5dc.csv"},
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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


# ------------------------------------------------------------------ data / plans
def host_input(w: dict, n: int) -> np.ndarray:
    """The workload's input on the host: the reference scenario stream
    (bit-exact, parallel) or the config-5 stand-in."""
    from paper_2007_11919_b200.synthetic import image_like, scenario
    if w["data"] == "image":
        return image_like(n, seed=0)
    x = scenario(n, w["p"], w["h"], seed=0)
    return x.astype(np.float32) if w["dtype"] == "f32" else x


def make_plan(w: dict, n: int, seed: int = 0):
    from paper_2007_11919_b200 import plans
    if w["algo"] == "divide":
        return plans.plan_divide_conquer(n, w["l"], w["c"], seed)
    if w["algo"] == "fast":
        return plans.plan_fast(n, w["l"], w["s"], seed)
    return plans.interpolation_sample(n, w["l"], seed)


def make_run(w: dict, x, plan):
    from paper_2007_11919_b200 import DivideRun, FastRun, InterpolationRun
    if w["algo"] == "divide":
        return DivideRun(x, plan, w["r"], w["c"])
    if w["algo"] == "fast":
        return FastRun(x, plan, w["r"])
    return InterpolationRun(x, plan, w["r"])


class ShardedRun:
    """bench adapter for the distributed classes (N > 1)."""

    def __init__(self, w, x_local, n, plan, comm, x_landmarks=None):
        from paper_2007_11919_b200 import distributed as dd
        be = dd.GpuBackend(x_local.device)
        if w["algo"] == "divide":
            self.impl = dd.ShardedDivide(be, x_local, plan, w["r"], comm)
        elif w["algo"] == "fast":
            self.impl = dd.ShardedFast(be, x_local, plan, w["r"], comm)
        else:
            self.impl = dd.ShardedInterpolation(be, x_local, n, plan, w["r"], comm, x_landmarks)
        self.res = None

    def launch(self):
        self.res = self.impl.launch()

    def finish(self, return_device=True):
        from paper_2007_11919_b200 import MdsConfiguration
        r = self.res.finish()
        return MdsConfiguration(r.out, r.estimates, r.gof_g1, r.gof_g2)


# ------------------------------------------------------------------ work models
def piece_sizes(w: dict, plan) -> list:
    if w["algo"] == "divide":
        return [len(q) for q in plan.subsets]
    if w["algo"] == "fast":
        from paper_2007_11919_b200.plans import flatten_fast
        return list(np.diff(flatten_fast(plan).piece_off))
    return [w["l"]]


def kernel_work(w: dict, n: int, plan, kernel: str, krylov_dims=None, executed=0.0,
                p_eff=None) -> dict | None:
    """Algorithmic work of ONE step's launches of `kernel` (DESIGN.md §3 work
    models): flops for compute-bound kernels (fp64), bytes for streaming ones.
    p_eff: the width the kernels actually ran at (column compaction of wide
    inputs drops the all-zero columns, k_compact.cu); the bytes of the passes
    over the input keep the stored width p."""
    p, r = w["p"], w["r"]
    pe = int(p_eff or p)
    esize = 4 if w["dtype"] == "f32" else 8
    sizes = piece_sizes(w, plan)
    form0 = [m for m in sizes if pe < m]
    form1 = [m for m in sizes if pe >= m]
    if kernel in ("gram_piece_kernel", "gram_tile_async_kernel", "gram_dmma_kernel"):
        return {"bound": "tensor", "flops": float(sum(m * pe * (pe + 1) for m in form0)),
                "model": "SYRK m*p*(p+1) per form-0 piece (p x p Gram of the centred rows; "
                         f"p = {pe} active columns)"}
    if kernel in ("gram_rows_async_kernel", "gram_kernel"):
        return {"bound": "tensor", "flops": float(sum(m * (m + 1) * pe for m in form1)),
                "model": f"SYRK m*(m+1)*p per form-1 piece (m x m Gram; p = {pe} active columns)"}
    if kernel == "bgemm_dmma_kernel" and executed > 0:
        return {"bound": "tensor", "flops": float(executed),
                "model": "executed block-Krylov products, 2*M*N*K per task of a piece not yet "
                         "converged (counted by the launcher)"}
    if kernel == "bgemm_stream_kernel" and executed > 0:
        return {"bound": "hbm", "bytes": float(executed),
                "model": "executed streamed block-Krylov products (Z = A Q, P = Q^T Z, Q -= Q P, "
                         "H = Q^T Z, Y = Q S): each operand read once + the result written, "
                         "8*(M*K + K*N + M*N) bytes per task (counted by the launcher)"}
    if kernel == "lanczos_smem_kernel" and krylov_dims is not None:
        fl = 0.0
        for m, steps in zip(sizes, krylov_dims):
            k = min(m, pe)
            if steps > 0:
                j = np.arange(int(steps))
                fl += float(np.sum(2.0 * k * k + 4.0 * k * (j + 1) + 6.0 * k))
        return {"bound": "tensor", "flops": fl,
                "limiter": "latency (dependent Krylov steps, per-step barriers; fp64 FMA work "
                           "is a few % of the pipe)",
                "model": "sum over Krylov steps of 2k^2 (matvec) + 4k(j+1) (one CGS pass) "
                         "+ 6k (three-term part)"}
    if kernel in ("gower_affine_kernel", "gower_bulk_kernel"):
        return {"bound": "hbm", "bytes": float(n * pe * esize + n * r * 8),
                "model": f"n*p*sizeof(in) + n*r*8 (one read of every row, one write; p = {pe})"}
    if kernel == "subtract_mean_kernel":
        return {"bound": "hbm", "bytes": float(2 * n * r * 8),
                "model": "read + write of the n x r output"}
    if kernel == "piece_out_kernel":
        c = w.get("c") or 0
        own = sum(sizes) - (c * (len(sizes) - 1) if w["algo"] == "divide" else 0)
        return {"bound": "hbm", "bytes": float(own * (pe * esize + 2 * 8) + n * r * 8),
                "model": "every output row's input row gathered once (p*sizeof(in)) + its "
                         "two int64 indices + the n x r write"}
    if kernel in ("points_kernel", "points_piece_kernel"):
        tot = sum(sizes)
        if w["algo"] in ("divide", "fast") and pe <= 104:
            return None          # alignment sets / anchor only: not the per-row pass
        return {"bound": "hbm", "bytes": float(tot * pe * esize + tot * r * 8),
                "model": "rows*p*sizeof(in) + rows*r*8"}
    if kernel == "dc_stitch_kernel":
        tot = sum(sizes)
        return {"bound": "hbm", "bytes": float(tot * r * 8 + n * r * 8 + n * 8),
                "model": "read piece points + write n x r + read row indices"}
    if kernel == "nonzero_cols_kernel":
        return {"bound": "hbm", "bytes": float(n * p * esize),
                "model": "one read of the input (active-column flags)"}
    return None


def step_bytes(w: dict, n: int) -> float:
    """One-pass algorithmic traffic of a whole step: every input row read once,
    the n x r configuration written once, one int64 plan index per row."""
    esize = 4 if w["dtype"] == "f32" else 8
    idx = 0 if w["algo"] == "interpolate" else 8
    return float(n * (w["p"] * esize + w["r"] * 8 + idx))


# ------------------------------------------------------------------ CPU oracle sample
def oracle_kwargs(w):
    kw = dict(l=w["l"])
    if w["algo"] == "divide":
        kw["c"] = w["c"]
    if w["algo"] == "fast":
        kw["s"] = w["s"]
    return kw


def oracle_sample(w: dict, x_host: np.ndarray, budget_s: float, cores: int, tuned: bool = True):
    """Time the oracle (oracle/mds_oracle.py, the reference's numpy path) on a
    bounded prefix of the workload's rows with the same p, l, c/s, r.
    tuned: a pool of `cores` threads, BLAS 1 thread (the reference's tuned
    setting); otherwise the reference defaults (threads=None, BLAS default).
    Returns (points/s, sample description, rows)."""
    from threadpoolctl import threadpool_limits

    from oracle import mds_oracle as orc

    algo = w["algo"]
    kw = oracle_kwargs(w)
    n = x_host.shape[0]
    if algo == "fast":
        n_s = min(n, (w["l"] // w["s"]) * 400)   # one level-1 subtree: 50 leaves + alignment
    elif algo == "divide":
        n_s = min(n, max(4 * w["l"], 4 * cores * (w["l"] - w["c"])))
    else:
        n_s = min(n, max(4 * w["l"], 100_000))
    threads = cores if tuned else None

    def once(m):
        t0 = time.perf_counter()
        if tuned:
            with threadpool_limits(1):
                orc.run(algo, x_host[:m], w["r"], seed=0, threads=threads, **kw)
        else:
            orc.run(algo, x_host[:m], w["r"], seed=0, threads=threads, **kw)
        return time.perf_counter() - t0

    dt = once(n_s)
    if dt < budget_s * 0.5 and n_s < n and algo != "fast":
        n_s = int(min(n, n_s * max(1.0, budget_s / max(dt, 1e-3))))
        dt = once(n_s)
    setting = (f"{cores}-thread pool, BLAS 1 thread (tuned)" if tuned else
               "reference defaults: threads=None (pool of min(pieces, cores)), BLAS default threads")
    desc = f"oracle {algo} on the first {n_s} rows (same p,l,c/s,r; seed 0), {setting}"
    return n_s / dt, desc, n_s


# ------------------------------------------------------------------ arms
def workload_config(name, w, gpus, n, scaling):
    cfg = {"workload": f"{name}: {w['algo']} n={n} p={w['p']} {w['dtype']} l={w['l']}"
                       + (f" c={w['c']}" if w['c'] else "") + (f" s={w['s']}" if w['s'] else "")
                       + f" r={w['r']}",
           "algorithm": w["algo"], "n": n, "n_per_gpu": n // gpus if scaling == "strong" else w["n"],
           "p": w["p"], "l": w["l"], "r": w["r"], "input_dtype": w["dtype"],
           "parallelism": f"dp{gpus} ({'rows' if w['algo'] == 'interpolate' else 'partitions'} "
                          f"sharded, {scaling} scaling)",
           "l2_flush": "inputs larger than L2 (126 MB): no flush",
           "compute_precision": "fp64 throughout (fp32 inputs widened in-kernel)",
           "input": ("reference scenario stream (simulation.py:68-80), seed 0"
                     if w["data"] == "gaussian" else "config-5 image-like stand-in, seed 0")}
    if w["c"]:
        cfg["c"] = w["c"]
    if w["s"]:
        cfg["s"] = w["s"]
    return cfg


def run_reference(args, w):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    nh = min(w["n"], 200_000 if w["data"] == "image" else 300_000)
    xh = host_input(w, nh)
    rate, desc, n_s = oracle_sample(dict(w, n=nh), xh, 6.0, cores)
    from threadpoolctl import threadpool_limits

    from oracle import mds_oracle as orc
    kw = oracle_kwargs(w)
    times = []
    with threadpool_limits(1):
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            orc.run(w["algo"], xh[:n_s], w["r"], seed=0, threads=cores, **kw)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = n_s / t
    scaling = scaling_mode(args, w)
    n = w["n"] if scaling == "strong" else w["n"] * args.gpus
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, w, args.gpus, n, scaling),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def scaling_mode(args, w) -> str:
    if args.scaling != "auto":
        return args.scaling
    return "strong" if w.get("strong") else "weak"


def parity_block(name: str, w: dict, points, est, g1, g2) -> dict | None:
    """Compare this run's result with the fixture made by the reference itself."""
    import full_configs as fc
    if name == "interp1":
        from conftest import golden
        g = golden("cfg1_interp")
        P = np.asarray(points, dtype=np.float64)
        s = np.sign(np.sum(P * g["points"], axis=0))
        s[s == 0] = 1
        return {"fixture": "tests/golden/cfg1_interp.npz (reference, full size)",
                "points_rel_err": float(np.linalg.norm(P * s - g["points"]) /
                                        np.linalg.norm(g["points"])),
                "estimates_rel_err": float(np.linalg.norm(np.asarray(est) - g["estimates"]) /
                                           np.linalg.norm(g["estimates"])),
                "g1_abs_err": abs(float(g1) - float(g["g1"]))}
    if name not in fc.FULL:
        return None
    rep = fc.compare(name, points, est, g1, g2)
    rep["tolerance"] = "north star: 1e-6 relative Frobenius after sign fix, eigenvalues 1e-6"
    return rep


def distribute_rows(w, x_host, plan, n, comm, dev):
    """Rank 0 holds the global host input; every rank receives the rows of its
    share (distributed.local_rows order) over NCCL.  Returns (x_local device,
    x_local host copy, landmark rows on rank 0 for interpolation)."""
    import torch
    import torch.distributed as dist

    from paper_2007_11919_b200 import _device as D
    from paper_2007_11919_b200 import distributed as dd
    dt = torch.float32 if w["dtype"] == "f32" else torch.float64
    p = w["p"]
    rows_k = [dd.local_rows(w["algo"], plan, n, comm.world, k) for k in range(comm.world)]
    mine = None
    if comm.rank == 0:
        xg = D.from_host(np.ascontiguousarray(x_host), dev)
        for k in range(comm.world):
            part = xg.index_select(0, torch.from_numpy(rows_k[k]).to(dev))
            if k == 0:
                mine = part
            else:
                dist.send(part, dst=k)
        land = xg.index_select(0, torch.from_numpy(np.asarray(plan)).to(dev)) \
            if w["algo"] == "interpolate" else None
        del xg
    else:
        mine = torch.empty((len(rows_k[comm.rank]), p), dtype=dt, device=dev)
        dist.recv(mine, src=0)
        land = None
    torch.cuda.synchronize(dev)
    return mine, mine.cpu().numpy(), land


def run_ours(args, w):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    force = os.environ.get("MDSX_BENCH_SHARDED") == "1"   # exercise the N>1 path on one GPU
    sharded = ws > 1 or force
    if sharded:
        if "RANK" not in os.environ:          # MDSX_BENCH_SHARDED=1 without a launcher: world size 1
            import socket
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0"),
                         ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", str(port))):
                os.environ.setdefault(k, v)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2007_11919_b200 import (AlgorithmParams, InterpPlan, divide_and_conquer_mds,
                                       fast_mds, interpolation_mds)
    from paper_2007_11919_b200 import _device as D
    from paper_2007_11919_b200 import distributed as dd

    peaks = measured_peaks(dev)
    scaling = scaling_mode(args, w)
    n = w["n"] if scaling == "strong" else w["n"] * ws
    t0 = time.perf_counter()
    plan = make_plan(w, n)
    planner_ms = (time.perf_counter() - t0) * 1e3
    x_host = host_input(w, n) if rank == 0 else None
    comm = dd.Comm(device=dev) if sharded else None
    if sharded:
        x, x_local_host, land = distribute_rows(w, x_host, plan, n, comm, dev)
        run = ShardedRun(w, x, n, plan, comm, land)
    else:
        x = D.from_host(np.ascontiguousarray(x_host), dev)
        run = make_run(w, x, plan)
    h = D.handle(dev)
    log(f"[rank {rank}] n={n} local rows {x.shape[0]} {x.dtype}; planner {planner_ms:.1f} ms; "
        f"warmup {args.warmup}")
    for _ in range(args.warmup):
        run.launch()
    torch.cuda.synchronize()
    run.finish(return_device=True)          # statuses OK (raises otherwise)

    stream = torch.cuda.current_stream(dev)
    l0 = h.launches()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    smi_idx = int(vis.split(",")[local]) if vis and vis.split(",")[local].isdigit() else local
    with ClockSampler(smi_idx) as clk:
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            run.launch()
        ev1.record(stream)
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
    launches = h.launches() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    if sharded:
        tm = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms = float(tm.item())
    cfg_out = run.finish(return_device=True)
    value = n / (ms / 1e3)

    # per-kernel timing pass (not the measurement): the same steps with every
    # kernel on ONE stream (MDSX_PIPE_SERIAL), so a launch's event time is its
    # own duration, not time shared with the other pipeline stream
    os.environ["MDSX_PIPE_SERIAL"] = "1"
    h.timing_report()
    h.timing(True)
    tsteps = max(1, min(args.steps, 5))
    for _ in range(tsteps):
        run.launch()
    torch.cuda.synchronize()
    h.timing(False)
    kernels = h.timing_report(with_work=True)
    del os.environ["MDSX_PIPE_SERIAL"]
    try:       # Krylov dimension per piece (solver diagnostics in the status records)
        st = D.decode_status(run.status)
        krylov = [float(v) for v in st["value"]]
    except AttributeError:
        krylov = None

    # column compaction of wide inputs (k_compact.cu): the width the kernels ran at
    p_eff = getattr(getattr(run, "compact", None), "active", None)
    roof, per_kernel = None, {}
    total_k = sum(v[0] for v in kernels.values()) or 1.0
    dom = max(kernels, key=lambda k: kernels[k][0]) if kernels else None
    ranked = sorted(kernels, key=lambda k: -kernels[k][0])
    # The roofline block describes the largest kernel by time.  A latency-bound
    # kernel (work model with a "limiter": dependent steps, not throughput)
    # has no meaningful fraction of a throughput roofline, so unless it takes
    # more than half of the kernel time the block goes to the largest
    # throughput-bound kernel and names the latency-bound one beside it.
    works = {}
    for kname in ranked:
        works[kname] = kernel_work(w, n if not sharded else x.shape[0], plan, kname, krylov,
                                   kernels[kname][2] / tsteps, p_eff=p_eff) if not sharded else None
    modelled = [k for k in ranked if works[k]]
    headline = modelled[0] if modelled else None
    latency_top = None
    if headline and "limiter" in works[headline] and kernels[headline][0] / total_k <= 0.5:
        alt = [k for k in modelled if "limiter" not in works[k]]
        if alt:
            latency_top = headline
            headline = alt[0]
    for kname in ranked:
        ms_k, cnt, executed = kernels[kname]
        wk = works[kname]
        if not wk:
            continue
        t = ms_k / tsteps / 1e3                     # seconds per step of this kernel
        ent = {"ms_per_step": ms_k / tsteps, "launches_per_step": cnt / tsteps,
               "share_of_kernel_time": ms_k / total_k}
        if wk["bound"] == "hbm":
            ent["GB/s"] = wk["bytes"] / t / 1e9
            ent["frac_hbm"] = ent["GB/s"] / peaks["hbm_gbs"]
        if "flops" in wk:
            ent["TFLOP/s"] = wk["flops"] / t / 1e12
            ent["frac_fp64"] = ent["TFLOP/s"] / peaks["fp64_tflops"]
        per_kernel[kname] = ent
        if kname == headline:
            if wk["bound"] == "hbm":
                roof = {"kernel": kname, "bound": "hbm", "achieved": ent["GB/s"],
                        "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ent["frac_hbm"],
                        "peak_src": peaks["hbm_src"]}
            else:
                roof = {"kernel": kname, "bound": "tensor", "achieved": ent["TFLOP/s"],
                        "peak": peaks["fp64_tflops"], "unit": "TFLOP/s", "frac": ent["frac_fp64"],
                        "precision": "fp64 (DMMA / DFMA share one pipe)",
                        "peak_src": peaks["fp64_src"]}
            roof.update(traffic=None, work_model=wk["model"],
                        avg_launch_ms=ms_k / cnt, launches_per_step=cnt / tsteps,
                        share_of_kernel_time=ms_k / total_k,
                        timing="serialised pass (MDSX_PIPE_SERIAL: all chunks on one stream), "
                               "CUDA events on the launching stream")
            if "limiter" in wk:
                roof["limiter"] = wk["limiter"]
            if latency_top:
                roof["largest_by_time"] = {
                    "kernel": latency_top, "ms_per_step": kernels[latency_top][0] / tsteps,
                    "share_of_kernel_time": kernels[latency_top][0] / total_k,
                    "limiter": works[latency_top]["limiter"]}
            elif kname != dom:
                roof["note"] = f"dominant kernel {dom} has no work model; largest modelled kernel"
            if roof["frac"] < 0.02 and "limiter" not in roof:
                # a handful of CTAs (one landmark / anchor piece, a 1e4-row problem):
                # the launch is bounded by its own latency chain, not by a throughput peak
                roof["limiter"] = ("latency (few CTAs: the serial landmark / anchor setup of a small "
                                   "problem; no throughput roofline applies)")
            traffic = TRAFFIC.get((args.workload, kname))
            if traffic:
                roof["traffic"] = traffic["bytes"]          # per launch, like `achieved`
                roof["traffic_src"] = traffic["src"]
    for ent in per_kernel.values():
        for key in ("frac_hbm", "frac_fp64"):
            if ent.get(key, 0) > 1.2:
                ent["suspect"] = f"{key} above 1.2: work model overstates this kernel"
    step_roof = {"bytes_per_step": step_bytes(w, n if not sharded else x.shape[0]),
                 "model": "one read of every input row + one write of n x r + one int64 plan "
                          "index per row (D&C / fast)"}
    step_roof["achieved_GBs"] = step_roof["bytes_per_step"] / (ms / 1e3) / 1e9
    step_roof["frac_hbm"] = step_roof["achieved_GBs"] / peaks["hbm_gbs"]

    # ---- e2e through the public API (host input, numpy result)
    e2e = None
    params = AlgorithmParams(r=w["r"], l=w["l"], c=w["c"], s=w["s"], seed=0)
    parity = None
    if not args.no_e2e and not sharded:
        del run
        torch.cuda.empty_cache()
        fn = {"divide": divide_and_conquer_mds, "fast": fast_mds,
              "interpolate": interpolation_mds}[w["algo"]]
        kw = dict(plan=plan if w["algo"] != "interpolate" else InterpPlan([plan], n, w["l"], 0),
                  device=dev)
        n_idx = len(plan) if w["algo"] == "interpolate" else (
            sum(len(q) for q in plan.subsets) if w["algo"] == "divide" else 2 * n)

        def e2e_of(host_in, k):
            res = None
            for _ in range(2):    # steady state: one result alive while the next call runs
                res = fn(host_in, params, **kw)
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(k):
                res = fn(host_in, params, **kw)
            torch.cuda.synchronize()
            return (time.perf_counter() - t) / k, res

        # the contract's e2e: the public API on a page-locked host tensor (H2D of
        # the input at PCIe speed); the drop-in case, a pageable numpy array as a
        # scalemds user passes it (staged by mdsx_h2d), is reported beside it
        pinned = torch.empty(x_host.shape, dtype=torch.from_numpy(x_host[:1]).dtype, pin_memory=True)
        pinned.numpy()[...] = x_host
        k_e2e = max(1, min(args.steps, 5))
        e2e_s, res = e2e_of(pinned, k_e2e)
        del pinned
        e2e = {"value": n / e2e_s, "unit": UNIT, "ms_per_step": e2e_s * 1e3,
               "h2d_bytes_per_step": int(x_host.nbytes + 8 * n_idx),
               "d2h_bytes_per_step": int(n * w["r"] * 8), "steps": k_e2e,
               "path": f"paper_2007_11919_b200.{fn.__name__}(page-locked host tensor, plan=...) "
                       "-> numpy points"}
        e2e_np, res = e2e_of(x_host, max(1, min(args.steps, 3)))
        e2e["numpy_input"] = {"value": n / e2e_np, "ms_per_step": e2e_np * 1e3,
                              "path": f"paper_2007_11919_b200.{fn.__name__}(numpy array (pageable), "
                                      "plan=...): input staged by mdsx_h2d"}
        parity = parity_block(args.workload, w, res.points, res.eigenvalue_estimates,
                              res.gof_g1, res.gof_g2)
    elif not args.no_e2e and sharded:
        # per rank: its own rows from pageable host memory -> device, the
        # sharded step, the gather of n x r to rank 0 and its D2H
        from paper_2007_11919_b200.distributed import gather_points
        k_e2e = max(1, min(args.steps, 3))
        dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(k_e2e):
            xd = D.from_host(x_local_host, dev)
            if w["algo"] == "interpolate":
                land = D.from_host(np.ascontiguousarray(x_host[plan]), dev) if rank == 0 else None
                run2 = ShardedRun(w, xd, n, plan, comm, land)
            else:
                run2 = ShardedRun(w, xd, n, plan, comm)
            run2.launch()
            pts = gather_points(run2.res, n, comm)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t) / k_e2e
        tm = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        e2e_s = float(tm.item())
        hb = torch.tensor([x_local_host.nbytes], device=dev, dtype=torch.float64)
        dist.all_reduce(hb)
        e2e = {"value": n / e2e_s, "unit": UNIT, "ms_per_step": e2e_s * 1e3,
               "h2d_bytes_per_step": int(hb.item()), "d2h_bytes_per_step": int(n * w["r"] * 8),
               "steps": k_e2e,
               "path": "paper_2007_11919_b200.distributed (each rank H2Ds its own rows from "
                       "pageable host memory; NCCL gather of n x r to rank 0, D2H there)"}
        if rank == 0 and ws == 1:
            parity = parity_block(args.workload, w, pts, run2.res.estimates,
                                  run2.res.gof_g1, run2.res.gof_g2)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        nh = min(n, 300_000)
        xs = x_host[:nh]
        rate, desc, _ = oracle_sample(dict(w, n=nh), xs, 8.0, cores, tuned=True)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc,
               "cpu_model": cpu_model()}
        if not args.no_cpu_default:
            rate_d, desc_d, _ = oracle_sample(dict(w, n=nh), xs, 8.0, cores, tuned=False)
            cpu["reference_defaults"] = {"value": rate_d, "unit": UNIT, "sample": desc_d}

    companions = None
    if rank == 0 and ws == 1 and not sharded and args.workload == "dc2" and not args.no_companions:
        # the metric names three algorithms: the default line also carries the
        # config-3 (fast) and config-4 (interpolation) runs, each its own process
        torch.cuda.empty_cache()
        companions = {wl: companion_line(wl, args) for wl in ("fast3", "interp4")}

    if rank == 0:
        config = workload_config(args.workload, w, ws, n, scaling)
        if p_eff is not None:
            config["active_columns"] = int(p_eff)
            config["column_compaction"] = ("all-zero columns dropped inside every step "
                                           "(k_compact.cu: one detection pass + one gather)"
                                           if p_eff < 0.9 * w["p"] else "none (too few zero columns)")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config,
            "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e,
            "parity": parity, "clocks": clk.summary(), "gpu_launches": launches,
            "planner_ms": planner_ms,
            "host": {"cpu_model": cpu_model(), "cores": os.cpu_count()},
            "kernel_rooflines": per_kernel,
            "kernels_ms_per_step_serialised": {k: v[0] / tsteps for k, v in sorted(kernels.items())},
            "peaks": peaks,
            "companions": companions,
            "fit": {"g1": cfg_out.gof_g1,
                    "estimates": [float(v) for v in cfg_out.eigenvalue_estimates]},
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()
    return 0


def companion_line(wl: str, args) -> dict:
    """One more workload in its own process (same timing rules, no CPU leg),
    condensed for the ``companions`` block of the default line."""
    cmd = [sys.executable, str(Path(__file__).resolve()), "--workload", wl, "--steps",
           str(max(1, min(args.steps, 5))), "--warmup", str(args.warmup), "--no-cpu",
           "--no-companions"]
    if args.no_e2e:
        cmd.append("--no-e2e")
    t0 = time.perf_counter()
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=400)
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:      # noqa: BLE001 - reported in the line, the headline stands
        return {"error": f"{type(e).__name__}: {e}"[:300]}
    keep = ("value", "unit", "ms_per_step", "steps", "warmup", "scaling", "roofline",
            "step_roofline", "e2e", "parity", "clocks", "gpu_launches", "planner_ms")
    res = {k: d.get(k) for k in keep}
    res["workload"] = d["config"]["workload"]
    res["wall_s"] = time.perf_counter() - t0
    return res


def check_launch(args):
    """--check-launch: the self-launch plumbing only (rendezvous + one
    collective); gloo on CPU, NCCL when every rank has a GPU."""
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    use_nccl = torch.cuda.is_available() and torch.cuda.device_count() >= ws
    dist.init_process_group("nccl" if use_nccl else "gloo")
    dev = torch.device("cuda", local) if use_nccl else torch.device("cpu")
    t = torch.tensor([rank], dtype=torch.int64, device=dev)
    out = [torch.empty_like(t) for _ in range(ws)]
    dist.all_gather(out, t)
    if rank == 0:
        print(json.dumps({"check": "launch", "n_gpus": ws, "ranks_seen": [int(v) for v in out],
                          "backend": dist.get_backend()}), flush=True)
    dist.destroy_process_group()
    return 0


def self_launch(args) -> int:
    """--gpus N > 1 without torchrun: start N ranks with torch's launcher."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    log(f"self-launch: {' '.join(cmd)}")
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="dc2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu-default", action="store_true",
                    help="skip the reference-defaults CPU sample (oversubscribed BLAS)")
    ap.add_argument("--check-launch", action="store_true")
    ap.add_argument("--no-companions", action="store_true",
                    help="default workload only: skip the fast3 / interp4 companion runs")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    w = WORKLOADS[args.workload]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not (
            args.impl == "reference"):
        return self_launch(args)
    if args.check_launch:
        return check_launch(args)
    if args.impl == "reference":
        return run_reference(args, w)
    return run_ours(args, w)


if __name__ == "__main__":
    sys.exit(main())
