"""Roofline of the dense seams (K1 distance matrix, K2 double centering):

    python tools/dense_bench.py [m] [p]        -> one JSON line

m x m squared distances of the first m rows of the config-2 scenario stream
(fp64 and its float32 cast), the cross distances of two m/2 halves and the
double centering of the m x m result, each timed with CUDA events on the
launching stream (5 runs after 2 warm-ups, best and mean).  The matrices are
larger than L2.  Work models: K1 self = m^2 p flops (the lower triangle of
2 m^2 p) against the fp64 tensor peak (cuBLAS DGEMM measured in this run) and
m^2 * 8 bytes written against HBM; K1 cross = 2 ma mb p; K2 = one read of the
matrix for the row means + one read + one write for the centring (3 m^2 * 8
bytes).  MDSX_SQDIST_SYNC=1 / MDSX_DCENTER_FLAT=1 select the previous
(unpipelined / untiled) kernels for the A/B columns.
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2007_11919_b200 import _device as D
from paper_2007_11919_b200.synthetic import scenario


def sqdist_self(x, out):
    n, p = x.shape
    D.handle(x.device).call("mdsx_sqdist_self", x.data_ptr(), D.dtype_code(x), p, n, p,
                            out.data_ptr(), n, D.stream_ptr(x.device))
    return out


def sqdist_cross(a, b, out):
    D.handle(a.device).call("mdsx_sqdist_cross", a.data_ptr(), a.shape[1], a.shape[0], b.data_ptr(),
                            b.shape[1], b.shape[0], D.dtype_code(a), a.shape[1], out.data_ptr(),
                            b.shape[0], D.stream_ptr(a.device))
    return out


def double_center(d, q):
    D.handle(d.device).call("mdsx_double_center", d.data_ptr(), d.shape[0], q.data_ptr(),
                            D.stream_ptr(d.device))
    return q


def timed(fn, runs=5, warm=2):
    for _ in range(warm):
        out = fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(runs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), sum(ts) / len(ts), out


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    dev = torch.device("cuda", 0)
    peaks = bench.measured_peaks(dev)
    x64 = torch.from_numpy(scenario(m, p, 10, seed=0)).to(dev)
    x32 = x64.float()
    res = {"m": m, "p": p, "peaks": peaks, "kernels": {}}
    h = m // 2
    xa, xb = x64[:h].contiguous(), x64[h:].contiguous()
    bufs = {t: (D.empty((m, m), dev), D.empty((m, m), dev), D.empty((h, m - h), dev)) for t in ("", "_previous")}

    def entry(name, ms, flops=None, nbytes=None, note=None):
        e = {"ms_best": ms[0], "ms_mean": ms[1]}
        if flops:
            e["TFLOP/s"] = flops / ms[0] / 1e9
            e["frac_fp64"] = e["TFLOP/s"] / peaks["fp64_tflops"]
        if nbytes:
            e["GB/s"] = nbytes / ms[0] / 1e6
            e["frac_hbm"] = e["GB/s"] / peaks["hbm_gbs"]
        if note:
            e["model"] = note
        res["kernels"][name] = e

    for tag, env in (("", {}), ("_previous", {"MDSX_SQDIST_SYNC": "1", "MDSX_DCENTER_FLAT": "1"})):
        for k, v in env.items():
            os.environ[k] = v
        for nm, x in (("f64", x64), ("f32", x32)):
            b, a, d = timed(lambda: sqdist_self(x, bufs[tag][0]))
            entry(f"sqdist_self_{nm}{tag}", (b, a), flops=float(m) * m * p, nbytes=float(m) * m * 8,
                  note="m^2 p flops (lower triangle), m^2*8 bytes written")
        b, a, d = timed(lambda: sqdist_self(x64, bufs[tag][0]))      # fp64 result for the centring
        b, a, c = timed(lambda: sqdist_cross(xa, xb, bufs[tag][2]))
        entry(f"sqdist_cross_f64{tag}", (b, a), flops=2.0 * h * h * p, nbytes=float(h) * h * 8,
              note="2 ma mb p flops, ma*mb*8 bytes written")
        b, a, q = timed(lambda: double_center(d, bufs[tag][1]))
        entry(f"double_center{tag}", (b, a), nbytes=3.0 * m * m * 8,
              note="row means (one read) + centring (one read, one write): 3 m^2 * 8 bytes")
        if not tag:
            d_new, q_new = d, q
            res["cross_vs_self_block"] = float((c - d[:h, h:]).abs().max())
        else:
            res["previous_vs_new"] = {
                "sqdist_max_abs_diff": float((d - d_new).abs().max()),
                "dcenter_max_abs_diff": float((q - q_new).abs().max())}
        for k in env:
            del os.environ[k]
    # parity of the new kernels against numpy on a corner
    xs = x64[:512].cpu().numpy()
    ref = ((xs[:, None, :] - xs[None, :, :]) ** 2).sum(-1)
    res["sqdist_vs_numpy_512"] = float(np.abs(d_new[:512, :512].cpu().numpy() - ref).max())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
