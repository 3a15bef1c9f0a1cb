"""A/B of the Gower stream with and without the per-tile column sums
(mdsx_gower_tiles vs mdsx_gower_interpolate) on config 4's shape.  GPU box:
    python tools/gower_tiles_ab.py [n] [p] [f32|f64]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2007_11919_b200 import _device as D
from paper_2007_11919_b200 import distributed as dd

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 100
dt = torch.float32 if (sys.argv[3] if len(sys.argv) > 3 else "f32") == "f32" else torch.float64
r, l = 10, 2000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
x = torch.rand((n, p), generator=g, device=dev, dtype=torch.float32).to(dt)
be = dd.GpuBackend(dev)
head = torch.zeros(be.head_len(l, p, r), dtype=torch.float64, device=dev)
idx = torch.randperm(n, device=dev)[:l].sort().values
be.landmark_head(x.index_select(0, idx), r, head)
out = torch.empty((n, r), dtype=torch.float64, device=dev)
tr = be.tile_rows(x, r)
tsum = torch.empty(((n + tr - 1) // tr, r), dtype=torch.float64, device=dev)
print(f"n={n} p={p} {dt} tile_rows={tr}")


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for rep in range(2):
    a = timeit(lambda: be.gower_rows(head, l, r, x, out))
    b = timeit(lambda: be.gower_tiles(head, l, r, x, out, tsum))
    print(f"plain {a:.4f} ms   tiles {b:.4f} ms   ({(b / a - 1) * 100:+.1f}%)")
