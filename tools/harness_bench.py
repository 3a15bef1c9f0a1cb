"""Harness metrics on the GPU box: device
aligned_correlations (n = 1e6, r = 10, device-resident inputs) vs the
reference's NumPy path, and gof_sweep (one solve at h_cap) vs the per-h loop."""
import dataclasses
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2007_11919_b200 as m

spec = m.ScenarioSpec(n=1_000_000, k=100, h=10, seed=0)
data = m.generate_scenario(spec, 0)
x = torch.from_numpy(data).cuda()
cfg = m.divide_and_conquer_mds(x, m.AlgorithmParams(r=10, l=1000, c=20), return_device=True)
for _ in range(3):
    m.aligned_correlations(cfg, x[:, :10])
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    c = m.aligned_correlations(cfg, x[:, :10])
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"device aligned_correlations n=1e6 r=10: {(t1 - t0) / 20 * 1e3:.3f} ms per call "
      f"(incl. the r-vector readback)")
pts = cfg.points.cpu().numpy()
dom = data[:, :10]
t0 = time.perf_counter()
tc = dom - dom.mean(axis=0)
sc = pts - pts.mean(axis=0)
u, _, vt = np.linalg.svd(tc.T @ sc)
rot = vt.T @ u.T
tr = (dom - pts @ rot).mean(axis=0)
res = dom - pts @ rot - tr
loss = float(np.sum(res * res))
al = pts @ rot + tr
a = al - al.mean(axis=0)
ref = np.einsum("ij,ij->j", a, tc) / (np.sqrt(np.einsum("ij,ij->j", a, a)) *
                                      np.sqrt(np.einsum("ij,ij->j", tc, tc)))
t1 = time.perf_counter()
print(f"reference numpy path (fit + apply + correlations): {(t1 - t0) * 1e3:.1f} ms; "
      f"max |diff| {np.abs(ref - c).max():.2e}")

small = m.generate_scenario(m.ScenarioSpec(n=200_000, k=30, h=6, seed=1), 0)
xs = torch.from_numpy(small).cuda()
prm = m.AlgorithmParams(r=1, l=1000, c=30)
m.gof_sweep(xs, "divide", prm, 0.9)
torch.cuda.synchronize()
t0 = time.perf_counter()
h1 = m.gof_sweep(xs, "divide", prm, 0.999)
torch.cuda.synchronize()
t1 = time.perf_counter()
h2 = None
for h in range(1, 31):
    if m.run_algorithm("divide", xs, dataclasses.replace(prm, r=h)).gof_g1 >= 0.999:
        h2 = h
        break
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"gof_sweep divide n=2e5 k=30 target 0.999: one solve {(t1 - t0) * 1e3:.1f} ms -> h={h1}; "
      f"per-h loop {(t2 - t1) * 1e3:.1f} ms -> h={h2}")
