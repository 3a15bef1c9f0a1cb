"""Where does the end-to-end D&C call spend its time? (config 2)

    python tools/e2e_breakdown.py
Times each stage of divide_and_conquer_mds(pinned host array) with a device
synchronize between stages (so the stages do not overlap as they would in the
real call; the sum is an upper bound)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2007_11919_b200 as mds
from paper_2007_11919_b200 import _device as D
from paper_2007_11919_b200 import plans
from paper_2007_11919_b200.algorithms import DivideRun

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
x = torch.randn(1_000_000, 100, generator=g, dtype=torch.float64, device=dev)
x[:, :10] *= 15.0 ** 0.5          # BASELINE config 2 distribution
host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
host.copy_(x)
plan = plans.plan_divide_conquer(1_000_000, 1000, 20, 0)
prm = mds.AlgorithmParams(r=10, l=1000, c=20, seed=0)
for _ in range(3):
    mds.divide_and_conquer_mds(host, prm, plan=plan, device=dev)
torch.cuda.synchronize()


def t(f, k=5):
    torch.cuda.synchronize()
    s = time.perf_counter()
    for _ in range(k):
        r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - s) / k * 1e3, r


print("full e2e ms %.2f" % t(lambda: mds.divide_and_conquer_mds(host, prm, plan=plan, device=dev))[0])
print("to_device_matrix (800 MB H2D) ms %.2f" % t(lambda: D.to_device_matrix(host, dev))[0])
xd = D.to_device_matrix(host, dev)
print("flatten_subsets ms %.2f" % t(lambda: plans.flatten_subsets(plan.subsets))[0])
rows, off = plans.flatten_subsets(plan.subsets)
print("index_tensor (%d MB) ms %.2f" % (rows.nbytes >> 20, t(lambda: D.index_tensor(rows, dev))[0]))
ms, run = t(lambda: DivideRun(xd, plan, 10, 20))
print("DivideRun init ms %.2f" % ms)
print("launch+sync ms %.2f" % t(lambda: run.launch())[0])
print("decode_status ms %.2f" % t(lambda: D.decode_status(run.status))[0])
print("finish(device) ms %.2f" % t(lambda: run.finish(True))[0])
print("finish(host) ms %.2f" % t(lambda: run.finish(False))[0])
print("to_host 80 MB ms %.2f" % t(lambda: D.to_host(run.out))[0])

if "--profile" in sys.argv:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        mds.divide_and_conquer_mds(host, prm, plan=plan, device=dev)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
