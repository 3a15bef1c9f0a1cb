"""Histogram of the Lanczos Krylov dimension per piece (status value) for a workload."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench
from paper_2007_11919_b200 import _device as D

for name in sys.argv[1:] or ["dc2"]:
    w = dict(bench.WORKLOADS[name])
    dev = torch.device("cuda", 0)
    x = bench.make_data(w, dev, 0)
    plan = bench.make_plan(w, 0)
    run = bench.make_run(w, x, plan)
    run.launch()
    torch.cuda.synchronize()
    st = D.decode_status(run.status)
    v = st["value"]
    print(name, "pieces", len(v), "codes", np.unique(st["code"], return_counts=True))
    u, c = np.unique(v, return_counts=True)
    print("  krylov dims:", dict(zip(u.tolist(), c.tolist())))
