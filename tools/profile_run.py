"""Run one workload step (after one warm-up) for ncu captures:
    python tools/profile_run.py dc2 [n]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench
from paper_2007_11919_b200 import _device as D

name = sys.argv[1] if len(sys.argv) > 1 else "dc2"
w = dict(bench.WORKLOADS[name])
n = int(sys.argv[2]) if len(sys.argv) > 2 else w["n"]
dev = torch.device("cuda", 0)
x = D.from_host(np.ascontiguousarray(bench.host_input(w, n)), dev)
plan = bench.make_plan(w, n)
run = bench.make_run(w, x, plan)
for _ in range(2):
    run.launch()
torch.cuda.synchronize()
cfg = run.finish(return_device=True)
print("ok", name, n, cfg.gof_g1)
