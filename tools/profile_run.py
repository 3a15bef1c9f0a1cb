"""Run one workload step (after one warm-up) for ncu captures:
    python tools/profile_run.py dc2 [n]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench

name = sys.argv[1] if len(sys.argv) > 1 else "dc2"
w = dict(bench.WORKLOADS[name])
if len(sys.argv) > 2:
    w["n"] = int(sys.argv[2])
dev = torch.device("cuda", 0)
x = bench.make_data(w, dev, 0)
plan = bench.make_plan(w, 0)
run = bench.make_run(w, x, plan)
for _ in range(2):
    run.launch()
torch.cuda.synchronize()
cfg = run.finish(return_device=True)
print("ok", name, w["n"], cfg.gof_g1)
