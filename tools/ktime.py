"""Per-kernel times (serialised pass, CUDA events per launch) of one workload,
without result checks -- for A/B experiments with run-time switches:
    MDSX_X=1 python tools/ktime.py dc2 [steps] [n]"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench
from paper_2007_11919_b200 import _device as D

name = sys.argv[1] if len(sys.argv) > 1 else "dc2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = dict(bench.WORKLOADS[name])
if len(sys.argv) > 3:
    w["n"] = int(sys.argv[3])
dev = torch.device("cuda", 0)
x = D.from_host(np.ascontiguousarray(bench.host_input(w, w["n"])), dev)
plan = bench.make_plan(w, w["n"])
run = bench.make_run(w, x, plan)
h = D.handle(dev)
for _ in range(3):
    run.launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    run.launch()
e1.record()
torch.cuda.synchronize()
step = e0.elapsed_time(e1) / steps
os.environ["MDSX_PIPE_SERIAL"] = "1"
h.timing_report()
h.timing(True)
for _ in range(steps):
    run.launch()
torch.cuda.synchronize()
h.timing(False)
k = h.timing_report()
tot = sum(v[0] for v in k.values()) / steps
print(f"{name} step {step:.3f} ms  serial sum {tot:.3f} ms  " + "  ".join(
    f"{n.replace('_kernel', '')}={v[0] / steps:.3f}" for n, v in sorted(k.items(), key=lambda t: -t[1][0])
    if v[0] / steps > 0.01))
