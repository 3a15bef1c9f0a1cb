"""Per-launch timeline of one pipelined step (CUDA events around every launch,
both pipeline streams): start/end per kernel relative to the step's first
launch, and the union of busy time.
    python tools/timeline.py dc2 [n]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench
from paper_2007_11919_b200 import _device as D

name = sys.argv[1] if len(sys.argv) > 1 else "dc2"
w = dict(bench.WORKLOADS[name])
if len(sys.argv) > 2:
    w["n"] = int(sys.argv[2])
dev = torch.device("cuda", 0)
x = D.from_host(np.ascontiguousarray(bench.host_input(w, w["n"])), dev)
plan = bench.make_plan(w, w["n"])
run = bench.make_run(w, x, plan)
h = D.handle(dev)
for _ in range(3):
    run.launch()
torch.cuda.synchronize()
h.timing_report()
h.timing(True)
run.launch()
torch.cuda.synchronize()
h.timing(False)
tr = h.timing_trace()
h.timing_report()
end = max(b for _, _, b in tr)
print(f"{name}: {len(tr)} launches, step span {end:.3f} ms (with per-launch event overhead)")
for k, a, b in sorted(tr, key=lambda t: t[1]):
    bar = " " * int(60 * a / end) + "#" * max(1, int(60 * (b - a) / end))
    print(f"{a:7.3f} {b:7.3f} {b - a:6.3f}  {k[:28]:28s} |{bar}")
