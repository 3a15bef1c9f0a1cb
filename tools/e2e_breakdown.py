"""Where does the end-to-end D&C call spend its time? (config 2)"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2007_11919_b200 as mds
from paper_2007_11919_b200 import plans
from paper_2007_11919_b200.algorithms import DivideRun

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(0)
x = torch.randn(1_000_000, 100, generator=g, dtype=torch.float64, device=dev)
x[:, :10] *= 15.0 ** 0.5          # BASELINE config 2 distribution
host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True); host.copy_(x)
plan = plans.plan_divide_conquer(1_000_000, 1000, 20, 0)
prm = mds.AlgorithmParams(r=10, l=1000, c=20, seed=0)
for _ in range(2):
    mds.divide_and_conquer_mds(host, prm, plan=plan, device=dev)
torch.cuda.synchronize()
def t(f, k=3):
    torch.cuda.synchronize(); s = time.perf_counter()
    for _ in range(k): r = f()
    torch.cuda.synchronize(); return (time.perf_counter() - s) / k * 1e3, r
print("full e2e ms", t(lambda: mds.divide_and_conquer_mds(host, prm, plan=plan, device=dev))[0])
print("H2D 800MB ms", t(lambda: host.to(dev, non_blocking=True))[0])
xd = host.to(dev)
print("flatten ms", t(lambda: plans.flatten_subsets(plan.subsets))[0])
ms, run = t(lambda: DivideRun(xd, plan, 10, 20))
print("DivideRun init ms", ms)
print("launch ms (wall)", t(lambda: run.launch())[0])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record(); run.launch(); e1.record(); torch.cuda.synchronize()
print("launch ms (events)", e0.elapsed_time(e1))
s0 = time.perf_counter(); run.launch(); s1 = time.perf_counter(); torch.cuda.synchronize(); s2 = time.perf_counter()
print("launch host-enqueue ms", (s1 - s0) * 1e3, "then drain ms", (s2 - s1) * 1e3)
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.draw,pcie.link.gen.current,pcie.link.width.current", "--format=csv"], capture_output=True, text=True).stdout)
print("finish(host) ms", t(lambda: run.finish(False))[0])
print("finish(device) ms", t(lambda: run.finish(True))[0])
out = run.out
print("D2H 80MB pageable ms", t(lambda: out.cpu())[0])
pin = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
print("D2H 80MB pinned ms", t(lambda: pin.copy_(out, non_blocking=True))[0])
