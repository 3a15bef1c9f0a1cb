"""Kernel breakdown of one step, unsharded vs the sharded path at world size 1
(torch.profiler over CUDA activity, so torch ops and NCCL show up beside the
mdsx kernels).  GPU box:
    python tools/shard_profile.py dc2 fast3 interp4"""
import os
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import torch.distributed as dist
from torch.profiler import ProfilerActivity, profile

import bench
from paper_2007_11919_b200 import _device as D
from paper_2007_11919_b200 import distributed as dd

STEPS = 3


def table(run, label):
    for _ in range(3):
        run.launch()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(10):
        run.launch()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 10
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(STEPS):
            run.launch()
        torch.cuda.synchronize()
    tot, cnt = defaultdict(float), defaultdict(int)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name[:60]
            tot[k] += e.device_time / 1e3 / STEPS
            cnt[k] += 1
    print(f"== {label}: {ms:.3f} ms/step (events); kernel sum {sum(tot.values()):.3f} ms")
    for k in sorted(tot, key=lambda k: -tot[k])[:25]:
        print(f"   {tot[k]:8.4f} ms  x{cnt[k] / STEPS:5.1f}  {k}")


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    comm = dd.Comm(device=dev)
    for name in sys.argv[1:] or ["dc2"]:
        w = dict(bench.WORKLOADS[name])
        n = w["n"]
        plan = bench.make_plan(w, n)
        xh = bench.host_input(w, n)
        x = D.from_host(np.ascontiguousarray(xh), dev)
        table(bench.make_run(w, x, plan), f"{name} unsharded")
        del x
        xl, _, land = bench.distribute_rows(w, xh, plan, n, comm, dev)
        table(bench.ShardedRun(w, xl, n, plan, comm, land), f"{name} sharded (world 1)")
        del xl, land
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
