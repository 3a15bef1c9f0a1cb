"""The sharded divide-and-conquer path on the GPU backend at world size 1
(NCCL, one B200): mdsx_divide_conquer_sharded gathers the subsets'
contributions through its host callback and re-centres inside the call, so
the rank's configuration must equal the unsharded call bitwise.  (The N > 1
logic runs in tests/test_distributed.py on gloo; one GPU cannot host two NCCL
ranks.)"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1(cuda):
    import torch
    import torch.distributed as dist
    created = False
    if not dist.is_initialized():
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                world_size=1, device_id=torch.device("cuda", 0))
        created = True
    yield
    if created:
        dist.destroy_process_group()


def test_sharded_divide_equals_unsharded(nccl1):
    import torch
    import paper_2007_11919_b200 as mds
    from paper_2007_11919_b200 import distributed as dd
    from paper_2007_11919_b200.synthetic import scenario
    x = scenario(120_000, 20, 4, seed=9)
    prm = mds.AlgorithmParams(r=4, l=500, c=10, seed=2)
    plan = mds.plan_divide_conquer(x.shape[0], prm.l, prm.c, prm.seed)
    dev = torch.device("cuda", 0)
    comm = dd.Comm(device=dev)
    sh = dd.dc_shard(plan, comm.world, comm.rank)
    xl = torch.from_numpy(np.ascontiguousarray(x[sh.local_rows])).to(dev)
    res = dd.sharded_divide_and_conquer(dd.GpuBackend(dev), xl, x.shape[0], prm, comm, plan=plan)
    got = np.empty((x.shape[0], prm.r))
    got[sh.local_rows[res.report_lo:]] = res.out[res.report_lo:].cpu().numpy()
    ref = mds.divide_and_conquer_mds(x, prm, plan=plan)
    assert np.array_equal(got, ref.points)
    assert np.array_equal(res.estimates, ref.eigenvalue_estimates)
    assert res.gof_g1 == ref.gof_g1


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_sharded_interpolation_equals_unsharded(nccl1, dtype):
    """The tile route (per-tile Gower sums, per-landmark corrections, one fold)
    at world size 1 against the single call (per-CTA column sums): the same
    points up to the summation order of the column mean."""
    import torch
    import paper_2007_11919_b200 as mds
    from paper_2007_11919_b200 import distributed as dd
    from paper_2007_11919_b200.synthetic import scenario
    n = 300_000
    x = scenario(n, 24, 4, seed=5).astype(dtype)
    prm = mds.AlgorithmParams(r=5, l=700, seed=3)
    sample = mds.plans.interpolation_sample(n, prm.l, prm.seed)
    dev = torch.device("cuda", 0)
    comm = dd.Comm(device=dev)
    be = dd.GpuBackend(dev)
    xd = torch.from_numpy(x).to(dev)
    sh = dd.interp_shard(n, sample, comm.world, comm.rank)
    assert be.tile_rows(xd, prm.r) > 0
    run = dd.ShardedInterpolation(be, xd[sh.lo:sh.hi], n, sample, prm.r, comm,
                                  x_landmarks=xd.index_select(0, torch.from_numpy(sample).to(dev)))
    assert run.tr > 0
    res = run.launch().finish()
    ref = mds.interpolation_mds(x, prm)
    got = res.out.cpu().numpy()
    assert np.abs(got - ref.points).max() <= 1e-13 * np.abs(ref.points).max()
    assert np.array_equal(res.estimates, ref.eigenvalue_estimates)
    # the re-centring is the only difference: centred columns
    assert np.abs(got.mean(axis=0)).max() < 1e-12 * np.abs(got).max()


def test_sharded_fast_equals_unsharded(nccl1):
    """mdsx_fast_mds_sharded at world size 1: the leaf contributions gathered
    through the callback give the single call's mean -> bitwise equal."""
    import torch
    import paper_2007_11919_b200 as mds
    from paper_2007_11919_b200 import distributed as dd
    from paper_2007_11919_b200.synthetic import scenario
    x = scenario(150_000, 20, 4, seed=4)
    prm = mds.AlgorithmParams(r=4, l=600, s=8, seed=3)
    plan = mds.plans.plan_fast(x.shape[0], prm.l, prm.s, prm.seed)
    dev = torch.device("cuda", 0)
    comm = dd.Comm(device=dev)
    sh = dd.fast_shard(plan, comm.world, comm.rank)
    xl = torch.from_numpy(np.ascontiguousarray(x[sh.local_rows])).to(dev)
    run = dd.ShardedFast(dd.GpuBackend(dev), xl, plan, prm.r, comm)
    res = run.launch().finish()
    got = np.empty((x.shape[0], prm.r))
    got[sh.local_rows[:sh.n_own]] = res.out.cpu().numpy()
    ref = mds.fast_mds(x, prm, plan=plan)
    assert np.array_equal(got, ref.points)
    assert np.array_equal(res.estimates, ref.eigenvalue_estimates)
    assert res.gof_g1 == ref.gof_g1
