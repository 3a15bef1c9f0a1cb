"""Multi-rank path on CPU: torch.distributed with gloo, world size 1 and 2.

The sharding, collectives (all-gather, broadcast) and plan-order aggregation
of paper_2007_11919_b200.distributed run unchanged; the per-rank compute is an
oracle-backed backend (test infrastructure) in place of the GPU backend.
Checks: the sharded result equals the single-process reference algorithm, and
world size 1 and 2 give bitwise identical configurations."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mds_oracle as orc
from paper_2007_11919_b200 import AlgorithmParams
from paper_2007_11919_b200 import distributed as dd
from paper_2007_11919_b200.synthetic import scenario

STATUS = np.dtype([("code", np.int32), ("index", np.int32), ("value", np.float64)])


class OracleBackend:
    """Per-rank compute by the CPU oracle (same contract as GpuBackend)."""

    def __init__(self, x):
        self.x = np.asarray(x, dtype=np.float64)

    def own_segment_sums(self, out, r):
        return self.segment_sums(out, self._own, r)

    def shift_own(self, out, mean):
        self.shift(out, np.concatenate(self._own), mean)

    def range_sums(self, out, offsets, r):
        return np.stack([out[offsets[j]:offsets[j + 1]].sum(axis=0) for j in range(len(offsets) - 1)]) \
            if len(offsets) > 1 else np.zeros((0, r))

    def shift_all(self, out, mean):
        out -= mean

    def dc_subplan(self, subsets, c, r, key=None):
        self._own = [subsets[0]] + [s[c:] for s in subsets[1:]]
        embs = [orc.mds_from_data(self.x[s], r) for s in subsets]
        out = np.zeros((self.x.shape[0], r))
        out[subsets[0]] = embs[0].points
        anchor = embs[0].points[:c]
        for s, e in zip(subsets[1:], embs[1:]):
            out[s[c:]] = orc.procrustes_apply(e.points[c:], orc.procrustes_fit(anchor, e.points[:c]))
        est = np.stack([e.estimates for e in embs])
        gof = np.array([[e.g1, e.g2] for e in embs])
        return out, est, gof, np.zeros(len(subsets), dtype=STATUS)

    def fast_subtrees(self, plan, lo, hi, r, key=None):
        from paper_2007_11919_b200.plans import flatten_fast_shard
        flat = flatten_fast_shard(plan, lo, hi)
        off = flat.piece_off
        npc = len(off) - 1
        pts = np.zeros((int(off[-1]), r))
        est = np.zeros((npc, r))
        gof = np.zeros((npc, 2))
        for j in range(npc):
            e = orc.mds_from_data(self.x[flat.piece_rows[off[j]:off[j + 1]]], r)
            pts[off[j]:off[j + 1]] = e.points
            est[j] = e.estimates
            gof[j] = [e.g1, e.g2]
        for lv in flat.levels:
            for t in range(len(lv.start)):
                a, b = lv.job_off[t], lv.job_off[t + 1]
                T = orc.procrustes_fit(pts[lv.tgt_rows[a:b]], pts[lv.src_rows[a:b]])
                s0, ln = lv.start[t], lv.length[t]
                pts[s0:s0 + ln] = orc.procrustes_apply(pts[s0:s0 + ln], T)
        out = pts[:len(flat.order)]
        return out, flat, est, gof, np.zeros(npc, dtype=STATUS)

    def segment_sums(self, out, segments, r):
        return np.stack([out[s].sum(axis=0) for s in segments])

    def shift(self, out, rows, mean):
        out[rows] -= mean

    def take(self, out, rows):
        return out[rows].copy()

    def take_all(self, out):
        return np.array(out, copy=True)

    def place(self, out, local, values):
        out[local] = values

    def context_len(self, l, r):
        return l + r * r + l * self.x.shape[1] + l * r + l * r

    def landmark_context(self, sample, r):
        base = orc.mds_from_data(self.x[sample], r)
        ctx = orc.gower_ctx(self.x[sample], base.points)
        packed = np.concatenate([ctx.q_diag, ctx.covariance.ravel(), ctx.base_rows.ravel(),
                                 ctx.base_config.ravel(), base.points.ravel()])
        return packed, base.estimates, base.g1, base.g2

    def gower_rows(self, packed, l, r, lo, hi):
        p = self.x.shape[1]
        o = 0
        q = packed[o:o + l]; o += l
        cov = packed[o:o + r * r].reshape(r, r); o += r * r
        rows = packed[o:o + l * p].reshape(l, p); o += l * p
        cfg = packed[o:o + l * r].reshape(l, r)
        ctx = orc.GowerCtx(cfg, q, cov, rows)
        return orc.gower_project(ctx, self.x[lo:hi])


def _worker(rank, world, port, algo, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = scenario(2600, 8, 4, seed=9)
        comm = dd.Comm()
        be = OracleBackend(x)
        if algo == "divide":
            prm = AlgorithmParams(r=4, l=300, c=10, seed=2)
            res = dd.sharded_divide_and_conquer(be, x.shape[0], prm, comm)
        elif algo == "fast":
            prm = AlgorithmParams(r=4, l=300, s=8, seed=2)
            res = dd.sharded_fast(be, x.shape[0], prm, comm)
        else:
            prm = AlgorithmParams(r=4, l=400, seed=2)
            dd.SUM_BLOCK = 256                     # several blocks per rank at test size
            res = dd.sharded_interpolation(be, x.shape[0], prm, comm)
        full = dd.gather_points(res, x.shape[0], 4, comm)
        if rank == 0:
            np.savez(path, points=full, est=res.estimates, g=np.array([res.gof_g1, res.gof_g2]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, algo):
    path = tempfile.mktemp(suffix=".npz")
    mp.spawn(_worker, args=(world, _free_port(), algo, path), nprocs=world, join=True)
    with np.load(path) as z:
        out = {k: z[k] for k in z.files}
    os.unlink(path)
    return out


@pytest.mark.parametrize("algo", ["divide", "interpolate", "fast"])
def test_sharded_matches_reference_and_is_world_size_independent(algo):
    x = scenario(2600, 8, 4, seed=9)
    if algo == "divide":
        ref = orc.divide_conquer(x, 4, l=300, c=10, seed=2, threads=1)
    elif algo == "fast":
        ref = orc.run("fast", x, 4, l=300, s=8, seed=2, threads=1)
    else:
        ref = orc.interpolation(x, 4, l=400, seed=2, threads=1)
    one = _run(1, algo)
    two = _run(2, algo)
    assert np.array_equal(one["points"], two["points"])          # bitwise across world sizes
    assert np.array_equal(one["g"], two["g"]) and np.array_equal(one["est"], two["est"])
    err = np.linalg.norm(two["points"] - ref.points) / np.linalg.norm(ref.points)
    assert err <= 1e-12, err
    assert np.allclose(two["est"], ref.estimates, rtol=1e-13)
    assert abs(two["g"][0] - ref.g1) <= 1e-14 and abs(two["g"][1] - ref.g2) <= 1e-14


def test_shard_partition():
    for count in (0, 1, 7, 1020):
        for world in (1, 2, 3, 8):
            spans = [dd.shard(count, world, k) for k in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
