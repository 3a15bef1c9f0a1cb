"""Multi-rank path on CPU: torch.distributed with gloo, world sizes 1, 2 and 3.

The sharding, collectives (all-gather of record tensors, broadcast of the
landmark head, gather of the result) and the plan-order aggregation of
paper_2007_11919_b200.distributed run unchanged; each rank holds only its own
input rows (``distributed.local_rows``), and the per-rank compute is an
oracle-backed backend (test infrastructure) in place of the GPU backend.
Checks: the sharded result equals the single-process reference algorithm,
every world size gives bitwise identical configurations, and a failing piece
or a non-finite row on a rank other than 0 makes EVERY rank raise the same
exception (no rank is left waiting in a collective)."""

import os
import socket
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mds_oracle as orc
from paper_2007_11919_b200 import AlgorithmParams, plans
from paper_2007_11919_b200 import distributed as dd
from paper_2007_11919_b200.synthetic import scenario

ROOT = Path(__file__).resolve().parent.parent
STATUS = np.dtype([("code", np.int32), ("index", np.int32), ("value", np.float64)])


def _status_rows(codes):
    st = np.zeros(len(codes), dtype=STATUS)
    st["code"] = codes
    return torch.from_numpy(st.view(np.uint8).view(np.float64).reshape(-1, 2).copy())


def _emb(rows, r):
    """Oracle classical MDS of rows, or a status code when the oracle raises."""
    if not np.isfinite(rows).all():
        return None, 3
    try:
        return orc.mds_from_data(rows, r), 0
    except orc.OracleError as exc:
        return None, 5 if exc.kind == "DegenerateRankError" else 4


class OracleBackend:
    """Per-rank compute by the CPU oracle (same contract as GpuBackend)."""

    HEAD_FIXED = 6
    device = torch.device("cpu")

    def index(self, a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64))

    fail_local = None          # local subset index whose status is forced to DegenerateRank

    def dc_run(self, x, row_idx, piece_off, c, r, out, est, gof, status):
        x, ridx = x.numpy(), row_idx.numpy()
        subsets = [ridx[piece_off[j]:piece_off[j + 1]] for j in range(len(piece_off) - 1)]
        res = [_emb(x[s], r) for s in subsets]
        if self.fail_local is not None:
            res[self.fail_local] = (None, 5)
        status.copy_(_status_rows([code for _, code in res]))
        out.fill_(np.nan)
        if res[0][0] is None:
            return
        e0 = res[0][0]
        out[torch.from_numpy(subsets[0])] = torch.from_numpy(e0.points)
        anchor = e0.points[:c]
        for j, (s, (e, code)) in enumerate(zip(subsets, res)):
            if e is None:
                continue
            est[j] = torch.from_numpy(e.estimates)
            gof[j] = torch.tensor([e.g1, e.g2], dtype=torch.float64)
            if j:
                pts = orc.procrustes_apply(e.points[c:], orc.procrustes_fit(anchor, e.points[:c]))
                out[torch.from_numpy(s[c:])] = torch.from_numpy(pts)

    def range_sums(self, out, off, nseg, sums):
        o = off.numpy()
        for j in range(nseg):
            sums[j] = out[o[j]:o[j + 1]].sum(dim=0)

    def shift_rows(self, out, mean):
        out -= mean

    def scatter_rows(self, src, idx, out):
        out[idx] = src

    def head_len(self, l, p, r):
        return 6 + r + (l + r * r + l * p + l * r) + l * r

    def landmark_head(self, xl, r, head):
        xl = xl.numpy()
        l, p = xl.shape
        e, code = _emb(xl, r)
        head.zero_()
        head[2 + r:4 + r] = _status_rows([code])[0]
        if e is None:
            return
        ctx = orc.gower_ctx(xl, e.points)
        packed = np.concatenate([ctx.q_diag, ctx.covariance.ravel(), ctx.base_rows.ravel(),
                                 ctx.base_config.ravel()])
        head[0], head[1] = e.g1, e.g2
        head[2:2 + r] = torch.from_numpy(e.estimates)
        head[6 + r:6 + r + packed.size] = torch.from_numpy(packed)
        head[6 + r + packed.size:] = torch.from_numpy(e.points.ravel())

    def gower_rows(self, head, l, r, x, out):
        x = x.numpy()
        p = x.shape[1]
        h = head.numpy()[6 + r:]
        q = h[:l]
        cov = h[l:l + r * r].reshape(r, r)
        rows = h[l + r * r:l + r * r + l * p].reshape(l, p)
        cfg = h[l + r * r + l * p:l + r * r + l * p + l * r].reshape(l, r)
        if not np.isfinite(x).all():
            out.zero_()
            return torch.tensor(1.0, dtype=torch.float64)
        ctx = orc.GowerCtx(cfg, q, cov, rows)
        # fixed 64-row chunks (rank blocks start at multiples of SUM_BLOCK): the
        # same BLAS calls for a row whatever the world size
        for a in range(0, x.shape[0], 64):
            out[a:a + 64] = torch.from_numpy(orc.gower_project(ctx, x[a:a + 64]))
        return torch.tensor(0.0, dtype=torch.float64)

    def fast_run_sharded(self, run, n_total, nleaves_total, gather):
        """The contribution route's host side: per-leaf column sums gathered in
        global leaf order, the mean over n_total rows taken off every row."""
        pts, est, gof, status = self.fast_run(run)
        off = run[1].piece_off
        nl = run[1].n_leaves
        local = torch.stack([pts[off[j]:off[j + 1]].sum(dim=0) for j in range(nl)])
        glob = gather(local)
        pts[:off[nl]] -= glob.sum(dim=0) / n_total
        return pts, est, gof, status

    TILE = 64

    def tile_rows(self, x, r):
        return self.TILE

    def gower_tiles(self, head, l, r, x, out, tsum):
        flag = self.gower_rows(head, l, r, x, out)
        for t in range(tsum.shape[0]):
            tsum[t] = out[t * self.TILE:(t + 1) * self.TILE].sum(dim=0)
        return flag

    def landmark_overwrite(self, base, sel, pos, out, corr):
        corr.zero_()
        corr[sel] = base[sel] - out[pos]
        out[pos] = base[sel]

    def interp_recenter(self, tiles, corr, n, out):
        out -= (tiles.sum(dim=0) + corr.sum(dim=0)) / n

    def fast_prepare(self, x, plan, flat, r):
        return (x.numpy(), flat, r)

    def fast_run(self, run):
        x, flat, r = run
        off = flat.piece_off
        npc = len(off) - 1
        pts = np.zeros((int(off[-1]), r))
        est = np.zeros((npc, r))
        gof = np.zeros((npc, 2))
        codes = []
        for j in range(npc):
            e, code = _emb(x[flat.piece_rows[off[j]:off[j + 1]]], r)
            codes.append(code)
            if e is not None:
                pts[off[j]:off[j + 1]] = e.points
                est[j] = e.estimates
                gof[j] = [e.g1, e.g2]
        for lv in flat.levels:
            for t in range(len(lv.start)):
                a, b = lv.job_off[t], lv.job_off[t + 1]
                T = orc.procrustes_fit(pts[lv.tgt_rows[a:b]], pts[lv.src_rows[a:b]])
                s0, ln = lv.start[t], lv.length[t]
                pts[s0:s0 + ln] = orc.procrustes_apply(pts[s0:s0 + ln], T)
        return (torch.from_numpy(pts), torch.from_numpy(est), torch.from_numpy(gof),
                _status_rows(codes))


N = 2600


def _data(poison=None):
    x = scenario(N, 8, 4, seed=9)
    if poison is not None:
        x[poison, 3] = np.nan
    return x


def _params(algo):
    if algo == "divide":
        return AlgorithmParams(r=4, l=300, c=10, seed=2)
    if algo == "fast":
        return AlgorithmParams(r=4, l=300, s=8, seed=2)
    return AlgorithmParams(r=4, l=400, seed=2)


def _worker(rank, world, port, algo, path, poison, fail):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dd.SUM_BLOCK = 256                         # several blocks per rank at test size
        x = _data(poison)
        prm = _params(algo).resolved(algo)
        comm = dd.Comm()
        be = OracleBackend()
        if fail is not None and fail[0] == rank:
            be.fail_local = fail[1]
        if algo == "divide":
            plan = plans.plan_divide_conquer(N, prm.l, prm.c, prm.seed)
        elif algo == "fast":
            plan = plans.plan_fast(N, prm.l, prm.s, prm.seed)
        else:
            plan = plans.interpolation_sample(N, prm.l, prm.seed)
        rows = dd.local_rows(algo, plan, N, world, rank)
        xl = torch.from_numpy(np.ascontiguousarray(x[rows]))
        try:
            if algo == "divide":
                res = dd.sharded_divide_and_conquer(be, xl, N, prm, comm, plan=plan)
            elif algo == "fast":
                res = dd.sharded_fast(be, xl, N, prm, comm, plan=plan)
            else:
                land = torch.from_numpy(x[plan]) if rank == 0 else None
                res = dd.sharded_interpolation(be, xl, N, prm, comm, sample=plan, x_landmarks=land)
        except Exception as exc:                   # every rank must raise the same
            np.savez(f"{path}.{rank}.err.npz", kind=type(exc).__name__, msg=str(exc))
            return
        full = dd.gather_points(res, N, comm)
        if rank == 0:
            np.savez(path, points=full, est=res.estimates, g=np.array([res.gof_g1, res.gof_g2]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, algo, poison=None, fail=None):
    path = tempfile.mktemp(suffix=".npz")
    mp.spawn(_worker, args=(world, _free_port(), algo, path, poison, fail), nprocs=world,
             join=True)
    errs = [f"{path}.{k}.err.npz" for k in range(world)]
    if any(os.path.exists(e) for e in errs):
        out = []
        for e in errs:
            with np.load(e) as z:
                out.append((str(z["kind"]), str(z["msg"])))
            os.unlink(e)
        return {"errors": out}
    with np.load(path) as z:
        out = {k: z[k] for k in z.files}
    os.unlink(path)
    return out


@pytest.mark.parametrize("algo", ["divide", "interpolate", "fast"])
def test_sharded_matches_reference_and_is_world_size_independent(algo):
    x = _data()
    if algo == "divide":
        ref = orc.divide_conquer(x, 4, l=300, c=10, seed=2, threads=1)
    elif algo == "fast":
        ref = orc.run("fast", x, 4, l=300, s=8, seed=2, threads=1)
    else:
        ref = orc.interpolation(x, 4, l=400, seed=2, threads=1)
    runs = [_run(w, algo) for w in (1, 2, 3)]
    for other in runs[1:]:
        assert np.array_equal(runs[0]["points"], other["points"])    # bitwise across world sizes
        assert np.array_equal(runs[0]["g"], other["g"])
        assert np.array_equal(runs[0]["est"], other["est"])
    got = runs[1]
    err = np.linalg.norm(got["points"] - ref.points) / np.linalg.norm(ref.points)
    assert err <= 1e-12, err
    assert np.allclose(got["est"], ref.estimates, rtol=1e-13)
    assert abs(got["g"][0] - ref.g1) <= 1e-14 and abs(got["g"][1] - ref.g2) <= 1e-14


@pytest.mark.parametrize("algo", ["divide", "interpolate", "fast"])
def test_non_finite_row_on_last_rank_raises_everywhere(algo, monkeypatch):
    """A NaN in a row only the last rank reads: every rank raises
    InvalidInputError (the verdict is taken from the all-gathered records)."""
    monkeypatch.setattr(dd, "SUM_BLOCK", 256)            # as in the workers
    prm = _params(algo).resolved(algo)
    if algo == "divide":
        plan = plans.plan_divide_conquer(N, prm.l, prm.c, prm.seed)
    elif algo == "fast":
        plan = plans.plan_fast(N, prm.l, prm.s, prm.seed)
    else:
        plan = plans.interpolation_sample(N, prm.l, prm.seed)
    rows0 = set(dd.local_rows(algo, plan, N, 2, 0).tolist())
    if algo == "interpolate":
        rows0 |= set(plan.tolist())
    only1 = [i for i in dd.local_rows(algo, plan, N, 2, 1).tolist() if i not in rows0]
    out = _run(2, algo, poison=only1[len(only1) // 2])
    assert [e[0] for e in out["errors"]] == ["InvalidInputError"] * 2, out


def test_degenerate_piece_on_last_rank_raises_everywhere():
    """A subset owned by rank 1 fails (the backend reports DegenerateRank for
    it): both ranks raise the same DegenerateRankError naming that subset."""
    prm = _params("divide").resolved("divide")
    plan = plans.plan_divide_conquer(N, prm.l, prm.c, prm.seed)
    lo, _ = dd.shard(plan.p - 1, 2, 1)
    out = _run(2, "divide", fail=(1, 2))                 # rank 1, its second local subset
    kinds = [e[0] for e in out["errors"]]
    msgs = [e[1] for e in out["errors"]]
    assert kinds == ["DegenerateRankError"] * 2, out
    assert msgs[0] == msgs[1] and f"subset {1 + lo + 2}:" in msgs[0], msgs


def test_shard_partition():
    for count in (0, 1, 7, 1020):
        for world in (1, 2, 3, 8):
            spans = [dd.shard(count, world, k) for k in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


@pytest.mark.parametrize("algo", ["divide", "fast", "interpolate"])
def test_local_rows_cover_the_input_once(algo):
    """The ranks' reported rows partition 0..n-1 and the local matrices add
    up to about one copy of the input (anchor / alignment rows aside)."""
    prm = _params(algo).resolved(algo)
    n = 50_000
    if algo == "divide":
        plan = plans.plan_divide_conquer(n, prm.l, prm.c, prm.seed)
    elif algo == "fast":
        plan = plans.plan_fast(n, prm.l, prm.s, prm.seed)
    else:
        plan = plans.interpolation_sample(n, prm.l, prm.seed)
    for world in (1, 2, 4):
        total = sum(len(dd.local_rows(algo, plan, n, world, k)) for k in range(world))
        extra = {"divide": prm.l, "fast": 2 * prm.l, "interpolate": 0}[algo]
        assert n <= total <= n + world * extra


@pytest.mark.parametrize("world", [2, 4])
def test_bench_self_launch(world):
    """bench.py --gpus N without WORLD_SIZE starts N ranks itself (torch
    distributed launcher on 127.0.0.1) and rank 0 reports n_gpus = N; the
    launch check runs the rendezvous and a collective over gloo on CPU."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(world),
                          "--check-launch"], capture_output=True, text=True, timeout=300,
                         env=env, cwd=str(ROOT))
    assert res.returncode == 0, res.stderr[-2000:]
    import json
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == world and line["ranks_seen"] == list(range(world))


def _gather_worker(rank, world, port, path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = plans.plan_divide_conquer(30_000, 400, 10, 3)
        comm = dd.Comm()
        sd = dd.ShardedDivide.__new__(dd.ShardedDivide)       # layout fields only
        sd.plan, sd.comm = plan, comm
        sd.sh = dd.dc_shard(plan, world, rank)
        sd.first = 0 if rank == 0 else 1
        sd.kmax = 1 + dd.shard(plan.p - 1, world, 0)[1]
        ids = torch.tensor(sd.sh.pieces, dtype=torch.float64)[:, None]
        rows = torch.cat([ids, ids * 10.0 + rank * (ids == 0)], dim=1)  # anchor row differs per rank
        out = sd._gather_sorted(rows)
        np.save(f"{path}.{rank}.npy", out.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_record_gather_layout(world):
    """ShardedDivide._gather_sorted (the GPU backend's contribution and record
    gather): every subset's row exactly once, in global subset order, the
    anchor's from rank 0, identical on every rank."""
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "g")
        mp.spawn(_gather_worker, args=(world, _free_port(), path), nprocs=world, join=True)
        outs = [np.load(f"{path}.{k}.npy") for k in range(world)]
    p = plans.plan_divide_conquer(30_000, 400, 10, 3).p
    for o in outs:
        assert np.array_equal(o, outs[0])
    assert np.array_equal(outs[0][:, 0], np.arange(p))
    assert np.array_equal(outs[0][:, 1], np.arange(p) * 10.0)
