"""Pin the CPU oracle (oracle/mds_oracle.py) against the reference's own
outputs (tests/golden/*.npz written by make_golden.py from scalemds).  The
oracle is the checker for every GPU parity test, so it must reproduce the
reference first: plans bit-exact, arrays to round-off."""

import hashlib

import numpy as np
import pytest

from conftest import golden, sign_fixed_rel_err
from oracle import mds_oracle as orc
from paper_2007_11919_b200 import synthetic


def digest(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
        h.update(np.int64(a.size).tobytes())
        h.update(a.tobytes())
    return h.hexdigest()


def close(cfg, ref, tol=1e-9):
    assert sign_fixed_rel_err(cfg.points, ref["points"]) <= tol
    assert np.allclose(cfg.estimates, ref["estimates"], rtol=tol, atol=0)
    assert abs(cfg.g1 - float(ref["g1"])) <= tol and abs(cfg.g2 - float(ref["g2"])) <= tol


class TestPrimitives:
    def test_distances_and_centering(self):
        g = golden("fn_small")
        assert np.abs(orc.sqdist_self(g["d40"]) - g["dist_self"]).max() <= 1e-12
        assert np.abs(orc.sqdist_cross(g["a43"], g["b63"]) - g["dist_cross"]).max() <= 1e-12
        assert np.abs(orc.center_delta(g["dist_self"]) - g["dcenter"]).max() <= 1e-12

    def test_classical(self):
        g = golden("fn_small")
        e = orc.mds_from_data(g["x60"], 3)
        assert np.abs(e.points - g["c_points"]).max() <= 1e-10
        assert np.allclose(e.estimates, g["c_est"], rtol=1e-12)
        n = orc.mds_from_delta(g["ne"], 2)
        assert np.abs(n.points - g["ne_points"]).max() <= 1e-10
        assert abs(n.g1 - g["ne_g"][0]) <= 1e-12 and abs(n.g2 - g["ne_g"][1]) <= 1e-12

    def test_procrustes_and_gower(self):
        g = golden("fn_small")
        t = orc.procrustes_fit(g["pt"], g["ps"])
        assert np.abs(t.rotation - g["pf_rot"]).max() <= 1e-12
        ctx = orc.gower_ctx(g["base"], g["base_points"])
        assert np.abs(ctx.q_diag - g["ctx_q"]).max() <= 1e-12 * np.abs(g["ctx_q"]).max()
        assert np.abs(orc.gower_project(ctx, g["newrows"]) - g["gower"]).max() <= 1e-12 * 10


class TestAlgorithms:
    def test_config1(self):
        ref = golden("cfg1_interp")
        x = orc.scenario(10_000, 10, 2, seed=0)
        assert np.array_equal(x[:5], ref["x_head"])
        subsets = orc.plan_interp(10_000, 500, 0)
        assert digest(subsets) == str(ref["plan_digest"])
        close(orc.interpolation(x, 2, l=500, seed=0, threads=1), ref)

    def test_divide_and_fast(self):
        x = orc.scenario(5000, 100, 10, seed=0)
        close(orc.divide_conquer(x, 10, l=1000, c=20, seed=0, threads=1), golden("dc_n5000"))
        close(orc.fast(x, 10, l=1000, s=20, seed=0, threads=1), golden("fast_n5000"))

    def test_fast_deep(self):
        x = orc.scenario(3000, 10, 5, seed=4)
        close(orc.fast(x, 5, l=100, s=10, seed=4, threads=1), golden("fast_deep"))

    def test_interp_fp32(self):
        x = orc.scenario(8000, 100, 10, seed=0).astype(np.float32)
        close(orc.interpolation(x, 10, l=2000, seed=0, threads=1), golden("interp_f32_n8000"))

    @pytest.mark.parametrize("name,kw", [("divide", dict(l=1000, c=20)),
                                         ("fast", dict(l=1000, s=20)),
                                         ("interpolate", dict(l=1000))])
    def test_image_like(self, name, kw):
        x = synthetic.image_like(3000, seed=0)
        close(orc.run(name, x, 10, seed=0, threads=1, **kw), golden(f"img_{name}_n3000"), tol=1e-8)

    def test_generator_matches_package_generator(self):
        assert np.array_equal(orc.scenario(700, 9, 3, seed=5, rep=2),
                              synthetic.scenario(700, 9, 3, seed=5, rep=2))


class TestOraclePlans:
    """The oracle's planners against the reference's partition contracts and
    the (digest-pinned) product planner, including the short-remainder merge."""

    def test_divide_merge_case(self):
        conn, subs = orc.plan_divide(285, 100, 10, 1)
        assert [len(s) for s in subs] == [100, 100, 105]
        merged = np.concatenate([conn] + [s[10:] for s in subs])
        assert np.array_equal(np.sort(merged), np.arange(285))

    @pytest.mark.parametrize("n,l,c,seed", [(1300, 650, 20, 1), (285, 100, 10, 1), (5000, 1000, 20, 0),
                                            (1000, 400, 20, 5), (999, 300, 7, 3)])
    def test_divide_matches_product_planner(self, n, l, c, seed):
        from paper_2007_11919_b200.plans import plan_divide_conquer
        _, subs = orc.plan_divide(n, l, c, seed)
        ref = plan_divide_conquer(n, l, c, seed).subsets
        assert len(subs) == len(ref) and all(np.array_equal(a, b) for a, b in zip(subs, ref))

    def test_interp_and_fast_match_product_planner(self):
        from paper_2007_11919_b200.plans import plan_fast, plan_interpolation
        for n, l, seed in [(10, 4, 0), (1001, 100, 2), (3000, 1000, 3)]:
            a = orc.plan_interp(n, l, seed)
            b = plan_interpolation(n, l, seed).subsets
            assert all(np.array_equal(x, y) for x, y in zip(a, b))
        ta, tb = orc.plan_fast_tree(5000, 100, 10, 4), plan_fast(5000, 100, 10, 4).root
        def walk(x, y):
            assert np.array_equal(x.indices, y.indices)
            if x.positions is not None:
                assert np.array_equal(x.positions, y.sampling_positions)
            assert len(x.children) == len(y.children)
            for cx, cy in zip(x.children, y.children):
                walk(cx, cy)
        walk(ta, tb)
