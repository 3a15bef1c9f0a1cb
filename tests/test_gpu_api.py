"""The reference's own test suite (tests/test_linalg.py, test_classical.py,
test_procrustes.py, test_algorithms.py) re-expressed against the GPU-backed
drop-in API.  Same inputs, same assertions, same exception types/messages.
Deliberate difference (documented in DESIGN.md §3): classical_mds_from_data
uses the Gram-of-centred-rows path, so it equals classical_mds(Delta) to
round-off (1e-12) rather than bitwise."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mds(cuda):
    import paper_2007_11919_b200 as m
    return m


def naive_sq(data):
    n, k = data.shape
    out = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            out[i, j] = sum((data[i, s] - data[j, s]) ** 2 for s in range(k))
    return out


def aligned_corr(mds, cfg, dominant):
    """simulation.py:83-108 on the GPU Procrustes."""
    fit = mds.fit_procrustes(dominant, cfg.points)
    al = mds.apply_procrustes(cfg.points, fit)
    a = al - al.mean(axis=0)
    d = dominant - dominant.mean(axis=0)
    return np.einsum("ij,ij->j", a, d) / np.sqrt(np.einsum("ij,ij->j", a, a) * np.einsum("ij,ij->j", d, d))


class TestDistances:
    def test_345(self, mds):
        assert np.array_equal(mds.euclidean_distance_matrix(np.array([[0.0, 0.0], [3.0, 4.0]])),
                              [[0.0, 25.0], [25.0, 0.0]])

    def test_single_row(self, mds):
        assert np.array_equal(mds.euclidean_distance_matrix([[7.0]]), [[0.0]])

    def test_naive_loop(self, mds):
        data = np.random.default_rng(0).standard_normal((5, 3))
        assert np.abs(mds.euclidean_distance_matrix(data) - naive_sq(data)).max() <= 1e-12

    def test_symmetric_zero_diag_nonneg(self, mds):
        d = mds.euclidean_distance_matrix(np.random.default_rng(1).standard_normal((40, 6)))
        assert np.array_equal(d, d.T) and np.all(np.diagonal(d) == 0.0) and d.min() >= 0.0

    @pytest.mark.parametrize("m,mb,p,dtype", [(200, 130, 37, np.float64), (65, 64, 16, np.float64),
                                              (300, 77, 100, np.float32), (1, 129, 5, np.float64)])
    def test_tensor_tiles_ragged(self, mds, m, mb, p, dtype):
        """DMMA distance tiles: ragged rows / features, fp32 storage, several
        tiles; self distances exactly symmetric (mirrored lower triangle)."""
        rng = np.random.default_rng(m + p)
        a = rng.standard_normal((m, p)).astype(dtype)
        b = rng.standard_normal((mb, p)).astype(dtype)
        a64, b64 = a.astype(np.float64), b.astype(np.float64)
        ref = np.maximum((a64 * a64).sum(1)[:, None] + (b64 * b64).sum(1)[None, :] - 2 * a64 @ b64.T, 0)
        got = mds.cross_squared_distances(a, b)
        assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
        d = mds.euclidean_distance_matrix(a)
        assert np.array_equal(d, d.T) and np.all(np.diagonal(d) == 0.0)
        assert np.abs(d - naive_sq(a64)).max() <= 1e-12 * max(1.0, d.max())

    @pytest.mark.parametrize("m,mb,p,dtype", [(333, 190, 38, np.float64), (257, 65, 100, np.float64),
                                              (400, 129, 36, np.float32), (130, 64, 4, np.float64),
                                              (129, 200, 52, np.float32)])
    def test_pipelined_tiles(self, mds, m, mb, p, dtype):
        """The cp.async ring kernel (rows 16-byte aligned): 128 x 64 tiles with
        ragged last tiles in both directions, a last feature chunk that stops at
        p, fp32 storage; exactly symmetric self distances; the self matrix of the
        stacked rows holds the cross block."""
        rng = np.random.default_rng(7 * m + p)
        a = (rng.standard_normal((m, p)) * 3.0).astype(dtype)
        b = (rng.standard_normal((mb, p)) * 3.0).astype(dtype)
        a64, b64 = a.astype(np.float64), b.astype(np.float64)
        ref = ((a64[:, None, :] - b64[None, :, :]) ** 2).sum(-1)
        got = mds.cross_squared_distances(a, b)
        assert np.abs(got - ref).max() <= 1e-12 * max(1.0, ref.max())
        d = mds.euclidean_distance_matrix(np.vstack([a, b]))
        assert np.array_equal(d, d.T) and np.all(np.diagonal(d) == 0.0) and d.min() >= 0.0
        assert np.abs(d[:m, m:] - ref).max() <= 1e-12 * max(1.0, ref.max())
        self_ref = ((a64[:, None, :] - a64[None, :, :]) ** 2).sum(-1)
        assert np.abs(d[:m, :m] - self_ref).max() <= 1e-12 * max(1.0, d.max())

    def test_non_finite_and_guard(self, mds):
        with pytest.raises(mds.InvalidInputError):
            mds.euclidean_distance_matrix([[1.0, np.nan]])
        with pytest.raises(mds.ParamError, match="exact-size guard"):
            mds.euclidean_distance_matrix(np.zeros((11, 2)), exact_guard=10)

    def test_cross(self, mds):
        assert np.array_equal(mds.cross_squared_distances([[0.0]], [[3.0], [4.0]]), [[9.0, 16.0]])
        a = np.random.default_rng(2).standard_normal((6, 4))
        assert np.abs(np.diagonal(mds.cross_squared_distances(a, a))).max() <= 1e-12
        rng = np.random.default_rng(3)
        a, b = rng.standard_normal((4, 3)), rng.standard_normal((6, 3))
        st = mds.euclidean_distance_matrix(np.vstack([a, b]))
        assert np.abs(mds.cross_squared_distances(a, b) - st[:4, 4:]).max() <= 1e-12
        with pytest.raises(mds.ShapeError):
            mds.cross_squared_distances(np.zeros((2, 3)), np.zeros((2, 4)))


class TestDoubleCenter:
    def test_hand_values(self, mds):
        assert np.allclose(mds.double_center([[0.0, 1.0], [1.0, 0.0]]),
                           [[0.25, -0.25], [-0.25, 0.25]], atol=1e-15)
        assert np.array_equal(mds.double_center(np.zeros((3, 3))), np.zeros((3, 3)))

    def test_collinear_and_gram(self, mds):
        coords = np.array([-4.0, -1.0, 5.0]) / 3.0
        delta = mds.euclidean_distance_matrix(np.array([[0.0], [1.0], [3.0]]))
        assert np.abs(mds.double_center(delta) - np.outer(coords, coords)).max() <= 1e-12
        data = np.random.default_rng(4).standard_normal((30, 5)) * 3.0
        c = data - data.mean(axis=0)
        q = mds.double_center(mds.euclidean_distance_matrix(data))
        assert np.abs(q - c @ c.T).max() <= 1e-9 * np.abs(c @ c.T).max()
        assert np.array_equal(q, q.T)

    def test_annihilates_ones(self, mds):
        q = mds.double_center(mds.euclidean_distance_matrix(np.random.default_rng(5).standard_normal((25, 4))))
        assert np.abs(q @ np.ones(25)).max() <= 1e-9 * 25 * np.abs(q).max()

    @pytest.mark.parametrize("m", [64, 129, 200, 513])
    def test_tile_pairs(self, mds, m):
        """64 x 64 tile pairs with ragged edges, odd m (scalar row means) and even
        m (16-byte loads), against the formula of linalg.py:116-121 in numpy."""
        rng = np.random.default_rng(m)
        x = rng.standard_normal((m, 7)) * 2.0
        delta = ((x[:, None, :] - x[None, :, :]) ** 2).sum(-1)
        delta = 0.5 * (delta + delta.T)
        mu = delta.mean(axis=1)
        ref = -0.5 * (delta - mu[:, None] - mu[None, :] + delta.mean())
        ref = 0.5 * (ref + ref.T)
        q = mds.double_center(delta)
        assert np.array_equal(q, q.T)
        assert np.abs(q - ref).max() <= 1e-12 * np.abs(ref).max()

    def test_invalid_delta(self, mds):
        with pytest.raises(mds.InvalidInputError, match="symmetric"):
            mds.double_center([[0.0, 1.0], [2.0, 0.0]])
        with pytest.raises(mds.InvalidInputError, match="diagonal"):
            mds.double_center([[1.0, 1.0], [1.0, 0.0]])
        with pytest.raises(mds.InvalidInputError, match="negative"):
            mds.double_center([[0.0, -1.0], [-1.0, 0.0]])


class TestClassical:
    def test_collinear(self, mds):
        cfg = mds.classical_mds(mds.euclidean_distance_matrix(np.array([[0.0], [1.0], [3.0]])), 1)
        coords = np.array([-4.0, -1.0, 5.0]) / 3.0
        col = cfg.points[:, 0]
        assert min(np.abs(col - coords).max(), np.abs(col + coords).max()) <= 1e-12
        assert cfg.eigenvalue_estimates[0] == pytest.approx(14.0 / 9.0, rel=1e-12)
        assert cfg.gof_g1 == 1.0 and cfg.gof_g2 == 1.0

    def test_degenerate_and_range(self, mds):
        with pytest.raises(mds.DegenerateRankError):
            mds.classical_mds(np.zeros((4, 4)), 1)
        delta = mds.euclidean_distance_matrix(np.random.default_rng(1).standard_normal((20, 2)))
        with pytest.raises(mds.DegenerateRankError, match="3"):
            mds.classical_mds(delta, 3)
        with pytest.raises(mds.ParamError):
            mds.classical_mds(np.zeros((3, 3)), 3)
        with pytest.raises(mds.ParamError, match="exact-size guard"):
            mds.classical_mds(np.zeros((12, 12)), 1, exact_guard=10)
        with pytest.raises(mds.ParamError):
            mds.classical_mds_from_data(np.array([[1.0, 2.0]]), 1)

    def test_round_trip(self, mds):
        data = np.random.default_rng(0).standard_normal((50, 5))
        delta = mds.euclidean_distance_matrix(data)
        back = mds.euclidean_distance_matrix(mds.classical_mds(delta, 5).points)
        assert np.abs(back - delta).max() <= 1e-8

    def test_variance_centering_nesting(self, mds):
        data = np.random.default_rng(2).standard_normal((60, 4))
        cfg = mds.classical_mds_from_data(data, 4)
        var = (cfg.points ** 2).sum(axis=0) / 60
        assert np.abs(var - cfg.eigenvalue_estimates).max() <= 1e-9 * cfg.eigenvalue_estimates[0]
        assert np.abs(cfg.points.mean(axis=0)).max() <= 1e-9 * cfg.points.std(axis=0).min()
        delta = mds.euclidean_distance_matrix(np.random.default_rng(4).standard_normal((30, 6)))
        wide, narrow = mds.classical_mds(delta, 5), mds.classical_mds(delta, 2)
        assert np.array_equal(wide.points[:, :2], narrow.points)

    def test_rotation_invariance_and_recovery(self, mds):
        rng = np.random.default_rng(5)
        data = rng.standard_normal((40, 5))
        basis, _ = np.linalg.qr(rng.standard_normal((5, 5)))
        a = mds.classical_mds_from_data(data, 3)
        b = mds.classical_mds_from_data(data @ basis, 3)
        assert np.abs(a.eigenvalue_estimates - b.eigenvalue_estimates).max() <= 1e-9
        rng = np.random.default_rng(6)
        raw = rng.standard_normal((40, 4))
        raw -= raw.mean(axis=0)
        u, _, _ = np.linalg.svd(raw, full_matrices=False)
        d = u * np.array([8.0, 4.0, 2.0, 1.0])
        cfg = mds.classical_mds_from_data(d, 4)
        for i in range(4):
            assert min(np.abs(cfg.points[:, i] - d[:, i]).max(), np.abs(cfg.points[:, i] + d[:, i]).max()) <= 1e-9

    def test_composition_to_roundoff(self, mds):
        data = np.random.default_rng(7).standard_normal((100, 10))
        a = mds.classical_mds_from_data(data, 3)
        b = mds.classical_mds(mds.euclidean_distance_matrix(data), 3)
        assert np.abs(a.points - b.points).max() <= 1e-11
        assert abs(a.gof_g1 - b.gof_g1) <= 1e-12

    def test_g1_equals_g2_euclidean(self, mds):
        rng = np.random.default_rng(1004)
        for _ in range(20):
            n, k = int(rng.integers(20, 80)), int(rng.integers(2, 8))
            cfg = mds.classical_mds_from_data(rng.standard_normal((n, k)) * rng.uniform(0.1, 10.0), min(k, n - 1))
            assert cfg.gof_g1 == cfg.gof_g2


class TestProcrustes:
    ROT90 = np.array([[0.0, -1.0], [1.0, 0.0]])

    def test_identity_rotation_translation(self, mds):
        x = np.random.default_rng(0).standard_normal((10, 3))
        fit = mds.fit_procrustes(x, x)
        assert np.abs(fit.rotation - np.eye(3)).max() <= 1e-10 and fit.loss <= 1e-10
        x = np.random.default_rng(1).standard_normal((12, 2))
        fit = mds.fit_procrustes(x, x @ self.ROT90)
        assert np.abs(fit.rotation - self.ROT90.T).max() <= 1e-12 and fit.loss <= 1e-18
        assert np.abs(mds.apply_procrustes(x @ self.ROT90, fit) - x).max() <= 1e-10
        x = np.random.default_rng(2).standard_normal((8, 2))
        fit = mds.fit_procrustes(x, x + np.array([5.0, -3.0]))
        assert np.allclose(fit.translation, [-5.0, 3.0], atol=1e-12)

    def test_shape_and_degenerate(self, mds):
        with pytest.raises(mds.ShapeError):
            mds.fit_procrustes(np.zeros((4, 2)), np.zeros((4, 3)))
        with pytest.raises(mds.ShapeError):
            mds.fit_procrustes(np.zeros((1, 2)), np.zeros((1, 2)))
        fit = mds.fit_procrustes(np.ones((5, 2)), np.ones((5, 2)))
        assert fit.degenerate
        assert np.abs(fit.rotation @ fit.rotation.T - np.eye(2)).max() <= 1e-10

    def test_random_recovery_and_kristof(self, mds):
        rng = np.random.default_rng(3)
        for r in (2, 5, 10):
            for _ in range(3):
                x = rng.standard_normal((30, r))
                q, _ = np.linalg.qr(rng.standard_normal((r, r)))
                moved = x @ q + rng.standard_normal(r) * 3.0
                fit = mds.fit_procrustes(x, moved)
                assert fit.loss <= 1e-18 * max(1.0, (x ** 2).sum())
                assert np.abs(mds.apply_procrustes(moved, fit) - x).max() <= 1e-10
        rng = np.random.default_rng(5)
        t, s = rng.standard_normal((20, 3)), rng.standard_normal((20, 3))
        best = mds.fit_procrustes(t, s)
        assert abs(abs(np.linalg.det(best.rotation)) - 1.0) <= 1e-10
        for _ in range(200):
            q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
            res = t - s @ q - (t - s @ q).mean(axis=0)
            assert best.loss <= np.sum(res * res) + 1e-12

    def test_apply_identity_bitwise(self, mds):
        pts = np.random.default_rng(9).standard_normal((11, 3))
        ident = mds.ProcrustesTransform(rotation=np.eye(3), translation=np.zeros(3), loss=0.0)
        assert np.array_equal(mds.apply_procrustes(pts, ident), pts)
        with pytest.raises(mds.ShapeError):
            mds.apply_procrustes(np.zeros((4, 2)), ident)


class TestGower:
    @pytest.fixture
    def ctx(self, mds):
        base = np.random.default_rng(21).standard_normal((200, 10)) * 2.0
        cfg = mds.classical_mds_from_data(base, 5)
        return base, cfg, mds.gower_context(base, cfg.points)

    def test_self_single_centroid(self, mds, ctx):
        base, cfg, c = ctx
        assert np.abs(mds.gower_interpolate(c, base) - cfg.points).max() <= 1e-8
        assert np.abs(mds.gower_interpolate(c, base[42:43]) - cfg.points[42]).max() <= 1e-8
        got = mds.gower_interpolate(c, base.mean(axis=0, keepdims=True))
        assert np.linalg.norm(got) <= 1e-6 * np.abs(cfg.points).max()

    def test_errors(self, mds, ctx):
        _, _, c = ctx
        with pytest.raises(mds.ShapeError):
            mds.gower_interpolate(c, np.zeros((3, 4)))
        base = np.random.default_rng(22).standard_normal((50, 5))
        cfg = mds.classical_mds_from_data(base, 3)
        crushed = cfg.points.copy()
        crushed[:, 2] *= 1e-9
        with pytest.raises(mds.NumericalError, match="condition"):
            mds.gower_context(base, crushed)


@pytest.fixture(scope="module")
def scenario_data(cuda):
    from paper_2007_11919_b200.synthetic import scenario
    return scenario(3000, 10, 5, seed=17)


ALGS = [("divide", dict(r=5, l=400, c=10, seed=7)), ("interpolate", dict(r=5, l=1000, seed=7)),
        ("fast", dict(r=5, l=1000, s=10, seed=7))]


# tests/test_acceptance.py:110-164 of the reference: the desk grid (n = 1e4, k = 10,
# h = 5, 10 replications, seed 20 240); its eigenvalue-bias vectors as recorded by the
# reference run (pkg/test_output.txt:230, printed to 2 decimals).
DESK_BIAS = {
    "interpolate": [1.67, 0.81, 0.17, -0.66, -1.44],
    "divide": [3.04, 1.58, 0.39, -0.78, -2.06],
    "fast": [5.15, 2.04, -0.34, -2.39, -4.57],
}
DESK_PARAMS = {"interpolate": dict(r=5, l=1000), "divide": dict(r=5, l=400, c=10),
               "fast": dict(r=5, l=1000, s=10)}


@pytest.mark.parametrize("name", ["interpolate", "divide", "fast"])
def test_desk_grid_matches_reference_record(mds, name):
    from paper_2007_11919_b200.synthetic import scenario
    est, corr = [], []
    for rep in range(10):
        x = scenario(10_000, 10, 5, seed=20_240, rep=rep)
        cfg = mds.run_algorithm(name, x, mds.AlgorithmParams(seed=rep, **DESK_PARAMS[name]))
        est.append(cfg.eigenvalue_estimates)
        corr.append(aligned_corr(mds, cfg, x[:, :5]))
    bias = np.mean(est, axis=0) - 15.0
    assert np.allclose(bias, DESK_BIAS[name], atol=0.0051), (name, np.round(bias, 3))
    floor = {"interpolate": 0.999, "divide": 0.99, "fast": 0.95}[name]
    assert np.mean(corr) >= floor


class TestAlgorithms:
    def test_dc_recovery_shape_centering(self, mds, scenario_data):
        cfg = mds.divide_and_conquer_mds(scenario_data, mds.AlgorithmParams(r=5, l=400, c=10, seed=3))
        assert aligned_corr(mds, cfg, scenario_data[:, :5]).min() >= 0.99
        assert cfg.points.shape == (3000, 5)
        assert np.abs(cfg.points.mean(axis=0)).max() <= 1e-6 * cfg.points.std(axis=0).min()
        assert np.all(np.diff(cfg.eigenvalue_estimates) <= 0) and cfg.gof_g1 <= cfg.gof_g2

    def test_connecting_rows_from_first_subset(self, mds, scenario_data):
        cfg = mds.divide_and_conquer_mds(scenario_data, mds.AlgorithmParams(r=5, l=400, c=10, seed=3))
        plan = mds.plan_divide_conquer(3000, 400, 10, seed=3)
        first = mds.classical_mds_from_data(scenario_data[plan.subsets[0]], 5)
        delta = cfg.points[plan.subsets[0]] - first.points
        assert np.abs(delta - delta.mean(axis=0)).max() <= 1e-12

    def test_degenerate_subset_reported(self, mds):
        rank2 = np.random.default_rng(0).standard_normal((2000, 2)) @ \
            np.random.default_rng(1).standard_normal((2, 6))
        with pytest.raises(mds.DegenerateRankError, match="subset"):
            mds.divide_and_conquer_mds(rank2, mds.AlgorithmParams(r=4, l=400, c=8, seed=0))

    def test_non_finite_rejected(self, mds, scenario_data):
        bad = scenario_data.copy()
        bad[1234, 3] = np.inf
        for name, prm in ALGS:
            with pytest.raises(mds.InvalidInputError):
                mds.run_algorithm(name, bad, mds.AlgorithmParams(**prm))

    def test_interp_gof_from_sample(self, mds, scenario_data):
        cfg = mds.interpolation_mds(scenario_data, mds.AlgorithmParams(r=5, l=1000, seed=3))
        plan = mds.plan_interpolation(3000, 1000, seed=3)
        first = mds.classical_mds_from_data(scenario_data[plan.subsets[0]], 5)
        assert cfg.gof_g1 == first.gof_g1 and cfg.gof_g2 == first.gof_g2
        assert np.array_equal(cfg.eigenvalue_estimates, first.eigenvalue_estimates)
        assert aligned_corr(mds, cfg, scenario_data[:, :5]).min() >= 0.995

    def test_fast(self, mds, scenario_data):
        cfg = mds.fast_mds(scenario_data, mds.AlgorithmParams(r=5, l=1000, s=10, seed=3))
        assert aligned_corr(mds, cfg, scenario_data[:, :5]).min() >= 0.95
        assert cfg.gof_g1 <= cfg.gof_g2 and np.all(np.diff(cfg.eigenvalue_estimates) <= 0)
        from paper_2007_11919_b200.synthetic import scenario
        data = scenario(600, 6, 3, seed=5)
        cfg = mds.fast_mds(data, mds.AlgorithmParams(r=3, l=60, s=20, seed=5))
        assert cfg.points.shape == (600, 3) and aligned_corr(mds, cfg, data[:, :3]).min() >= 0.8

    @pytest.mark.parametrize("name,prm", ALGS)
    def test_local_isometry_and_seed(self, mds, scenario_data, name, prm):
        cfg = mds.run_algorithm(name, scenario_data, mds.AlgorithmParams(**prm))
        assert np.isfinite(cfg.points).all()
        pairs = np.random.default_rng(0).integers(0, 3000, size=(100, 2))
        o = np.sqrt(((scenario_data[pairs[:, 0], :5] - scenario_data[pairs[:, 1], :5]) ** 2).sum(1))
        e = np.sqrt(((cfg.points[pairs[:, 0]] - cfg.points[pairs[:, 1]]) ** 2).sum(1))
        assert np.corrcoef(o, e)[0, 1] >= 0.95
        import dataclasses
        b = mds.run_algorithm(name, scenario_data, dataclasses.replace(mds.AlgorithmParams(**prm), seed=99))
        if name == "interpolate":
            assert not np.array_equal(cfg.points, b.points)
        assert aligned_corr(mds, b, scenario_data[:, :5]).min() >= 0.95

    def test_device_resident_api(self, mds, scenario_data):
        import torch
        x = torch.from_numpy(scenario_data).cuda()
        cfg = mds.divide_and_conquer_mds(x, mds.AlgorithmParams(r=5, l=400, c=10, seed=3),
                                         return_device=True)
        assert isinstance(cfg.points, torch.Tensor) and cfg.points.is_cuda
        host = mds.divide_and_conquer_mds(scenario_data, mds.AlgorithmParams(r=5, l=400, c=10, seed=3))
        assert np.array_equal(cfg.points.cpu().numpy(), host.points)


class TestProcrustesBatched:
    """The batched fit kernels (Newton-Schulz polar factor with the
    lane-group Jacobi kernel taking the fits it does not converge on, for
    r <= 16; the warp kernel above) against the oracle restatement of
    procrustes.py:46-78 on many jobs at once: every r up to 16, uneven job
    sizes, rank-deficient cross products (collinear / constant sources),
    near-singular and strongly anisotropic ones."""

    @staticmethod
    def _batch(mds, tgts, srcs, r):
        import torch
        from paper_2007_11919_b200 import _device as D
        dev = D.require_device(None)
        sizes = [len(t) for t in tgts]
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        tt = torch.from_numpy(np.ascontiguousarray(np.concatenate(tgts))).to(dev)
        ss = torch.from_numpy(np.ascontiguousarray(np.concatenate(srcs))).to(dev)
        rows = torch.arange(int(off[-1]), dtype=torch.int64, device=dev)
        nj = len(tgts)
        rot, tr = D.empty((nj, r, r), dev), D.empty((nj, r), dev)
        loss, deg = D.empty((nj,), dev), torch.empty(nj, dtype=torch.int32, device=dev)
        D.handle(dev).call("mdsx_procrustes_fit", tt.data_ptr(), rows.data_ptr(), ss.data_ptr(),
                           rows.data_ptr(), off.ctypes.data, nj, r, rot.data_ptr(), tr.data_ptr(),
                           loss.data_ptr(), deg.data_ptr(), D.stream_ptr(dev))
        return rot.cpu().numpy(), tr.cpu().numpy(), loss.cpu().numpy(), deg.cpu().numpy()

    @pytest.mark.parametrize("r", list(range(1, 17)))
    def test_matches_oracle(self, mds, r, monkeypatch):
        from oracle import mds_oracle as orc
        rng = np.random.default_rng(100 + r)
        tgts, srcs = [], []
        for j in range(77):
            k = int(rng.integers(max(2, r), 3 * r + 4))
            t = rng.standard_normal((k, r)) * rng.uniform(0.1, 20.0)
            if j % 11 == 3 and r > 1:      # rank-deficient source: one column repeated
                s = rng.standard_normal((k, r))
                s[:, -1] = s[:, 0]
            elif j % 11 == 7:              # constant source: zero cross product
                s = np.ones((k, r))
            elif j % 11 in (5, 9):         # spread singular values: near-singular (Jacobi
                q, _ = np.linalg.qr(rng.standard_normal((r, r)))     # redo) / anisotropic
                sv = np.logspace(0, -9 if j % 11 == 5 else -2, r)
                s = (t - t.mean(axis=0)) @ q * sv + rng.standard_normal(r)
            else:
                q, _ = np.linalg.qr(rng.standard_normal((r, r)))
                s = t @ q + rng.standard_normal((k, r)) * 0.1 + rng.standard_normal(r)
            tgts.append(t)
            srcs.append(s)
        rot, tr, loss, deg = self._batch(mds, tgts, srcs, r)
        monkeypatch.setenv("MDSX_FIT_WARP", "1")
        rot_w, tr_w, loss_w, deg_w = self._batch(mds, tgts, srcs, r)
        for j, (t, s) in enumerate(zip(tgts, srcs)):
            ref = orc.procrustes_fit(t, s)
            assert bool(deg[j]) == ref.degenerate == bool(deg_w[j])
            scale = max(1.0, np.abs(t).max())
            # orthogonality and the optimal loss hold whatever completion a degenerate fit takes
            assert np.abs(rot[j] @ rot[j].T - np.eye(r)).max() <= 1e-10
            assert abs(loss[j] - ref.loss) <= 1e-9 * max(ref.loss, scale ** 2 * len(t))
            res = t - s @ rot[j] - tr[j]
            assert abs(np.sum(res * res) - loss[j]) <= 1e-9 * max(loss[j], scale ** 2)
            if not ref.degenerate:
                assert np.abs(rot[j] - ref.rotation).max() <= 1e-9
                assert np.abs(rot[j] - rot_w[j]).max() <= 1e-12
                assert np.abs(tr[j] - ref.translation).max() <= 1e-9 * scale


def test_fast_finish_c_abi(cuda):
    """mdsx_fast_finish (include/mdsx.h): out[order[i]] = P[i] @ T_j + t_j - mean
    for the rows i of job j, mean = column mean of the result — against numpy,
    with uneven job sizes (several CTAs per job) and a random row order."""
    import torch
    from paper_2007_11919_b200 import _device as D
    rng = np.random.default_rng(77)
    r = 7
    sizes = np.array([1, 5000, 2300, 3, 1024, 2049])
    n = int(sizes.sum())
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    P = rng.standard_normal((n, r)) * 3.0 + 1.5
    rots = np.stack([np.linalg.qr(rng.standard_normal((r, r)))[0] for _ in sizes])
    trans = rng.standard_normal((len(sizes), r)) * 10.0
    order = rng.permutation(n).astype(np.int64)
    want = np.empty((n, r))
    for j in range(len(sizes)):
        want[order[off[j]:off[j + 1]]] = P[off[j]:off[j + 1]] @ rots[j] + trans[j]
    want -= want.mean(axis=0)
    dev = D.require_device(None)
    Pd = torch.from_numpy(P).to(dev)
    rd = torch.from_numpy(np.ascontiguousarray(rots)).to(dev)
    td = torch.from_numpy(np.ascontiguousarray(trans)).to(dev)
    od = torch.from_numpy(order).to(dev)
    out = D.empty((n, r), dev)
    D.handle(dev).call("mdsx_fast_finish", Pd.data_ptr(), r, off.ctypes.data, len(sizes),
                       rd.data_ptr(), td.data_ptr(), od.data_ptr(), n, out.data_ptr(),
                       D.stream_ptr(dev))
    got = out.cpu().numpy()
    assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max()
    assert np.abs(got.mean(axis=0)).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("nbytes,dtype", [(5 << 20, np.float64), ((100 << 20) + 24, np.float64),
                                          ((37 << 20) + 4, np.float32)])
def test_staged_h2d(cuda, nbytes, dtype):
    """mdsx_h2d: pageable host -> device through the pinned chunk rings of the
    host thread pool, exact, with odd sizes (last chunk partial) and the
    source overwritten right after the call returns."""
    from paper_2007_11919_b200 import _device as D
    count = nbytes // np.dtype(dtype).itemsize
    src = np.random.default_rng(count).standard_normal(count).astype(dtype)
    want = src.copy()
    got = D.from_host(src, cuda)
    src[:] = -1.0                                     # the call has finished reading the source
    assert np.array_equal(got.cpu().numpy(), want)


def test_two_threads_share_a_handle(cuda):
    """Two host threads on two torch streams call the library through ONE
    handle (shared workspace and staging): each result equals its
    single-threaded run bitwise (calls are serialised and stream-ordered)."""
    import threading

    import torch
    import paper_2007_11919_b200 as mds_
    from paper_2007_11919_b200.synthetic import scenario
    xs = [scenario(40_000, 30, 5, seed=s) for s in (1, 2)]
    prm = [mds_.AlgorithmParams(r=5, l=700, c=12, seed=3), mds_.AlgorithmParams(r=5, l=900, seed=4)]
    names = ["divide", "interpolate"]
    want = [mds_.run_algorithm(nm, x, p) for nm, x, p in zip(names, xs, prm)]
    got = [None, None]

    def work(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(4):
                got[i] = mds_.run_algorithm(names[i], xs[i], prm[i])

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for a, b in zip(got, want):
        assert np.array_equal(a.points, b.points)
        assert np.array_equal(a.eigenvalue_estimates, b.eigenvalue_estimates)


@pytest.mark.parametrize("n,kind", [(1, "rand"), (2, "rand"), (3, "rand"), (113, "rand"),
                                    (300, "centred_delta"), (257, "clustered"), (640, "low_rank"),
                                    (1500, "rand")])
def test_sym_eigvals_against_lapack(cuda, n, kind):
    """mdsx_sym_eigvals (Householder tridiagonalisation + bisection, no library
    call) against LAPACK dsyevd: every eigenvalue within 1e-12 ||A||, for
    indefinite, clustered (repeated) and rank-deficient spectra."""
    import torch
    from paper_2007_11919_b200 import _device as D
    rng = np.random.default_rng(n)
    if kind == "rand":
        a = rng.standard_normal((n, n))
        a = a + a.T
    elif kind == "centred_delta":                 # doubly centred non-Euclidean delta
        x = rng.standard_normal((n, 5))
        d = ((x[:, None, :] - x[None, :, :]) ** 2).sum(-1) + rng.uniform(0, 0.3, (n, n))
        d = (d + d.T) / 2
        np.fill_diagonal(d, 0)
        j = np.eye(n) - 1.0 / n
        a = -0.5 * j @ d @ j
    elif kind == "clustered":
        q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = np.repeat([5.0, -2.0, 1e-3, 0.0], (n + 3) // 4)[:n]
        a = (q * lam) @ q.T
        a = (a + a.T) / 2
    else:
        y = rng.standard_normal((n, 7))
        a = y @ y.T
    want = np.linalg.eigvalsh(a)
    ad = torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    w = D.empty((n,), cuda)
    D.handle(cuda).call("mdsx_sym_eigvals", ad.data_ptr(), n, w.data_ptr(), D.stream_ptr(cuda))
    got = w.cpu().numpy()
    scale = max(np.abs(want).max(), 1e-300)
    assert np.abs(got - want).max() <= 1e-12 * scale * max(1.0, n / 500), (
        np.abs(got - want).max() / scale)
    assert np.array_equal(ad.cpu().numpy(), a)      # input untouched
