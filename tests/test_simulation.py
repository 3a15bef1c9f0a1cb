"""The reference's metric tests (tests/test_simulation.py) re-expressed against
the drop-in ``simulation`` module (device metrics), plus parity of the device
aligned_correlations with a NumPy restatement of simulation.py:83-108 and of
the single-solve gof_sweep with the reference's per-h loop."""

import dataclasses

import numpy as np
import pytest

from paper_2007_11919_b200 import AlgorithmParams, MetricError, ParamError
from paper_2007_11919_b200.synthetic import scenario


def ref_aligned(points, dominant):
    """NumPy restatement of simulation.py:83-108 (fit_procrustes + apply +
    centred Pearson), the oracle for the device metric."""
    t = dominant - dominant.mean(axis=0)
    s = points - points.mean(axis=0)
    u, _, vt = np.linalg.svd(t.T @ s)
    rot = vt.T @ u.T
    a = points @ rot
    a = a - a.mean(axis=0)
    return np.einsum("ij,ij->j", a, t) / (np.sqrt(np.einsum("ij,ij->j", a, a)) *
                                          np.sqrt(np.einsum("ij,ij->j", t, t)))


@pytest.mark.gpu
class TestAlignedCorrelations:
    @pytest.fixture()
    def config(self, cuda):
        from paper_2007_11919_b200 import classical_mds_from_data
        data = scenario(400, 6, 3, seed=9)
        return classical_mds_from_data(data, 3), data[:, :3]

    def test_identity_rotation_reflection(self, config):
        from paper_2007_11919_b200 import aligned_correlations
        cfg, dom = config
        assert np.allclose(aligned_correlations(dataclasses.replace(cfg, points=dom.copy()), dom),
                           1.0, atol=1e-12)
        basis, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((3, 3)))
        assert np.allclose(aligned_correlations(dataclasses.replace(cfg, points=dom @ basis), dom),
                           1.0, atol=1e-9)
        assert np.allclose(aligned_correlations(dataclasses.replace(cfg, points=-dom), dom),
                           1.0, atol=1e-9)

    def test_invariant_under_rigid_motion(self, config):
        from paper_2007_11919_b200 import aligned_correlations
        cfg, dom = config
        basis, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((3, 3)))
        moved = dataclasses.replace(cfg, points=cfg.points @ basis + [4.0, -1.0, 0.5])
        assert np.abs(aligned_correlations(moved, dom) - aligned_correlations(cfg, dom)).max() <= 1e-9

    def test_zero_variance_column(self, config):
        from paper_2007_11919_b200 import aligned_correlations
        cfg, dom = config
        flat = dom.copy()
        flat[:, 1] = 2.5
        with pytest.raises(MetricError):
            aligned_correlations(cfg, flat)

    @pytest.mark.parametrize("n,r,f32", [(400, 3, False), (100_003, 10, False), (5000, 16, True),
                                         (2, 1, False)])
    def test_parity_with_numpy(self, cuda, n, r, f32):
        import torch
        from paper_2007_11919_b200 import aligned_correlations
        from paper_2007_11919_b200.results import MdsConfiguration
        rng = np.random.default_rng(n + r)
        data = rng.standard_normal((n, r + 3)) * 3.0 + 7.0
        if f32:
            data = data.astype(np.float32)
        dom = data[:, :r]
        pts = dom.astype(np.float64) @ np.linalg.qr(rng.standard_normal((r, r)))[0] + \
            0.3 * rng.standard_normal((n, r)) + 11.0
        cfg = MdsConfiguration(pts, np.ones(r), 1.0, 1.0)
        want = ref_aligned(pts, dom.astype(np.float64))
        got = aligned_correlations(cfg, dom)
        assert np.abs(got - want).max() <= 1e-12 * max(1, n / 1e4)
        # device tensors (strided column view of the data matrix) give the same
        xd = torch.from_numpy(data).cuda()
        got2 = aligned_correlations(cfg, xd[:, :r])
        assert np.array_equal(got, got2)


@pytest.mark.gpu
class TestGofSweep:
    def _dominant(self, seed):
        data = np.random.default_rng(seed).standard_normal((1500, 5))
        data[:, 0] *= np.sqrt(95.0)
        data[:, 1:] *= np.sqrt(5.0 / 4.0)
        return data

    def test_reference_cases(self, cuda):
        from paper_2007_11919_b200 import gof_sweep
        assert gof_sweep(self._dominant(8), "classical", AlgorithmParams(r=1), 0.8) == 1
        assert gof_sweep(self._dominant(9), "divide", AlgorithmParams(r=1, l=400), 0.8) == 1
        iso = np.random.default_rng(10).standard_normal((2000, 10))
        assert gof_sweep(iso, "classical", AlgorithmParams(r=1), 0.8) == 8
        full = np.random.default_rng(11).standard_normal((500, 6))
        assert gof_sweep(full, "classical", AlgorithmParams(r=1), 1.0) == 6
        with pytest.raises(ParamError, match="unreachable"):
            gof_sweep(np.random.default_rng(11).standard_normal((2000, 6)), "divide",
                      AlgorithmParams(r=1, l=400, c=3), 0.99)
        with pytest.raises(ParamError):
            gof_sweep(np.zeros((20, 2)), "classical", AlgorithmParams(r=1), 0.0)

    @pytest.mark.parametrize("algo,kw", [("classical", {}), ("divide", dict(l=500, c=12)),
                                         ("interpolate", dict(l=600)), ("fast", dict(l=800, s=12))])
    def test_curve_matches_per_h_runs(self, cuda, algo, kw):
        """One run at h_cap gives every G1(h) of the reference's per-h loop."""
        from paper_2007_11919_b200 import g1_curve, run_algorithm
        data = scenario(4000, 12, 4, seed=2)
        params = AlgorithmParams(r=1, **kw)
        curve = g1_curve(data, algo, params, 10)
        for h in range(1, 11):
            g = run_algorithm(algo, data, dataclasses.replace(params, r=h)).gof_g1
            assert abs(curve[h - 1] - g) <= 1e-12, (h, curve[h - 1], g)
