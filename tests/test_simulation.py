"""The reference's tests/test_simulation.py re-expressed against the drop-in
``simulation`` module (device metrics), plus parity of the device
aligned_correlations with a NumPy restatement of simulation.py:83-108 and of
the single-solve gof_sweep with the reference's per-h loop."""

import csv
import dataclasses

import numpy as np
import pytest

from paper_2007_11919_b200 import (AlgorithmParams, MetricError, ParamError, ScenarioSpec,
                                   eigenvalue_error_stats, generate_scenario)

REF_SRC = "/root/reference/pkg/src"


class TestGenerateScenario:
    def test_dominant_and_noise_variance(self):
        data = generate_scenario(ScenarioSpec(n=100_000, k=4, h=2, seed=0), 0)
        assert 14.5 <= data[:, 0].var() <= 15.5
        assert 0.97 <= data[:, 3].var() <= 1.03

    def test_columns_uncorrelated(self):
        data = generate_scenario(ScenarioSpec(n=100_000, k=4, h=2, seed=1), 0)
        corr = np.corrcoef(data, rowvar=False)
        assert np.abs(corr[~np.eye(4, dtype=bool)]).max() <= 0.02

    def test_deterministic_per_seed_and_replication(self):
        spec = ScenarioSpec(n=200, k=3, h=1, seed=5)
        assert np.array_equal(generate_scenario(spec, 2), generate_scenario(spec, 2))
        assert not np.array_equal(generate_scenario(spec, 2), generate_scenario(spec, 3))

    def test_validation(self):
        with pytest.raises(ParamError):
            generate_scenario(ScenarioSpec(n=100, k=3, h=4, seed=0), 0)
        with pytest.raises(ParamError):
            generate_scenario(ScenarioSpec(n=5, k=3, h=1, seed=0), 0)

    @pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference absent")
    def test_bit_exact_against_reference(self):
        import importlib
        import sys
        sys.path.insert(0, REF_SRC)
        try:
            ref = importlib.import_module("scalemds.simulation")
        finally:
            sys.path.remove(REF_SRC)
        for kw in (dict(n=1000, k=10, h=3, seed=5), dict(n=101, k=7, h=2, seed=1,
                                                          dominant_sd=2.0, noise_sd=0.5)):
            for rep in (0, 3):
                assert np.array_equal(generate_scenario(ScenarioSpec(**kw), rep),
                                      ref.generate_scenario(ref.ScenarioSpec(**kw), rep))


class TestEigenvalueErrorStats:
    def test_exact_estimates(self):
        bias, mse = eigenvalue_error_stats(np.full((5, 3), 15.0))
        assert np.array_equal(bias, np.zeros(3)) and np.array_equal(mse, np.zeros(3))

    def test_pairs_and_single(self):
        bias, mse = eigenvalue_error_stats(np.array([[14.0], [16.0]]))
        assert bias[0] == 0.0 and mse[0] == 1.0
        bias, mse = eigenvalue_error_stats(np.array([[12.0]]))
        assert bias[0] == -3.0 and mse[0] == 9.0

    def test_mse_dominates_squared_bias(self):
        est = np.random.default_rng(2).normal(15.0, 2.0, size=(40, 4))
        bias, mse = eigenvalue_error_stats(est)
        assert np.all(mse >= bias ** 2 - 1e-9)


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
        data = generate_scenario(ScenarioSpec(n=400, k=6, h=3, seed=9), 0)
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


def read_rows(path):
    with open(path, newline="") as handle:
        return list(csv.DictReader(handle))


@pytest.mark.gpu
class TestRunCellStudy:
    def test_metrics_shape_and_bounds(self, cuda):
        from paper_2007_11919_b200 import run_cell
        spec = ScenarioSpec(n=300, k=4, h=2, replications=3, seed=13)
        metrics, rows = run_cell(spec, "classical")
        assert metrics.correlations.shape == (3, 2) and metrics.eigenvalue_estimates.shape == (3, 2)
        assert metrics.elapsed_s.shape == (3,) and len(rows) == 6
        assert np.all(np.abs(metrics.correlations) <= 1.0)

    def test_failed_replication_keeps_going(self, cuda):
        from paper_2007_11919_b200 import run_cell
        spec = ScenarioSpec(n=300, k=4, h=2, replications=2, seed=14)
        metrics, rows = run_cell(spec, "divide", params=AlgorithmParams(r=2, l=150, c=1))
        assert metrics.correlations.shape == (0, 2) and len(rows) == 2
        assert all(row["error"] for row in rows)

    def test_study_rows_resume_reproducible(self, cuda, tmp_path):
        from paper_2007_11919_b200 import run_study
        spec = ScenarioSpec(n=300, k=4, h=3, replications=2, seed=4)
        path = run_study([spec], ["classical", "interpolate"], tmp_path / "a",
                         params={"interpolate": AlgorithmParams(r=3, l=150)})
        rows = read_rows(path)
        assert len(rows) == 2 * 2 * 3 and {row["dim"] for row in rows} == {"1", "2", "3"}
        again = run_study([spec], ["classical", "interpolate"], tmp_path / "a").read_bytes()
        assert again == path.read_bytes()                      # resumed from the cells
        b = run_study([spec], ["classical", "interpolate"], tmp_path / "b",
                      params={"interpolate": AlgorithmParams(r=3, l=150)})

        def strip(p):
            return [{k: v for k, v in row.items() if k != "elapsed_s"} for row in read_rows(p)]
        assert strip(path) == strip(b)

    def test_cell_failure_recorded_not_fatal(self, cuda, tmp_path):
        from paper_2007_11919_b200 import run_study
        spec = ScenarioSpec(n=200, k=3, h=2, replications=1, seed=7)
        rows = read_rows(run_study([spec], ["bogus", "classical"], tmp_path))
        errors = [row for row in rows if row["error"]]
        assert len(errors) == 1 and "bogus" in errors[0]["error"]
        assert len(rows) - len(errors) == 2


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
        data = generate_scenario(ScenarioSpec(n=4000, k=12, h=4, seed=2), 0)
        params = AlgorithmParams(r=1, **kw)
        curve = g1_curve(data, algo, params, 10)
        for h in range(1, 11):
            g = run_algorithm(algo, data, dataclasses.replace(params, r=h)).gof_g1
            assert abs(curve[h - 1] - g) <= 1e-12, (h, curve[h - 1], g)
