"""Column compaction of wide inputs (k_compact.cu): the algorithms on a
matrix with all-zero columns must return the configuration of the matrix
without them (exact-zero terms only) and match the oracle; non-finite values
in an otherwise zero column are still reported."""

import numpy as np
import pytest

from conftest import sign_fixed_rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mds(cuda):
    import paper_2007_11919_b200 as m
    return m


def _wide(n, p_active, p_zero, seed, dtype=np.float64):
    from paper_2007_11919_b200.synthetic import scenario
    core = scenario(n, p_active, 6, seed=seed)
    rng = np.random.default_rng(seed)
    cols = np.sort(rng.choice(p_active + p_zero, p_active, replace=False))
    x = np.zeros((n, p_active + p_zero), dtype=dtype)
    x[:, cols] = core
    return x, cols


@pytest.mark.parametrize("algo,prm", [
    ("divide", dict(r=6, l=600, c=12, seed=2)),
    ("interpolate", dict(r=6, l=500, seed=4)),
    ("fast", dict(r=6, l=900, s=12, seed=5)),
])
def test_compacted_equals_narrow_and_oracle(mds, algo, prm):
    from oracle import mds_oracle as orc
    x, cols = _wide(9_000, 112, 48, seed=7)
    p = mds.AlgorithmParams(**prm)
    got = mds.run_algorithm(algo, x, p)
    narrow = np.zeros((x.shape[0], 112))            # the active columns, 16-byte rows
    narrow[:, :] = x[:, cols]
    ref_gpu = mds.run_algorithm(algo, narrow, p)
    assert sign_fixed_rel_err(got.points, ref_gpu.points) < 1e-12
    ref = orc.run(algo, narrow, prm["r"], l=prm["l"], c=prm.get("c"), s=prm.get("s"),
                            seed=prm["seed"], threads=8)
    assert sign_fixed_rel_err(got.points, ref.points) < 1e-9
    assert np.allclose(got.eigenvalue_estimates, ref.estimates, rtol=1e-9)


def test_compaction_fp32_and_nonfinite(mds):
    from paper_2007_11919_b200.errors import InvalidInputError
    x, cols = _wide(6_000, 120, 60, seed=3, dtype=np.float32)
    p = mds.AlgorithmParams(r=5, l=700, c=10, seed=1)
    got = mds.divide_and_conquer_mds(x, p)
    narrow = np.ascontiguousarray(x[:, cols])
    assert sign_fixed_rel_err(got.points, mds.divide_and_conquer_mds(narrow, p).points) < 1e-12
    zero_col = np.setdiff1d(np.arange(x.shape[1]), cols)[0]
    x[123, zero_col] = np.nan                       # a NaN keeps its column active
    with pytest.raises(InvalidInputError):
        mds.divide_and_conquer_mds(x, p)
