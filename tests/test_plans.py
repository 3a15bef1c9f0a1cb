"""Host planner: bit-exact with the reference (digests of the reference's own
plans at BASELINE sizes, tests/golden/plan_digests.npz) and the reference's
partition tests (tests/test_partition.py) re-run against this planner."""

import json

import numpy as np
import pytest

from conftest import golden
from paper_2007_11919_b200 import ParamError, fast_stats, plans
from paper_2007_11919_b200.plans import (flatten_fast, flatten_subsets, interpolation_sample,
                                         plan_divide_conquer, plan_fast, plan_interpolation)
from test_oracle import digest


def leaves_digest(plan):
    return digest([leaf.indices for leaf in plan.leaves()])


def positions_digest(plan):
    out, stack = [], [plan.root]
    while stack:
        node = stack.pop()
        if node.sampling_positions is not None:
            out.append(node.sampling_positions)
        stack.extend(reversed(node.children))
    return digest(out)


class TestBaselinePlansBitExact:
    def test_divide_config2(self):
        g = golden("plan_digests")
        plan = plan_divide_conquer(1_000_000, 1000, 20, 0)
        assert plan.p == int(g["dc_1e6_p"]) == 1021
        assert digest(plan.subsets) == str(g["dc_1e6"])

    def test_fast_config3(self):
        g = golden("plan_digests")
        plan = plan_fast(1_000_000, 1000, 20, 0)
        assert leaves_digest(plan) == str(g["fast_1e6_leaves"])
        assert positions_digest(plan) == str(g["fast_1e6_positions"])
        assert digest([plan.root.indices]) == str(g["fast_1e6_root"])

    @pytest.mark.slow
    def test_interp_config4(self):
        g = golden("plan_digests")
        plan = plan_interpolation(10_000_000, 2000, 0)
        assert plan.p == int(g["interp_1e7_p"])
        assert digest(plan.subsets) == str(g["interp_1e7"])
        assert np.array_equal(interpolation_sample(10_000_000, 2000, 0), plan.subsets[0])

    def test_config5_plans(self):
        g = golden("plan_digests")
        assert digest(plan_divide_conquer(814_255, 1000, 20, 0).subsets) == str(g["dc_cfg5"])
        fp = plan_fast(814_255, 1000, 20, 0)
        assert leaves_digest(fp) == str(g["fast_cfg5_leaves"])
        assert positions_digest(fp) == str(g["fast_cfg5_positions"])
        assert digest(plan_interpolation(814_255, 1000, 0).subsets) == str(g["interp_cfg5"])


def assert_exact_cover(arrays, n):
    merged = np.concatenate([np.asarray(a) for a in arrays])
    assert len(merged) == n and np.array_equal(np.sort(merged), np.arange(n))


class TestReferencePartitionContracts:
    """tests/test_partition.py of the reference, against this planner."""

    def test_divide_sizes_and_merge(self):
        assert plan_divide_conquer(1000, 400, 20, seed=0).p == 3
        assert [len(s) for s in plan_divide_conquer(1000, 400, 20, seed=5).subsets] == [400, 400, 240]
        plan = plan_divide_conquer(285, 100, 10, seed=1)
        assert [len(s) for s in plan.subsets] == [100, 100, 105]
        assert_exact_cover([plan.connecting_indices] + [s[10:] for s in plan.subsets], 285)

    def test_divide_passthrough_and_errors(self):
        plan = plan_divide_conquer(300, 400, 20, seed=0)
        assert plan.p == 1 and np.array_equal(plan.subsets[0], np.arange(300))
        with pytest.raises(ParamError):
            plan_divide_conquer(100, 10, 10, seed=0)

    def test_divide_audit_1e6(self):
        plan = plan_divide_conquer(1_000_000, 400, 20, seed=123)
        for s in plan.subsets:
            assert np.array_equal(s[:20], plan.connecting_indices)
        assert_exact_cover([plan.connecting_indices] + [s[20:] for s in plan.subsets], 1_000_000)

    def test_json_round_trips(self):
        plan = plan_divide_conquer(50, 20, 4, seed=2)
        assert json.loads(plan.to_json())["subsets"] == [s.tolist() for s in plan.subsets]
        fp = plan_fast(50, 20, 5, seed=2)
        assert len(json.loads(fp.to_json())["tree"]["children"]) == 4

    def test_interp_sizes(self):
        assert [len(s) for s in plan_interpolation(10, 4, seed=0).subsets] == [4, 4, 2]
        for n, l in [(10, 4), (1001, 100), (999, 100), (1000, 100)]:
            assert plan_interpolation(n, l, seed=0).p == -(-n // l)
        plan = plan_interpolation(100_000, 1000, seed=11)
        assert_exact_cover(plan.subsets, 100_000)
        with pytest.raises(ParamError):
            plan_interpolation(10, 1, seed=0)

    def test_fast_structure_and_stats(self):
        for n, l, s in [(20_000, 700, 20), (5_000, 300, 10), (999, 100, 7)]:
            plan = plan_fast(n, l, s, seed=4)
            st = plan.stats()
            pure = fast_stats(n, l, s)
            assert (st.leaf_count, st.depth) == (pure.leaf_count, pure.depth)
            assert_exact_cover([leaf.indices for leaf in plan.leaves()], n)
        d = fast_stats(1_000_000, 700, 20)
        assert d.leaf_count == 42_875 and d.depth == 3 and abs(d.mean_leaf_size - 23.32) < 0.01
        s = fast_stats(1_000_000, 800, 20)
        assert s.leaf_count == 1600 and s.mean_leaf_size == 625.0 and s.depth == 2
        with pytest.raises(ParamError):
            plan_fast(100, 30, 20, seed=0)


class TestFlatteners:
    def test_subsets(self):
        rows, off = flatten_subsets([np.array([3, 1]), np.array([0, 2, 4])])
        assert rows.tolist() == [3, 1, 0, 2, 4] and off.tolist() == [0, 2, 5]

    def test_fast_flat_consistent(self):
        plan = plan_fast(5000, 100, 10, seed=4)
        flat = flatten_fast(plan)
        assert np.array_equal(flat.order, plan.root.indices)
        leaves = plan.leaves()
        assert flat.n_leaves == len(leaves)
        assert np.array_equal(flat.piece_rows[:5000], plan.root.indices)
        # every job's source rows index its child's range; targets index alignment pieces
        for lv in flat.levels:
            for t in range(len(lv.start)):
                src = lv.src_rows[lv.job_off[t]:lv.job_off[t + 1]]
                assert src.min() >= lv.start[t] and src.max() < lv.start[t] + lv.length[t]
                tgt = lv.tgt_rows[lv.job_off[t]:lv.job_off[t + 1]]
                assert tgt.min() >= 5000
        assert sorted(flat.eval_order) == list(range(len(flat.piece_off) - 1))


def test_native_permutation_and_choices_match_numpy():
    """mdsx_plan_permute / mdsx_plan_choices (the native planner) against
    numpy's Generator on PCG64: identical outputs AND identical generator
    state afterwards (including the buffered 32-bit half), for populations
    that take numpy's Floyd and tail-shuffle paths."""
    from paper_2007_11919_b200 import plans
    rng = np.random.default_rng(5)
    for trial in range(400):
        seed = int(rng.integers(0, 1 << 30))
        g1 = np.random.Generator(np.random.PCG64(seed))
        g2 = np.random.Generator(np.random.PCG64(seed))
        if trial % 2:                                  # leave a buffered 32-bit half
            g1.integers(0, 7)
            g2.integers(0, 7)
        n = int(rng.choice([5000, 4096, 20000, 123457]))
        a = np.arange(n, dtype=np.int64) * 3
        assert np.array_equal(plans._permutation(g1, a), g2.permutation(a))
        s = int(rng.integers(1, 60))
        pops = [max(int(q), s + 1) for q in rng.choice(
            [rng.integers(1, 100), rng.integers(100, 12000), rng.integers(10000, 200000),
             50 * s, 50 * s + 1], size=int(rng.integers(1, 5)))]
        got = plans._choices_sorted(g1, pops, s)
        want = [np.sort(g2.choice(q, size=min(s, q), replace=False)) for q in pops]
        assert all(np.array_equal(x, y) for x, y in zip(got, want))
        assert g1.bit_generator.state == g2.bit_generator.state
