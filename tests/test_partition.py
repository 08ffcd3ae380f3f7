"""partition.balance vs the reference examples and brute force (acceptance #4)."""

import numpy as np
import pytest

from oracle.partition import brute_force_balance, objective
from paper_2210_09147_b200 import partition


def test_examples():
    assert partition.balance([3, 1, 1, 3], 2) == ([2, 2], 4)
    assert partition.balance([3, 1, 1, 3], 1) == ([4], 8)
    assert partition.balance([3, 1, 1, 3], 4) == ([1, 1, 1, 1], 3)


def test_d_greater_than_l():
    with pytest.raises(ValueError, match="D=5 > L=4"):
        partition.balance([1, 1, 1, 1], 5)


def test_optimality_vs_brute_force():
    rng = np.random.default_rng(0)
    for _ in range(500):
        L = int(rng.integers(1, 13))
        D = int(rng.integers(1, L + 1))
        costs = list(rng.integers(0, 20, L).astype(float))
        counts, best = partition.balance(costs, D)
        ref_counts, ref_best = brute_force_balance(costs, D)
        assert best == ref_best
        assert counts == ref_counts  # leftmost tie-breaking
        cuts = np.cumsum(counts)[:-1]
        assert objective(costs, cuts) == best


def test_transfer_term_charged_downstream():
    rng = np.random.default_rng(1)
    for _ in range(200):
        L = int(rng.integers(2, 10))
        D = int(rng.integers(1, L + 1))
        costs = list(rng.integers(0, 10, L).astype(float))
        tr = list(rng.integers(0, 5, L).astype(float))
        counts, best = partition.balance(costs, D, tr)
        ref_counts, ref_best = brute_force_balance(costs, D, tr)
        assert best == ref_best and counts == ref_counts


def test_monotone_in_d():
    rng = np.random.default_rng(2)
    for _ in range(100):
        L = int(rng.integers(1, 12))
        costs = list(rng.integers(0, 20, L).astype(float))
        vals = [partition.balance(costs, D)[1] for D in range(1, L + 1)]
        assert all(a >= b for a, b in zip(vals, vals[1:]))


def test_mlp_costs_and_c5_plan():
    """Config 5 (uneven widths) is balanced on algorithmic bytes."""
    dims = [1024, 2048, 4096, 8192, 8192, 4096, 2048, 1024] * 3 + [1024]
    costs, boundary = partition.mlp_costs(dims)
    assert len(costs) == 24 and costs[3] == 12 * 8192 * 8192
    for D in (2, 4, 8):
        counts, best = partition.balance(costs, D)
        assert sum(counts) == 24 and len(counts) == D
        assert best >= sum(costs) / D


# ---- CostProfile / balance_profile / assign_workers

def _profile(f, b=None, bb=None, tpb=0.0, hc=None):
    L = len(f)
    return partition.CostProfile(list(f), list(b if b is not None else [0.0] * L),
                                 list(bb if bb is not None else [0] * L), tpb, list(hc or []))


def test_balance_profile_modes_and_prediction():
    prof = _profile([3, 1, 1, 3], [0, 0, 0, 0])
    plan = partition.balance_profile(prof, 2, "inference")
    assert plan.layer_counts() == [2, 2] and plan.predicted_stage_cost == [4, 4]
    # learning adds the backward cost
    prof = _profile([1, 1, 1, 1], [5, 0, 0, 0])
    plan = partition.balance_profile(prof, 2, "learning")
    assert plan.layer_counts() == [1, 3] and max(plan.predicted_stage_cost) == 6
    # transfer charged downstream: bytes * seconds/byte on the stage after the boundary
    prof = _profile([2, 2, 2, 2], bb=[0, 100, 0, 0], tpb=0.01)
    plan = partition.balance_profile(prof, 2, "inference")
    assert plan.predicted_stage_cost[1] == 4 + (1.0 if plan.layer_counts()[0] == 2 else 0.0)
    with pytest.raises(ValueError):
        partition.balance_profile(prof, 2, "training")


def test_cost_profile_invariants():
    with pytest.raises(ValueError):
        _profile([1, -1])
    with pytest.raises(ValueError):
        partition.CostProfile([1, 1], [1], [0, 0], 0.0)


def test_assign_workers_examples():
    plan = partition.balance_profile(_profile([1, 1, 1, 1]), 4, "inference")
    assert partition.assign_workers(plan, _profile([1, 1, 1, 1], hc=[2, 2, 2, 2])).worker_assignment == [0, 1, 2, 3]
    # host_copy_cost [5, 1, 1, 5]: stage 1 and stage D on workers 2 and 3 (1-based)
    a = partition.assign_workers(plan, _profile([1, 1, 1, 1], hc=[5, 1, 1, 5])).worker_assignment
    assert {a[0], a[3]} == {1, 2} and sorted(a) == [0, 1, 2, 3]
    # 4 stages on 2 workers -> round-robin [1, 2, 1, 2] (0-based [0, 1, 0, 1])
    assert partition.assign_workers(plan, _profile([1, 1, 1, 1], hc=[1, 1]), n_workers=2).worker_assignment == [0, 1, 0, 1]
