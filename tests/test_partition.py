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
