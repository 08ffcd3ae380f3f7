"""partition oracle: brute-force min-max contiguous split. TEST INFRASTRUCTURE ONLY.

Restates the objective of SPEC.md:147-156 and the optimality property of
SPEC.md:168. The search is exhaustive over all C(L-1, D-1) partitions, which
is feasible for L <= 12. Ties go to the leftmost boundary.
The cost of block h is the sum of cost[i] over the block, plus
transfer[b_{h-1}] when h > 1. transfer[j] is the cost of a boundary placed
after layer j, and it is charged to the downstream stage.
"""

from __future__ import annotations

import itertools


def objective(costs, cuts, transfer=None):
    """Max stage cost for boundaries `cuts` (layer counts before each cut, strictly increasing)."""
    bounds = [0] + list(cuts) + [len(costs)]
    worst = 0.0
    for h in range(len(bounds) - 1):
        c = sum(costs[bounds[h]:bounds[h + 1]])
        if h > 0 and transfer is not None:
            c += transfer[bounds[h] - 1]
        worst = max(worst, c)
    return worst


def brute_force_balance(costs, D, transfer=None):
    L = len(costs)
    if D > L:
        raise ValueError(f"D={D} > L={L}")
    best, best_cuts = None, None
    for cuts in itertools.combinations(range(1, L), D - 1):  # lexicographic = leftmost first
        v = objective(costs, cuts, transfer)
        if best is None or v < best:
            best, best_cuts = v, cuts
    return [b - a for a, b in zip((0,) + best_cuts, best_cuts + (L,))], best
