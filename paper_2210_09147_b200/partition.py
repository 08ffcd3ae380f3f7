"""Stage balancing (reference `partition` module).

balance() is the min-max contiguous partition of SPEC.md:147-156. It is
computed by dynamic programming; ties go to the leftmost boundaries, and
the transfer term is charged to the downstream stage.
mlp_costs() is the byte-cost profile that the B200 path is bound by.
Per-layer cost is the algorithmic HBM bytes per tick: 12 n_in n_out learning
(one W read in the forward pass, one W read and write in the fused
backward+update), 4 n_in n_out inference. This stands in for the timed
medians of profile_costs because every kernel here is
HBM-bound.
"""

from __future__ import annotations

from functools import lru_cache


def balance(costs, D, transfer=None):
    """Layer counts of the min-max contiguous split of `costs` into D blocks.

    Returns (counts, max_stage_cost). For a boundary placed after layer j,
    transfer[j] is added to the cost of the stage that starts at j+1.
    """
    L = len(costs)
    if D < 1:
        raise ValueError("D must be >= 1")
    if D > L:
        raise ValueError(f"D={D} > L={L} (SPEC.md:151)")
    pre = [0.0]
    for c in costs:
        pre.append(pre[-1] + c)

    def block(i, j):  # layers [i, j)
        c = pre[j] - pre[i]
        if i > 0 and transfer is not None:
            c += transfer[i - 1]
        return c

    @lru_cache(maxsize=None)
    def best(i, h):  # min max cost splitting [i, L) into h blocks
        if h == 1:
            return block(i, L)
        return min(max(block(i, j), best(j, h - 1)) for j in range(i + 1, L - h + 2))

    opt = best(0, D)
    counts, i = [], 0
    for h in range(D, 1, -1):  # leftmost boundary that still achieves the optimum
        for j in range(i + 1, L - h + 2):
            if block(i, j) <= opt and best(j, h - 1) <= opt:
                counts.append(j - i)
                i = j
                break
    counts.append(L - i)
    best.cache_clear()
    return counts, opt


def mlp_costs(dims, learn=True):
    """Bytes per tick per fused dense layer, and boundary bytes (fp32, M=1)."""
    per = 12 if learn else 4
    costs = [per * dims[i] * dims[i + 1] for i in range(len(dims) - 1)]
    boundary = [4 * dims[i + 1] for i in range(len(dims) - 1)]
    return costs, boundary
