"""balance_pipeline_partitions.

The paper times host copies and per-layer compute, then splits the layers so
that the stages' times are similar. On B200 every stage kernel is bound by HBM
bandwidth, so the per-layer cost used here is the algorithmic bytes per tick
(partition.mlp_costs) rather than a timed median. The split is the min-max
contiguous DP, with leftmost ties. The result is a
module-count list over the Sequential, e.g. [8, 10, 12, 11], in which each
Linear keeps the activation that follows it.
"""

from __future__ import annotations

from .. import partition
from ..model import fuse
from .convert import sequential_to_model


def balance_pipeline_partitions(net, devices, n_stages, learn=True):
    model = sequential_to_model(net)
    return balance_model(model, n_stages, learn)


def balance_model(model, n_stages, learn=True):
    units, owner = fuse(model)
    dims = [model.layers[units[0][0]].in_dim] + [model.layers[u[0]].out_dim for u in units]
    costs, _ = partition.mlp_costs(dims, learn)
    unit_counts, _ = partition.balance(costs, n_stages)
    # expand fused-unit counts back to module counts
    unit_modules = [0] * len(units)
    for o in owner:
        unit_modules[o] += 1
    out, u = [], 0
    for c in unit_counts:
        out.append(sum(unit_modules[u:u + c]))
        u += c
    return out
