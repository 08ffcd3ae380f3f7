"""profile_costs on the B200: timed per-layer medians from the tick
kernel's device trace, then balance + assign_workers over the measured profile."""

import numpy as np
import pytest

from paper_2210_09147_b200 import model as mdl, partition

pytestmark = pytest.mark.gpu


def test_profile_costs_measures_wide_layers_as_costlier():
    # unit 1 (2048 x 2048, 16 MB) streams 8x the weight bytes of units 0 and 2 (2 MB each)
    m = mdl.mlp([256, 2048, 2048, 256, 256], act="relu", seed=0)
    prof = partition.profile_costs(m, np.ones(256, np.float32), iters=5, warmup_iters=2)
    L = len(m.dense_layers)
    assert len(prof.fwd_cost) == L and len(prof.bwd_cost) == L and len(prof.boundary_bytes) == L
    assert all(c > 0 for c in prof.fwd_cost) and all(c > 0 for c in prof.bwd_cost)
    assert prof.boundary_bytes == [4 * 2048, 4 * 2048, 4 * 256, 4 * 256]
    assert prof.transfer_cost_per_byte > 0 and len(prof.host_copy_cost) >= 1
    assert sum(prof.unit_layers) == len(m.layers)
    # the 2048 x 2048 unit is the costliest in learning mode
    learn = [f + b for f, b in zip(prof.fwd_cost, prof.bwd_cost)]
    assert int(np.argmax(learn)) == 1, learn
    plan = partition.balance_profile(prof, 2, "learning")
    assert sum(plan.layer_counts()) == len(m.layers) and len(plan.predicted_stage_cost) == 2
    plan = partition.assign_workers(plan, prof, n_workers=2)
    assert sorted(plan.worker_assignment) == [0, 1]
