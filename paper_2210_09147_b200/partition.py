"""Stage balancing (reference `partition` module).

balance() is the min-max contiguous partition of SPEC.md:147-156. It is
computed by dynamic programming; ties go to the leftmost boundaries, and
the transfer term is charged to the downstream stage.

Two ways to get a CostProfile:
- profile_costs(): the SPEC's timed medians, measured on the B200 from the
  tick kernel's per-step device timestamps;
- byte_profile(): the algorithmic HBM bytes per tick each unit moves (12
  n_in n_out learning: one W read in the forward pass, one W read and write
  in the fused backward+update; 4 n_in n_out inference), a CPU-only stand-in
  that ranks stages the same way because every kernel here is HBM-bound.
balance_profile() splits a profile into D stages and assign_workers() places
the stages on GPUs.
"""

from __future__ import annotations

import os
import statistics
import time
from dataclasses import dataclass, field
from functools import lru_cache

from .model import canonical_loss


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


# --------------------------------------------------------------------------------------------
# CostProfile / profile_costs / balance_profile / assign_workers
# --------------------------------------------------------------------------------------------

@dataclass
class CostProfile:
    """SPEC.md:129-131. One entry per fused dense unit (dense + its activation: a stage
    boundary never splits the pair). Seconds and bytes."""
    fwd_cost: list
    bwd_cost: list
    boundary_bytes: list            # payload if the boundary is placed after unit i
    transfer_cost_per_byte: float   # between workers (NVLink peer, or on-device copy)
    host_copy_cost: list = field(default_factory=list)  # per worker: input + output host transfers
    unit_layers: list = None        # Model.layers per unit (dense [+ activation]); None = 1 each

    def __post_init__(self):
        L = len(self.fwd_cost)
        if len(self.bwd_cost) != L or len(self.boundary_bytes) != L:
            raise ValueError("CostProfile: one entry per layer/boundary")
        if any(c < 0 for c in list(self.fwd_cost) + list(self.bwd_cost) + list(self.boundary_bytes)) \
                or self.transfer_cost_per_byte < 0 or any(c < 0 for c in self.host_copy_cost):
            raise ValueError("CostProfile: all costs must be >= 0")


def byte_profile(model, M=1, seconds_per_byte=1.0 / 7.0e12):
    """CPU-only CostProfile from algorithmic bytes (module docstring); costs in seconds at
    `seconds_per_byte` (default: B200 HBM at ~7 TB/s). The split does not depend on the scale."""
    from .model import fuse
    units, owner = fuse(model)
    dims = [model.layers[units[0][0]].in_dim] + [model.layers[u[0]].out_dim for u in units]
    L = len(units)
    fwd = [4.0 * dims[i] * dims[i + 1] * seconds_per_byte for i in range(L)]
    bwd = [8.0 * dims[i] * dims[i + 1] * seconds_per_byte for i in range(L)]
    boundary = [4 * M * d for d in dims[1:]]
    unit_layers = [0] * L
    for u in owner:
        unit_layers[u] += 1
    return CostProfile(fwd, bwd, boundary, 0.0, [], unit_layers)


def balance_profile(profile: CostProfile, D, mode="learning"):
    """balance(profile, D, mode) of SPEC.md:147-156: min-max contiguous split where a stage
    costs sum(fwd) (inference) or sum(fwd + bwd) (learning) plus the transfer term of its
    incoming boundary (charged downstream). Returns a StagePlan over fused
    units with predicted_stage_cost filled."""
    from .model import StagePlan
    if mode not in ("inference", "learning"):
        raise ValueError("mode must be 'inference' or 'learning'")
    cost = [f + (b if mode == "learning" else 0.0) for f, b in zip(profile.fwd_cost, profile.bwd_cost)]
    transfer = [bb * profile.transfer_cost_per_byte for bb in profile.boundary_bytes]
    counts, _ = balance(cost, D, transfer)
    ul = profile.unit_layers or [1] * len(cost)
    lc, a = [], 0
    for c in counts:  # unit counts -> Model.layers counts
        lc.append(sum(ul[a:a + c]))
        a += c
    plan = StagePlan.from_counts(lc)
    pred, a = [], 0
    for h, c in enumerate(counts):
        pred.append(sum(cost[a:a + c]) + (transfer[a - 1] if h > 0 else 0.0))
        a += c
    plan.predicted_stage_cost = pred
    return plan


def assign_workers(plan, profile: CostProfile, n_workers=None):
    """the first and the last stage go to the workers with the lowest
    measured host_copy_cost (they copy from / to the host); the other stages round-robin.
    Several stages may share a worker. Ties keep the stable (lowest index) order."""
    D = plan.D
    W = n_workers if n_workers is not None else (len(profile.host_copy_cost) or D)
    hc = list(profile.host_copy_cost) if profile.host_copy_cost else [0.0] * W
    if len(hc) < W:
        hc = hc + [0.0] * (W - len(hc))
    if W >= D and len(set(hc[:W])) == 1:
        assign = list(range(D))  # uniform costs: identity
    elif W >= D:
        order = sorted(range(W), key=lambda w: (hc[w], w))
        assign = [None] * D
        assign[0] = order[0]
        if D > 1:
            assign[D - 1] = order[1]
        rest = [w for w in range(W) if w not in (assign[0], assign[D - 1])]
        for h in range(1, D - 1):
            assign[h] = rest[(h - 1) % len(rest)]
    else:
        assign = [h % W for h in range(D)]  # more stages than workers: round-robin
    plan.worker_assignment = assign
    return plan


def profile_costs(model, sample_input, iters=5, warmup_iters=2, device=0):
    """SPEC.md:138-146 on the B200: per-layer forward / backward times are the medians of
    the device-side step timestamps of the tick kernel (pt_set_trace, CTA 0) over `iters`
    ticks after `warmup_iters`, on a D=1 pipeline of the model on GPU `device`; boundary
    bytes come from the shapes (fp32); the transfer cost is a measured device-to-device
    copy (NVLink peer copy when a second GPU is visible); the host copy cost is a measured
    H2D of the input plus D2H of the output on every visible GPU."""
    import numpy as np
    import torch
    from .engine import Pipeline
    from .model import fuse
    if iters < 3:
        raise ValueError("profile_costs needs iters >= 3 (median of timed runs)")
    units, owner = fuse(model)
    L = len(units)
    si = np.asarray(sample_input, np.float32)
    M = 1 if si.ndim == 1 else si.shape[0]
    dims = [model.layers[units[0][0]].in_dim] + [model.layers[u[0]].out_dim for u in units]
    T = warmup_iters + iters
    old_tile = os.environ.get("PT_TILE")
    os.environ["PT_TILE"] = "0"  # the per-step trace is the tick kernel's (layer-wise steps)
    try:
      with torch.cuda.device(device):
        xs = np.tile(si.reshape(1, M, -1), (T, 1, 1)).astype(np.float32)
        ys = np.zeros((T, M, 1 if canonical_loss(model.loss) == "softmax_ce" else dims[-1]), np.float32)
        if M == 1:
            xs, ys = xs[:, 0], ys[:, 0]
        p = Pipeline(model, [len(model.layers)], "sgd", 1e-9, si, ys[0])
        p.run(xs[:warmup_iters], ys[:warmup_iters])
        p.sync()
        p.set_trace(0, 1 << 16)
        p.run(xs[warmup_iters:], ys[warmup_iters:])
        p.sync()
        cons, _, _ = p.get_trace()
        p.close()
    finally:
        if old_tile is None:
            os.environ.pop("PT_TILE", None)
        else:
            os.environ["PT_TILE"] = old_tile
    # step boundaries: F of unit i starts at code 1, B of unit i at code 11 (units in
    # reverse), the tick ends at code 20 (pt_kernels.cuh trace codes)
    fwd = [[] for _ in range(L)]
    bwd = [[] for _ in range(L)]
    ticks, cur = [], []
    for code, ns in cons:
        if code in (1, 11, 20):
            cur.append((code, ns))
        if code == 20:
            ticks.append(cur)
            cur = []
    for tk in ticks:
        marks = [ns for _, ns in tk]
        if len(marks) != 2 * L + 1:
            continue
        for i in range(L):
            fwd[i].append((marks[i + 1] - marks[i]) * 1e-9)
            j = 2 * L - 1 - i  # backward of unit i is the (L + (L-1-i))-th mark
            bwd[i].append((marks[j + 1] - marks[j]) * 1e-9)
    if not ticks or not fwd[0]:
        raise RuntimeError("profile_costs: no complete tick in the device trace")
    fwd_m = [statistics.median(v) for v in fwd]
    bwd_m = [statistics.median(v) for v in bwd]
    if max(fwd_m + bwd_m) == 0:
        raise RuntimeError("profile_costs: timing resolution insufficient; use a larger input (SPEC.md:143)")
    boundary = [4 * M * d for d in dims[1:]]
    # transfer cost per byte: a 64 MB copy, peer when possible
    n = 16 << 20
    src = torch.empty(n, dtype=torch.float32, device=f"cuda:{device}")
    peer = torch.cuda.device_count() > 1
    dst = torch.empty(n, dtype=torch.float32, device=f"cuda:{(device + 1) % torch.cuda.device_count()}")
    dst.copy_(src)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        dst.copy_(src)
    torch.cuda.synchronize()
    per_byte = (time.perf_counter() - t0) / (5 * 4 * n) / (1.0 if peer else 2.0)  # D2D reads + writes
    host = []
    for w in range(torch.cuda.device_count()):
        hi = torch.empty(M * dims[0], dtype=torch.float32).pin_memory()
        ho = torch.empty(M * dims[-1], dtype=torch.float32).pin_memory()
        di = torch.empty_like(hi, device=f"cuda:{w}")
        do = torch.empty_like(ho, device=f"cuda:{w}")
        samples = []
        for _ in range(max(3, iters)):
            torch.cuda.synchronize(w)
            t0 = time.perf_counter()
            di.copy_(hi, non_blocking=True)
            ho.copy_(do, non_blocking=True)
            torch.cuda.synchronize(w)
            samples.append(time.perf_counter() - t0)
        host.append(statistics.median(samples))
    unit_layers = [0] * L
    for u in owner:
        unit_layers[u] += 1
    return CostProfile(fwd_m, bwd_m, boundary, per_byte, host, unit_layers)
