"""One process per GPU: each rank owns a contiguous range of stages (by default
stage rank+1). Neighbouring ranks exchange CUDA IPC handles of their stage
comm blocks through torch.distributed. After that, the tick kernels store
activations and gradients straight into the neighbour's memory over NVLink.

This replaces the paper's per-device CUDA streams and device-to-device copies
(PAPER.md:577, 584-595). No data-path collective is involved, only
point-to-point peer stores.
"""

from __future__ import annotations

import torch.distributed as dist

from .engine import Pipeline


def stage_range(rank, world, D):
    """Contiguous, balanced assignment of D stages to `world` ranks -> (first, count)."""
    if D < world:
        raise ValueError(f"{D} stages cannot occupy {world} ranks")
    base, extra = divmod(D, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def exchange_ipc(pipe, group=None):
    """All-gather every rank's exported stage blobs and import the neighbours'."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    first, count = pipe.local_first, pipe.local_count
    mine = {h: pipe.ipc_export(h) for h in range(first + 1, first + count + 1)}
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    blobs = {}
    for d in gathered:
        blobs.update(d)
    want = []
    if first > 0:
        want.append(first)              # upstream neighbour: stage `first` (1-based)
    if first + count < pipe.D:
        want.append(first + count + 1)  # downstream neighbour
    for h in want:
        if h not in blobs:
            raise RuntimeError(f"rank {rank}: stage {h} was not exported by any rank")
        pipe.ipc_import(blobs[h])
    return want


def build_distributed(model, plan, optimizer="sgd", lr=1e-3, sample_input=None, sample_target=None,
                      group=None, **kw):
    """pipeline_build for one rank of a one-process-per-GPU job (torchrun)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    from .model import StagePlan
    D = len(plan) if isinstance(plan, (list, tuple)) else StagePlan.D.fget(plan)
    pipe = Pipeline(model, plan, optimizer, lr, sample_input, sample_target,
                    local_stages=stage_range(rank, world, D), **kw)
    exchange_ipc(pipe, group)
    dist.barrier(group)
    return pipe
