"""Multi-GPU replica plumbing (host side).  One process per GPU; under torchrun every rank runs an
independent simulation at its own point of a bias-field sweep (the anticrossing sweep of an
analysis like the paper's Fig. 3e), so the data path needs no collective.  The only
cross-rank operations are the timing reduction (max over ranks) and the gather of results.
torch.distributed is plumbing here (NCCL on GPUs, gloo in the CPU tests)."""
from __future__ import annotations

import numpy as np


def sweep_points(center, n, rel=0.1):
    """n bias magnitudes evenly spanning center*(1 +- rel) (a single point for n == 1)."""
    if n == 1:
        return [float(center)]
    return [float(v) for v in np.linspace(center * (1 - rel), center * (1 + rel), n)]


def replica_bias(bext, world, rank, rel=0.1):
    """Rank `rank`'s external field: bext rescaled to its sweep point (direction kept)."""
    b = np.asarray(bext, float)
    nrm = float(np.linalg.norm(b))
    if nrm == 0 or world == 1:
        return tuple(b)
    return tuple(b / nrm * sweep_points(nrm, world, rel)[rank])


def max_over_ranks(value, device=None):
    """Max of a float over all ranks (device timing rule: the job takes as long as its slowest
    rank).  Works with NCCL (cuda tensors) and gloo (cpu tensors)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(obj):
    """All ranks' python objects (e.g. per-replica spectra peaks), in rank order."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out
