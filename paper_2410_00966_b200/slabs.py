"""z-slab decomposition plumbing (host side).  One process per GPU; rank r holds
the planes plane_range(nz, world, r) of the grid.  The exchanges themselves (one-plane halos,
the demag all-to-all transpose, the W-partials all-gather, the relax max-torque all-reduce) run
inside libmcq over its own NCCL communicator; torch.distributed only carries the 128-byte NCCL
unique id from rank 0 to the others (NCCL on GPUs, gloo in the CPU tests)."""
from __future__ import annotations


def plane_range(nz, world, rank):
    """Global z planes [z0, z1) of `rank` (world must divide nz, include/mcq.h mcq_dist)."""
    if world < 1 or nz % world:
        raise ValueError(f"world={world} must divide nz={nz}")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    n = nz // world
    return rank * n, (rank + 1) * n


def cell_range(grid, world, rank):
    """Cells [i0, i1) of the global x-fastest array that `rank` reads / writes."""
    nx, ny, nz = grid
    z0, z1 = plane_range(nz, world, rank)
    return z0 * nx * ny, z1 * nx * ny


def slab_dist(rank, world, device=-1, stream=None, nccl_id=None):
    """mcq_dist dict for rank `rank` of a `world`-slab context.  Rank 0 creates the NCCL unique
    id (mcq_nccl_get_unique_id) and torch.distributed broadcasts it, unless `nccl_id` is given."""
    if world == 1:
        return {"rank": 0, "world": 1, "device": device, "stream": stream}
    if nccl_id is None:
        import torch.distributed as dist
        box = [None]
        if rank == 0:
            from . import mcq_nccl_get_unique_id
            box[0] = mcq_nccl_get_unique_id()
        dist.broadcast_object_list(box, src=0)
        nccl_id = box[0]
    if not isinstance(nccl_id, (bytes, bytearray)) or len(nccl_id) != 128:
        raise ValueError("nccl_id must be 128 bytes")
    return {"rank": int(rank), "world": int(world), "device": int(device), "stream": stream,
            "nccl_id": bytes(nccl_id)}
