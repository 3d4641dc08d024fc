"""Multi-GPU plumbing (host side): one process per GPU, launched by torchrun.

The data-parallel split follows the paper's OpenMP design -- "the dataset is
to be divided among the number of threads" -- as contiguous
ceiling-partition shards (datagen.shard_range).  Each rank keeps its shard in
HBM; the only exchange per iteration is one allreduce of the K*(d+1)+1
partials (sums, counts, inertia), done by the library's own NCCL communicator
inside the iteration's CUDA graph.  This module only creates that
communicator: rank 0 draws an NCCL unique id, torch.distributed broadcasts it
(any backend, gloo included), every rank calls kmeans_comm_init.
"""
from __future__ import annotations

from . import datagen
from . import kmeans as km


def check_shards(global_N: int, world: int) -> None:
    """Every rank must own at least one point: the ceiling partition leaves the
    last ranks empty when (world - 1) * ceil(N / world) >= N (e.g. N = 5 over
    4 ranks), and an empty rank would fail kmeans_create while its peers
    enter the collectives.  Raises the same ValueError on every rank (the test
    needs no communication)."""
    if world < 1 or global_N < 1:
        raise ValueError(f"need global_N >= 1 and world >= 1 (got {global_N}, {world})")
    c = -(-global_N // world)
    if (world - 1) * c >= global_N:
        raise ValueError(f"global_N={global_N} over {world} ranks leaves rank {world - 1} "
                         "without points (contiguous ceiling partition)")


def shard(global_N: int, world: int, rank: int) -> tuple[int, int]:
    """[a, b) owned by `rank` (contiguous ceiling partition); ValueError on
    every rank if some rank would own no point (check_shards)."""
    check_shards(global_N, world)
    return datagen.shard_range(global_N, world, rank)


def broadcast_unique_id(rank: int, group=None) -> bytes:
    """Rank 0's NCCL unique id, broadcast over torch.distributed."""
    import torch.distributed as dist
    obj = [km.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_comm(rank: int, world: int, device: int, group=None) -> int:
    """Create the library's NCCL communicator for this rank (collective).

    NCCL_ALGO / NCCL_PROTO are pinned (unless the caller set them) so the
    allreduce's summation order -- and so every centroid bit -- is the same
    from run to run."""
    import os
    os.environ.setdefault("NCCL_ALGO", "Ring")
    os.environ.setdefault("NCCL_PROTO", "Simple")
    uid = broadcast_unique_id(rank, group)
    return km.comm_init(world, uid, rank, device)


def enable_p2p(ctx, group=None) -> bool:
    """Switch a communicator context to the P2P exchange (kmeans_p2p_handle /
    kmeans_p2p_open): the IPC handles are all-gathered over torch.distributed.
    All-or-nothing: if any rank cannot map its peers, every rank stays on the
    NCCL allreduce.  Returns whether the exchange is on."""
    import torch.distributed as dist
    h = ctx.p2p_handle()
    world = dist.get_world_size(group)
    handles = [None] * world
    dist.all_gather_object(handles, h, group=group)
    try:
        ctx.p2p_open(handles)
        ok = True
    except Exception:
        ok = False
    oks = [None] * world
    dist.all_gather_object(oks, ok, group=group)
    if not all(oks):
        if ok:
            ctx.p2p_disable()
        return False
    return True
