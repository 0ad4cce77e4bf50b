"""Multi-GPU use of the C-ABI: one process per GPU (torchrun), axis-0 slabs (north_star: "Large
grids are slab-partitioned along axis 0 ... Each RK stage does an NCCL send/recv halo exchange over
NVLink, and an allreduce-max of alpha per step"; §4.2 P:288 -- every node of a stage is
independent).

torch.distributed is plumbing only: it starts the ranks and broadcasts the 128-byte NCCL id; the
halo exchange and the range allreduce run inside libodp.so (odp_grid_partition / odp_hj_solve).
"""
from __future__ import annotations

import os
from typing import Optional, Tuple

from .capi import Grid, comm_unique_id, partition_extent


def env_ranks() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1 process = rank 0 of 1)."""
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def slabs(N0: int, world: int):
    """Every rank's (first plane, plane count) -- odp_partition_extent for all ranks."""
    return [partition_extent(N0, world, r) for r in range(world)]


def broadcast_uid(uid: Optional[bytes], rank: int) -> bytes:
    """Rank 0's NCCL id to every rank over the default torch.distributed group (any backend)."""
    import torch
    import torch.distributed as dist
    obj = [uid if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    assert isinstance(obj[0], (bytes, bytearray)) and len(obj[0]) == 128
    return bytes(obj[0])


def partitioned_grid(w, rank: int, world: int, device: int, force_comm: bool = False) -> Grid:
    """odp_grid_create + odp_grid_partition for this rank; collective when world > 1 (or force_comm)."""
    g = Grid(w.N, w.lo, w.hi, w.periodic_mask)
    if world > 1 or force_comm:
        uid = comm_unique_id() if rank == 0 else None
        if world > 1:
            uid = broadcast_uid(uid, rank)
        g.partition(rank, world, uid, device)
    return g


def local_v0(w, rank: int, world: int, seed=None):
    """This rank's slab of the workload's V0 (bitwise the slice of the whole array)."""
    from inputs import make_v0
    return make_v0(w, seed=seed, i0=partition_extent(w.N[0], world, rank))
