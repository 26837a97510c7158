"""Host-side plumbing for one-process-per-GPU runs (torchrun): rank discovery, the NCCL id
handshake for sw_mesh_create, batch slicing per data-parallel replica, and max-over-ranks
timing. The data path itself (collectives inside the step) is NCCL inside the C++ executor;
torch.distributed (gloo) only carries these small host messages."""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass
class RankInfo:
    rank: int
    world: int
    local_rank: int


def rank_info() -> RankInfo:
    return RankInfo(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                    int(os.environ.get("LOCAL_RANK", "0")))


def init_host_group(info: RankInfo):
    """gloo group for host messages (None when world == 1)."""
    if info.world == 1:
        return None
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=info.rank, world_size=info.world)
    return dist


def share_nccl_id(dist, rank: int) -> bytes | None:
    """Rank 0 creates the NCCL unique id (sw_nccl_unique_id) and broadcasts it."""
    if dist is None:
        return None
    from . import engine

    obj = [engine.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(dist, x: float) -> float:
    """The step time of the job is the slowest rank's."""
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def replica_rows(global_batch: np.ndarray, dp: int, dp_index: int) -> np.ndarray:
    """slice_batch_inputs (spmd.hpp:751-769) for one input: equal leading-dim chunks."""
    rows = global_batch.shape[0]
    if dp < 1 or not 0 <= dp_index < dp:
        raise ValueError(f"slice_batch_inputs: bad slice {dp_index}/{dp}")
    if rows % dp != 0:
        raise ValueError(f"slice_batch_inputs: input with shape {list(global_batch.shape)} cannot be "
                         f"cut into {dp} batch slices")
    chunk = rows // dp
    return global_batch[dp_index * chunk:(dp_index + 1) * chunk]


def mesh_coords(device: int, dp: int, mp: int):
    """(dp_index, mp_index) of a device id; device_id = dp_index * mp + mp_index (mesh.hpp:25)."""
    return device // mp, device % mp


def mp_group(dp_index: int, mp: int):
    return [dp_index * mp + j for j in range(mp)]


def dp_group(mp_index: int, dp: int, mp: int):
    return [i * mp + mp_index for i in range(dp)]
