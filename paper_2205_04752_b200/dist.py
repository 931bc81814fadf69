"""Transports for the block-row sharded matvec (HMatrix.attach_comm /
attach_nccl).

torch_transport(): the host-callback transport over a torch.distributed
process group with CPU tensors (gloo) -- for hosts without NCCL and for the
world-2/4 tests that run several ranks against one visible GPU (each rank a
process; the collectives run on the host, so no kernel waits on another
rank's kernel).  On an NVLink box use HMatrix.attach_nccl instead: the
library's own NCCL communicator on the context's stream.
"""
from __future__ import annotations

import numpy as np


def torch_transport(group=None):
    import torch
    import torch.distributed as dist

    def broadcast(buf: np.ndarray, root: int) -> None:
        t = torch.from_numpy(buf)
        dist.broadcast(t, src=root, group=group)

    def allgather(send: np.ndarray, recv: np.ndarray) -> None:
        n = send.size
        r = torch.from_numpy(recv)
        outs = [r[k * n:(k + 1) * n] for k in range(recv.size // n)]
        dist.all_gather(outs, torch.from_numpy(send.copy()), group=group)

    return broadcast, allgather


def exchange_unique_id(rank: int, uid: bytes | None, group=None) -> bytes:
    """Hands rank 0's NCCL unique id to every rank over torch.distributed."""
    import torch.distributed as dist
    box = [uid if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return box[0]
