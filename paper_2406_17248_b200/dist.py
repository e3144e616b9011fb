"""Multi-GPU launch plumbing: one process per GPU (torchrun), torch.distributed only to broadcast
the NCCL unique id; every state-vector operation then runs in libsv.so (NCCL over NVLink)."""
from __future__ import annotations

import os

from . import _sv


def create_sharded(n_qubits: int):
    """Creates this rank's shard handle of an n-qubit state sharded over WORLD_SIZE ranks
    (RANK / WORLD_SIZE from the environment; torch.distributed must be initialised). Returns a
    StateVector (world 1: a plain single-GPU handle)."""
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world == 1:
        return _sv.StateVector(n_qubits)
    obj = [_sv.sv_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    h = _sv.sv_create_sharded(n_qubits, rank, world, obj[0])
    return _sv.StateVector(n_qubits, handle=h)
