"""Distributed bootstrap: one process per GPU, torch.distributed only as plumbing (C5).

Rank 0 asks libsv for an NCCL unique id; torch.distributed broadcasts the 128 bytes; every rank
then calls sv_create_dist on its own device.  All state-vector work happens in libsv.so.
"""
from __future__ import annotations

import numpy as np

from ._lib import StateVector, nccl_unique_id


def create_distributed(n_qubits: int, chunk_bits: int, precision: str = "fp64", group=None) -> StateVector:
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world & (world - 1):
        raise ValueError("world size must be a power of two")
    uid = nccl_unique_id() if rank == 0 else bytes(128)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor(np.frombuffer(uid, dtype=np.uint8).copy(), dtype=torch.uint8, device=dev)
    dist.broadcast(t, src=0, group=group)
    uid = bytes(t.cpu().numpy().tobytes())
    return StateVector(n_qubits, chunk_bits, precision, rank=rank, world=world, nccl_id=uid)
