"""Multi-GPU plumbing (one process per GPU, torch.distributed for bootstrap only).

The sweep-sharded path (include/louvain.h) runs inside the library over an
NCCL communicator the library owns; this module creates it by broadcasting an NCCL
unique id over a torch process group, and offers the host helpers the benchmark uses
(max over ranks, barrier, shard ranges).  Marshalling only.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import check


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def init_process_group(backend: str = "nccl"):
    import torch.distributed as dist

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group(backend)
    return dist.get_rank(), dist.get_world_size()


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(_lib.load().louvain_nccl_unique_id(buf))
    return bytes(buf)


def broadcast_bytes(data: bytes | None, src: int = 0, group=None, device=None) -> bytes:
    """Broadcast a 128-byte blob from `src` over a torch process group (gloo or nccl)."""
    import torch
    import torch.distributed as dist

    t = torch.zeros(128, dtype=torch.uint8, device=device or "cpu")
    if dist.get_rank(group) == src if group is not None else dist.get_rank() == src:
        t.copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
    dist.broadcast(t, src=src, group=group)
    return bytes(t.cpu().numpy().tobytes())


def nccl_comm(device: int, group=None):
    """Create the library's NCCL communicator across the ranks of `group`."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    uid = nccl_unique_id() if rank == 0 else None
    dev = "cuda" if dist.get_backend(group) == "nccl" else None
    uid = broadcast_bytes(uid, 0, group, device=dev)
    comm = C.c_void_p()
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    check(_lib.load().louvain_nccl_init(buf, world, rank, device, C.byref(comm)))
    return comm.value, rank, world


def destroy_comm(comm):
    if comm:
        _lib.load().louvain_nccl_destroy(C.c_void_p(comm))


def shard_bounds(row_ptr, world: int) -> np.ndarray:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    out = np.empty(world + 1, dtype=np.int64)
    check(_lib.load().louvain_shard_bounds(rp.ctypes.data, len(rp) - 1, int(world), out.ctypes.data))
    return out


def allmax(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], device=device or "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
