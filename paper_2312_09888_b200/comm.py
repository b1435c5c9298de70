"""Communicator for the sort-last composite (the paper's
``initialize(MPI_Comm*, nek_data)`` argument).

One process per GPU.  The NCCL unique id made by rank 0 is distributed
either through an already-initialised ``torch.distributed`` group (plumbing
only) or through an atomically renamed file -- the reference's port-file
handshake (harness.py:186-189).  The composite itself runs inside
libnekb200 on the communicator created here.
"""
from __future__ import annotations

import os
import time

from .context import Context


class Communicator:
    def __init__(self, ctx: Context, rank: int, size: int, uid: bytes):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.ctx = ctx
        self.rank = int(rank)
        self.size = int(size)
        if self.size > 1:
            ctx.comm_init(uid, self.size, self.rank)

    @classmethod
    def from_torch(cls, ctx: Context | None = None, group=None) -> "Communicator":
        import torch.distributed as dist

        rank, size = dist.get_rank(group), dist.get_world_size(group)
        if ctx is None:
            ctx = Context(int(os.environ.get("LOCAL_RANK", rank)))
        obj = [Context.nccl_unique_id() if (rank == 0 and size > 1) else b"\0" * 128]
        if size > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(ctx, rank, size, obj[0])

    @classmethod
    def from_file(cls, ctx: Context, rank: int, size: int, path: str, timeout: float = 120.0) -> "Communicator":
        if size == 1:
            return cls(ctx, 0, 1, b"\0" * 128)
        if rank == 0:
            uid = Context.nccl_unique_id()
            tmp = f"{path}.tmp{os.getpid()}"
            with open(tmp, "wb") as f:
                f.write(uid)
            os.replace(tmp, path)        # atomic publish
        else:
            t0 = time.time()
            while not os.path.exists(path):
                if time.time() - t0 > timeout:
                    raise TimeoutError(f"no NCCL id at {path}")
                time.sleep(0.01)
            with open(path, "rb") as f:
                uid = f.read()
        return cls(ctx, rank, size, uid)

    def close(self) -> None:
        if self.size > 1:
            self.ctx.comm_destroy()
