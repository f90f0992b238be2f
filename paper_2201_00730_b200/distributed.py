"""Multi-GPU plumbing for the row-sharded Sinkhorn (BASELINE config 3).

One process per GPU (torchrun).  ``NcclComm`` builds an NCCL communicator
inside the extension from a unique id that rank 0 creates and
torch.distributed broadcasts (any backend); ``shard_rows`` fixes the
contiguous row partition.  The per-iteration exchange itself (one
ncclAllGather of per-column log-sum-exp pairs) lives in csrc/sinkhorn.cu.
Batched configs (2, 4, 5) shard by problem with no communication:
``shard_problems``.
"""

from __future__ import annotations

import ctypes

from . import _lib


def shard_rows(n, world):
    """Contiguous balanced row counts [world] (the first n % world get one more)."""
    base, extra = divmod(int(n), int(world))
    return [base + (1 if r < extra else 0) for r in range(world)]


def row_offset(n, world, rank):
    return sum(shard_rows(n, world)[:rank])


def shard_problems(batch, world, rank):
    """[start, stop) of this rank's problems for the batched configs."""
    counts = shard_rows(batch, world)
    start = sum(counts[:rank])
    return start, start + counts[rank]


def broadcast_bytes(payload, src=0, group=None):
    """Broadcast a bytes object from ``src`` over torch.distributed."""
    import torch.distributed as dist

    obj = [payload]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


class NcclComm:
    """NCCL communicator owned by the extension (context manager)."""

    def __init__(self, world, rank, group=None):
        lib = _lib.load()
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _lib.check(lib.uot_nccl_unique_id(uid), "uot_nccl_unique_id")
        raw = broadcast_bytes(uid.raw if rank == 0 else None, src=0, group=group)
        uid = ctypes.create_string_buffer(raw, 128)
        handle = ctypes.c_void_p(0)
        _lib.check(lib.uot_nccl_comm_init(uid, int(world), int(rank), ctypes.byref(handle)),
                   "uot_nccl_comm_init")
        self.handle = handle
        self.world = int(world)
        self.rank = int(rank)

    def close(self):
        if self.handle is not None and self.handle.value:
            _lib.load().uot_nccl_comm_destroy(self.handle)
        self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
