"""Multi-GPU subtree sharding helpers (argument marshalling only; see include/hodlr.h, hodlr_dist).

Dist.from_torch(): one process per GPU under torch.distributed -- rank 0 creates the ncclUniqueId through
the library and broadcasts it with torch.distributed (PyTorch is the process-group plumbing); the library
then runs its own NCCL communicator on the handle's stream.
Group / run_virtual_ranks(): P virtual ranks as host threads of one process on one device (the library's
in-process transport), so the sharded path can be exercised on a single GPU.
"""
from __future__ import annotations

import ctypes as C
import threading

from . import hodlr as hb


class Group:
    """In-process group of nranks virtual ranks (hodlr_group_create)."""

    def __init__(self, nranks: int):
        self.nranks = int(nranks)
        p = C.c_void_p(0)
        hb._check(hb.load().hodlr_group_create(self.nranks, C.byref(p)))
        self.ptr = p.value

    def mode(self, m: int):
        """0 normal, 1 record the next sharded run's exchanges, 2 solo replay of rank 0 (scaling projection)."""
        hb._check(hb.load().hodlr_group_mode(self.ptr, int(m)))

    def close(self):
        if self.ptr:
            hb.load().hodlr_group_destroy(self.ptr)
            self.ptr = 0


class Dist:
    """One rank's view of a sharded factorization: rank, nranks and the transport (NCCL id or Group)."""

    def __init__(self, rank: int, nranks: int, nccl_id: bytes | None = None, group: Group | None = None):
        if (nccl_id is None) == (group is None):
            raise ValueError("exactly one of nccl_id and group")
        self.rank, self.nranks, self.group = int(rank), int(nranks), group
        self._id = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None

    def struct(self) -> hb.hodlr_dist:
        return hb.hodlr_dist(self.rank, self.nranks,
                             C.cast(self._id, C.c_void_p) if self._id is not None else None,
                             self.group.ptr if self.group is not None else None)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        hb._check(hb.load().hodlr_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch(cls, id_factory=None) -> "Dist":
        """Collective over the default torch.distributed group: rank 0 makes the id, everyone receives it."""
        import torch.distributed as dist
        rank, ws = dist.get_rank(), dist.get_world_size()
        obj = [(id_factory or cls.nccl_unique_id)() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(rank, ws, nccl_id=obj[0])


def run_virtual_ranks(nranks: int, fn, group: Group | None = None):
    """Run fn(rank, Dist) for every virtual rank on its own host thread (one shared Group, created here unless
    given); returns the list of results in rank order and re-raises the first exception."""
    g = group or Group(nranks)
    out, errs = [None] * nranks, [None] * nranks

    def body(r):
        try:
            out[r] = fn(r, Dist(r, nranks, group=g))
        except BaseException as e:       # noqa: BLE001 -- reported below
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if group is None:
        g.close()
    for e in errs:
        if e is not None:
            raise e
    return out
