"""Multi-process z-slab jobs over CUDA IPC (include/abft_stencil.h,
abft_stencil_ipc_export / _link): plumbing only.  torch.distributed carries
the IPC blobs and the name of the host-shared progress slots; the halo itself
moves inside the sm_100a kernels (stores into the neighbours' mapped buffers).

    ctx = IpcContext(rank, world)                # once per process group
    st = abft.from_problem(p, u0, P, z_begin=z0, z_count=zc, rank=rank, nranks=world)
    ctx.link(st)                                 # collective: export, exchange, link, barrier
    st.step(n)                                   # every rank, same n
"""
from __future__ import annotations

import ctypes as C
import os
import uuid
from multiprocessing import shared_memory

import torch.distributed as dist

from . import abft


class IpcContext:
    """The job's host-shared slots (one abft_ipc_slot per rank, a /dev/shm
    segment created by rank 0) and the collective link of a handle."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world
        nbytes = C.sizeof(abft.abft_ipc_slot) * world
        name = [f"abft_{os.getpid()}_{uuid.uuid4().hex[:12]}" if rank == 0 else None]
        if rank == 0:
            self.shm = shared_memory.SharedMemory(name=name[0], create=True, size=nbytes)
            C.memset(C.addressof(C.c_char.from_buffer(self.shm.buf)), 0, nbytes)
        dist.broadcast_object_list(name, src=0)
        if rank != 0:
            self.shm = shared_memory.SharedMemory(name=name[0])
            # the segment is rank 0's to unlink; keep this process's resource
            # tracker from unlinking it (again) at exit
            from multiprocessing import resource_tracker
            resource_tracker.unregister(self.shm._name, "shared_memory")
        self._owner = rank == 0
        self._view = C.c_char.from_buffer(self.shm.buf)   # exports the mapping; dropped in close()
        self.addr = C.addressof(self._view)
        dist.barrier()

    def link(self, st: abft.Stencil) -> bool:
        """Collective: every rank exports, the blobs are all-gathered, each rank
        links to its neighbours, barrier (no rank steps before all linked).
        Returns True on every rank if every rank linked; on False the handles
        are unlinked and the caller picks another transport (NCCL)."""
        import torch
        from .dist import neighbours
        err = None
        try:
            blob = abft.ipc_export(st)
        except Exception as ex:   # noqa: BLE001 -- reported collectively below
            blob, err = None, ex
        blobs = [None] * self.world
        dist.all_gather_object(blobs, blob)
        if err is None and all(b is not None for b in blobs):
            lo_r, hi_r = neighbours(self.rank, self.world, periodic=st.cfg.bc == abft.ABFT_BC_PERIODIC)
            try:
                abft.ipc_link(st, blobs[lo_r] if lo_r is not None else None,
                              blobs[hi_r] if hi_r is not None else None, self.addr)
            except Exception as ex:   # noqa: BLE001
                err = ex
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        ok = torch.tensor([0 if (err is not None or any(b is None for b in blobs)) else 1], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        self.error = err
        dist.barrier()
        return bool(ok.item())

    def close(self) -> None:
        """Collective: after every rank destroyed its handles."""
        dist.barrier()
        self.addr = None
        self._view = None
        self.shm.close()
        if self._owner:
            self.shm.unlink()
