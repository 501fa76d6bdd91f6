"""Env sharding across GPUs ("a set of environments" per GPU).

Environments are independent, so each rank owns a contiguous env range and no
collective runs inside the solver.  The only exchange is the optional all-gather
of the marker fields to the policy rank: tac_markers writes the rank's
slot of one gather buffer and an in-place all_gather_into_tensor (NCCL over
NVLink / NVSwitch on GPUs; gloo in the CPU tests) fills the other slots.
"""
from __future__ import annotations


def env_range(rank: int, world: int, n_total: int):
    """Contiguous [start, stop) of env ids owned by `rank` (ragged splits allowed)."""
    if not (0 <= rank < world) or n_total < 0:
        raise ValueError("bad rank / world / n_total")
    base, rem = divmod(n_total, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


class MarkerGather:
    """Gather buffer [world * n_local, n_markers, ncomp]; `slot` is this rank's view.

    Requires equal n_local on every rank (weak scaling, or strong scaling with
    n_total divisible by world), as all_gather_into_tensor does."""

    def __init__(self, n_local, n_markers, ncomp, rank, world, device, group=None):
        import torch
        self.rank, self.world, self.group = rank, world, group
        self.buffer = torch.empty((world * n_local, n_markers, ncomp), dtype=torch.float32, device=device)
        self.slot = self.buffer[rank * n_local:(rank + 1) * n_local]

    def gather(self):
        import torch.distributed as dist
        if self.world == 1 and not dist.is_initialized():
            return self.buffer
        try:
            dist.all_gather_into_tensor(self.buffer, self.slot, group=self.group)
        except (RuntimeError, NotImplementedError):  # backends without the fused collective
            parts = list(self.buffer.chunk(self.world))
            dist.all_gather(parts, self.slot.clone(), group=self.group)
        return self.buffer


class _BorrowedComm:
    """torch.distributed's own NCCL communicator (ProcessGroupNCCL._comm_ptr), borrowed: one
    communicator per process, owned and destroyed by torch."""

    def __init__(self, ptr, nranks, rank):
        import ctypes
        self.handle, self.nranks, self.rank = ctypes.c_void_p(ptr), nranks, rank

    def close(self):
        pass


def torch_nccl_comm(device):
    """The default process group's NCCL communicator for `device`, or None (gloo, not yet
    initialised -- pass device_id to init_process_group for an eager one -- or a torch without
    ProcessGroupNCCL._comm_ptr)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_backend() != "nccl":
        return None
    try:
        pg = dist.distributed_c10d._get_default_group()
        ptr = pg._get_backend(torch.device(device))._comm_ptr()
    except Exception:
        return None
    return _BorrowedComm(ptr, dist.get_world_size(), dist.get_rank()) if ptr else None


class NativeMarkerGather:
    """The same gather through the C ABI (tac_gather_markers: tac_markers into this rank's slot +
    an in-place ncclAllGather on the caller's stream).  The communicator is torch.distributed's
    own when it is NCCL (one communicator per process), else one created by
    tac_nccl_comm_create with the unique id sent over the existing group.  Requires equal
    n_local on every rank."""

    def __init__(self, sim, n_local, n_markers, ncomp, rank, world, device, borrow=True):
        import torch
        import torch.distributed as dist
        from .tac import NcclComm, nccl_unique_id
        dev = torch.device(device)
        self.comm = torch_nccl_comm(dev) if borrow else None
        if self.comm is None:
            uid = [nccl_unique_id() if rank == 0 else None]
            if dist.is_initialized():
                dist.broadcast_object_list(uid, src=0)
            self.comm = NcclComm(uid[0], world, rank, dev.index if dev.index is not None else 0)
        self.sim, self.ncomp = sim, ncomp
        self.buffer = torch.empty((world * n_local, n_markers, ncomp), dtype=torch.float32, device=dev)
        self.slot = self.buffer[rank * n_local:(rank + 1) * n_local]

    def gather(self):
        return self.sim.gather_markers(self.comm, self.buffer, self.ncomp)

    def close(self):
        self.comm.close()
