"""Guest sharding across the GPUs of one box.

Guests share nothing on the data path (walks read only their own tables and
the replicated host-private region; copies write only their own slots), so
the batch scheduler needs no collective: guest g is owned by rank
g mod world, every rank processes its guests' op batches, and per-guest
results return to rank 0 by point-to-point sends (NCCL: peer copies over
NVLink / NVSwitch; gloo: host memory, used by the CPU tests).  Timing is the
max over ranks.
"""

from __future__ import annotations

from typing import Callable, Iterable


def owned_guests(n_guests: int, rank: int, world: int) -> list[int]:
    """Guests rank ``rank`` of ``world`` owns (round robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return [g for g in range(n_guests) if g % world == rank]


def owner_of(guest: int, world: int) -> int:
    return guest % world


def run_owned(n_guests: int, rank: int, world: int, work: Callable[[int], dict]) -> dict[int, dict]:
    """Run ``work(guest)`` for every owned guest; returns {guest: result}
    where a result is a dict of tensors of fixed, guest-independent shape
    per key (so peers can pre-allocate receive buffers)."""
    return {g: work(g) for g in owned_guests(n_guests, rank, world)}


def gather_to_rank0(results: dict[int, dict], n_guests: int, rank: int, world: int,
                    like: Callable[[int], dict]) -> dict[int, dict] | None:
    """Return every guest's result to rank 0 (point-to-point, in guest order).

    ``like(guest)`` builds an empty result of the right shapes/dtypes on
    rank 0 for a remote guest.  Non-zero ranks return None.
    """
    import torch.distributed as dist

    if world == 1:
        return dict(results)
    host = _host_backend()  # gloo: stage device tensors through host memory
    out: dict[int, dict] = {}
    for g in range(n_guests):
        src = owner_of(g, world)
        if rank == 0:
            if src == 0:
                out[g] = results[g]
                continue
            buf = like(g)
            for key in sorted(buf):
                if host and buf[key].is_cuda:
                    tmp = buf[key].cpu()
                    dist.recv(tmp, src=src)
                    buf[key].copy_(tmp)
                else:
                    dist.recv(buf[key], src=src)
            out[g] = buf
        elif rank == src:
            for key in sorted(results[g]):
                t = results[g][key].contiguous()
                dist.send(t.cpu() if host else t, dst=0)
    return out if rank == 0 else None


def _host_backend() -> bool:
    """True when the process group cannot move device tensors (gloo)."""
    import torch.distributed as dist

    return dist.get_backend() != "nccl"


def max_over_ranks(values: Iterable[float], world: int, device=None) -> list[float]:
    """Element-wise max over ranks (the bench's timing rule).  ``device`` is
    where the reduction tensor lives under NCCL; gloo reduces on the host."""
    import torch

    vals = list(values)
    import torch.distributed as dist

    if world == 1 or not dist.is_initialized():  # one rank, or one rank's share run alone
        return vals

    t = torch.tensor(vals, dtype=torch.float64, device=None if _host_backend() else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


class SharedHostBuffer:
    """One host buffer every rank of the box maps (the rank-0 result return
    of the end-to-end path): rank 0 creates it in /dev/shm
    (or /tmp when /dev/shm is too small), every rank maps it MAP_SHARED and
    registers it with CUDA (cudaHostRegister), so each rank's device-to-host
    copies of its own guests' results land directly in the buffer rank 0
    reads -- the return costs one barrier, no extra copy and no collective.
    """

    def __init__(self, nbytes: int, rank: int, world: int, tag: str = "pv"):
        import os
        import shutil
        import uuid

        import torch
        import torch.distributed as dist

        self.nbytes = max(int(nbytes), 8)
        self.rank = rank
        path = [None]
        if rank == 0:
            base = "/dev/shm"
            if not os.path.isdir(base) or shutil.disk_usage(base).free < 2 * self.nbytes:
                base = "/tmp"
            path[0] = os.path.join(base, f"{tag}_{os.getpid()}_{uuid.uuid4().hex[:8]}")
            with open(path[0], "wb") as f:
                f.truncate(self.nbytes)
        if world > 1:
            dist.broadcast_object_list(path, src=0)
        self.path = path[0]
        self.bytes = torch.from_file(self.path, shared=True, size=self.nbytes, dtype=torch.uint8)
        rc = torch.cuda.cudart().cudaHostRegister(self.bytes.data_ptr(), self.nbytes, 0)
        self.registered = int(rc) == 0
        if not self.registered:
            raise RuntimeError(f"cudaHostRegister of the shared result buffer failed ({rc})")
        self.world = world

    def view(self, dtype, offset_elems: int, count: int):
        """A typed view of ``count`` elements at element offset ``offset_elems``."""
        return self.bytes.view(dtype)[offset_elems:offset_elems + count]

    def close(self) -> None:
        import os

        import torch
        import torch.distributed as dist

        if self.registered:
            torch.cuda.cudart().cudaHostUnregister(self.bytes.data_ptr())
            self.registered = False
        if self.world > 1 and dist.is_initialized():
            dist.barrier()
        if self.rank == 0 and self.path and os.path.exists(self.path):
            os.unlink(self.path)


class PeerResultBuffer:
    """The job's lane words in rank 0's HBM: rank 0
    allocates ``nbytes`` with an IPC handle (pv_peer_alloc), every other rank
    maps it (pv_peer_open: a device pointer into rank 0's memory over NVLink /
    NVSwitch) and hands a slice of it to its walk as the output, so each word
    is stored into rank 0's memory by the kernel that computes it -- the
    result return is fused into the walk (no gather step, no collective).
    ``ptr`` is this rank's device address of the buffer."""

    def __init__(self, nbytes: int, rank: int, world: int):
        import ctypes

        import torch.distributed as dist

        from . import _native as N

        lib = N.lib()
        self.rank, self.world, self.nbytes = rank, world, int(nbytes)
        ptr = ctypes.c_void_p()
        handle = (ctypes.c_uint8 * 64)()
        box = [None]
        if rank == 0:
            N.check(lib.pv_peer_alloc(self.nbytes, ctypes.byref(ptr), handle), "pv_peer_alloc")
            box[0] = bytes(handle)
        if world > 1:
            dist.broadcast_object_list(box, src=0)
        if rank != 0:
            h = (ctypes.c_uint8 * 64).from_buffer_copy(box[0])
            N.check(lib.pv_peer_open(h, ctypes.byref(ptr)), "pv_peer_open")
        self.ptr = int(ptr.value)

    def copy_out(self, dst_ptr: int, offset: int, nbytes: int, stream: int) -> None:
        """Stream-ordered copy of ``nbytes`` at byte ``offset`` of the buffer to ``dst_ptr``."""
        from . import _native as N

        N.check(N.lib().pv_memcpy(dst_ptr, self.ptr + offset, nbytes, stream), "pv_memcpy")

    def close(self) -> None:
        """Unmap (ranks > 0) after a barrier; rank 0 frees after every rank unmapped."""
        import torch
        import torch.distributed as dist

        from . import _native as N

        torch.cuda.synchronize()
        if self.world > 1 and dist.is_initialized():
            dist.barrier()
        if self.rank != 0:
            N.lib().pv_peer_close(self.ptr)
        if self.world > 1 and dist.is_initialized():
            dist.barrier()
        if self.rank == 0:
            N.lib().pv_peer_free(self.ptr)
        self.ptr = 0
