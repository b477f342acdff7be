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
