"""Grid-point sharding across GPUs (one process per GPU, torch.distributed).

Every phase of the solver is a pure function of the phase-start snapshot
(reference solver.py:16-20), so the points of a stage are split into
contiguous shards, each rank sweeps its shard, and ONE all-gather per phase
(NCCL over NVLink/NVSwitch) rebuilds the full controller on every rank.  The
objective's per-point terms are all-gathered the same way and every rank runs
the identical serial trapezoid, so J -- and therefore the adaptive split and
the termination test -- is bitwise identical on all ranks without a
broadcast.  Results are bitwise independent of the rank count.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

__all__ = ["Sharding", "LOCAL", "from_process_group"]


@dataclass(frozen=True)
class Sharding:
    rank: int = 0
    world: int = 1
    group: object = None  # torch.distributed ProcessGroup (None = default / single process)

    def __post_init__(self):
        if not (0 <= self.rank < self.world):
            raise ValueError(f"rank {self.rank} outside world of {self.world}")

    # -- partition ---------------------------------------------------------
    def chunk(self, d: int) -> int:
        return -(-int(d) // self.world)

    def bounds(self, d: int) -> tuple[int, int]:
        """Contiguous [begin, end) of this rank (the last shard may be short or empty)."""
        c = self.chunk(d)
        begin = min(self.rank * c, d)
        return begin, min(begin + c, d)

    def out_buffer(self, d: int, device) -> torch.Tensor:
        """A float64 buffer sized chunk*world so the all-gather is in place."""
        return torch.empty(self.chunk(d) * self.world, dtype=torch.float64, device=device)

    # -- collectives -------------------------------------------------------
    def allgather_(self, buf: torch.Tensor) -> None:
        """In-place all-gather of each rank's chunk of ``buf`` (no-op for one rank)."""
        if self.world == 1:
            return
        import torch.distributed as dist

        c = buf.numel() // self.world
        if buf.is_cuda and dist.get_backend(self.group) == "gloo":
            # CPU-collective plumbing (multi-process tests on one GPU); NCCL in production
            host = buf.cpu()
            dist.all_gather_into_tensor(host, host[self.rank * c:(self.rank + 1) * c], group=self.group)
            buf.copy_(host)
            return
        dist.all_gather_into_tensor(buf, buf[self.rank * c:(self.rank + 1) * c], group=self.group)

    def allreduce_min_(self, t: torch.Tensor) -> None:
        if self.world == 1:
            return
        import torch.distributed as dist

        if t.is_cuda and dist.get_backend(self.group) == "gloo":
            host = t.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.MIN, group=self.group)
            t.copy_(host)
            return
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)


LOCAL = Sharding()


def from_process_group(group=None) -> Sharding:
    """Sharding for the current torch.distributed process group."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return LOCAL
    return Sharding(rank=dist.get_rank(group), world=dist.get_world_size(group), group=group)
