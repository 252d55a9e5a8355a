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

    # -- work-balanced partitions -------------------------------------------
    def plan(self, d: int, weights: torch.Tensor | None = None) -> tuple:
        """Shard boundaries (world+1 ints).  With ``weights`` (int64 per-point
        work estimates, identical on every rank because they derive from the
        same snapshot) the cumulative work is split evenly; otherwise equal
        point counts.  Boundaries never change a result bit.  (Reads the cuts
        back: the solver queues ``plan_cuts`` instead and reads them with a
        synchronisation it makes anyway.)"""
        d = int(d)
        if self.world == 1:
            return (0, d)
        if weights is None:
            return self.equal_plan(d)
        return self.plan_from_cuts(d, self.plan_cuts(weights).cpu().tolist())

    def equal_plan(self, d: int) -> tuple:
        c = self.chunk(d)
        return tuple(min(r * c, d) for r in range(self.world)) + (d,)

    def plan_cuts(self, weights: torch.Tensor) -> torch.Tensor:
        """The world-1 interior cuts of the weight-balanced plan, on the
        weights' device (no synchronisation)."""
        cum = torch.cumsum(weights.to(torch.int64), 0)
        targets = (cum[-1] * torch.arange(1, self.world, device=cum.device, dtype=torch.int64)) // self.world
        return torch.searchsorted(cum, targets, right=True)

    def plan_from_cuts(self, d: int, cuts) -> tuple:
        out = [0]
        for c in cuts:
            out.append(min(max(int(c), out[-1]), d))
        out.append(int(d))
        return tuple(out)

    def shard(self, bounds: tuple) -> tuple[int, int]:
        return bounds[self.rank], bounds[self.rank + 1]

    def padded_buffer(self, bounds: tuple, device) -> torch.Tensor:
        """The phase output in the natural layout (grid point i at index i),
        padded to chunk*world doubles so an equal-split plan all-gathers in place."""
        d = bounds[-1]
        return torch.empty(max(self.chunk(d) * self.world, 1), dtype=torch.float64, device=device)

    def rank_ptr(self, buf: torch.Tensor, bounds: tuple) -> int:
        """Base pointer such that base[i] (i in this rank's shard) is its output slot."""
        return buf.data_ptr()

    def gather(self, buf: torch.Tensor, bounds: tuple, d: int) -> torch.Tensor:
        """All-gather every rank's shard of ``buf`` (natural layout) in place and
        return the contiguous length-d vector: no compaction copy.  Equal-split
        plans use one all_gather_into_tensor; work-balanced (uneven) plans one
        uneven all_gather (NCCL: grouped broadcasts straight into place)."""
        if self.world == 1:
            return buf[:d]
        if tuple(bounds) == self.equal_plan(d):
            self.allgather_(buf)
            return buf[:d]
        self.allgather_uneven_(buf, bounds)
        return buf[:d]

    # -- collectives -------------------------------------------------------
    def allgather_uneven_(self, buf: torch.Tensor, bounds: tuple) -> None:
        """buf[bounds[r]:bounds[r+1]] of rank r to every rank, in place."""
        import torch.distributed as dist

        b, e = self.shard(bounds)
        if dist.get_backend(self.group) == "gloo":
            # gloo has no uneven all-gather: pad each shard to the longest on the
            # host (CPU-collective plumbing for tests; NCCL in production)
            cm = max(1, max(bounds[r + 1] - bounds[r] for r in range(self.world)))
            host = buf.cpu()
            slots = torch.zeros(cm * self.world, dtype=host.dtype)
            slots[self.rank * cm:self.rank * cm + (e - b)] = host[b:e]
            dist.all_gather_into_tensor(slots, slots[self.rank * cm:(self.rank + 1) * cm].clone(), group=self.group)
            for r in range(self.world):
                host[bounds[r]:bounds[r + 1]] = slots[r * cm:r * cm + bounds[r + 1] - bounds[r]]
            if buf.is_cuda:
                buf.copy_(host)
            return
        outs = [buf[bounds[r]:bounds[r + 1]] for r in range(self.world)]
        dist.all_gather(outs, buf[b:e], group=self.group)

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
