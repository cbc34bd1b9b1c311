"""Multi-GPU plumbing for the benchmark: one process per GPU, batch-sharded.

The TKD layer is independent per image, so data parallelism has
no data-path collective: every rank runs its own shard and the only
collectives are a barrier around the timed region and the max-over-ranks of the
measured time.  Backend "nccl" on GPUs, "gloo" for the CPU tests.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_ranks() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, device: torch.device | None = None) -> tuple[int, int]:
    rank, world, _ = env_ranks()
    if world > 1 and not dist.is_initialized():
        kw = {"device_id": device} if (device is not None and backend == "nccl") else {}
        dist.init_process_group(backend, **kw)
    return rank, world


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def max_over_ranks(value: float, device: torch.device | str = "cpu") -> float:
    """The job's time is the slowest rank's (timing rule: max over ranks)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device: torch.device | str = "cpu") -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def shard(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous batch slice (start, count) of rank; sizes differ by at most 1."""
    if global_batch < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


class BatchShard:
    """Contiguous slice of a global batch owned by this rank, and the gather of the
    per-rank results (e.g. logits) back into global-batch order -- the one collective of
    batch-sharded inference ("an optional final ncclAllGather of
    logits").  Shards may differ in size by one image: every rank pads its result to
    the largest shard, all-gathers, and the padding is dropped."""

    def __init__(self, global_batch: int, world: int | None = None, rank: int | None = None):
        if world is None or rank is None:
            r, w, _ = env_ranks()
            world = w if world is None else world
            rank = r if rank is None else rank
        self.global_batch, self.world, self.rank = global_batch, world, rank
        self.start, self.count = shard(global_batch, world, rank)
        self.max_count = -(-global_batch // world)
        self.bounds = [shard(global_batch, world, r) for r in range(world)]

    def gather(self, local: torch.Tensor) -> torch.Tensor:
        """local: [count, ...] on this rank -> [global_batch, ...] on every rank."""
        if local.shape[0] != self.count:
            raise ValueError(f"rank {self.rank} holds {local.shape[0]} rows, shard is {self.count}")
        if self.world == 1 or not (dist.is_initialized() and dist.get_world_size() > 1):
            return local
        pad = local.new_zeros((self.max_count, *local.shape[1:]))
        pad[:self.count] = local
        if dist.get_backend() == "nccl":
            buf = local.new_empty((self.world * self.max_count, *local.shape[1:]))
            dist.all_gather_into_tensor(buf, pad)
            parts = buf.view(self.world, self.max_count, *local.shape[1:])
        else:  # gloo: list form
            parts = [torch.empty_like(pad) for _ in range(self.world)]
            dist.all_gather(parts, pad)
        return torch.cat([parts[r][:n] for r, (_, n) in enumerate(self.bounds)], dim=0)


def finalize() -> None:
    if dist.is_initialized():
        dist.destroy_process_group()
