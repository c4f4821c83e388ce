"""Multi-GPU plumbing: batch sharding across ranks and the all-reduce of the loss sum.

Utterances are independent ("batch items are embarrassingly parallel"), so the only
cross-GPU exchange the path has is the sum of the per-utterance losses (BASELINE.json north_star (5)):
each rank reduces its shard's losses on the device (``rnnt_loss_sum``, fixed order, fp64) and one
``all_reduce(SUM)`` of that 8-byte scalar runs over NCCL (NVLink 5 / NVSwitch).  No joint-tensor bytes
cross GPUs; gradients stay local for the joint network's backward.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_world():
    """(rank, world_size, local_rank) from the torchrun environment (1-process defaults)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str = "nccl"):
    rank, world, local = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", rank=rank, world_size=world,
                                    device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world, local


def device_index(local_rank: int, backend: str = "nccl") -> int:
    """CUDA device of a rank: its local rank (one process per GPU).  Under gloo several ranks may share a GPU
    (harness tests on a one-GPU box): local rank modulo the visible device count."""
    if backend == "nccl":
        return local_rank
    return local_rank % max(1, torch.cuda.device_count())


def contiguous_shard(n_global: int, rank: int, world: int):
    """Global utterance ids of ``rank``: a contiguous block; block sizes differ by at most one."""
    base, extra = divmod(n_global, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def lpt_shard(costs, world: int):
    """Greedy longest-processing-time assignment of utterances (cost ~ T_b (U_b+1) V) to ranks.

    Deterministic: ties broken by utterance id, then by rank id.  Returns one sorted id list per rank.
    """
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0] * world
    out = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += costs[i]
    return [sorted(ids) for ids in out]


def allreduce_loss_sum(loss_sum: torch.Tensor, group=None) -> torch.Tensor:
    """In-place all-reduce(SUM) of the per-rank fp64 loss sum (a no-op for a single process)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(loss_sum, op=dist.ReduceOp.SUM, group=group)
    return loss_sum


def sum_over_ranks(value: float, device) -> float:
    """Sum of a host scalar over ranks (the units all ranks processed)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(value: float, device) -> float:
    """Max of a host scalar over ranks (used for the step time: the slowest rank defines throughput)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
