"""Multi-GPU plumbing for GPU-AR (one process per GPU, torch.distributed).

The path partitions: selections are independent and a
selection's outputs depend only on (seed, global index s, epoch, alpha), so ranks own
contiguous global ranges and never exchange data on the hot path.  The only collectives:

* C1 ``broadcast_vector``: one shared propensity vector from rank 0 (NCCL over NVLink);
* C2 ``reduce_validation``: sum of the uint64 validation histograms + totals to rank 0;
* C3 ``max_over_ranks``: the bench's per-rank device time -> the job's time.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(K_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous range of global selections owned by `rank`: (s0, K_local).  The first
    K_total % world ranks take one extra selection; ranges tile [0, K_total) exactly."""
    if world < 1 or not 0 <= rank < world or K_total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(K_total, world)
    s0 = rank * base + min(rank, extra)
    return s0, base + (1 if rank < extra else 0)


def weak_shard(K_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank owns K_per_rank selections starting at rank * K_per_rank."""
    return rank * K_per_rank, K_per_rank


def broadcast_vector(alpha: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """C1: every rank ends with rank `src`'s propensity vector (in place)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(alpha, src=src, group=group)
    return alpha


def reduce_validation(hist: torch.Tensor, totals: torch.Tensor, dst: int = 0, group=None):
    """C2: sum the per-rank histograms (M+1 bins, bin M = rejected) and totals
    (sum of trials, #rejected) onto rank `dst` (in place there)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if hist.is_cuda and dist.get_backend(group) != "nccl":
            # gloo has no reduce for CUDA tensors; all_reduce gives dst the same sum
            dist.all_reduce(hist, group=group)
            dist.all_reduce(totals, group=group)
        else:
            dist.reduce(hist, dst=dst, group=group)
            dist.reduce(totals, dst=dst, group=group)
    return hist, totals


def max_over_ranks(value: float, device: torch.device | str = "cpu", group=None) -> float:
    """C3: the maximum of a per-rank scalar (e.g. elapsed device time)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
