"""Data-parallel execution over independent stacks (BASELINE configs 2/3).

Stacks are independent Tucker problems, so multi-GPU work is sharded by stack
with no data-path collective ("C3 ... zero communication";
C1/C2/C4 "replicas only"). One process per GPU (torchrun); the only
collectives are the timing barrier and the max-over-ranks reduction of the
elapsed time, which is what makes the whole-job throughput honest.
"""

from __future__ import annotations

from typing import Callable, Sequence

__all__ = ["assign_stacks", "reduce_max", "aggregate_throughput", "run_stacks"]


def assign_stacks(n_stacks: int, rank: int, world: int) -> list[int]:
    """Round-robin stack ids for this rank (disjoint, covering, balanced +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"invalid rank {rank} for world size {world}")
    return list(range(rank, n_stacks, world))


def reduce_max(value: float, device=None) -> float:
    """Max of a scalar over all ranks of the default process group (gloo on
    CPU tensors, nccl on CUDA tensors); identity without a process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank: Sequence[int], max_seconds: float) -> float:
    """Whole-job units/s: every rank's units over the slowest rank's time."""
    if max_seconds <= 0:
        raise ValueError("elapsed time must be positive")
    return float(sum(units_per_rank)) / max_seconds


def run_stacks(stack_ids: Sequence[int], solve: Callable[[int], object]) -> list:
    """Solve this rank's stacks in order (stack i -> solve(i))."""
    return [solve(i) for i in stack_ids]
