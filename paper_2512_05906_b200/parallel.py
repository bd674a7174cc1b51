"""Trial-parallel multi-GPU driver.

Trials of one network are independent until the loss: B_global trials shard
across ranks (contiguous blocks), each rank runs its block through its own
engine with no communication, and one all-reduce (NCCL over NVLink on B200;
gloo on CPU for the tests) sums loss, dL/dw, dL/dd and dL/d amplitude.  Drive
seeds are global (trial t uses seed0 + t), so the result is independent of the
number of ranks up to the summation order of the final reduce.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_trials(global_trials: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced block (start, count) of trials for `rank`."""
    if global_trials < world:
        raise ValueError(f"{global_trials} trials cannot shard over {world} ranks")
    base, extra = divmod(global_trials, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


@dataclass
class ShardResult:
    loss: float
    grad_w: torch.Tensor
    grad_d: torch.Tensor
    grad_amp: Optional[torch.Tensor]
    trials: Tuple[int, int]


def sharded_value_and_grad(compute: Callable[[int, int], Tuple[float, torch.Tensor, torch.Tensor,
                                                              Optional[torch.Tensor]]],
                           global_trials: int, group=None) -> ShardResult:
    """Run `compute(start, count)` on this rank's block, then sum across ranks.

    `compute` returns (loss, grad_w, grad_d, grad_amp or None) for the trials
    [start, start+count) — the engine's forward + reverse on B200, or the oracle
    in the CPU tests.  No collective happens before the final reduce."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    start, count = shard_trials(global_trials, world, rank)
    loss, gw, gd, ga = compute(start, count)
    if world > 1:
        dev = gw.device
        lt = torch.tensor([loss], dtype=torch.float64, device=dev)
        dist.all_reduce(lt, group=group)
        dist.all_reduce(gw, group=group)
        dist.all_reduce(gd, group=group)
        if ga is not None:
            dist.all_reduce(ga, group=group)
        loss = float(lt.item())
    return ShardResult(loss, gw, gd, ga, (start, count))
