"""Data parallelism over tokens for the exit-head step (host orchestration).

EE-Tuning's exits are independent and every token contributes independently to
an exit's loss, so the step shards along the flat token axis:
rank r owns tokens [r*N/P, (r+1)*N/P).  The only exchanges are

  1. the global number of valid tokens W (one int64 all-reduce), so every
     rank normalises its loss and gradients by the *global* W (A16);
  2. each exit's fp32 parameter gradients (sum all-reduce), issued
     asynchronously right after that exit's backward so it overlaps the next
     exit's compute on the GPU (NCCL runs on its own stream);
  3. the per-exit partial losses (sum all-reduce) for reporting.

The compute is injected (`run_exit`), so the same orchestration drives the CUDA
library on GPUs (NCCL) and is tested on CPUs with the oracle (gloo,
tests/test_dp_gloo.py).
"""

from __future__ import annotations

from typing import Callable, Iterable

import torch
import torch.distributed as dist


def shard_range(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous token shard of `rank` (sizes differ by at most one)."""
    base, rem = divmod(n_global, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def data_parallel_step(n_exits: int, count_local: Callable[[], torch.Tensor],
                       run_exit: Callable[[int, torch.Tensor], None],
                       grads_of: Callable[[int], Iterable[torch.Tensor]],
                       loss: torch.Tensor, optimizer_step: Callable[[], None] | None = None,
                       group=None) -> torch.Tensor:
    """One data-parallel EE-Tuning step.

    count_local() -> int64 tensor [1] with the local valid-token count;
    run_exit(i, W) computes exit i's loss (into loss[i]) and gradients on the
    local tokens, normalised by the global count W; grads_of(i) yields exit i's
    gradient tensors; optimizer_step() applies the update after all reductions.
    Returns the global count W.
    """
    W = count_local()
    dist.all_reduce(W, group=group)
    handles = []
    for i in range(n_exits):
        run_exit(i, W)
        for t in grads_of(i):
            handles.append(dist.all_reduce(t, group=group, async_op=True))
    handles.append(dist.all_reduce(loss, group=group, async_op=True))
    for h in handles:
        h.wait()
    if optimizer_step is not None:
        optimizer_step()
    return W
