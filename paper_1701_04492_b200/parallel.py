"""Multi-GPU plumbing for the type-II path (one process per GPU, torch.distributed).

The rank-K sum shards two ways:

* batch sharding (weak scaling): every rank executes whole transforms on its
  own slice of a batch of coefficient vectors, sharing the same samples x —
  no data-path collective;
* r-term sharding (strong scaling): rank g evaluates the contiguous block of
  terms [K g / G, K (g+1) / G) of ONE transform (nufft_plan2_exec_terms) and
  the partial f vectors are summed with one reduce (NCCL over NVLink on
  GPUs; gloo in the CPU tests).  The partition mirrors the reference's thread
  split of r ranges (transforms.hpp:181-193), with ranks in place of threads.
"""
from __future__ import annotations

from typing import Callable


def term_range(K: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of rank terms owned by `rank` (transforms.hpp:187-188)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return K * rank // world, K * (rank + 1) // world


def batch_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice of a batch of transforms owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return batch * rank // world, batch * (rank + 1) // world


def reduce_terms(partial, dst: int = 0, group=None):
    """Sum the per-rank partial f (in place on `dst`) — the one collective of r-sharding."""
    import torch.distributed as dist
    dist.reduce(partial, dst=dst, group=group)
    return partial


def exec_rsplit(partial_fn: Callable[[int, int], object], K: int, dst: int = 0, group=None):
    """partial_fn(r0, r1) -> tensor with the partial sum over terms [r0, r1);
    returns the reduced tensor (complete on rank `dst`)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = term_range(K, world, rank)
    return reduce_terms(partial_fn(r0, r1), dst=dst, group=group)
