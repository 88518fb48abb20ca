"""Mask-sharded multi-GPU orchestration (one process per GPU).

The C(g,m) masks are independent (Supp. S:5.3 P:454), so rank r of
P processes the masks whose global index (level by level m = 0..M,
lexicographic within a level) is congruent to r mod P — the rule
gakco_set_shard implements in libgakco.so. Each rank accumulates a partial
int64 C (upper triangle); one reduce(SUM) over the process group (NCCL int64 on
B200s) gives rank 0 the full C, and rank 0 runs the epilogue (gakco_finalize).
"""
from __future__ import annotations

from itertools import combinations


def masks(g: int, M: int):
    """Global mask order: (m, removed positions) for m = 0..M, lexicographic."""
    out = []
    for m in range(M + 1):
        out.extend((m, rem) for rem in combinations(range(g), m))
    return out


def shard_masks(g: int, M: int, rank: int, world: int):
    """Masks of rank `rank` of `world` (global index = rank mod world)."""
    return [mk for i, mk in enumerate(masks(g, M)) if i % world == rank]


def sharded_kernel_matrix(C, N, accumulate, finalize, group=None, reduce_op=None):
    """One step of the sharded path.

    accumulate(C): add this rank's masks into the zeroed C (gakco_accumulate);
    finalize(C):   rank 0 only, after the reduction (gakco_finalize).
    The reduction is torch.distributed.reduce(C, dst=0, SUM) when a process
    group is initialised with more than one rank.
    """
    import torch.distributed as dist
    C.zero_()
    accumulate(C)
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if world > 1:
        dist.reduce(C, dst=0, op=reduce_op or dist.ReduceOp.SUM, group=group)
    if rank == 0:
        finalize(C)
    return rank
