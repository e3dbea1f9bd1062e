"""Multi-GPU plumbing for batched sweeps: one process per GPU, contiguous
seed shards, one reduction per step over torch.distributed (NCCL on GPUs,
gloo for the CPU tests). The compute never exchanges data; only the
per-rank statistics (layout: include/commsched.h CS_DSTATS_*) are combined.
"""
from __future__ import annotations


def shard(seed_lo: int, count: int, rank: int, world: int) -> tuple[int, int]:
    """Rank's contiguous seed range [lo, lo + n) of seeds [seed_lo, seed_lo + count)."""
    per = (count + world - 1) // world
    lo = seed_lo + rank * per
    n = max(0, min(per, count - rank * per))
    return lo, n


def reduce_stats(i64, f64, rank: int, world: int, slots=None):
    """In-place all-reduce of one step's statistics.

    i64[0] (min key) and i64[1] (max key) are gathered through per-rank slots
    of a zeroed vector and one SUM all-reduce, the counters/histograms
    i64[2:] with a second SUM, the float sums f64 with a third. Keys are
    (m << key_bits) | offset with offsets relative to the GLOBAL seed base,
    so the minimum resolves ties to the lowest seed across ranks."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return i64, f64
    if slots is None:
        slots = torch.zeros(2 * world, dtype=torch.int64, device=i64.device)
    slots.zero_()
    # an idle rank's min key is all ones (-1 as int64): it must not win
    slots[rank] = torch.where(i64[0] < 0, torch.full_like(i64[0], (1 << 63) - 1), i64[0])
    slots[world + rank] = i64[1]
    dist.all_reduce(slots)
    dist.all_reduce(i64[2:])
    dist.all_reduce(f64)
    i64[0] = slots[:world].min()
    i64[1] = slots[world:].max()
    return i64, f64
