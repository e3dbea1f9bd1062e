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


def reduce_stats(i64, f64, rank: int, world: int, buf=None):
    """In-place all-reduce of one step's statistics: ONE SUM all-reduce.

    Every rank writes into a zeroed int64 vector: its min key i64[0] and max
    key i64[1] into per-rank slots, its counters and histograms i64[2:] into
    a shared region, and the bit patterns of its float sums f64 into per-rank
    slots; after the SUM each slot holds exactly one rank's value, so the
    min/max and the float sums (in rank order, deterministic) are finished
    locally. Keys are (m << key_bits) | offset with offsets relative to the
    GLOBAL seed base, so the minimum resolves ties to the lowest seed across
    ranks."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return i64, f64
    n_i = i64.numel() - 2
    n_f = f64.numel()
    size = 2 * world + n_i + n_f * world
    if buf is None or buf.numel() < size:
        buf = torch.zeros(size, dtype=torch.int64, device=i64.device)
    buf.zero_()
    # an idle rank's min key is all ones (-1 as int64): it must not win
    buf[rank] = torch.where(i64[0] < 0, torch.full_like(i64[0], (1 << 63) - 1), i64[0])
    buf[world + rank] = i64[1]
    buf[2 * world:2 * world + n_i] = i64[2:]
    fo = 2 * world + n_i
    buf[fo + rank * n_f:fo + (rank + 1) * n_f] = f64.contiguous().view(torch.int64)
    dist.all_reduce(buf[:size])
    i64[0] = buf[:world].min()
    i64[1] = buf[world:2 * world].max()
    i64[2:] = buf[2 * world:2 * world + n_i]
    f64.copy_(buf[fo:fo + world * n_f].view(torch.float64).view(world, n_f).sum(0))
    return i64, f64
