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


MIN_KEYS = (0, 4)  # CS_DSTATS_I64 words holding min keys (makespan, iteration time)
MAX_KEYS = (1, 5)  # ... and max keys; every other word is summed


def packed_words(world: int) -> int:
    """include/commsched.h CS_PACKED_WORDS."""
    return 6 * world + 2006


def reduce_stats_device(lib, i64, f64, rank: int, world: int, buf, stream: int = 0):
    """The same reduction on CUDA tensors through the library's pack/unpack
    kernels (cs_sweep_stats_pack / _unpack): two tiny launches around the one
    all-reduce, all on `stream` (a cudaStream_t)."""
    import torch.distributed as dist
    if world == 1:
        return i64, f64
    n = packed_words(world)
    lib.call("cs_sweep_stats_pack", i64.data_ptr(), f64.data_ptr(), rank, world, buf.data_ptr(), stream)
    dist.all_reduce(buf[:n])
    lib.call("cs_sweep_stats_unpack", buf.data_ptr(), world, i64.data_ptr(), f64.data_ptr(), stream)
    return i64, f64


def reduce_stats(i64, f64, rank: int, world: int, buf=None):
    """In-place all-reduce of one step's statistics: ONE SUM all-reduce.

    Every rank writes into a zeroed int64 vector: its min/max keys (words 0,
    4 / 1, 5) into per-rank slots, its counters and histograms into a shared
    region, and the bit patterns of its float sums f64 into per-rank slots;
    after the SUM each slot holds exactly one rank's value, so the min/max and
    the float sums (in rank order, deterministic) are finished locally. Keys
    are (m << key_bits) | offset with offsets relative to the GLOBAL seed
    base, so the minimum resolves ties to the lowest seed across ranks."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return i64, f64
    keys = MIN_KEYS + MAX_KEYS
    n_i = i64.numel()
    n_f = f64.numel()
    kw = len(keys) * world
    size = kw + n_i + n_f * world
    if buf is None or buf.numel() < size:
        buf = torch.zeros(size, dtype=torch.int64, device=i64.device)
    buf.zero_()
    big = torch.full_like(i64[0], (1 << 63) - 1)
    for j, k in enumerate(keys):
        v = i64[k]
        if k in MIN_KEYS:  # an idle rank's min key is all ones (-1 as int64): it must not win
            v = torch.where(v < 0, big, v)
        buf[j * world + rank] = v
    body = i64.clone()
    for k in keys:
        body[k] = 0
    buf[kw:kw + n_i] = body
    fo = kw + n_i
    buf[fo + rank * n_f:fo + (rank + 1) * n_f] = f64.contiguous().view(torch.int64)
    dist.all_reduce(buf[:size])
    i64.copy_(buf[kw:kw + n_i])
    for j, k in enumerate(keys):
        slots = buf[j * world:(j + 1) * world]
        i64[k] = slots.min() if k in MIN_KEYS else slots.max()
    f64.copy_(buf[fo:fo + world * n_f].view(torch.float64).view(world, n_f).sum(0))
    return i64, f64
