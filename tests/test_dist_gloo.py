"""World-size-2 gloo test of the multi-GPU host logic (CPU): contiguous seed
shards cover the range exactly once, and the one-step statistics reduction
(paper_1803_03288_b200/dist.py) equals the single-process result, with
argmin ties resolved to the lowest seed across ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_03288_b200 import dist as pdist

BINS = 1000


def stats_of(ms: np.ndarray, seeds: np.ndarray, base: int):
    """Reference statistics in the CS_DSTATS layout for given makespans."""
    i64 = np.zeros(2008, dtype=np.int64)
    f64 = np.zeros(2, dtype=np.float64)
    if len(ms) == 0:
        i64[0] = -1
        return i64, f64
    off = seeds - base
    kmin = (ms.astype(np.uint64) << np.uint64(26)) | off.astype(np.uint64)
    kmax = (ms.astype(np.uint64) << np.uint64(26)) | (np.uint64((1 << 26) - 1) - off.astype(np.uint64))
    i64[0] = int(kmin.min())
    i64[1] = int(kmax.max())
    i64[2] = int(ms.sum())
    i64[3] = len(ms)
    for b in (ms % BINS):
        i64[8 + b] += 1
    f64[0] = float((ms.astype(np.float64) ** 2).sum())
    return i64, f64


def _worker(rank, world, port, ms, base, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, n = pdist.shard(base, len(ms), rank, world)
    seeds = np.arange(lo, lo + n)
    i64, f64 = stats_of(ms[lo - base:lo - base + n], seeds, base)
    ti, tf = torch.from_numpy(i64.copy()), torch.from_numpy(f64.copy())
    pdist.reduce_stats(ti, tf, rank, world)
    if rank == 0:
        q.put((ti.numpy().copy(), tf.numpy().copy()))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shards_partition_the_range():
    for count in (0, 1, 7, 1000, 1 << 24):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                lo, n = pdist.shard(5, count, r, world)
                covered.extend(range(lo, lo + n)) if count < 10000 else covered.append((lo, n))
            if count < 10000:
                assert covered == list(range(5, 5 + count))
            else:
                assert sum(n for _, n in covered) == count


@pytest.mark.parametrize("count", [11, 1000])
def test_gloo_reduction_matches_single_process(count):
    rng = np.random.default_rng(count)
    ms = rng.integers(1000, 1200, size=count).astype(np.int64)
    ms[count // 2] = ms[count - 1] = 900  # tie across ranks: lowest seed must win
    base = 77
    want_i, want_f = stats_of(ms, np.arange(base, base + count), base)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ms, base, q)) for r in range(2)]
    for p in procs:
        p.start()
    got_i, got_f = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got_i, want_i)
    assert np.allclose(got_f, want_f)
    assert (int(got_i[0]) & ((1 << 26) - 1)) + base == base + count // 2
