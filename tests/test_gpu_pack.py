"""cs_sweep_stats_pack / _unpack (the multi-process drivers' one-all-reduce
statistics reduction) against the sequential single-plan result: three
"ranks" sweep contiguous shards into their own statistics, the packed
buffers are summed (what the SUM all-reduce does), and the unpacked words
equal one sweep over the whole range."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model,expand", [("resnet_v2_50_inference", None), ("vgg16_training", (4, 1, 100))])
def test_pack_unpack_equals_single_sweep(lib, model, expand):
    import torch
    from paper_1803_03288_b200 import capi, dist as pdist
    g = lib.model(model, 1)
    if expand:
        g = g.expand(*expand)
    o = g.declared()
    plan = capi.SweepPlan.create(g, o)
    n, world, lo = 300_000, 3, 5

    def stats(seed_lo, count):
        i64 = torch.zeros(capi.DSTATS_I64, dtype=torch.int64, device="cuda")
        f64 = torch.zeros(capi.DSTATS_F64, dtype=torch.float64, device="cuda")
        plan.reset(0, i64.data_ptr(), f64.data_ptr())
        plan.run(seed_lo, count, lo, 0, None, i64.data_ptr(), f64.data_ptr())
        return i64, f64

    total = torch.zeros(pdist.packed_words(world), dtype=torch.int64, device="cuda")
    for r in range(world):
        s_lo, s_n = pdist.shard(lo, n, r, world)
        i64, f64 = stats(s_lo, s_n)
        buf = torch.full((pdist.packed_words(world),), 7, dtype=torch.int64, device="cuda")  # pack zeroes it
        lib.call("cs_sweep_stats_pack", i64.data_ptr(), f64.data_ptr(), r, world, buf.data_ptr(), None)
        total += buf
    i64 = torch.zeros(capi.DSTATS_I64, dtype=torch.int64, device="cuda")
    f64 = torch.zeros(capi.DSTATS_F64, dtype=torch.float64, device="cuda")
    lib.call("cs_sweep_stats_unpack", total.data_ptr(), world, i64.data_ptr(), f64.data_ptr(), None)
    w_i64, w_f64 = stats(lo, n)
    got = plan.finish(i64.cpu().numpy(), f64.cpu().numpy(), lo)
    want = plan.finish(w_i64.cpu().numpy(), w_f64.cpu().numpy(), lo)
    for k in ("count", "min_us", "argmin_seed", "max_us", "argmax_seed", "sum_us", "iter_min_us",
              "iter_argmin_seed", "iter_max_us", "iter_argmax_seed", "iter_sum_us"):
        assert got[k] == want[k], k
    assert np.array_equal(got["e_hist"], want["e_hist"]) and np.array_equal(got["straggler_hist"],
                                                                             want["straggler_hist"])
    assert abs(got["sumsq_us"] - want["sumsq_us"]) <= 1e-9 * want["sumsq_us"]
