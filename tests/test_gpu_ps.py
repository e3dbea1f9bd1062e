"""Clusters whose parameter-server ops take time: the send phase
(cluster_ps_kernel — closed-form workers, then an exact replica of the
reference's rounds over the PS core and the released channels) against the
reference library's own per-seed loop: full makespans, per-worker
makespans, statistics; gated, reorder noise, ungated; and the exact event
replica forced on the same inputs."""
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref(tmp_path, text, seeds, noise=None, ungated=False):
    import oracle
    gp, sp, op = tmp_path / "g.json", tmp_path / "s.bin", tmp_path / "m.bin"
    gp.write_text(text)
    np.asarray(seeds, dtype=np.uint64).tofile(sp)
    cmd = [oracle.REF_SWEEP, "sweeplist", str(gp), "declared", str(sp), "0", str(op)]
    if noise is not None:
        cmd.append(repr(float(noise)))
    subprocess.run(cmd, capture_output=True, text=True, check=True)
    return np.fromfile(op, dtype=np.int64)


def _clusters(lib):
    return [
        ("vgg16 x4 ps100", lib.model("vgg16_training", 1).expand(4, 1, 100)),
        ("vgg16 x3 ps1", lib.model("vgg16_training", 1).expand(3, 1, 1)),
        ("resnet50 x2 ps7", lib.model("resnet_v2_50_inference", 1).expand(2, 1, 7)),
        ("chain x2 ps3", lib.generate("chain", 6, 2, "1/2", 11).expand(2, 1, 3)),
        ("layered x4 ps250", lib.generate("layered", 12, 4, "1", 3).expand(4, 1, 250)),
        ("chain x5 ps100", lib.generate("chain", 40, 1, "2", 8).expand(5, 1, 100)),
        ("vgg16 x4 / 2 PS ps100", lib.model("vgg16_training", 1).expand(4, 2, 100)),
        ("resnet50 x3 / 3 PS ps7", lib.model("resnet_v2_50_inference", 1).expand(3, 3, 7)),
        ("layered x2 / 4 PS ps250", lib.generate("layered", 12, 4, "1", 3).expand(2, 4, 250)),
    ]


def test_ps_plan_taken(lib):
    for name, c in _clusters(lib):
        assert c.sweep_path(c.declared())["path"] == "cluster_ps_kernel", name


@pytest.mark.parametrize("noise", [None, 0.3])
def test_ps_sweep_matches_reference(lib, ref, tmp_path, noise):
    from paper_1803_03288_b200.capi import policy
    for name, c in _clusters(lib):
        o = c.declared()
        n = 6000
        res = c.sweep_random(o, 1, n, policy(True, 0, noise or 0.0), makespans=True, worker_makespans=True)
        k = 600
        raw = _ref(tmp_path, c.serialize(), np.arange(1, k + 1, dtype=np.uint64), noise)
        nw = res["worker_makespans"].shape[1]
        assert np.array_equal(res["makespans"][:k], raw[:k]), name
        assert np.array_equal(res["worker_makespans"][:k].ravel(), raw[k:k + k * nw]), name
        ms, wm = res["makespans"], res["worker_makespans"]
        it = wm.max(axis=1)
        assert res["min_us"] == ms.min() and res["argmin_seed"] == 1 + int(np.argmin(ms)), name
        assert res["iter_min_us"] == it.min() and res["iter_argmin_seed"] == 1 + int(np.argmin(it)), name
        assert res["iter_max_us"] == it.max() and res["iter_sum_us"] == int(it.sum()), name
        assert res["sum_us"] == int(ms.sum()) and (ms >= it).all()


def test_ps_equals_forced_event_replica(lib, monkeypatch):
    from paper_1803_03288_b200.capi import policy
    for name, c in _clusters(lib)[:4] + _clusters(lib)[6:]:
        for pol in (None, policy(False, 0, 0.0), policy(True, 0, 1.0)):
            text = c.serialize()
            a = lib.graph(text)
            ra = a.sweep_random(a.declared(), 11, 3000, pol, makespans=True, worker_makespans=True)
            monkeypatch.setenv("TICTAC_SWEEP_FORCE_EXACT", "1")
            b = lib.graph(text)
            ob = b.declared()
            assert b.sweep_path(ob, pol)["path"] == "event_sim_kernel"
            rb = b.sweep_random(ob, 11, 3000, pol, makespans=True, worker_makespans=True)
            monkeypatch.delenv("TICTAC_SWEEP_FORCE_EXACT")
            assert np.array_equal(ra["makespans"], rb["makespans"]), name
            assert np.array_equal(ra["worker_makespans"], rb["worker_makespans"]), name
            for k in ("min_us", "argmin_seed", "max_us", "argmax_seed", "sum_us", "iter_min_us",
                      "iter_argmin_seed", "iter_max_us", "iter_argmax_seed", "iter_sum_us"):
                assert ra[k] == rb[k], (name, k)
            assert np.array_equal(ra["e_hist"], rb["e_hist"]) and np.array_equal(ra["straggler_hist"],
                                                                                  rb["straggler_hist"])


@pytest.mark.parametrize("cluster", [True, False])
def test_exact_sweep_stats_reduced_on_device(lib, monkeypatch, cluster):
    """The exact path's statistics come from the device reduction
    (event_stats_kernel / event_argext_kernel) with no per-run read-back:
    a stats-only call over more than one 2^20-run chunk equals numpy over the
    makespans a second call returns, and the closed form's statistics."""
    from paper_1803_03288_b200.capi import policy
    if cluster:
        text = lib.generate("chain", 6, 2, "1/2", 11).expand(2, 1, 3).serialize()
        pol = None
    else:
        text = lib.generate("layered", 8, 3, "1/3", 5).serialize()
        pol = policy(True, 0, 0.3)
    n = (1 << 20) + 4321
    fast = lib.graph(text)
    rf = fast.sweep_random(fast.declared(), 7, n, pol, makespans=True, worker_makespans=cluster)
    monkeypatch.setenv("TICTAC_SWEEP_FORCE_EXACT", "1")
    g = lib.graph(text)
    o = g.declared()
    assert g.sweep_path(o, pol)["path"] == "event_sim_kernel"
    only = g.sweep_random(o, 7, n, pol)
    full = g.sweep_random(o, 7, n, pol, makespans=True, worker_makespans=cluster)
    ms = full["makespans"]
    assert np.array_equal(ms, rf["makespans"])
    assert only["count"] == n
    assert only["min_us"] == ms.min() and only["argmin_seed"] == 7 + int(np.argmin(ms))
    assert only["max_us"] == ms.max() and only["argmax_seed"] == 7 + int(np.argmax(ms))
    assert only["sum_us"] == int(ms.sum())
    assert abs(only["sumsq_us"] - float((ms.astype(np.float64) ** 2).sum())) <= 1e-9 * only["sumsq_us"]
    keys = ["min_us", "argmin_seed", "max_us", "argmax_seed", "sum_us", "count"]
    if cluster:
        it = full["worker_makespans"].max(axis=1)
        assert only["iter_min_us"] == it.min() and only["iter_argmin_seed"] == 7 + int(np.argmin(it))
        assert only["iter_max_us"] == it.max() and only["iter_argmax_seed"] == 7 + int(np.argmax(it))
        assert np.array_equal(full["worker_makespans"], rf["worker_makespans"])
        keys += ["iter_min_us", "iter_argmin_seed", "iter_max_us", "iter_argmax_seed", "iter_sum_us"]
    for k in keys:
        assert only[k] == full[k] == rf[k], k
    for h in ("e_hist", "straggler_hist"):
        assert np.array_equal(only[h], rf[h]), h
