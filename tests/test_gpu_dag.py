"""General worker DAGs on the closed form (SURVEY Appendix A.2 without nested
recv-ancestor sets): dag_sweep_kernel against the reference library itself
(oracle/_ref) — random sweeps with and without reorder noise, cluster
workers, explicit orders, single simulations and brute force — and, with the
program forced onto nested graphs, against the chain-class kernel."""
import json
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BRANCHY = ["resnet_v2_50_inference_branchy", "inception_v3_training_branchy", "resnet_v2_101_training_branchy"]
SP = [("seriesparallel", 30, 1, "1", 42), ("seriesparallel", 100, 2, "1/2", 7), ("seriesparallel", 244, 1, "1", 3)]


def _ref_list(tmp_path, text, seeds, noise=None):
    import oracle
    gp, sp, op = tmp_path / "g.json", tmp_path / "s.bin", tmp_path / "m.bin"
    gp.write_text(text)
    np.asarray(seeds, dtype=np.uint64).tofile(sp)
    cmd = [oracle.REF_SWEEP, "sweeplist", str(gp), "declared", str(sp), "0", str(op)]
    if noise is not None:
        cmd.append(repr(float(noise)))
    subprocess.run(cmd, capture_output=True, text=True, check=True)
    return np.fromfile(op, dtype=np.int64)


def _graphs(lib):
    return [lib.model(m, 1) for m in BRANCHY] + [lib.generate(*s) for s in SP]


def test_dag_plan_on_non_nested_graphs(lib):
    from paper_1803_03288_b200.capi import SweepPlan
    for g in _graphs(lib):
        info = SweepPlan.create(g, g.declared()).info()
        assert info["kernel"] in ("dag_pair_kernel", "dag_sweep_kernel"), info
        assert info["joins"] > 0


@pytest.mark.parametrize("noise", [None, 0.1, 1.0])
def test_dag_sweep_matches_reference(lib, ref, tmp_path, noise):
    from paper_1803_03288_b200.capi import policy
    for g in _graphs(lib):
        o = g.declared()
        n = 20_000
        res = g.sweep_random(o, 1, n, policy(True, 0, noise or 0.0), makespans=True)
        ms = res["makespans"]
        seeds = np.arange(1, 2_001 if noise is None else 501, dtype=np.uint64)
        want = _ref_list(tmp_path, g.serialize(), seeds, noise)
        assert np.array_equal(ms[: len(seeds)], want), (g.name(), noise)
        assert res["min_us"] == ms.min() and res["argmin_seed"] == 1 + int(np.argmin(ms))
        U, L = g.bounds(o)
        assert (ms >= L).all() and (ms <= U).all()


def test_dag_config4_size_sweep_matches_reference(lib, ref, tmp_path):
    """The branchy config-4-sized DAG (5,380 ops / 244 recvs) over 2^24 seeds:
    seeds 1..10^4 plus 10^4 spread over the range against the reference."""
    g = lib.model("resnet_v2_101_training_branchy", 1)
    o = g.declared()
    n = 1 << 24
    res = g.sweep_random(o, 1, n, None, makespans=True)
    ms = res["makespans"]
    spread = np.unique(np.linspace(1, n, 10_000, dtype=np.uint64))
    seeds = np.concatenate([np.arange(1, 10_001, dtype=np.uint64), spread])
    want = _ref_list(tmp_path, g.serialize(), seeds)
    assert np.array_equal(ms[(seeds - 1).astype(np.int64)], want)
    U, L = g.bounds(o)
    bins = np.minimum((1000 * (U - ms)) // (U - L), 999)
    assert np.array_equal(res["e_hist"], np.bincount(bins, minlength=1000))
    assert res["min_us"] == ms.min() and res["argmin_seed"] == 1 + int(np.argmin(ms))
    assert res["max_us"] == ms.max() and res["sum_us"] == int(ms.sum())


def test_dag_forced_on_nested_graphs_equals_chain_kernel(lib, monkeypatch):
    """TICTAC_SWEEP_FORCE_DAG compiles nested graphs into the join program
    too: identical makespans and statistics to the chain-class kernel."""
    from paper_1803_03288_b200.capi import SweepPlan, policy
    specs = ["resnet_v2_50_inference", "vgg16_training", "layered:2000:200"]
    for spec in specs:
        for pol in (None, policy(True, 0, 0.3)):
            g1 = lib.model(spec, 1)
            a = g1.sweep_random(g1.declared(), 5, 50_000, pol, makespans=True)
            monkeypatch.setenv("TICTAC_SWEEP_FORCE_DAG", "1")
            g2 = lib.model(spec, 1)
            assert SweepPlan.create(g2, g2.declared()).info()["kernel"] in ("dag_pair_kernel", "dag_sweep_kernel")
            b = g2.sweep_random(g2.declared(), 5, 50_000, pol, makespans=True)
            monkeypatch.delenv("TICTAC_SWEEP_FORCE_DAG")
            assert np.array_equal(a["makespans"], b["makespans"]), spec
            for k in ("min_us", "argmin_seed", "max_us", "argmax_seed", "sum_us"):
                assert a[k] == b[k], (spec, k)
            assert np.array_equal(a["e_hist"], b["e_hist"])


def test_dag_cluster_workers_match_reference(lib, ref, tmp_path):
    """Branchy workers expanded to 4 workers / 1 PS with zero-time PS ops:
    full makespans and per-worker makespans against the reference."""
    for m in ("vgg16_training_branchy", "resnet_v2_50_inference_branchy"):
        c = lib.model(m, 1).expand(4, 1, 0)
        o = c.declared()
        n = 4_000
        res = c.sweep_random(o, 1, n, None, makespans=True, worker_makespans=True)
        raw = _ref_list(tmp_path, c.serialize(), np.arange(1, 501, dtype=np.uint64))
        assert np.array_equal(res["makespans"][:500], raw[:500]), m
        assert np.array_equal(res["worker_makespans"][:500].ravel(), raw[500:]), m
        assert res["min_us"] == res["makespans"].min() == res["iter_min_us"]
        assert (res["makespans"] == res["worker_makespans"].max(axis=1)).all()


def test_dag_orders_simulate_and_brute_force_match_reference(lib, ref):
    from paper_1803_03288_b200.capi import policy
    rng = np.random.default_rng(3)
    for g in _graphs(lib)[:4]:
        text = g.serialize()
        rg = ref.graph(text)
        o, ro = g.declared(), rg.declared()
        R = g.recv_count()
        orders = np.stack([rng.permutation(R) for _ in range(64)]).astype(np.int32)
        ms, vi = g.simulate_orders(o, orders)
        ids = sorted(json.loads(text)["ops"], key=lambda op: op["id"])
        rids = [op["id"] for op in ids if op["kind"] == "recv"]
        for k in range(0, 64, 9):
            pri = {rids[c]: i for i, c in enumerate(orders[k])}
            s = ref.schedule_parse(json.dumps({"graph": g.name(), "algorithm": "random",
                                               "priorities": pri}))
            assert ms[k] == rg.simulate(ro, s, policy(True, 0, 0.0)).makespan()
            assert vi[k] == 0
        for algo in ("tac", "tic"):
            s = g.tac(o) if algo == "tac" else g.tic("amended")
            rs = rg.tac(ro) if algo == "tac" else rg.tic("amended")
            assert g.simulate(o, s).makespan() == rg.simulate(ro, rs).makespan(), (g.name(), algo)
    for spec in (("seriesparallel", 8, 1, "1", 1000), ("seriesparallel", 6, 1, "1/2", 1003)):
        text = lib.generate(*spec).serialize()
        g, rg = lib.graph(text), ref.graph(text)
        assert g.brute_force_text(g.declared(), None, 8) == rg.brute_force_text(rg.declared(), None, 8), spec


def test_dag_pair_kernel_equals_single_warp_kernel(lib, monkeypatch):
    """dag_pair_kernel (random sweeps; the warps of a block share one set of
    positions/bins columns, 2 / 3 / 4 / 6 of them) against dag_sweep_kernel
    forced with TICTAC_DAG_NO_PAIR: identical makespans and statistics, with
    noise and on cluster workers."""
    from paper_1803_03288_b200.capi import policy
    for knob in ("TICTAC_DAG_NO_PAIR", "TICTAC_DAG_WARPS"):  # (a variant run may set them globally)
        monkeypatch.delenv(knob, raising=False)
    cases = [(lambda: lib.model("resnet_v2_101_training_branchy", 1), None),
             (lambda: lib.generate("seriesparallel", 300, 1, "1", 11), policy(True, 0, 0.2)),
             (lambda: lib.model("vgg16_training_branchy", 1).expand(3, 1, 0), None)]
    for make, pol in cases:
        a = make()
        assert a.sweep_path(a.declared(), pol or policy(True, 0, 0.0))["kernel"] == "dag_pair_kernel"
        ra = a.sweep_random(a.declared(), 3, 100_003, pol, makespans=True, worker_makespans=a.is_cluster())
        monkeypatch.setenv("TICTAC_DAG_NO_PAIR", "1")
        b = make()
        assert b.sweep_path(b.declared(), pol or policy(True, 0, 0.0))["kernel"] == "dag_sweep_kernel"
        rb = b.sweep_random(b.declared(), 3, 100_003, pol, makespans=True, worker_makespans=b.is_cluster())
        monkeypatch.delenv("TICTAC_DAG_NO_PAIR")
        others = [rb]
        for warps in ("2", "3", "4", "6"):  # warps sharing one phase-B set
            monkeypatch.setenv("TICTAC_DAG_WARPS", warps)
            c = make()
            others.append(c.sweep_random(c.declared(), 3, 100_003, pol, makespans=True,
                                         worker_makespans=c.is_cluster()))
            monkeypatch.delenv("TICTAC_DAG_WARPS")
        for rb in others:
            assert np.array_equal(ra["makespans"], rb["makespans"])
            if a.is_cluster():
                assert np.array_equal(ra["worker_makespans"], rb["worker_makespans"])
            for k in ("min_us", "argmin_seed", "max_us", "argmax_seed", "sum_us"):
                assert ra[k] == rb[k], k
            assert np.array_equal(ra["e_hist"], rb["e_hist"])
