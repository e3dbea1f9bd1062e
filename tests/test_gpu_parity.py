"""GPU parity: the product library (CUDA path) against the reference's own
known answers and against the reference library built from
/root/reference (oracle/_ref), byte for byte, through the same C ABI."""
import json
import os

import numpy as np
import pytest

import corpus
from paper_1803_03288_b200.capi import CsError, policy

pytestmark = pytest.mark.gpu


def outcome(fn):
    try:
        return ("ok", fn())
    except CsError as e:
        return ("err", e.code, e.message)


# ---------------------------------------------------------------- KATs ----

def test_toy_simulation_kats(lib, toy_text):
    """test_sim.cpp:43-103 and capi_tests.cpp:236-283 known answers."""
    g = lib.graph(toy_text)
    o = g.declared()
    fwd = lib.schedule_parse('{"graph":"toy","algorithm":"tic","priorities":{"recv1":0,"recv2":1}}')
    r = g.simulate(o, fwd)
    assert r.makespan() == 9 and r.violations() == 0
    ev = {e["op"]: (e["start_us"], e["end_us"]) for e in json.loads(r.json())["events"]}
    assert ev == {"recv1": (0, 3), "recv2": (3, 4), "op1": (3, 7), "op2": (7, 9)}
    assert json.loads(r.json())["busy"] == {"w0/channel/net0": 4, "w0/compute/cpu0": 6}
    rev = lib.schedule_parse('{"graph":"toy","algorithm":"tic","priorities":{"recv1":1,"recv2":0}}')
    r2 = g.simulate(o, rev)
    ev2 = {e["op"]: (e["start_us"], e["end_us"]) for e in json.loads(r2.json())["events"]}
    assert r2.makespan() == 10 and ev2["recv2"][1] == 1 and ev2["op1"][0] == 4 and ev2["op2"][0] == 8
    tie = lib.schedule_parse('{"graph":"toy","algorithm":"tic","priorities":{"recv1":0,"recv2":0}}')
    for seed in range(6):
        rt = g.simulate(o, tie, policy(True, seed, 0.0))
        chan = [e["op"] for e in json.loads(rt.json())["events"] if "channel" in e["resource"]]
        assert rt.makespan() == 9 and chan == ["recv1", "recv2"]
    orders = set()
    for seed in range(16):
        ru = g.simulate(o, None, policy(False, seed, 0.0))
        assert ru.makespan() in (9, 10)
        orders.add(tuple(e["op"] for e in json.loads(ru.json())["events"] if "channel" in e["resource"]))
    assert len(orders) == 2
    rn = g.simulate(o, fwd, policy(True, 0, 1.0))
    chan = [e["op"] for e in json.loads(rn.json())["events"] if "channel" in e["resource"]]
    assert chan == ["recv2", "recv1"] and rn.makespan() == 10 and rn.violations() == 1


def test_forced_release_kat(lib):
    """test_sim.cpp:126-145: recv1 outranks recv2 but waits on it."""
    doc = {"name": "g", "partition": "cluster", "ops": [
        {"id": "recv1", "kind": "recv", "resource": {"device": "w0", "unit": "channel", "name": "net0"}, "time_us": 2},
        {"id": "recv2", "kind": "recv", "resource": {"device": "w0", "unit": "channel", "name": "net0"}, "time_us": 3},
        {"id": "c", "kind": "compute", "resource": {"device": "w0", "unit": "compute", "name": "cpu0"}, "time_us": 1}],
        "edges": [["recv2", "c"], ["c", "recv1"]]}
    g = lib.graph(json.dumps(doc))
    s = lib.schedule_parse('{"graph":"g","algorithm":"tic","priorities":{"recv1":0,"recv2":1}}')
    r = g.simulate(g.declared(), s)
    chan = [e["op"] for e in json.loads(r.json())["events"] if "channel" in e["resource"]]
    assert r.makespan() == 6 and chan == ["recv2", "recv1"] and r.violations() == 2


def test_toy_schedule_and_metrics_kats(lib, toy_text):
    """test_schedule.cpp:37-82, test_properties.cpp:40-79, test_metrics.cpp."""
    g = lib.graph(toy_text)
    o = g.declared()
    assert g.tic("amended").priorities() == {"recv1": 0, "recv2": 1}
    assert g.tic("amended").total_order()
    assert g.tic("literal").priorities() == {"recv1": 0, "recv2": 0}
    assert not g.tic("literal").total_order()
    assert g.tac(o).priorities() == {"recv1": 0, "recv2": 1}
    lit, amd = g.properties(o, "literal"), g.properties(o, "amended")
    assert lit["M"] == {"op1": 3, "op2": 4, "recv1": 3, "recv2": 1}
    assert lit["P"] == {"recv1": 4, "recv2": 0}
    assert lit["M_plus"] == {"recv1": 4, "recv2": 4} and amd["M_plus"] == {"recv1": 3, "recv2": 4}
    assert amd["dep"]["op2"] == ["recv1", "recv2"]
    assert g.bounds(o) == (10, 6)
    r = g.simulate(o, g.tac(o))
    m = json.loads(g.metrics_text(o, r))
    assert m == {"U_us": 10, "L_us": 6, "m_us": 9, "E": {"num": 1, "den": 4},
                 "S": {"num": 2, "den": 3}, "straggler": None}
    bf = json.loads(g.brute_force_text(o))
    assert bf == {"order": ["recv1", "recv2"], "makespan_us": 9, "distribution": [9, 10]}
    with pytest.raises(CsError) as e:
        g.brute_force_text(o, None, 1)
    assert e.value.code == 4


def test_dense_tic_ranks_and_unbounded(lib):
    """test_schedule.cpp:55-73 and test_properties.cpp:81-92."""
    def op(i, k, unit, t):
        return {"id": i, "kind": k, "resource": {"device": "w0", "unit": unit,
                                                   "name": "net0" if unit == "channel" else "cpu0"}, "time_us": t}
    doc = {"name": "g", "partition": "worker",
           "ops": [op("r1", "recv", "channel", 1), op("r2", "recv", "channel", 1), op("r3", "recv", "channel", 1),
                   op("c1", "compute", "compute", 5), op("c2", "compute", "compute", 5)],
           "edges": [["r1", "c1"], ["r2", "c2"]]}
    g = lib.graph(json.dumps(doc))
    s = g.tic()
    assert s.priorities() == {"r1": 0, "r2": 0, "r3": 1} and not s.total_order()
    doc2 = {"name": "g", "partition": "worker", "ops": [op("r1", "recv", "channel", 2), op("r2", "recv", "channel", 5)], "edges": []}
    g2 = lib.graph(json.dumps(doc2))
    p = g2.properties(g2.declared())
    assert p["M_plus"] == {"r1": None, "r2": None} and p["P"]["r1"] == 0


# ------------------------------------------------ byte parity vs reference --

def _both(lib, ref, text, fn):
    a = outcome(lambda: fn(lib, lib.graph(text)))
    b = outcome(lambda: fn(ref, ref.graph(text)))
    assert a == b, (a[:2], b[:2])
    return a


@pytest.mark.parametrize("kind", ["worker", "cluster", "model"])
def test_schedules_match_reference(lib, ref, kind):
    graphs = {"worker": corpus.worker_graphs, "cluster": corpus.cluster_graphs,
              "model": corpus.model_graphs}[kind](lib)
    for name, text in graphs:
        for mode in ("amended", "literal"):
            _both(lib, ref, text, lambda L, g: g.tic(mode).serialize() + str(g.tic(mode).total_order()))
        _both(lib, ref, text, lambda L, g: g.tac(g.declared()).serialize())
        for seed in (0, 1, 7, 123456789):
            _both(lib, ref, text, lambda L, g: g.random(seed).serialize())
        if kind != "model":
            for mode in ("amended", "literal"):
                _both(lib, ref, text, lambda L, g: g.properties_text(g.declared(), mode))


@pytest.mark.parametrize("kind", ["worker", "cluster", "model"])
def test_simulation_matches_reference(lib, ref, kind):
    graphs = {"worker": corpus.worker_graphs, "cluster": corpus.cluster_graphs,
              "model": corpus.model_graphs}[kind](lib)
    pols = [None, policy(True, 3, 0.0), policy(False, 5, 0.0), policy(True, 9, 0.3), policy(True, 2, 1.0)]
    for name, text in graphs:
        def run(L, g, algo, pol):
            o = g.declared()
            s = {"none": None, "tic": g.tic(), "tac": g.tac(o), "random": g.random(17)}[algo]
            r = g.simulate(o, s, pol)
            out = r.json() + r.chrome_trace() + g.metrics_text(o, r) + str(r.violations())
            if g.is_cluster():
                out += r.iteration_json()
            return out
        for algo in ("none", "tic", "tac", "random"):
            for pol in pols:
                _both(lib, ref, text, lambda L, g: run(L, g, algo, pol))


def test_brute_force_matches_reference(lib, ref):
    for name, text in corpus.worker_graphs(lib)[:7]:
        for pol in (None, policy(True, 4, 0.0), policy(True, 1, 0.5)):
            _both(lib, ref, text, lambda L, g: g.brute_force_text(g.declared(), pol, 8))


def test_brute_force_closed_form(lib, ref):
    """Closed-form brute force (lexicographic unranking on the device):
    byte-equal to the reference at R = 8; at R = 10 consistent with sampled
    orders and with an exact simulation of the reported optimum."""
    for shape, layers, params in (("chain", 8, 1), ("layered", 4, 2)):
        text = lib.generate(shape, layers, params, "1", 21).serialize()
        _both(lib, ref, text, lambda L, g: g.brute_force_text(g.declared(), None, 8))
    g = lib.generate("chain", 10, 1, "1/2", 5)
    o = g.declared()
    bf = json.loads(g.brute_force_text(o, None, 10))
    sched = lib.schedule_parse(json.dumps({"graph": g.name(), "algorithm": "random",
                                           "priorities": {r: i for i, r in enumerate(bf["order"])}}))
    r = g.simulate(o, sched)
    assert r.makespan() == bf["makespan_us"] == json.loads(r.json())["makespan_us"]
    sample = g.sweep_random(o, 1, 20000, None, makespans=True)["makespans"]
    assert sample.min() >= bf["makespan_us"]
    assert set(int(x) for x in np.unique(sample)) <= set(bf["distribution"])


def test_sweep_matches_reference(lib, ref):
    """cs_sweep_random == the CLI sweep loop over the reference ABI."""
    for name, text in corpus.worker_graphs(lib) + corpus.model_graphs(lib):
        g = lib.graph(text)
        o = g.declared()
        res = g.sweep_random(o, 1, 300, None, makespans=True)
        rg = ref.graph(text)
        ro = rg.declared()
        want = []
        for s in range(1, 301):
            want.append(rg.simulate(ro, rg.random(s), policy(True, s, 0.0)).makespan())
        want = np.array(want)
        assert np.array_equal(res["makespans"], want), name
        assert res["min_us"] == want.min() and res["argmin_seed"] == 1 + int(np.argmin(want))
        assert res["sum_us"] == want.sum() and res["count"] == 300


def test_cluster_sweep_matches_reference(lib, ref):
    for name, text in corpus.cluster_graphs(lib):
        g = lib.graph(text)
        o = g.declared()
        res = g.sweep_random(o, 1, 100, None, makespans=True, worker_makespans=True)
        rg = ref.graph(text)
        ro = rg.declared()
        for i, s in enumerate(range(1, 101)):
            r = rg.simulate(ro, rg.random(s), policy(True, s, 0.0))
            it = json.loads(r.iteration_json())
            assert res["makespans"][i] == r.makespan()
            assert list(res["worker_makespans"][i]) == list(it["per_worker_makespan_us"].values())


@pytest.mark.parametrize("model", ["resnet_v2_50_inference", "vgg16_training"])
def test_event_sim_lane_modes_agree(lib, orc, monkeypatch, model):
    """The event replica's two run shapes (warp per run / thread per run,
    TICTAC_EVENT_LANES) give identical results outside the closed form, and
    spread samples match the oracle's simulator."""
    g = lib.model(model, 1)
    if model == "vgg16_training":
        g = g.expand(2, 1, 0)
    o = g.declared()
    og = orc.OracleGraph(json.loads(g.serialize()))
    R = g.recv_count()
    rng = np.random.default_rng(3)
    orders = np.argsort(rng.random((3000, R)), axis=1).astype(np.int32)
    cases = [("sweep", policy(False, 0, 0.0)), ("sweep", policy(True, 0, 0.2)),
             ("orders", policy(False, 11, 0.0)), ("orders", policy(True, 11, 0.3))]
    for kind, pol in cases:
        out = {}
        for lanes in ("32", "1"):
            monkeypatch.setenv("TICTAC_EVENT_LANES", lanes)
            if kind == "sweep":
                r = g.sweep_random(o, 5, 3000, pol, makespans=True,
                                   worker_makespans=g.is_cluster())
                out[lanes] = [r["makespans"]] + ([r["worker_makespans"]] if g.is_cluster() else [])
            else:
                out[lanes] = list(g.simulate_orders(o, orders, pol))
        for a, b in zip(out["32"], out["1"]):
            assert np.array_equal(a, b), (kind, pol.counter_gate, pol.reorder_noise)
    # oracle spot checks of the thread-per-run shape (ungated random sweeps,
    # exact replica forced: these orders would otherwise take the closed form)
    monkeypatch.setenv("TICTAC_EVENT_LANES", "1")
    monkeypatch.setenv("TICTAC_SWEEP_FORCE_EXACT", "1")
    o = g.declared()  # a fresh oracle: a fresh (forced) plan
    assert g.sweep_path(o, policy(False, 0, 0.0))["path"] == "event_sim_kernel"
    ms = g.sweep_random(o, 5, 3000, policy(False, 0, 0.0), makespans=True)["makespans"]
    for k in (0, 1, 1234, 2999):
        pr = orc.schedule_for(og, "random", 5 + k)
        m, _ = og.simulate(pr, False, 5 + k, 0.0)
        assert ms[k] == m, k


def test_irregular_graphs_match_reference(lib, ref):
    """SURVEY §8f row 1's cases outside the closed form — several compute
    units and channels per device, sends, zero durations, cluster recvs with
    predecessors — byte-equal to the reference for every schedule kind and
    policy, brute force included."""
    pols = [None, policy(True, 3, 0.0), policy(False, 5, 0.0), policy(True, 9, 0.3), policy(True, 2, 1.0)]
    for name, text in corpus.irregular_graphs():
        for mode in ("amended", "literal"):
            _both(lib, ref, text, lambda L, g: g.tic(mode).serialize() + str(g.tic(mode).total_order()))
            _both(lib, ref, text, lambda L, g: g.properties_text(g.declared(), mode))
        _both(lib, ref, text, lambda L, g: g.tac(g.declared()).serialize())

        def run(L, g, algo, pol):
            o = g.declared()
            s = {"none": None, "tic": g.tic(), "tac": g.tac(o), "random": g.random(17)}[algo]
            r = g.simulate(o, s, pol)
            out = r.json() + r.chrome_trace() + g.metrics_text(o, r) + str(r.violations())
            if g.is_cluster():
                out += r.iteration_json()
            return out
        for algo in ("none", "tic", "tac", "random"):
            for pol in pols:
                _both(lib, ref, text, lambda L, g: run(L, g, algo, pol))
        if not lib.graph(text).is_cluster():
            for pol in (None, policy(False, 4, 0.0), policy(True, 1, 0.5)):
                _both(lib, ref, text, lambda L, g: g.brute_force_text(g.declared(), pol, 8))


@pytest.mark.parametrize("gated,noise", [(True, 0.0), (False, 0.0), (True, 0.25)])
def test_irregular_sweeps_match_reference(lib, ref, gated, noise):
    """Batched sweeps over the irregular corpus (thread-per-run replica at
    this batch size) == the reference's per-seed loop."""
    n = 2500
    for name, text in corpus.irregular_graphs():
        g = lib.graph(text)
        o = g.declared()
        cl = g.is_cluster()
        res = g.sweep_random(o, 1, n, policy(gated, 0, noise), makespans=True, worker_makespans=cl)
        rg = ref.graph(text)
        ro = rg.declared()
        for i in range(n):
            s = 1 + i
            r = rg.simulate(ro, rg.random(s), policy(gated, s, noise))
            assert res["makespans"][i] == r.makespan(), (name, s)
            if cl:
                it = json.loads(r.iteration_json())
                assert list(res["worker_makespans"][i]) == list(it["per_worker_makespan_us"].values())


def test_event_sim_backs_off_when_hbm_is_short(lib):
    """With most of HBM taken by another allocation, a large exact-path batch
    runs with fewer runs in flight instead of failing (fresh process, so the
    simulator's scratch pool starts empty)."""
    import subprocess
    import sys
    code = (
        "import sys, torch; sys.path.insert(0, '.')\n"
        "from paper_1803_03288_b200.capi import Lib, policy\n"
        "g = Lib().model('resnet_v2_101_training', 1); o = g.declared()\n"
        "assert g.sweep_path(o, policy(False, 0, 0.0))['path'] == 'event_sim_kernel'\n"
        "free, _ = torch.cuda.mem_get_info()\n"
        "hog = torch.empty(max(0, free - (3 << 30)), dtype=torch.uint8, device='cuda')\n"
        "r = g.sweep_random(o, 1, 100000, policy(False, 0, 0.0))\n"
        "print(r['count'], r['min_us'], r['argmin_seed'], r['sum_us'])\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TICTAC_SWEEP_FORCE_EXACT="1")  # the exact replica, not the closed form
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, check=True,
                         env=env)
    got = [int(x) for x in out.stdout.split()[-4:]]
    g = lib.model("resnet_v2_101_training", 1)
    r = g.sweep_random(g.declared(), 1, 100000, policy(False, 0, 0.0))
    assert got == [r["count"], r["min_us"], r["argmin_seed"], r["sum_us"]]


def test_concurrent_calls_on_shared_handles(lib):
    """SURVEY §8b threading contract: graphs, oracles and schedules are
    immutable, so concurrent calls on shared handles are safe. Eight threads
    hammer the same handles (sweeps on both paths, TAC/TIC, reports, brute
    force); every result equals the sequential one."""
    import threading
    g = lib.model("resnet_v2_50_inference", 1)
    o = g.declared()
    toy = lib.generate("chain", 7, 1, "1", 3)
    to = toy.declared()
    cl = lib.generate("seriesparallel", 7, 1, "1/2", 1003).expand(2, 1, 3)  # exact replica
    co = cl.declared()
    assert cl.sweep_path(co)["path"] == "event_sim_kernel"
    jobs = {
        "sweep": lambda: g.sweep_random(o, 1, 1 << 16, None)["sum_us"],
        "sweep_exact": lambda: cl.sweep_random(co, 1, 4096, None)["sum_us"],
        "tac": lambda: g.tac(o).serialize(),
        "tic": lambda: g.tic("literal").serialize(),
        "report": lambda: g.simulate(o, g.random(9), policy(True, 9, 0.0)).json(),
        "brute": lambda: toy.brute_force_text(to, None, 8),
    }
    want = {k: f() for k, f in jobs.items()}
    errors, got = [], []

    def worker(k):
        try:
            for name in list(jobs)[k % len(jobs):] + list(jobs)[:k % len(jobs)]:
                got.append((name, jobs[name]()))
        except Exception as e:  # reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert len(got) == 8 * len(jobs)
    for name, v in got:
        assert v == want[name], name


def test_plans_with_different_shared_memory_coexist(lib):
    """A small plan created after a large one must not shrink the large
    one's shared-memory limit (the limit is a per-kernel attribute)."""
    big = lib.model("resnet_v2_101_training", 1)
    bo = big.declared()
    want = big.sweep_random(bo, 1, 1 << 16)["sum_us"]
    for shape in ("chain", "layered"):  # fresh, smaller plans of the same kernel instance
        small = lib.generate(shape, 5, 1, "1", 2)
        small.sweep_random(small.declared(), 1, 1000)
        small.tac(small.declared())
        assert big.sweep_random(bo, 1, 1 << 16)["sum_us"] == want
        assert big.sweep_random(big.declared(), 1, 1 << 16)["sum_us"] == want


def test_cluster_brute_force_matches_reference(lib, ref):
    """cs_brute_force over a cluster graph's recvs (event replica, lexicographic
    permutations on the device) == the reference, for several policies."""
    for shape, layers, params, w, ps in (("chain", 2, 1, 2, 1), ("layered", 1, 2, 2, 1), ("chain", 3, 1, 2, 2)):
        text = lib.generate(shape, layers, params, "1", 5).expand(w, ps, 1).serialize()
        for pol in (None, policy(True, 3, 0.0), policy(True, 1, 0.5), policy(False, 2, 0.0)):
            _both(lib, ref, text, lambda L, g: g.brute_force_text(g.declared(), pol, 8))


def test_config3_cluster_schedules_and_reports_match_reference(lib, ref):
    """Config 3 (VGG-16-shaped DAG, 4 workers / 1 PS): TIC (both modes), TAC,
    random schedules (per-worker derived seeds), and the cluster report /
    iteration statistics, byte for byte against the reference."""
    text = lib.model("vgg16_training", 1).expand(4, 1, 0).serialize()
    for mode in ("amended", "literal"):
        _both(lib, ref, text, lambda L, g: g.tic(mode).serialize())
    _both(lib, ref, text, lambda L, g: g.tac(g.declared()).serialize())
    for seed in (1, 99):
        _both(lib, ref, text, lambda L, g: g.random(seed).serialize())

    def rep(L, g, algo):
        o = g.declared()
        s = {"tic": g.tic(), "tac": g.tac(o), "random": g.random(5)}[algo]
        r = g.simulate(o, s, policy(True, 5, 0.0))
        return r.iteration_json() + g.metrics_text(o, r) + str(r.makespan())
    for algo in ("tic", "tac", "random"):
        _both(lib, ref, text, lambda L, g: rep(L, g, algo))


@pytest.mark.parametrize("scale", [10**5, 10**7])
def test_sweep_with_huge_durations_matches_reference(lib, ref, scale):
    """Durations scaled so U >= 2^31 (the sweep's 64-bit fold) and U >= 2^37
    (outside the closed form's key range: the exact event replica) — sweep
    makespans and statistics equal the reference's per-seed loop."""
    base = json.loads(lib.model("resnet_v2_50_inference", 1).serialize())
    for op in base["ops"]:
        op["time_us"] = op["time_us"] * scale
        op.pop("bytes", None)
    text = json.dumps(base)
    g = lib.graph(text)
    o = g.declared()
    from paper_1803_03288_b200.capi import SweepPlan
    U, _ = g.bounds(o)
    if scale == 10**5:  # closed form with the 64-bit fold
        assert (1 << 31) <= U < (1 << 37)
        SweepPlan.create(g, o)
    else:  # beyond the closed form's key range: exact replica
        assert U >= (1 << 37)
        with pytest.raises(CsError):
            SweepPlan.create(g, o)
    res = g.sweep_random(o, 1, 200, None, makespans=True)
    rg = ref.graph(text)
    ro = rg.declared()
    want = np.array([rg.simulate(ro, rg.random(s), policy(True, s, 0.0)).makespan() for s in range(1, 201)])
    assert np.array_equal(res["makespans"], want)
    assert res["min_us"] == want.min() and res["argmin_seed"] == 1 + int(np.argmin(want))
    assert res["sum_us"] == want.sum()


def _zeroed(text, seed, frac=3):
    """Same graph with roughly every `frac`-th duration set to zero (same-round
    completions of zero-duration recvs and computes)."""
    import random
    d = json.loads(text)
    rnd = random.Random(seed)
    for op in d["ops"]:
        if rnd.randrange(frac) == 0:
            op["time_us"] = 0
            op.pop("bytes", None)
    return json.dumps(d)


def test_large_closure_path_matches_reference(lib, ref, orc):
    """Closures too large for one block's shared memory (roots written in
    parallel, the other rows in topological order from staged terms,
    including a row with more terms than one staged chunk): TIC in both
    modes and the property tables match the reference library; TAC (5,003
    rounds, beyond the reference's reach) matches the oracle's A.1 TAC."""
    for seed in (1, 2):
        text = corpus.wide_fanin(seed)
        for mode in ("amended", "literal"):
            _both(lib, ref, text, lambda L, g: g.tic(mode).serialize() + str(g.tic(mode).total_order()))
            _both(lib, ref, text, lambda L, g: g.properties_text(g.declared(), mode))
        g = lib.graph(text)
        og = orc.OracleGraph(json.loads(text))
        assert g.tac(g.declared()).priorities() == og.tac(incremental=True)


def test_large_closure_kernels_on_every_graph_kind(lib, ref, monkeypatch):
    """The large-closure kernels forced on the parity corpora — worker,
    cluster (recvs with predecessors: rows with their own bit and
    predecessor rows), model and irregular graphs: TIC, TAC and property
    tables still match the reference."""
    monkeypatch.setenv("TICTAC_CLOSURE_GLOBAL", "1")
    graphs = (corpus.worker_graphs(lib)[:4] + corpus.cluster_graphs(lib)[:3] + corpus.model_graphs(lib)[:2]
              + corpus.irregular_graphs())
    for _, text in graphs:
        for mode in ("amended", "literal"):
            _both(lib, ref, text, lambda L, g: g.tic(mode).serialize() + str(g.tic(mode).total_order()))
            _both(lib, ref, text, lambda L, g: g.properties_text(g.declared(), mode))
        _both(lib, ref, text, lambda L, g: g.tac(g.declared()).serialize())


def test_single_reports_specialised_replica(lib, ref, monkeypatch):
    """Event lists of single runs inside the closed form's regime come from
    the specialised two-resource replica (csk_event_a2): byte-identical to the
    generic replica and to the reference, for TIC (with ties), TAC and random
    schedules over many choice seeds, including graphs where a third of all
    durations are zero — from both of its kernels (graph re-laid in shared
    memory, or read from the global arrays)."""
    texts = [t for _, t in corpus.worker_graphs(lib)] + [lib.model("resnet_v2_50_inference", 1).serialize()]
    texts += [_zeroed(t, k) for k, t in enumerate(texts[:6])]
    for k, text in enumerate(texts):
        g = lib.graph(text)
        o = g.declared()
        scheds = {"tic": g.tic("literal"), "tac": g.tac(o), "random": g.random(k)}
        for name, s in scheds.items():
            for seed in (0, 1, 2, 17, 12345):
                pol = policy(True, seed, 0.0)
                monkeypatch.delenv("TICTAC_NO_A2", raising=False)
                a = g.simulate(o, s, pol)
                fast = (a.json(), a.chrome_trace(), a.makespan(), a.violations())
                monkeypatch.setenv("TICTAC_A2_GLOBAL", "1")  # the kernel over the global graph arrays
                c = g.simulate(o, s, pol)
                fallback = (c.json(), c.chrome_trace(), c.makespan(), c.violations())
                monkeypatch.delenv("TICTAC_A2_GLOBAL")
                monkeypatch.setenv("TICTAC_NO_A2", "1")
                b = g.simulate(o, s, pol)
                generic = (b.json(), b.chrome_trace(), b.makespan(), b.violations())
                assert fast == generic == fallback, (k, name, seed)
        monkeypatch.delenv("TICTAC_NO_A2", raising=False)
        if k % 3 == 0:
            for seed in (0, 5):
                _both(lib, ref, text, lambda L, g: g.simulate(
                    g.declared(), g.tic("literal"), policy(True, seed, 0.0)).json())


def test_simulate_orders_rejects_out_of_range_entries(lib):
    """cs_simulate_orders: rows must be permutations of the recv columns;
    entries outside [0, R) or repeated are parameter errors on both paths
    (validated by the closed-form kernel as it reads them, by the host before
    the event replica)."""
    g = lib.model("resnet_v2_50_inference", 1)
    o = g.declared()
    R = g.recv_count()
    orders = np.tile(np.arange(R, dtype=np.int32), (300, 1))
    ms, _ = g.simulate_orders(o, orders, policy(True, 1, 0.0))
    assert (ms > 0).all()
    for bad in (R, -1):
        broken = orders.copy()
        broken[123, 7] = bad
        for pol in (policy(True, 1, 0.0), policy(True, 1, 0.5)):  # closed form / event replica
            with pytest.raises(CsError) as e:
                g.simulate_orders(o, broken, pol)
            assert e.value.code == 4 and "order entry out of range" in e.value.message
    dup = orders.copy()
    dup[200, 3] = dup[200, 4]  # not a permutation
    for pol in (policy(True, 1, 0.0), policy(True, 1, 0.5)):
        with pytest.raises(CsError) as e:
            g.simulate_orders(o, dup, pol)
        assert e.value.code == 4 and "permutations" in e.value.message


def test_ungated_runs_through_the_closed_form_match_reference(lib, ref):
    """Ungated runs with distinct recv priorities behave exactly like gated
    noiseless ones (the channel still runs recvs back-to-back in priority
    order; reorder noise is ignored when ungated, sim.cpp:93-110), so they use
    the closed form: sweeps, single simulations and brute force against the
    reference — including TIC-literal schedules with ties, which stay on the
    event replica."""
    texts = [t for _, t in corpus.worker_graphs(lib)[:6]] + [lib.model("resnet_v2_50_inference", 1).serialize()]
    from paper_1803_03288_b200.capi import SweepPlan
    closed = 0
    for text in texts:
        g = lib.graph(text)
        o = g.declared()
        try:  # wherever the gated closed form applies, the ungated one does too
            SweepPlan.create(g, o, None)
        except CsError:
            pass
        else:
            SweepPlan.create(g, o, policy(False, 0, 0.4))
            closed += 1
        rg = ref.graph(text)
        ro = rg.declared()
        for noise in (0.0, 0.4):
            res = g.sweep_random(o, 1, 150, policy(False, 0, noise), makespans=True)
            want = np.array([rg.simulate(ro, rg.random(s), policy(False, s, noise)).makespan()
                             for s in range(1, 151)])
            assert np.array_equal(res["makespans"], want)
        for sched in ("tac", "tic_literal", "random"):
            def run(L, gg):
                oo = gg.declared()
                s = {"tac": lambda: gg.tac(oo), "tic_literal": lambda: gg.tic("literal"),
                     "random": lambda: gg.random(3)}[sched]()
                r = gg.simulate(oo, s, policy(False, 7, 0.2))
                return r.json() + str(r.makespan()) + str(r.violations())
            _both(lib, ref, text, run)
        if g.recv_count() <= 8:
            _both(lib, ref, text, lambda L, gg: gg.brute_force_text(gg.declared(), policy(False, 2, 0.0), 8))
    assert closed >= 3


@pytest.mark.parametrize("noise", [0.1, 0.5, 1.0])
def test_noisy_sweeps_through_the_closed_form_match_reference(lib, ref, noise):
    """Gated sweeps with reorder noise use the closed form on the noise-
    permuted gate sequence: makespans equal the reference's
    per-seed loop on worker graphs, model DAGs (one with more than 311 noise
    draws per run) and clusters (one noise stream across the workers'
    channels)."""
    from paper_1803_03288_b200.capi import SweepPlan
    texts = [t for _, t in corpus.worker_graphs(lib)[:5]] + [lib.model("resnet_v2_50_inference", 1).serialize()]
    texts += [t for _, t in corpus.cluster_graphs(lib)[:2]]
    texts.append(lib.model("layered:4000:400", 1).serialize())  # > 311 noise draws: the stream's second block
    pol = policy(True, 0, noise)
    closed = 0
    for text in texts:
        g = lib.graph(text)
        o = g.declared()
        try:
            SweepPlan.create(g, o, pol)
            closed += 1
        except CsError:
            pass
        res = g.sweep_random(o, 1, 120, pol, makespans=True)
        rg = ref.graph(text)
        ro = rg.declared()
        want = np.array([rg.simulate(ro, rg.random(s), policy(True, s, noise)).makespan() for s in range(1, 121)])
        assert np.array_equal(res["makespans"], want), g.name()
    assert closed >= 3


def test_handles_outlive_their_graph(lib, ref):
    """Oracles, schedules and reports stay valid after their graph handle is
    freed (the reference's keep strings; here they keep the graph alive):
    same bytes as the reference, freed in the same order."""
    text = lib.model("resnet_v2_50_inference", 1).serialize()
    out = {}
    for name, L in (("ours", lib), ("ref", ref)):
        g = L.graph(text)
        o, s = g.declared(), g.tac(g.declared())
        r = g.simulate(o, s, policy(True, 3, 0.0))
        L.L.cs_graph_free(g.h)  # the graph goes first
        g.h = None
        del g
        out[name] = (o.json(), s.serialize(), r.makespan(), r.json(), r.chrome_trace())
    assert out["ours"] == out["ref"]
