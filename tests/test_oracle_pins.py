"""Pin the CPU oracle (oracle/oracle.c) before trusting it: the reference's
own known-answer tests and the reference library built from
/root/reference (oracle/_ref). CPU only."""
import json

import numpy as np
import pytest

import corpus


def test_rng_kats(orc):
    """test_util.cpp:110-117, SURVEY §7 hard part 2 (measured KATs)."""
    assert orc.splitmix64(1234567) == 6457827717110365317
    assert orc.MT(1).next() == 2469588189546311528
    m = orc.MT(5489)
    for _ in range(9999):
        m.next()
    assert m.next() == 9981545732273789042
    m = orc.MT(7)
    seen = {m.bounded(5) for _ in range(2000)}
    assert seen == {0, 1, 2, 3, 4}
    assert orc.MT(1).bounded(1) == 0 and orc.MT(1).bounded(0) == 0
    u = orc.MT(9)
    assert all(0.0 <= u.unit() < 1.0 for _ in range(1000))


def test_toy_kats(orc, toy_text):
    """test_properties.cpp:31-79, test_schedule.cpp:37-82, test_sim.cpp:43-145."""
    g = orc.OracleGraph.from_json(toy_text)
    assert g.dependencies() == {"op1": ["recv1"], "op2": ["recv1", "recv2"], "recv1": ["recv1"],
                                "recv2": ["recv2"]}
    M, P, Mp = g.properties(mode="literal")
    assert M == {"op1": 3, "op2": 4, "recv1": 3, "recv2": 1} and P == {"recv1": 4, "recv2": 0}
    assert Mp == {"recv1": 4, "recv2": 4}
    assert g.properties(mode="amended")[2] == {"recv1": 3, "recv2": 4}
    M2, P2, Mp2 = g.properties(["recv2"])
    assert M2["op1"] == 0 and M2["op2"] == 1 and P2 == {"recv2": 2} and Mp2 == {"recv2": 1}
    assert g.tic("amended") == ({"recv1": 0, "recv2": 1}, True)
    assert g.tic("literal") == ({"recv1": 0, "recv2": 0}, False)
    assert g.tac() == {"recv1": 0, "recv2": 1} == g.tac(incremental=True)
    m, v, st, en = g.simulate({"recv1": 0, "recv2": 1}, events=True)
    assert (m, v) == (9, 0)
    assert dict(zip(g.ids, zip(st, en))) == {"recv1": (0, 3), "recv2": (3, 4), "op1": (3, 7), "op2": (7, 9)}
    assert g.simulate({"recv1": 1, "recv2": 0})[0] == 10
    assert g.simulate({"recv1": 0, "recv2": 1}, noise=1.0) == (10, 1)
    assert {g.simulate(None, gated=False, choice_seed=s)[0] for s in range(16)} == {9, 10}
    assert g.bounds() == (10, 6)


def test_precedes_cases(orc):
    """test_schedule.cpp:13-35 (ids as column indices a<b<c<...)."""
    L = orc.lib()
    INF = orc.INF
    a, b, c, d, e, f = range(6)
    assert L.orc_precedes(a, 4, 3, 3, b, 0, 1, 4) and not L.orc_precedes(b, 0, 1, 4, a, 4, 3, 3)
    assert L.orc_precedes(c, 2, 2, 5, d, 2, 2, 7) and not L.orc_precedes(d, 2, 2, 7, c, 2, 2, 5)
    assert L.orc_precedes(c, 2, 2, 5, e, 2, 2, 5) and not L.orc_precedes(e, 2, 2, 5, c, 2, 2, 5)
    assert L.orc_precedes(c, 2, 2, 5, f, 2, 2, INF) and not L.orc_precedes(f, 2, 2, INF, c, 2, 2, 5)


def _graphs(lib):
    # host-only generation (no GPU needed); identical bytes on both libraries
    return corpus.worker_graphs(lib) + corpus.cluster_graphs(lib) + corpus.model_graphs(lib)


def test_oracle_matches_reference_schedules(orc, ref, lib):
    for name, text in _graphs(lib):
        doc = json.loads(text)
        g = orc.OracleGraph(doc)
        rg = ref.graph(text)
        for mode in ("amended", "literal"):
            s = rg.tic(mode)
            assert orc.schedule_for(g, "tic", mode=mode) == s.priorities(), name
        assert orc.schedule_for(g, "tac") == rg.tac(rg.declared()).priorities(), name
        for seed in (0, 1, 99, 2**63 + 5):
            assert orc.schedule_for(g, "random", seed) == rg.random(seed).priorities(), name
        if doc["partition"] == "worker":
            assert g.tac(incremental=True) == g.tac() == g.tac(rows=True), name
            for mode in ("amended", "literal"):
                want = rg.properties(rg.declared(), mode)
                M, P, Mp = g.properties(mode=mode)
                assert (want["M"], want["P"], want["M_plus"]) == (M, P, Mp), name
                assert want["dep"] == g.dependencies(), name


def test_oracle_matches_reference_simulation(orc, ref, lib):
    from paper_1803_03288_b200.capi import policy
    for name, text in _graphs(lib):
        doc = json.loads(text)
        g = orc.OracleGraph(doc)
        rg = ref.graph(text)
        ro = rg.declared()
        for algo in ("none", "tic", "tac", "random"):
            sched = None if algo == "none" else (rg.random(5) if algo == "random" else
                                                 (rg.tic() if algo == "tic" else rg.tac(ro)))
            pr = None if sched is None else sched.priorities()
            for gated, seed, noise in ((True, 0, 0.0), (False, 3, 0.0), (True, 8, 0.4), (True, 1, 1.0)):
                r = rg.simulate(ro, sched, policy(gated, seed, noise))
                m, v, st, en = g.simulate(pr, gated, seed, noise, events=True)
                assert (m, v) == (r.makespan(), r.violations()), (name, algo, gated, seed, noise)
                ev = {e["op"]: (e["start_us"], e["end_us"]) for e in json.loads(r.json())["events"]}
                assert ev == {s: (int(a), int(b)) for s, a, b in zip(g.ids, st, en)}, name


def test_oracle_matches_reference_sweep(orc, ref, lib):
    import os
    import subprocess
    import tempfile
    for name, text in corpus.worker_graphs(lib)[:5] + corpus.model_graphs(lib)[:1]:
        g = orc.OracleGraph(json.loads(text))
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "g.json")
            open(p, "w").write(text)
            out = os.path.join(d, "m.bin")
            r = subprocess.run([orc.REF_SWEEP, "sweep", p, "declared", "1", "64", "2", out],
                               capture_output=True, text=True, check=True)
            want = np.fromfile(out, dtype=np.int64)
        got = [g.simulate(g.random_schedule(s), True, s, 0.0)[0] for s in range(1, 65)]
        assert list(want) == got, name
        assert json.loads(r.stdout)["sims"] == 64
