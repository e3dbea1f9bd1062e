"""GPU parity against the committed reference fixture
(tests/golden/reference_outputs.json, generated from the reference library by
tests/golden/make_golden.py) — needs no reference build at run time."""
import hashlib
import json
import os

import pytest

import corpus
from paper_1803_03288_b200.capi import policy

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_outputs.json")))
POLICIES = [("default", None), ("gated_s3", (True, 3, 0.0)), ("open_s5", (False, 5, 0.0)),
            ("noise_s9", (True, 9, 0.3)), ("noise_full", (True, 2, 1.0))]


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def _graphs(lib):
    return [(k, n, t) for k, fn in (("worker", corpus.worker_graphs), ("cluster", corpus.cluster_graphs),
                                    ("model", corpus.model_graphs)) for n, t in fn(lib)]


def test_fixture_covers_corpus(lib):
    names = {n for _, n, _ in _graphs(lib)}
    assert names == set(GOLD["graphs"])
    for k, n, t in _graphs(lib):
        assert GOLD["graphs"][n]["text_sha"] == sha(t), n


@pytest.mark.parametrize("kind", ["worker", "cluster", "model"])
def test_schedules_and_properties_match_fixture(lib, kind):
    for k, name, text in _graphs(lib):
        if k != kind:
            continue
        want = GOLD["graphs"][name]["out"]
        g = lib.graph(text)
        o = g.declared()
        assert sha(g.serialize()) == want["serialize"]
        assert g.tic("amended").serialize() == want["tic_amended"], name
        assert g.tic("literal").serialize() == want["tic_literal"], name
        assert g.tac(o).serialize() == want["tac"], name
        for s, v in want["random"].items():
            assert g.random(int(s)).serialize() == v, name
        if "properties" in want:
            for m, v in want["properties"].items():
                assert sha(g.properties_text(o, m)) == v, (name, m)


@pytest.mark.parametrize("kind", ["worker", "cluster", "model"])
def test_simulations_match_fixture(lib, kind):
    for k, name, text in _graphs(lib):
        if k != kind:
            continue
        want = GOLD["graphs"][name]["out"]
        g = lib.graph(text)
        o = g.declared()
        for algo in ("none", "tic", "tac", "random"):
            s = {"none": None, "tic": g.tic(), "tac": g.tac(o), "random": g.random(17)}[algo]
            for pname, p in POLICIES:
                r = g.simulate(o, s, policy(*p) if p else None)
                out = r.json() + r.chrome_trace() + g.metrics_text(o, r)
                if g.is_cluster():
                    out += r.iteration_json()
                w = want["simulate"][f"{algo}/{pname}"]
                assert (r.makespan(), r.violations()) == (w["makespan"], w["violations"]), (name, algo, pname)
                # closed-form makespan (when it applied) == the event replica's
                assert json.loads(r.json())["makespan_us"] == r.makespan()
                assert sha(out) == w["sha"], (name, algo, pname)
        if "brute_force" in want:
            assert g.brute_force_text(o, None, 8) == want["brute_force"], name


def test_sweeps_match_fixture(lib):
    n = GOLD["sweep_seeds"]
    for k, name, text in _graphs(lib):
        want = GOLD["graphs"][name]["out"]["sweep"]
        g = lib.graph(text)
        o = g.declared()
        res = g.sweep_random(o, 1, n, None, makespans=True, worker_makespans=True)
        if k == "cluster":
            assert [int(x) for x in res["makespans"]] == [w[0] for w in want], name
            assert [list(map(int, row)) for row in res["worker_makespans"]] == \
                   [list(w[1].values()) for w in want], name
        else:
            assert [int(x) for x in res["makespans"]] == want, name
