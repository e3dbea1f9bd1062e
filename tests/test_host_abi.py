"""CPU tests of the drop-in boundary: the library loads, exports every symbol
include/commsched.h declares (a superset of the reference's 40), and its
host-side behaviour (parsing, validation messages, serialisation, expansion,
generators, oracles, schedule documents) is byte-identical to the reference.
No compute entry point is called here unless a GPU is present."""
import hashlib
import json
import os
import re
import subprocess

import pytest

import corpus
from conftest import HAS_GPU, ROOT
from paper_1803_03288_b200.capi import REFERENCE_SYMBOLS, CsError, Lib

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_outputs.json")))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "commsched.h")).read()
    return sorted(set(re.findall(r"\b(cs_[a-z_]+)\s*\(", text)))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_library_exports_header(lib):
    syms = exported(lib.path)
    declared = header_symbols()
    assert len(declared) >= 50
    missing = [s for s in declared if s not in syms]
    assert not missing, missing
    assert all(s.startswith("cs_") for s in syms), "only cs_* symbols may be exported"


def test_reference_surface_is_covered(lib, ref):
    ref_syms = {s for s in exported(ref.path) if s.startswith("cs_")}
    assert len(ref_syms) == 40
    assert ref_syms <= exported(lib.path)
    assert set(REFERENCE_SYMBOLS) == ref_syms
    assert lib.version() == ref.version() == "0.1.0"


def _same(a, b):
    def run(f):
        try:
            return ("ok", f())
        except CsError as e:
            return ("err", e.code, e.message)
    ra, rb = run(a), run(b)
    assert ra == rb, (ra, rb)
    return ra


BAD_GRAPHS = [
    "{", "[]", "", '{"name":1}', '{"name":"a"}', '{"name":"a","partition":"x","ops":[]}',
    '{"name":"a","partition":"worker","ops":[]}', '{"name":"a","partition":"worker","ops":{}}',
    '{"name":"a","partition":"worker","zzz":1}',
    '{"name":"a","partition":"worker","ops":[1]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x"}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"teleport","resource":{"device":"d","unit":"compute","name":"c"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","resource":{"device":"d","unit":"gpu","name":"c"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","resource":{"device":"d","unit":"compute"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","time_us":1.5,"resource":{"device":"d","unit":"compute","name":"c"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","time_us":-1,"resource":{"device":"d","unit":"compute","name":"c"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","bytes":5,"resource":{"device":"d","unit":"compute","name":"c"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"recv","bytes":-5,"resource":{"device":"d","unit":"channel","name":"c"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","resource":{"device":"d","unit":"channel","name":"c"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}},'
    '{"id":"x","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}}]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}}],"edges":[["x","x"]]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}}],"edges":[["x"]]}',
    '{"name":"a","partition":"worker","ops":[{"id":"x","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}}],"edges":{}}',
    '{"name":"a","partition":"worker","ops":[{"id":"r","kind":"recv","resource":{"device":"d","unit":"channel","name":"n"}},'
    '{"id":"x","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}}],"edges":[["x","r"]]}',
    '{"name":"a","partition":"worker","ops":[{"id":"s","kind":"send","resource":{"device":"d","unit":"channel","name":"n"}},'
    '{"id":"x","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}}],"edges":[["s","x"]]}',
    '{"name":"a","partition":"cluster","ops":[{"id":"a","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}},'
    '{"id":"b","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}},'
    '{"id":"c","kind":"compute","resource":{"device":"d","unit":"compute","name":"c"}}],"edges":[["a","b"],["b","c"],["c","a"]]}',
    '{\n  "name": "a",\n  "ops": [1,,2]\n}',
]


def test_graph_validation_matches_reference(lib, ref):
    for text in BAD_GRAPHS:
        _same(lambda: lib.graph(text).serialize(), lambda: ref.graph(text).serialize())


def test_host_outputs_match_reference(lib, ref):
    for name, text in corpus.worker_graphs(lib) + corpus.cluster_graphs(lib) + corpus.model_graphs(lib):
        a, b = lib.graph(text), ref.graph(text)
        assert a.serialize() == b.serialize() == lib.graph(a.serialize()).serialize()
        assert a.topo_order() == b.topo_order()
        assert a.worker_devices() == b.worker_devices()
        assert (a.op_count(), a.edge_count(), a.recv_count(), a.is_cluster()) == \
               (b.op_count(), b.edge_count(), b.recv_count(), b.is_cluster())
        for mk in ("declared", "general"):
            assert getattr(a, mk)().json() == getattr(b, mk)().json()
        _same(lambda: a.bandwidth(1250).json(), lambda: b.bandwidth(1250).json())
        _same(lambda: a.bandwidth(0).json(), lambda: b.bandwidth(0).json())
        for d in a.worker_devices() + ["nowhere"]:
            _same(lambda: a.partition(d).serialize(), lambda: b.partition(d).serialize())
        if not a.is_cluster():
            for w, p, t in ((1, 1, 0), (3, 2, 7), (0, 1, 1), (2, 0, 1), (2, 1, -1)):
                _same(lambda: a.expand(w, p, t).serialize(), lambda: b.expand(w, p, t).serialize())
        assert hashlib.sha256(a.serialize().encode()).hexdigest() == GOLD["graphs"][name]["out"]["serialize"]


def test_generators_match_reference(lib, ref):
    cases = [(s, l, p, r, seed) for s in ("chain", "layered", "seriesparallel", "pretzel")
             for l in (0, 1, 4) for p in (0, 1, 3) for r in ("1", "2/3", "0.25", "-1", "x", "1/0", "0.0000001")
             for seed in (0, 9)]
    for c in cases:
        _same(lambda: lib.generate(*c).serialize(), lambda: ref.generate(*c).serialize())


def test_traces_and_schedule_documents_match_reference(lib, ref, toy_text):
    a, b = lib.graph(toy_text), ref.graph(toy_text)
    traces = [
        '{"op": "op1", "run": 0, "us": 4200}\n{"op": "op1", "run": 1, "us": 4000}\n'
        '{"op": "op2", "run": 0, "us": 2}\n{"op": "recv1", "run": 0, "us": 3}\n{"op": "recv2", "run": 0, "us": 1}\n',
        '{"op": "op1", "run": 0, "us": 1}', '\n\n  \n', '{"op": "op1", "run": -1, "us": 1}',
        '{"op": "op1", "run": 0, "us": -1}', '{"op": 1}', '{"op": "op1", "run": 0, "us": 1}\n{',
        '{"op": "op1", "run": 0, "us": 4}\n{"op": "op2", "run": 0, "us": 2}\n{"op": "recv1", "run": 0, "us": 3}\n'
        '{"op": "recv2", "run": 0, "us": 1}\n{"op": "ghost", "run": 0, "us": 9}',
    ]
    for t in traces:
        _same(lambda: a.traces(t).json(), lambda: b.traces(t).json())
    docs = ['{"graph": "toy", "algorithm": "tic", "priorities": {"recv1": 0, "recv2": 1}}',
            '{"graph": "g", "algorithm": "magic", "priorities": {"r": 0}}', "[]", "{",
            '{"graph": "g", "algorithm": "tic", "priorities": {"r": -1}}',
            '{"graph": "g", "algorithm": "tac", "priorities": {"r1": 0, "r2": 0}}',
            '{"graph": "g", "algorithm": "random", "priorities": {"b": 1, "a": 0}}',
            '{"graph": "g", "algorithm": "random", "priorities": {"b": 2, "a": 0}}',
            '{"graph": "g", "algorithm": "random", "priorities": {}}']
    for d in docs:
        _same(lambda: (lambda s: s.serialize() + str(s.total_order()))(lib.schedule_parse(d)),
              lambda: (lambda s: s.serialize() + str(s.total_order()))(ref.schedule_parse(d)))


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu(lib, toy_text):
    g = lib.graph(toy_text)
    o = g.declared()
    for f in (lambda: g.tac(o), lambda: g.tic(), lambda: g.random(1), lambda: g.simulate(o),
              lambda: g.properties(o), lambda: g.sweep_random(o, 1, 10)):
        with pytest.raises(CsError) as e:
            f()
        assert e.value.code == 1 and "CUDA" in e.value.message


def test_null_arguments(lib, ref):
    import ctypes as C
    for L in (lib, ref):
        h = C.c_void_p()
        with pytest.raises(CsError) as e:
            L.call("cs_graph_parse", None, C.byref(h))
        assert e.value.code == 2 and e.value.message == "null argument: json_text"
        with pytest.raises(CsError) as e:
            L.call("cs_simulate", None, None, None, None, C.byref(h))
        assert e.value.message == "null argument: graph"
