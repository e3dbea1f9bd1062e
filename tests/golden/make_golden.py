"""Regenerate tests/golden/reference_outputs.json from the REFERENCE library
(oracle/_ref/libcommsched_ref.so, built from /root/reference by
`make -C oracle ref`). Run in the build container:

    python tests/golden/make_golden.py

The fixture pins, per corpus graph (tests/corpus.py), the reference's exact
outputs: schedules (full JSON), and SHA-256 digests of the byte outputs of
property tables, simulation reports / chrome traces / metrics under several
policies, brute force, plus per-seed sweep makespans. GPU tests compare the
product library against it when the reference build is not present.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import corpus  # noqa: E402
import oracle  # noqa: E402
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

POLICIES = [("default", None), ("gated_s3", (True, 3, 0.0)), ("open_s5", (False, 5, 0.0)),
            ("noise_s9", (True, 9, 0.3)), ("noise_full", (True, 2, 1.0))]
SWEEP_SEEDS = 200


def sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


def outputs(L, text, kind):
    g = L.graph(text)
    o = g.declared()
    out = {"serialize": sha(g.serialize())}
    out["tic_amended"] = g.tic("amended").serialize()
    out["tic_literal"] = g.tic("literal").serialize()
    out["tac"] = g.tac(o).serialize()
    out["random"] = {str(s): g.random(s).serialize() for s in (0, 1, 7, 123456789)}
    if kind != "model":
        out["properties"] = {m: sha(g.properties_text(o, m)) for m in ("amended", "literal")}
    sims = {}
    for algo in ("none", "tic", "tac", "random"):
        s = {"none": None, "tic": g.tic(), "tac": g.tac(o), "random": g.random(17)}[algo]
        for pname, p in POLICIES:
            r = g.simulate(o, s, policy(*p) if p else None)
            text_out = r.json() + r.chrome_trace() + g.metrics_text(o, r)
            if g.is_cluster():
                text_out += r.iteration_json()
            sims[f"{algo}/{pname}"] = {"makespan": r.makespan(), "violations": r.violations(),
                                       "sha": sha(text_out)}
    out["simulate"] = sims
    if kind == "worker" and g.recv_count() <= 7:
        out["brute_force"] = g.brute_force_text(o, None, 8)
    ms = []
    for s in range(1, SWEEP_SEEDS + 1):
        r = g.simulate(o, g.random(s), policy(True, s, 0.0))
        ms.append(r.makespan())
        if g.is_cluster():
            ms[-1] = [r.makespan(), json.loads(r.iteration_json())["per_worker_makespan_us"]]
    out["sweep"] = ms
    return out


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle ref)"
    ref = Lib(oracle.REF_LIB)
    me = Lib()  # host-only generation (identical bytes, checked by tests)
    doc = {"reference": "libcommsched built from /root/reference/proj/src (oracle/Makefile)",
           "sweep_seeds": SWEEP_SEEDS, "graphs": {}}
    for kind, fn in (("worker", corpus.worker_graphs), ("cluster", corpus.cluster_graphs),
                     ("model", corpus.model_graphs)):
        for name, text in fn(me):
            doc["graphs"][name] = {"kind": kind, "text_sha": sha(text), "out": outputs(ref, text, kind)}
    path = os.path.join(HERE, "reference_outputs.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
