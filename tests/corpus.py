"""Deterministic graph corpus shared by the parity tests and the golden
generator (tests/golden/make_golden.py). Graphs are built with the reference
generators' semantics (synthetic.cpp, cluster.cpp) and the model-shaped
backbones; everything is emitted as reference-format JSON text so both
libraries read the same bytes."""
from __future__ import annotations

# (shape, layers, params, ratio, seed) — mirrors acceptance.cpp's corpora
SYNTH = [
    ("chain", 3, 1, "1", 5), ("chain", 6, 2, "1/2", 11), ("layered", 4, 3, "2", 7),
    ("layered", 2, 2, "1", 9), ("seriesparallel", 5, 1, "1", 1000),
    ("seriesparallel", 7, 1, "1/2", 1003), ("seriesparallel", 6, 2, "2", 77),
    ("layered", 12, 4, "1", 3), ("seriesparallel", 30, 1, "1", 42), ("chain", 40, 1, "2", 8),
]
CLUSTERS = [  # (synthetic index, workers, ps, ps_op_time)
    (3, 2, 1, 1), (0, 4, 1, 100), (2, 3, 2, 5), (7, 4, 1, 0),
]
MODELS = ["resnet_v2_50_inference", "vgg16_training"]


def worker_graphs(lib):
    out = []
    for s in SYNTH:
        g = lib.generate(*s)
        out.append((g.name(), g.serialize()))
    return out


def cluster_graphs(lib):
    out = []
    for idx, w, p, t in CLUSTERS:
        g = lib.generate(*SYNTH[idx]).expand(w, p, t)
        out.append((g.name(), g.serialize()))
    return out


def model_graphs(lib):
    return [(m, lib.model(m, 1).serialize()) for m in MODELS]


def _op(oid, kind, dev, unit, name, t):
    return {"id": oid, "kind": kind, "resource": {"device": dev, "unit": unit, "name": name}, "time_us": t}


def irregular_worker(seed: int, n_comp=14, n_recv=6, n_send=2, cpus=2, chans=2):
    """Worker partition outside the closed form's preconditions: several
    compute units and channels on one device, send ops, zero durations,
    multi-parent DAG. Seeded python RNG; reference-format JSON."""
    import json
    import random
    rnd = random.Random(seed)
    ops, edges = [], []
    recvs = [f"r{k:02d}" for k in range(n_recv)]
    comps = [f"c{k:02d}" for k in range(n_comp)]
    sends = [f"s{k:02d}" for k in range(n_send)]
    for r in recvs:
        ops.append(_op(r, "recv", "w0", "channel", f"net{rnd.randrange(chans)}", rnd.choice([0, 1, 2, 3, 5, 8])))
    for k, c in enumerate(comps):
        ops.append(_op(c, "compute", "w0", "compute", f"cpu{rnd.randrange(cpus)}", rnd.choice([0, 1, 2, 4, 6])))
        pool = recvs + comps[:k]
        for p in rnd.sample(pool, min(len(pool), rnd.randint(1, 3))):
            edges.append([p, c])
    for s in sends:
        ops.append(_op(s, "send", "w0", "channel", f"net{rnd.randrange(chans)}", rnd.choice([1, 2, 3])))
        for p in rnd.sample(comps, 2):
            edges.append([p, s])
    rnd.shuffle(ops)
    return json.dumps({"name": f"irregular-w{seed}", "partition": "worker", "ops": ops, "edges": edges})


def wide_fanin(seed: int, n_recv=5000):
    """Worker graph whose dependency closure takes the large (global-memory)
    path with every kind of closure term: an op fed by every recv (more terms
    than one shared-memory chunk), ops fed by the previous row, by earlier
    non-root rows and by recv subsets."""
    import json
    import random
    rnd = random.Random(seed)
    recvs = [f"r{k:04d}" for k in range(n_recv)]
    ops = [_op(r, "recv", "w0", "channel", "net0", rnd.randint(1, 9)) for r in recvs]
    comps = [f"c{k:02d}" for k in range(24)]
    edges = [[r, comps[0]] for r in recvs]
    for k, c in enumerate(comps):
        ops.append(_op(c, "compute", "w0", "compute", "cpu0", rnd.randint(0, 9)))
        if k == 0:
            continue
        preds = {comps[k - 1]} if k % 3 else set(rnd.sample(comps[:k], min(k, 2)))
        preds |= set(rnd.sample(recvs, rnd.randint(0, 40)))
        edges += [[p, c] for p in sorted(preds)]
    rnd.shuffle(ops)
    return json.dumps({"name": f"wide-fanin{seed}", "partition": "worker", "ops": ops, "edges": edges})


def irregular_cluster(seed: int, workers=2, n_comp=8, n_recv=4):
    """Cluster partition where worker recvs have predecessors (PS reads) and
    sends feed PS aggregation: recvs are not roots, per-worker resources
    differ in size."""
    import json
    import random
    rnd = random.Random(seed)
    ops, edges = [], []
    for k in range(n_recv):
        ops.append(_op(f"ps/read{k}", "ps_read", "ps0", "compute", "cpu0", rnd.choice([0, 1, 2])))
        ops.append(_op(f"ps/agg{k}", "ps_aggregate", "ps0", "compute", "cpu0", rnd.choice([1, 2])))
        ops.append(_op(f"ps/upd{k}", "ps_update", "ps0", "compute", "cpu0", 1))
        edges.append([f"ps/agg{k}", f"ps/upd{k}"])
    for w in range(workers):
        d = f"w{w}"
        comps = [f"{d}/c{k:02d}" for k in range(n_comp)]
        recvs = [f"{d}/r{k:02d}" for k in range(n_recv)]
        for k, r in enumerate(recvs):
            ops.append(_op(r, "recv", d, "channel", f"net{rnd.randrange(2)}", rnd.choice([1, 2, 3, 5])))
            edges.append([f"ps/read{k}", r])
        for k, c in enumerate(comps):
            ops.append(_op(c, "compute", d, "compute", f"cpu{rnd.randrange(2)}", rnd.choice([0, 1, 3, 4])))
            pool = recvs + comps[:k]
            for p in rnd.sample(pool, min(len(pool), rnd.randint(1, 2))):
                edges.append([p, c])
        for k in range(n_recv):
            s = f"{d}/s{k:02d}"
            ops.append(_op(s, "send", d, "channel", f"net{rnd.randrange(2)}", rnd.choice([1, 2])))
            edges.append([rnd.choice(comps), s])
            edges.append([s, f"ps/agg{k}"])
    return json.dumps({"name": f"irregular-c{seed}", "partition": "cluster", "ops": ops, "edges": edges})


def irregular_graphs():
    return ([(f"irregular-w{s}", irregular_worker(s)) for s in (1, 2, 3, 4)] +
            [("irregular-w5-wide", irregular_worker(5, n_comp=30, n_recv=9, n_send=3, cpus=3, chans=3))] +
            [(f"irregular-c{s}", irregular_cluster(s)) for s in (1, 2)] +
            [("irregular-w6-odd-names", odd_names(irregular_worker(6)))])


def odd_names(text: str) -> str:
    """Same graph with op ids / device / resource names that need JSON
    escaping (quote, backslash, control characters, DEL, non-ASCII)."""
    import json
    d = json.loads(text)
    suffix = ["\"q", "\\b", "\t", "\n", "\x01", "\x7f", "é", "→", "\x1f"]
    ren = {}
    for k, op in enumerate(d["ops"]):
        ren[op["id"]] = op["id"] + suffix[k % len(suffix)]
        op["id"] = ren[op["id"]]
        op["resource"]["device"] = op["resource"]["device"] + "µ"
        op["resource"]["name"] = op["resource"]["name"] + "\"x"
    d["edges"] = [[ren[a], ren[b]] for a, b in d["edges"]]
    d["name"] = d["name"] + "☃\\"
    return json.dumps(d)
