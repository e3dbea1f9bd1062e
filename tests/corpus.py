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
