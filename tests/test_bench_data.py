"""The committed benchmark inputs (bench_data/*.json.gz, read by both
bench.py arms) are exactly what the model generator emits."""
import gzip
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_bench_data_matches_generator(lib):
    import make_bench_data
    for m in make_bench_data.MODELS:
        with gzip.open(make_bench_data.path(m), "rb") as f:
            assert f.read().decode() == lib.model(m, 1).serialize(), m
