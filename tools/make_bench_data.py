"""Writes the benchmark's input DAGs (reference-format graph JSON, gzip) to
bench_data/: both bench.py arms read these bytes, so the reference arm never
loads this library. tests/test_bench_data.py checks they equal the
generator's output.

    python tools/make_bench_data.py
"""
import gzip
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_03288_b200.capi import Lib  # noqa: E402

MODELS = ["resnet_v2_101_training", "resnet_v2_101_training_branchy", "resnet_v2_50_inference"]


def path(model):
    return os.path.join(ROOT, "bench_data", f"{model}-s1.json.gz")


def main():
    lib = Lib()
    os.makedirs(os.path.join(ROOT, "bench_data"), exist_ok=True)
    for m in MODELS:
        with gzip.GzipFile(path(m), "wb", mtime=0) as f:
            f.write(lib.model(m, 1).serialize().encode())
        print(m, os.path.getsize(path(m)))


if __name__ == "__main__":
    main()
