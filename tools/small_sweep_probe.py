"""Per-call latency of small cs_sweep_random batches (config 1, 1,000 seeds)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib  # noqa: E402

g = Lib().model("resnet_v2_50_inference", 1)
o = g.declared()
for n in (1000, 100000):
    g.sweep_random(o, 1, n)
    t = time.perf_counter()
    for _ in range(200):
        g.sweep_random(o, 1, n)
    print(f"{n} seeds: {1e6 * (time.perf_counter() - t) / 200:.1f} us per call", flush=True)
