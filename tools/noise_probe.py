"""Noisy closed-form sweep throughput (config 4, gated, reorder noise)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

g = Lib().model("resnet_v2_101_training", 1)
o = g.declared()
for noise in (0.0, 0.1, 1.0):
    pol = policy(True, 0, noise)
    g.sweep_random(o, 1, 1 << 24, pol)
    t = time.perf_counter()
    g.sweep_random(o, 1, 1 << 24, pol)
    print(f"noise {noise}: {(1 << 24) / (time.perf_counter() - t) / 1e9:.3f} G sims/s", flush=True)
