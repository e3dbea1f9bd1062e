"""Batch-size crossover between the event replica's run shapes."""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
for m in ["resnet_v2_50_inference", "resnet_v2_101_training"]:
    g = L.model(m, 1)
    o = g.declared()
    for B in (148, 512, 1024, 2048, 4096, 16384):
        row = []
        for lanes in ("32", "1"):
            os.environ["TICTAC_EVENT_LANES"] = lanes
            g.sweep_random(o, 1, B, policy(False, 0, 0.0))
            t = time.perf_counter()
            g.sweep_random(o, 1, B, policy(False, 0, 0.0))
            row.append((time.perf_counter() - t) * 1e3)
        print(f"{m:24s} B={B:6d} warp/run {row[0]:8.1f} ms  thread/run {row[1]:8.1f} ms", flush=True)
