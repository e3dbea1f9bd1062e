"""Thread-per-run event replica: throughput vs warps (32-run groups) per SM."""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
os.environ["TICTAC_EVENT_LANES"] = "1"
B = 262144
for m in ["resnet_v2_50_inference", "resnet_v2_101_training"]:
    g = L.model(m, 1)
    o = g.declared()
    g.sweep_random(o, 1, B, policy(False, 0, 0.0))
    for per_sm in (1, 2, 4, 8, 16, 32, 8):
        os.environ["TICTAC_EVENT_GROUPS"] = str(per_sm)
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            g.sweep_random(o, 1, B, policy(False, 0, 0.0))
            ts.append((time.perf_counter() - t) * 1e3)
        print(f"{m:24s} groups/SM={per_sm:3d} " + " ".join(f"{x:8.1f}" for x in ts) + " ms", flush=True)
