"""Thread-per-run event replica: throughput vs warps (32-run groups) per SM,
for a worker DAG run ungated with tied priorities (unprioritized recvs) and
for config 3's full cluster makespans."""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
B = 262144
cases = []
g = L.model("resnet_v2_50_inference", 1)
cases.append(("resnet50 inference, no schedule", lambda: g.sweep_random(g.declared(), 1, B, policy(False, 0, 0.0))))
c = L.model("vgg16_training", 1).expand(4, 1, 0)
co = c.declared()
cases.append(("config3 cluster makespans", lambda: c.sweep_random(co, 1, B, None, makespans=True)))
for name, fn in cases:
    os.environ.pop("TICTAC_EVENT_GROUPS", None)
    fn()
    for per_sm in (0, 2, 4, 8, 16, 32):
        if per_sm:
            os.environ["TICTAC_EVENT_GROUPS"] = str(per_sm)
        else:
            os.environ.pop("TICTAC_EVENT_GROUPS", None)
        ts = []
        for _ in range(2):
            t = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t) * 1e3)
        print(f"{name:34s} groups/SM={per_sm or 'default':>7} " + " ".join(f"{x:8.1f}" for x in ts) + " ms",
              flush=True)
