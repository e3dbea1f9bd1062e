"""Event-sim batch throughput and agreement: warp per run (TICTAC_EVENT_LANES=32)
vs thread per run (=1) on sweeps outside the closed form."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536


def run(label, fn):
    out = {}
    for lanes in ("32", "1"):
        os.environ["TICTAC_EVENT_LANES"] = lanes
        fn()  # warm
        t = time.perf_counter()
        r = fn()
        dt = time.perf_counter() - t
        out[lanes] = r
        print(f"{label:48s} lanes={lanes:>2s} {dt * 1e3:9.1f} ms  {N / dt / 1e3:9.1f} k sims/s", flush=True)
    same = all(np.array_equal(a, b) for a, b in zip(out["32"], out["1"]))
    print(f"{label:48s} agree={same}", flush=True)
    assert same


for m in ["resnet_v2_50_inference", "inception_v3_training", "resnet_v2_101_training"]:
    g = L.model(m, 1)
    o = g.declared()
    run(f"{m} ungated", lambda: (g.sweep_random(o, 1, N, policy(False, 0, 0.0), makespans=True)["makespans"],))
    run(f"{m} noise0.1", lambda: (g.sweep_random(o, 1, N, policy(True, 0, 0.1), makespans=True)["makespans"],))
v = L.model("vgg16_training", 1).expand(4, 1, 0)
o = v.declared()
run("vgg16x4 cluster worker makespans",
    lambda: (v.sweep_random(o, 1, N, None, makespans=True, worker_makespans=True)["worker_makespans"],))
g = L.model("resnet_v2_101_training", 1)
o = g.declared()
rng = np.random.default_rng(1)
orders = np.argsort(rng.random((N, g.recv_count())), axis=1).astype(np.int32)
run("resnet_v2_101_training simulate_orders gated", lambda: g.simulate_orders(o, orders, policy(True, 7, 0.0)))
