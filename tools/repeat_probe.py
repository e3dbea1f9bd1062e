"""Repeated calls of every public batched/compute entry point on the same
handles: each should settle to a steady time (no growth from call to call)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
g = L.model("resnet_v2_101_training", 1)
o = g.declared()
c = L.model("vgg16_training", 1).expand(4, 1, 0)
co = c.declared()
orders = np.argsort(np.random.default_rng(1).random((1 << 16, g.recv_count())), axis=1).astype(np.int32)
calls = {
    "sweep 2^22": lambda: g.sweep_random(o, 1, 1 << 22),
    "sweep 2^20 + makespans": lambda: g.sweep_random(o, 1, 1 << 20, makespans=True),
    "sweep noisy 2^20": lambda: g.sweep_random(o, 1, 1 << 20, policy(True, 0, 0.1)),
    "simulate_orders 2^16": lambda: g.simulate_orders(o, orders, policy(True, 1, 0.0)),
    "cluster event sweep 2^14": lambda: c.sweep_random(co, 1, 1 << 14, None, makespans=True),
    "ungated-tied event sweep 2^12": lambda: g.sweep_random(o, 1, 1 << 12, policy(False, 0, 0.0)),
    "tac": lambda: g.tac(o),
    "tic": lambda: g.tic("amended"),
    "report": lambda: g.simulate(o, g.random(3), policy(True, 1, 0.0)).json(),
}
for name, fn in calls.items():
    ts = []
    for _ in range(6):
        t = time.perf_counter()
        fn()
        ts.append(1e3 * (time.perf_counter() - t))
    print(f"{name:32s}", " ".join(f"{x:8.3f}" for x in ts), "ms", flush=True)
