"""Latency/throughput probe of single cs_simulate calls and event-sim batches."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
for m in ["resnet_v2_50_inference", "resnet_v2_101_training"]:
    g = L.model(m, 1)
    o = g.declared()
    s = g.tac(o)
    g.simulate(o, s)
    t = time.perf_counter()
    for _ in range(20):
        r = g.simulate(o, s)
        r.makespan()
    print(m, "cs_simulate+makespan ms", (time.perf_counter() - t) / 20 * 1000, r.makespan())
    ts = []
    for _ in range(7):
        t = time.perf_counter()
        r = g.simulate(o, s)
        js = r.json()
        ts.append((time.perf_counter() - t) * 1000)
    print(m, " cs_simulate+report_json ms (median of 7, first)", sorted(ts)[3], ts[0])
    t = time.perf_counter()
    for seed in range(1, 51):
        g.simulate(o, g.random(seed), policy(True, seed, 0.0)).makespan()
    print(m, " reference sweep loop via ABI (50 seeds): ms/seed", (time.perf_counter() - t) / 50 * 1000)
    orders = np.array([list(range(g.recv_count()))] * 4096, dtype="int32")
    t = time.perf_counter()
    ms, vi = g.simulate_orders(o, orders, policy(False, 1, 0.0))
    print(" simulate_orders ungated 4096: s", time.perf_counter() - t)
v = L.model("vgg16_training", 1).expand(4, 1, 0)
o = v.declared()
t = time.perf_counter()
r = v.sweep_random(o, 1, 100000, None)
print("config3 fast 1e5:", time.perf_counter() - t, r["straggler_sum"] / r["count"], r["min_us"])
t = time.perf_counter()
r = v.sweep_random(o, 1, 2000, None, makespans=True)
print("config3 exact 2000:", time.perf_counter() - t)
