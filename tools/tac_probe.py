"""Small driver for profiling the TAC / event-simulator kernels (ncu)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
which = sys.argv[1] if len(sys.argv) > 1 else "tac"
g = L.model(sys.argv[2] if len(sys.argv) > 2 else "resnet_v2_101_training", 1)
o = g.declared()
t = time.perf_counter()
if which == "tac":
    s = g.tac(o)
    print("tac", len(s.priorities()), time.perf_counter() - t)
elif which == "tic":
    g.tic("amended")  # warm
    t = time.perf_counter()
    s = g.tic("amended")
    print("tic", time.perf_counter() - t)
else:
    s = g.tac(o)
    r = g.simulate(o, s, policy(True, 1, 0.0))
    js = r.json()  # materialises the event list: one exact replica run
    print("sim", r.makespan(), len(js), time.perf_counter() - t)
