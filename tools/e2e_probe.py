"""Per-call breakdown of the e2e path (fresh oracle + cs_sweep_random)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib  # noqa: E402

g = Lib().model("resnet_v2_101_training", 1)
g = g.lib.graph(g.serialize())
for k in range(4):
    t = time.perf_counter()
    o = g.declared()
    t1 = time.perf_counter()
    st = g.sweep_random(o, 1, 1 << 24)
    t2 = time.perf_counter()
    print(f"call {k}: oracle {1e3 * (t1 - t):.3f} ms, sweep {1e3 * (t2 - t1):.3f} ms", flush=True)
