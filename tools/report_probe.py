"""Single cs_simulate + report JSON: wall time split (kernel via TICTAC_EVENT_TRACE)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
for m in ("resnet_v2_50_inference", "resnet_v2_101_training"):
    g = L.model(m, 1)
    o = g.declared()
    s = g.random(1)
    for k in range(5):
        t0 = time.perf_counter()
        r = g.simulate(o, s, policy(True, 1, 0.0))
        t1 = time.perf_counter()
        js = r.json()
        t2 = time.perf_counter()
        print(m, k, f"simulate {1e3 * (t1 - t0):.3f} ms, json {1e3 * (t2 - t1):.3f} ms", flush=True)
