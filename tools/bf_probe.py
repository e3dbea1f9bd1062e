"""Brute force over all R! orders of a chain graph (closed form): repeated timings."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib  # noqa: E402

L = Lib()
for R in (8, 10, 12, 12, 12):
    g = L.generate("chain", R, 1, "1", 5)
    o = g.declared()
    for k in range(2):
        t = time.perf_counter()
        res = json.loads(g.brute_force_text(o, None, R))
        print(R, k, f"{time.perf_counter() - t:.4f} s", res["makespan_us"], len(res["distribution"]), flush=True)
