"""Event replica run shapes on the bench's replica workload (branchy VGG-16
workers x 4 / 1 PS with 100 us PS ops: outside every closed form). Times
cs_sweep_random per TICTAC_EVENT_LANES setting and checks the makespans agree.

    python tools/ev_shape_probe.py [count] [lanes ...]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
shapes = sys.argv[2:] or ["1", "32"]
L = Lib(os.environ["TICTAC_LIB"]) if os.environ.get("TICTAC_LIB") else Lib()
g = L.model("vgg16_training_branchy", 1).expand(4, 1, 100)
o = g.declared()
print({"ops": g.op_count() if hasattr(g, "op_count") else None, "path": g.sweep_path(o)}, flush=True)
ref = None
for lanes in shapes:
    os.environ["TICTAC_EVENT_LANES"] = lanes
    g.sweep_random(o, 1, 4096, makespans=True)
    t = time.perf_counter()
    r = g.sweep_random(o, 1, n, makespans=True)
    dt = time.perf_counter() - t
    ms = r["makespans"]
    same = None if ref is None else bool(np.array_equal(ref, ms))
    ref = ms if ref is None else ref
    print({"lanes": lanes, "sims": n, "seconds": round(dt, 4), "sims_per_s": round(n / dt),
           "min_us": r["min_us"], "argmin": r["argmin_seed"], "agree_with_first": same}, flush=True)
