"""Thread-per-run event replica: lane-interleaved vs per-run contiguous state
(TICTAC_EVENT_LAYOUT=32/1); results must agree."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
os.environ["TICTAC_EVENT_LANES"] = "1"
B = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
for m in ["resnet_v2_50_inference", "inception_v3_training", "resnet_v2_101_training"]:
    g = L.model(m, 1)
    o = g.declared()
    for pol, tag in ((policy(False, 0, 0.0), "ungated"), (policy(True, 0, 0.1), "noise0.1")):
        res = {}
        for lay in ("32", "1"):
            os.environ["TICTAC_EVENT_LAYOUT"] = lay
            g.sweep_random(o, 1, B, pol)
            t = time.perf_counter()
            r = g.sweep_random(o, 1, B, pol, makespans=True)
            dt = time.perf_counter() - t
            res[lay] = r["makespans"]
            print(f"{m:24s} {tag:9s} layout={lay:>2s} {dt * 1e3:8.1f} ms {B / dt / 1e3:8.1f} k sims/s", flush=True)
        assert np.array_equal(res["32"], res["1"])
