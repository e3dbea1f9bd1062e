"""Exact event replica (event_sim_kernel, thread per run) on config 3 with
100 us parameter-server ops: 2^18 seeds through cs_sweep_random."""
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib  # noqa: E402

import os
L = Lib(os.environ["TICTAC_LIB"]) if os.environ.get("TICTAC_LIB") else Lib()
c = L.model("vgg16_training", 1).expand(4, 1, 100)
o = c.declared()
print(c.sweep_path(o))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
c.sweep_random(o, 1, 4096)
t = time.perf_counter()
r = c.sweep_random(o, 1, n, None)
dt = time.perf_counter() - t
print({"sims": n, "seconds": dt, "sims_per_s": n / dt, "min_us": r["min_us"], "argmin": r["argmin_seed"]})
