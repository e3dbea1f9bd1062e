"""Throughput of the exact event replica (event_sim_kernel, thread per run)
through cs_sweep_random: config 3 with 100 us PS ops forced onto the
replica, and config 3 with two parameter servers (outside every closed
form). Prints sims/s per workload.

    python tools/ev_replica_probe.py [count]
"""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
L = Lib(os.environ["TICTAC_LIB"]) if os.environ.get("TICTAC_LIB") else Lib()
cases = [("config3 ps100 (replica forced)", lambda: L.model("vgg16_training", 1).expand(4, 1, 100), True),
         ("config3 2 PS ps100", lambda: L.model("vgg16_training", 1).expand(4, 2, 100), False)]
for name, mk, force in cases:
    if force:
        os.environ["TICTAC_SWEEP_FORCE_EXACT"] = "1"
    g = mk()
    o = g.declared()
    path = g.sweep_path(o)["path"]
    g.sweep_random(o, 1, 4096)
    t = time.perf_counter()
    r = g.sweep_random(o, 1, n)
    dt = time.perf_counter() - t
    os.environ.pop("TICTAC_SWEEP_FORCE_EXACT", None)
    print({"workload": name, "path": path, "sims": n, "seconds": round(dt, 4), "sims_per_s": n / dt,
           "min_us": r["min_us"], "argmin": r["argmin_seed"]}, flush=True)
