"""Single cs_simulate + report JSON: wall time split per call, this library
and (when oracle/_ref is built) the reference library.

    TICTAC_EVENT_TRACE=1 python tools/report_probe.py
"""
import os
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402
import oracle  # noqa: E402

libs = {"ours": Lib()}
if oracle.ref_available():
    libs["ref"] = Lib(oracle.REF_LIB)
for m in ("resnet_v2_50_inference", "resnet_v2_101_training"):
    text = libs["ours"].model(m, 1).serialize()
    for name, L in libs.items():
        g = L.graph(text)
        o = g.declared()
        s = g.random(1)
        for k in range(4):
            t0 = time.perf_counter()
            r = g.simulate(o, s, policy(True, 1, 0.0))
            t1 = time.perf_counter()
            js = r.json()
            t2 = time.perf_counter()
            r.makespan()
            print(m, name, k, f"simulate {1e3 * (t1 - t0):.3f} ms, json {1e3 * (t2 - t1):.3f} ms"
                  f" ({len(js)} chars)", flush=True)
