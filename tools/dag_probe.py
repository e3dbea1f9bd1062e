"""Kernel time of the device-resident sweep plan (cs_sweep_plan_run) on the
chain-class and general-DAG graphs: 2^24 seeds, CUDA events on the launching
stream, median of 5 after warm-up.

    python tools/dag_probe.py [model ...]      (TICTAC_LIB=path: another build of the library)
"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1803_03288_b200 import capi  # noqa: E402

models = sys.argv[1:] or ["resnet_v2_101_training", "resnet_v2_101_training_branchy",
                          "inception_v3_training_branchy", "seriesparallel:244"]
L = capi.Lib(os.environ["TICTAC_LIB"]) if os.environ.get("TICTAC_LIB") else capi.Lib()
n = 1 << 24
s = torch.cuda.current_stream()
d_i64 = torch.zeros(capi.DSTATS_I64, dtype=torch.int64, device="cuda")
d_f64 = torch.zeros(capi.DSTATS_F64, dtype=torch.float64, device="cuda")
for m in models:
    g = L.generate("seriesparallel", int(m.split(":")[1]), 1, "1", 3) if m.startswith("seriesparallel") else L.model(m, 1)
    o = g.declared()
    p = capi.SweepPlan.create(g, o)
    ts = []
    for k in range(8):
        p.reset(s.cuda_stream, d_i64.data_ptr(), d_f64.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        p.run(1, n, 1, s.cuda_stream, None, d_i64.data_ptr(), d_f64.data_ptr())
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts[3:])[2]
    st = p.finish(d_i64.cpu().numpy(), d_f64.cpu().numpy(), 1)
    info = p.info()
    print(json.dumps({"model": m, "kernel": info["kernel"], "R": info["recvs_per_worker"], "ops": info["ops"],
                      "joins": info.get("joins"), "ms": round(t, 3), "Msims_per_s": round(n / t / 1e3, 1),
                      "min_us": st["min_us"], "argmin": st["argmin_seed"]}), flush=True)
