"""Small invocation of every device kernel, for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_probe.py

Covers: graph upload, closure (shared and global), property/TIC/TAC kernels
(one-block shared-memory, one-block global, distributed, register-resident),
the closed-form sweep (statistics, explicit orders, generic engine, long
streams, cluster), lexicographic brute force, random orders, and the event
replica in both run shapes (warp per run, thread per run).

(compute-sanitizer is closed on the GPU pool this repository was built on;
the probe also runs bare, as a smoke test of every kernel.)"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

L = Lib()
small = os.environ.get("SANITIZE_SMALL") is not None


def env(**kv):
    for k, v in kv.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


g = L.generate("seriesparallel", 6, 2, "1", 7)
o = g.declared()
g.properties_text(o, "amended")
g.tic("literal")
g.tac(o)
env(TICTAC_TAC_NO_SMEM="1")
g.tac(o)
env(TICTAC_TAC_NO_SMEM=None, TICTAC_TAC_BLOCKS="2")
L.model("layered:2000:200", 1).tac(L.model("layered:2000:200", 1).declared())
env(TICTAC_TAC_BLOCKS=None)
m = L.model("resnet_v2_50_inference", 1)
mo = m.declared()
m.tac(mo)
m.sweep_random(mo, 1, 512 if small else 4096, None, makespans=True)
env(TICTAC_SWEEP_FORCE_SLOW="1")
m.sweep_random(mo, 1, 64, None)
env(TICTAC_SWEEP_FORCE_SLOW=None)
lr = L.model("layered:4000:400", 1)
lr.sweep_random(lr.declared(), 1, 64, None)
orders = np.argsort(np.random.default_rng(1).random((64, m.recv_count())), axis=1).astype(np.int32)
m.simulate_orders(mo, orders, policy(True, 3, 0.0))
m.simulate_orders(mo, orders, policy(False, 3, 0.0))  # event replica, warp per run
m.simulate(mo, m.random(5)).json()
env(TICTAC_EVENT_LANES="1")
m.sweep_random(mo, 1, 256 if small else 2048, policy(True, 0, 0.2), makespans=True)  # thread per run
env(TICTAC_EVENT_LANES=None)
c = L.model("vgg16_training", 1).expand(2, 1, 0)
co = c.declared()
c.sweep_random(co, 1, 256, None, worker_makespans=True)
c.sweep_random(co, 1, 64, None, makespans=True)
ch = L.generate("chain", 8, 1, "1", 5)
ch.brute_force_text(ch.declared(), None, 8)
ch.brute_force_text(ch.declared(), policy(True, 1, 0.5), 8)
L.model("layered:20000:2000", 1).random(3)
g.tac_traffic(o)
print("sanitize probe ok, launches", L.launches())
