"""cs_sweep_random with per-seed makespans requested: host-buffer read-back
cost against the statistics-only call (config 4)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

g = Lib().model("resnet_v2_101_training", 1)
o = g.declared()
for n, pol in ((1 << 22, None), (1 << 24, None), (1 << 22, policy(True, 0, 0.1))):
    for ms in (False, True, True):
        g.sweep_random(o, 1, 1 << 16, pol, makespans=ms)
        t = time.perf_counter()
        g.sweep_random(o, 1, n, pol, makespans=ms)
        dt = time.perf_counter() - t
        print(f"n=2^{n.bit_length() - 1} noise={pol.reorder_noise if pol else 0} makespans={ms}: "
              f"{1e3 * dt:.2f} ms, {n / dt / 1e9:.3f} G sims/s", flush=True)
