"""One exact-path sweep launch (thread per run) for profiling:
config 4, counter gate + reorder noise 0.1, 65536 seeds."""
import sys

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib, policy  # noqa: E402

g = Lib().model("resnet_v2_101_training", 1)
o = g.declared()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
r = g.sweep_random(o, 1, n, policy(True, 0, 0.1))
print(r["count"], r["min_us"], r["argmin_seed"])
