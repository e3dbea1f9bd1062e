"""One exact-path sweep launch (thread per run) for profiling: config 3
(VGG-16 x 4 workers / 1 PS), full cluster iteration makespans through the
exact event replica — the bench's `event_replica_config3_makespans`."""
import sys

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib  # noqa: E402

L = Lib()
c = L.model("vgg16_training", 1).expand(4, 1, 0)
o = c.declared()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
r = c.sweep_random(o, 1, n, None, makespans=True)
print(r["count"], r["min_us"], r["argmin_seed"])
