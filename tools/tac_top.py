"""TAC wall time at the config-5 top point (10^6 ops / 10^5 recvs), cold and warm."""
import sys
import time

sys.path.insert(0, ".")
from paper_1803_03288_b200.capi import Lib  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "layered:1000000:100000"
g = Lib().model(spec, 1)
o = g.declared()
for k in range(3):
    t = time.perf_counter()
    g.tac(o)
    print(spec, "call", k, round(time.perf_counter() - t, 4), flush=True)
