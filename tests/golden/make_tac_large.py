"""Oracle TAC orders for the config-5 layered sweep, where the reference
itself is infeasible (≈3e6 s at 1e5 ops, ≈7e9 s at 1e6). The
orders come from oracle/oracle.c's incremental TAC,
which tests/test_oracle_pins.py checks against both the literal restatement
and the reference library on every graph the reference can finish. Stored
as SHA-256 of the priorities JSON (schedule serialisation order).

    python tests/golden/make_tac_large.py [--top]
    python tests/golden/make_tac_large.py --tic   # TIC digests, every config-5 size

The orders come from the row-aliased form of the same restatement
(orc_tac_rows: the closure per row of ops sharing one dependency set, a
column-major retire), which reproduces orc_tac_incremental's digests at
10^4 and 10^5 and finishes the top point (10^6 ops / 10^5 recvs, --top) in
minutes; tests/test_oracle_pins.py checks all three forms on the corpus.
"""
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle  # noqa: E402
from paper_1803_03288_b200.capi import Lib  # noqa: E402


def main():
    specs = ["layered:10000:1000", "layered:100000:10000"]
    if "--top" in sys.argv:
        specs.append("layered:1000000:100000")
    path = os.path.join(HERE, "tac_large.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    lib = Lib()
    if "--tic" in sys.argv:  # TIC (both modes) at every config-5 size, the top included
        for spec in ["layered:10000:1000", "layered:100000:10000", "layered:1000000:100000"]:
            t = time.time()
            g = lib.model(spec, 1)
            og = oracle.OracleGraph(json.loads(g.serialize()))
            for mode in ("amended", "literal"):
                prio, total = og.tic(mode)
                text = json.dumps(prio, sort_keys=True)
                out[f"tic:{mode}:{spec}"] = {"sha256": hashlib.sha256(text.encode()).hexdigest(),
                                             "recvs": len(prio), "total_order": bool(total),
                                             "oracle_seconds": round(time.time() - t, 1)}
                print(spec, mode, out[f"tic:{mode}:{spec}"], flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)
        return
    for spec in specs:
        t = time.time()
        g = lib.model(spec, 1)
        og = oracle.OracleGraph(json.loads(g.serialize()))
        prio = og.tac(rows=True)
        text = json.dumps(prio, sort_keys=True)
        out[spec] = {"sha256": hashlib.sha256(text.encode()).hexdigest(), "recvs": len(prio),
                     "first": min(prio, key=prio.get), "oracle_seconds": round(time.time() - t, 1)}
        print(spec, out[spec], flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
