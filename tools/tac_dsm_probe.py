"""TAC wall time per kernel choice (each in a subprocess so the knob is read
at call time) on the config-5 layered sweep, with the committed oracle
digests checked.

    python tools/tac_dsm_probe.py [spec ...]
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
specs = sys.argv[1:] or ["layered:100000:10000", "layered:1000000:100000"]
golden = json.load(open(os.path.join(ROOT, "tests", "golden", "tac_large.json")))
code = ("import sys,time,json,hashlib; sys.path.insert(0,'.')\n"
        "from paper_1803_03288_b200.capi import Lib\n"
        "g=Lib().model(sys.argv[1],1); o=g.declared(); g.tac(o)\n"
        "ts=[]\n"
        "for _ in range(3):\n"
        "    t=time.perf_counter(); p=g.tac(o).priorities(); ts.append(time.perf_counter()-t)\n"
        "print(json.dumps({'s': sorted(ts)[1], 'sha': hashlib.sha256(json.dumps(p,sort_keys=True).encode()).hexdigest()}))\n")
for spec in specs:
    for name, env in (("default", {}), ("dsm off", {"TICTAC_TAC_DSM": "0"})):
        e = dict(os.environ, **env, TICTAC_TAC_TRACE="1")
        r = subprocess.run([sys.executable, "-c", code, spec], cwd=ROOT, capture_output=True, text=True, env=e)
        if r.returncode:
            print(spec, name, "FAILED", r.stderr[-400:], flush=True)
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        kern = [ln for ln in r.stderr.splitlines() if "DSMEM" in ln or "cluster" in ln or "blocks" in ln][-1:]
        print(spec, name, round(d["s"], 4), "s", "digest ok" if d["sha"] == golden[spec]["sha256"] else "DIGEST MISMATCH",
              kern, flush=True)
