"""The speculative TAC kernels (retire the lowest outstanding column while
checking that nothing beats it; undo and walk the find-first chain when
something does) against the one-block kernel, on graphs whose TAC chains are
not empty so the misspeculation path runs: the corpus worker / cluster /
model graphs, irregular workers and the same graphs with scrambled
durations. tac_cspec_kernel (one cluster; 32- and 64-bit values) is forced
with TICTAC_TAC_CSPEC=1, tac_spec_kernel (cooperative grid) with
TICTAC_TAC_BLOCKS."""
import json
import os
import random
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import json, sys
sys.path.insert(0, '.')
from paper_1803_03288_b200.capi import Lib
L = Lib()
out = []
for text in json.load(open(sys.argv[1])):
    g = L.graph(text)
    out.append(g.tac(g.declared()).priorities())
print(json.dumps(out))
"""


def _scrambled(text, seed):
    d = json.loads(text)
    rnd = random.Random(seed)
    for op in d["ops"]:
        op["time_us"] = rnd.choice([0, 1, 2, 3, 5, 8, 13, 40, 100])
        op.pop("bytes", None)
    return json.dumps(d)


def _graphs(lib):
    from corpus import cluster_graphs, irregular_worker, model_graphs, worker_graphs
    texts = [t for _, t in worker_graphs(lib) + cluster_graphs(lib) + model_graphs(lib)]
    texts += [irregular_worker(s) for s in range(6)]
    texts += [_scrambled(t, k) for k, t in enumerate(list(texts))]
    texts.append(lib.model("inception_v3_training_branchy", 1).serialize())
    texts.append(_scrambled(lib.model("resnet_v2_50_inference_branchy", 1).serialize(), 99))
    return texts


def _run(path, env_extra):
    # (the kernel knobs of the calling environment are dropped: each run
    # forces exactly the path it names)
    env = {k: v for k, v in os.environ.items() if not k.startswith("TICTAC_TAC")}
    env.update(TICTAC_TAC_TRACE="1", **env_extra)
    r = subprocess.run([sys.executable, "-c", CODE, path], cwd=ROOT, capture_output=True, text=True, env=env,
                       check=True, timeout=600)
    misses = [int(ln.rsplit(",", 1)[1].split()[0]) for ln in r.stderr.splitlines() if "misspeculated" in ln]
    return json.loads(r.stdout.strip().splitlines()[-1]), misses


def test_speculative_tac_matches_one_block(lib, tmp_path):
    texts = _graphs(lib)
    path = tmp_path / "graphs.json"
    path.write_text(json.dumps(texts))
    want, _ = _run(str(path), {"TICTAC_TAC_BLOCKS": "1"})
    total_misses = 0
    for name, env in (("cluster, 32-bit", {"TICTAC_TAC_CSPEC": "1"}),
                      ("cluster, 64-bit", {"TICTAC_TAC_CSPEC": "1", "TICTAC_TAC_WIDE": "1"}),
                      ("grid, 3 blocks", {"TICTAC_TAC_BLOCKS": "3"}),
                      ("grid, 64 blocks", {"TICTAC_TAC_BLOCKS": "64"})):
        got, misses = _run(str(path), env)
        for k, (a, b) in enumerate(zip(got, want)):
            assert a == b, (name, k)
        assert misses, name  # the speculative kernel ran
        total_misses += sum(misses)
        if name.startswith("cluster"):
            assert sum(misses) > 0, name  # and its misspeculation path did
    assert total_misses > 0
