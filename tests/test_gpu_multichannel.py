"""Workers with several channels (clusters with several parameter servers,
and worker graphs whose recvs arrive over two or three links) on the closed
form (chain_multi_kernel: per-channel prefix sums, T_cpu = max(S(0), max_r
c(r) + S(first[r]))): sweeps against the reference library's per-seed loop,
with and without reorder noise, plus single simulations (exact replica)."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref_sweep(ref, text, n, noise):
    from paper_1803_03288_b200.capi import policy
    rg = ref.graph(text)
    ro = rg.declared()
    ms, wms = [], []
    for s in range(1, n + 1):
        r = rg.simulate(ro, rg.random(s), policy(True, s, noise))
        ms.append(r.makespan())
        if rg.is_cluster():
            wms.append(list(json.loads(r.iteration_json())["per_worker_makespan_us"].values()))
    return np.array(ms), np.array(wms)


def _split_channels(text, k):
    """The worker graph with its recvs spread round-robin over k channels."""
    d = json.loads(text)
    recvs = sorted(op["id"] for op in d["ops"] if op["kind"] == "recv")
    idx = {r: i for i, r in enumerate(recvs)}
    for op in d["ops"]:
        if op["kind"] == "recv":
            op["resource"]["name"] = f"net{idx[op['id']] % k}"
    return json.dumps(d)


def _cases(lib):
    return [
        ("vgg16 x4 / 2 PS", lib.model("vgg16_training", 1).expand(4, 2, 0).serialize()),
        ("resnet50 x3 / 3 PS", lib.model("resnet_v2_50_inference", 1).expand(3, 3, 0).serialize()),
        ("layered x2 / 4 PS", lib.generate("layered", 12, 4, "1", 3).expand(2, 4, 0).serialize()),
        ("resnet50, 2 links", _split_channels(lib.model("resnet_v2_50_inference", 1).serialize(), 2)),
        ("inception, 3 links", _split_channels(lib.model("inception_v3_training", 1).serialize(), 3)),
    ]


@pytest.mark.parametrize("noise", [0.0, 0.3])
def test_multichannel_sweeps_match_reference(lib, ref, noise):
    from paper_1803_03288_b200.capi import policy
    for name, text in _cases(lib):
        g = lib.graph(text)
        o = g.declared()
        pol = policy(True, 0, noise)
        assert g.sweep_path(o, pol)["path"] == "chain_sweep_kernel", name
        n = 400
        res = g.sweep_random(o, 1, 20_000, pol, makespans=True, worker_makespans=g.is_cluster())
        want, wwant = _ref_sweep(ref, text, n, noise)
        assert np.array_equal(res["makespans"][:n], want), name
        if g.is_cluster():
            assert np.array_equal(res["worker_makespans"][:n], wwant), name
        ms = res["makespans"]
        assert res["min_us"] == ms.min() and res["argmin_seed"] == 1 + int(np.argmin(ms)), name


def test_multichannel_single_runs_match_reference(lib, ref):
    from paper_1803_03288_b200.capi import policy
    for name, text in _cases(lib)[3:]:
        g, rg = lib.graph(text), ref.graph(text)
        o, ro = g.declared(), rg.declared()
        for seed in (1, 9):
            pol = policy(True, seed, 0.2)
            a, b = g.simulate(o, g.random(seed), pol), rg.simulate(ro, rg.random(seed), pol)
            assert (a.makespan(), a.violations()) == (b.makespan(), b.violations()), name
            assert a.json() == b.json()
        orders = np.stack([np.random.default_rng(4).permutation(g.recv_count()) for _ in range(8)]).astype(np.int32)
        ms, _ = g.simulate_orders(o, orders, policy(True, 0, 0.0))
        rids = sorted(op["id"] for op in json.loads(text)["ops"] if op["kind"] == "recv")
        for k in range(8):
            pri = {rids[c]: i for i, c in enumerate(orders[k])}
            s = ref.schedule_parse(json.dumps({"graph": g.name(), "algorithm": "random", "priorities": pri}))
            assert ms[k] == rg.simulate(ro, s, policy(True, 0, 0.0)).makespan(), name
