"""Gated runs with reorder noise inside SURVEY A.2's regime stay on the
closed form for single simulations and explicit orders: the noise swaps are
applied to the gate order on the host and the violations are their count
(SURVEY A.4). Compared with the reference library: makespans, violations and
the report / metrics documents byte for byte."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRAPHS = ["resnet_v2_50_inference", "resnet_v2_50_inference_branchy", "vgg16_training"]


@pytest.mark.parametrize("noise", [0.05, 0.5, 1.0])
def test_noisy_simulate_matches_reference(lib, ref, noise):
    from paper_1803_03288_b200.capi import policy
    for m in GRAPHS:
        text = lib.model(m, 1).serialize()
        g, rg = lib.graph(text), ref.graph(text)
        o, ro = g.declared(), rg.declared()
        for seed in (0, 3, 11):
            for s, rs in ((g.random(seed), rg.random(seed)), (g.tac(o), rg.tac(ro)), (g.tic("amended"), rg.tic("amended"))):
                pol = policy(True, seed, noise)
                r, rr = g.simulate(o, s, pol), rg.simulate(ro, rs, pol)
                assert (r.makespan(), r.violations()) == (rr.makespan(), rr.violations()), (m, seed)
                assert g.metrics_text(o, r) == rg.metrics_text(ro, rr)
        r, rr = g.simulate(o, g.random(5), policy(True, 5, noise)), rg.simulate(ro, rg.random(5), policy(True, 5, noise))
        assert r.json() == rr.json() and r.chrome_trace() == rr.chrome_trace(), m


def test_noisy_orders_match_reference(lib, ref):
    from paper_1803_03288_b200.capi import policy
    rng = np.random.default_rng(7)
    for m in GRAPHS[:2]:
        text = lib.model(m, 1).serialize()
        g, rg = lib.graph(text), ref.graph(text)
        o, ro = g.declared(), rg.declared()
        R = g.recv_count()
        rids = sorted(op["id"] for op in json.loads(text)["ops"] if op["kind"] == "recv")
        orders = np.stack([rng.permutation(R) for _ in range(40)]).astype(np.int32)
        for pol in (policy(True, 9, 0.3), policy(True, 1234, 1.0)):
            ms, vi = g.simulate_orders(o, orders, pol)
            for k in range(0, 40, 7):
                pri = {rids[c]: i for i, c in enumerate(orders[k])}
                s = ref.schedule_parse(json.dumps({"graph": g.name(), "algorithm": "random", "priorities": pri}))
                r = rg.simulate(ro, s, pol)
                assert (ms[k], vi[k]) == (r.makespan(), r.violations()), (m, k)
