"""Edge cases of the general-DAG and send-phase kernels against the
reference library's per-seed loop: 64-bit folds (U >= 2^31), more than 255
recvs (16-bit shared-memory items), about a third of all durations zero
(same-round completions), cluster workers with reorder noise, and the
send phase on scaled and zeroed clusters."""
import json
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _scaled(text, scale):
    d = json.loads(text)
    for op in d["ops"]:
        op["time_us"] = op["time_us"] * scale
        op.pop("bytes", None)
    return json.dumps(d)


def _zeroed(text, seed, frac=3):
    d = json.loads(text)
    rnd = random.Random(seed)
    for op in d["ops"]:
        if rnd.randrange(frac) == 0:
            op["time_us"] = 0
            op.pop("bytes", None)
    return json.dumps(d)


def _check(lib, ref, text, n=300, noise=0.0, path=None):
    from paper_1803_03288_b200.capi import policy
    g = lib.graph(text)
    o = g.declared()
    pol = policy(True, 0, noise)
    if path:
        assert g.sweep_path(o, pol)["path"] == path
    res = g.sweep_random(o, 1, n, pol, makespans=True, worker_makespans=g.is_cluster())
    rg = ref.graph(text)
    ro = rg.declared()
    want, wwant = [], []
    for s in range(1, n + 1):
        r = rg.simulate(ro, rg.random(s), policy(True, s, noise))
        want.append(r.makespan())
        if g.is_cluster():
            wwant.append(list(json.loads(r.iteration_json())["per_worker_makespan_us"].values()))
    want = np.array(want)
    assert np.array_equal(res["makespans"], want)
    if g.is_cluster():
        assert np.array_equal(res["worker_makespans"], np.array(wwant))
    assert res["min_us"] == want.min() and res["argmin_seed"] == 1 + int(np.argmin(want))
    assert res["sum_us"] == want.sum()
    return g


def test_dag_64bit_fold(lib, ref):
    text = _scaled(lib.model("resnet_v2_50_inference_branchy", 1).serialize(), 10**5)
    g = _check(lib, ref, text, path="dag_sweep_kernel")
    U, _ = g.bounds(g.declared())
    assert U >= (1 << 31)


def test_dag_more_than_255_recvs(lib, ref):
    text = lib.generate("seriesparallel", 300, 1, "1", 11).serialize()
    g = _check(lib, ref, text, n=200, path="dag_sweep_kernel")
    assert g.recv_count() > 255
    _check(lib, ref, text, n=100, noise=0.4, path="dag_sweep_kernel")


@pytest.mark.parametrize("seed", [1, 2])
def test_dag_zero_durations(lib, ref, seed):
    for m in ("resnet_v2_50_inference_branchy", "inception_v3_training_branchy"):
        text = _zeroed(lib.model(m, 1).serialize(), seed)
        _check(lib, ref, text, n=200, path="dag_sweep_kernel")


def test_dag_cluster_with_noise(lib, ref):
    text = lib.model("vgg16_training_branchy", 1).expand(3, 1, 0).serialize()
    _check(lib, ref, text, n=300, noise=0.3, path="dag_sweep_kernel")


def test_send_phase_scaled_and_zeroed(lib, ref):
    base = lib.model("vgg16_training", 1).expand(3, 1, 50).serialize()
    _check(lib, ref, _scaled(base, 10**3), n=200, path="cluster_ps_kernel")  # U >= 2^31: 64-bit fold
    z = json.loads(_zeroed(base, 5))
    # keep every worker's last compute op positive (the send phase's
    # precondition); zero-duration sends, recvs and PS ops stay
    for op in z["ops"]:
        if op["kind"] == "compute":
            op["time_us"] = max(op["time_us"], 1)
    _check(lib, ref, json.dumps(z), n=200, path="cluster_ps_kernel")
    _check(lib, ref, json.dumps(z), n=200, noise=0.5, path="cluster_ps_kernel")
