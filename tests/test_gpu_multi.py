"""cs_sweep_random_multi: seeds sharded over this process's GPUs, statistics
combined by one NCCL all-reduce per round (csrc/host/nccl_reduce.cpp). Every
output must equal the single-GPU cs_sweep_random's. The 2-GPU cases run on
boxes with at least two devices (gpurun --gpus 2)."""
import ctypes
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _devices():
    cuda = ctypes.CDLL("libcuda.so.1")
    n = ctypes.c_int(0)
    cuda.cuInit(0)
    cuda.cuDeviceGetCount(ctypes.byref(n))
    return n.value


KEYS = ("count", "min_us", "argmin_seed", "max_us", "argmax_seed", "sum_us", "n_workers",
        "iter_min_us", "iter_argmin_seed", "iter_max_us", "iter_argmax_seed", "iter_sum_us")


def _same(a, b):
    for k in KEYS:
        assert a[k] == b[k], k
    assert np.array_equal(a["e_hist"], b["e_hist"])
    assert np.array_equal(a["straggler_hist"], b["straggler_hist"])
    assert abs(a["sumsq_us"] - b["sumsq_us"]) <= 1e-9 * max(1.0, abs(a["sumsq_us"]))
    for k in ("makespans", "worker_makespans"):
        if k in a:
            assert np.array_equal(a[k], b[k]), k


def _cases(lib):
    from paper_1803_03288_b200.capi import policy
    return [
        (lib.model("resnet_v2_101_training", 1), None, 1 << 20),             # chain-class kernel
        (lib.model("inception_v3_training_branchy", 1), None, 1 << 20),      # general-DAG kernel
        (lib.model("resnet_v2_50_inference", 1), policy(True, 0, 0.2), 300_000),  # reorder noise
        (lib.model("vgg16_training", 1).expand(4, 1, 0), None, 200_000),      # cluster, closed form
        (lib.generate("chain", 6, 2, "1/2", 11).expand(2, 1, 3), None, 50_000),  # cluster, PS send phase
        (lib.generate("seriesparallel", 7, 1, "1/2", 1003).expand(2, 1, 3), None, 5_000),  # event replica
    ]


@pytest.mark.parametrize("n_dev", [1, 2])
def test_multi_equals_single(lib, n_dev):
    if _devices() < n_dev:
        pytest.skip(f"needs {n_dev} GPUs")
    for g, pol, n in _cases(lib):
        o = g.declared()
        wm = g.is_cluster()
        a = g.sweep_random(o, 7, n, pol, makespans=True, worker_makespans=wm)
        b = g.sweep_random_multi(o, 7, n, n_dev, pol, makespans=True, worker_makespans=wm)
        _same(a, b)
        c = g.sweep_random_multi(o, 7, n, n_dev, pol)  # statistics only
        for k in KEYS:
            assert a[k] == c[k], k


def test_multi_rejects_bad_device_counts(lib):
    from paper_1803_03288_b200.capi import CsError, CS_ERR_PARAMETER
    g = lib.model("resnet_v2_50_inference", 1)
    for n in (0, _devices() + 1):
        with pytest.raises(CsError) as e:
            g.sweep_random_multi(g.declared(), 1, 10, n)
        assert e.value.code == CS_ERR_PARAMETER


def test_cli_gpus_flag_same_csv(lib, cli, tmp_path):
    if _devices() < 2:
        pytest.skip("needs 2 GPUs")
    gp = tmp_path / "g.json"
    gp.write_text(lib.model("resnet_v2_101_training_branchy", 1).serialize())
    outs = []
    for gpus in (1, 2):
        out = tmp_path / f"s{gpus}.csv"
        r = subprocess.run([cli, "sweep", "--graph", str(gp), "--algo", "random", "--seeds", "1..200000",
                            "--out", str(out), "--gpus", str(gpus)], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        outs.append((out.read_text(), r.stdout.strip().splitlines()[-1]))  # the summary line
    assert outs[0] == outs[1]


def test_torch_imports_after_multi_sweep():
    """The multi-GPU path loads NCCL before torch has been imported: it must
    be torch's own copy (TICTAC_NCCL_LIB, set by the binding), locally bound,
    so torch's later import resolves every NCCL symbol it needs."""
    import os
    import sys
    if _devices() < 2:
        pytest.skip("needs two GPUs")
    code = ("import sys; sys.path.insert(0, '.')\n"
            "from paper_1803_03288_b200.capi import Lib\n"
            "g = Lib().model('resnet_v2_50_inference', 1); o = g.declared()\n"
            "r = g.sweep_random_multi(o, 1, 20000, 2)\n"
            "import torch\n"
            "x = torch.ones(4, device='cuda'); print(int(x.sum().item()), r['count'])\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1].split() == ["4", "20000"]  # (NCCL may print its version first)
