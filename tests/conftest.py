"""Shared fixtures. `-m gpu` tests need a CUDA device and call the product
library through its C ABI; everything else runs on the CPU.

Checkers (oracle/, the reference build in oracle/_ref/) are test
infrastructure only."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

TOY = """{
  "name": "toy",
  "partition": "worker",
  "ops": [
    {"id": "op1", "kind": "compute",
     "resource": {"device": "w0", "unit": "compute", "name": "cpu0"},
     "time_us": 4},
    {"id": "op2", "kind": "compute",
     "resource": {"device": "w0", "unit": "compute", "name": "cpu0"},
     "time_us": 2},
    {"id": "recv1", "kind": "recv",
     "resource": {"device": "w0", "unit": "channel", "name": "net0"},
     "time_us": 3},
    {"id": "recv2", "kind": "recv",
     "resource": {"device": "w0", "unit": "channel", "name": "net0"},
     "time_us": 1}
  ],
  "edges": [["recv1", "op1"], ["op1", "op2"], ["recv2", "op2"]]
}"""


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _has_gpu() -> bool:
    try:
        import ctypes
        cuda = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int(0)
        return cuda.cuInit(0) == 0 and cuda.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def lib():
    from paper_1803_03288_b200 import capi
    if not os.path.exists(capi.PRODUCT_LIB):
        from paper_1803_03288_b200 import build
        build.build()
    return capi.Lib(capi.PRODUCT_LIB)


@pytest.fixture(scope="session")
def cli(lib):
    """The native sweep/bruteforce driver (paper_1803_03288_b200/tictac_sched)."""
    from paper_1803_03288_b200 import build
    if not os.path.exists(build.CLI):
        build.build()
    return build.CLI


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def ref():
    """The reference library itself (oracle/_ref), when it was built."""
    import oracle
    from paper_1803_03288_b200 import capi
    if not oracle.ref_available():
        if os.path.isdir("/root/reference/proj"):
            import subprocess
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
        else:
            pytest.skip("reference build (oracle/_ref) unavailable")
    return capi.Lib(oracle.REF_LIB)


@pytest.fixture(scope="session")
def toy_text():
    return TOY
