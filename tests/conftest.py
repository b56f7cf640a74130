import ctypes
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "multigpu: needs several GPUs on one node")


def _device_count() -> int:
    try:
        from paper_2005_03300_b200._lib import lib
        n = ctypes.c_int()
        lib.cagnet_device_count(ctypes.byref(n))
        return n.value
    except Exception:
        return 0


DEVICES = _device_count()


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    return oracle.Ref()


@pytest.fixture(scope="session")
def cg():
    import paper_2005_03300_b200 as cg
    return cg


@pytest.fixture
def need_gpus():
    def _need(k: int):
        if DEVICES < k:
            pytest.skip(f"needs {k} GPUs, found {DEVICES}")
    return _need
