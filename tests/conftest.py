import ctypes
import os
import sys

# The in-process world runs up to 8 ranks x 2 streams on one GPU: give every
# stream its own hardware work queue (set before any CUDA context exists).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# Lazy module loading may wait for a context synchronisation that a spinning
# peer rank on the same GPU never allows (see capi.cu cagnet_env_defaults).
os.environ.setdefault("CUDA_MODULE_DATA_LOADING", "EAGER")

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
    """need_gpus(P): a P-rank run needs one GPU (the in-process world runs
    every rank on it when there are fewer than P GPUs)."""
    def _need(k: int):
        if DEVICES < 1:
            pytest.skip("needs a GPU")
    return _need


def pytest_generate_tests(metafunc):
    """Multi-rank tests take a `comm` backend: "local" (every rank on one GPU,
    the in-process world) always; "nccl" (one GPU per rank) only where the
    node has several GPUs (per-test rank counts are checked by need_comm)."""
    if "comm" in metafunc.fixturenames:
        metafunc.parametrize("comm", ["local", "nccl"] if DEVICES >= 2 else ["local"])


@pytest.fixture
def need_comm():
    def _need(comm: str, k: int):
        if DEVICES < 1:
            pytest.skip("needs a GPU")
        if comm == "nccl" and DEVICES < k:
            pytest.skip(f"NCCL backend needs {k} GPUs, found {DEVICES}")
    return _need
