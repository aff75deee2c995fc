import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and the built libsvdk.so")
    config.addinivalue_line("markers", "slow: long-running (oracle at full config size)")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


@pytest.fixture(scope="session", autouse=True)
def _segv_trace():
    """Development: native backtrace on SIGSEGV (tools/debug/segv_trace.c), installed after
    pytest's faulthandler so both print. SVDK_SEGV_TRACE=<path to libsegv_trace.so>."""
    path = os.environ.get("SVDK_SEGV_TRACE")
    if path:
        import ctypes
        ctypes.CDLL(path).segv_trace_install()
    yield


@pytest.fixture(scope="session")
def port():
    from oracle.pyoracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def sk():
    if not HAS_GPU:
        pytest.skip("no GPU")
    from paper_1906_12085_b200 import svdkit
    return svdkit
