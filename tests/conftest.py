import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# parity runs pin the reference's scalar kernels and keep its
# sessions single-threaded (its multi-stream sessions race)
os.environ.setdefault("TBEAM_KERNELS", "scalar")
os.environ.setdefault("TBEAM_THREADS", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle.cpu import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build()
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.cpu import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return RefLib()
