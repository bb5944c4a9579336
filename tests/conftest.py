import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libnlg.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


REFERENCE = "/root/reference/pkg/src"


@pytest.fixture(scope="session")
def reference():
    """The read-only reference package, importable only in the build container."""
    if not os.path.isdir(REFERENCE):
        pytest.skip("reference tree not present (GPU box)")
    if REFERENCE not in sys.path:
        sys.path.insert(0, REFERENCE)
    import nlfem.assembly  # noqa: F401
    return sys.modules["nlfem.assembly"]
