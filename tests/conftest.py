import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE = "/root/reference/pkg/src"
# In the build container the reference is importable as `nlfem` (a drop-in
# user's environment): the package's exceptions then subclass nlfem.errors.
# The GPU box has no reference tree; the package stands alone there.
if os.path.isdir(REFERENCE) and REFERENCE not in sys.path:
    sys.path.append(REFERENCE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libnlg.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def reference():
    """The read-only reference package, importable only in the build container."""
    if not os.path.isdir(REFERENCE):
        pytest.skip("reference tree not present (GPU box)")
    if REFERENCE not in sys.path:
        sys.path.insert(0, REFERENCE)
    import nlfem.assembly  # noqa: F401
    return sys.modules["nlfem.assembly"]
