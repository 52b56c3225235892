import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


def _ref_available():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libembcomm_ref.so"))


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref).  Built here from /root/reference;
    the .so travels to the GPU box with the snapshot."""
    if not _ref_available():
        pytest.skip("oracle/_ref/libembcomm_ref.so not built (needs /root/reference once)")
    import oracle
    return oracle


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.orc_lib()
    return oracle


@pytest.fixture(scope="session")
def ec():
    import paper_2411_01611_b200 as ec
    return ec
