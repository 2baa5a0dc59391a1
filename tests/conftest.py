import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def ctx():
    import paper_2107_06876_b200 as lcn
    return lcn.Context(0, store_fp64=False)


@pytest.fixture(scope="session")
def ctx64():
    import paper_2107_06876_b200 as lcn
    return lcn.Context(0, store_fp64=True)
