import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: longer parity cases")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import OracleC
    return OracleC()


@pytest.fixture(scope="session")
def ref():
    """The reference itself (oracle/_ref), when it was built."""
    from oracle.pyoracle import REF_SO, ReferenceLib, build_reference
    if not os.path.exists(REF_SO):
        try:
            build_reference()
        except Exception:
            pass
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return ReferenceLib()


@pytest.fixture(scope="session")
def ea():
    """The product package with a live device context (GPU tests only)."""
    import paper_2112_05576_b200 as ea
    ea.default_context(0)
    return ea
