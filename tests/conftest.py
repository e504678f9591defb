import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: larger CPU cases")


@pytest.fixture(scope="session")
def ref():
    from oracle import refbind
    if not refbind.available():
        refbind.build()
    if not refbind.available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return refbind
