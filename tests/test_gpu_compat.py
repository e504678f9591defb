"""Drop-in check: the reference's C++ operator API (compiled reference) vs the
reference-shaped xmoe C++ API on the B200 (tests/cpp/compat_vs_ref.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin", "compat_vs_ref")


@pytest.mark.skipif(not os.path.exists(BIN), reason="compat_vs_ref not built (needs /root/reference headers)")
def test_compat_api_vs_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0
    assert "0 failed" in r.stdout
