"""Drop-in builds: the reference's OWN acceptance suite
(tests/acceptance.cpp) and verification harness (src/verify.cpp run_verify,
incl. its --perturb self-test) compiled unmodified and linked against xmoe's
reference-shaped adapter (tests/cpp/dropin.cpp) instead of the reference's
hot-path sources, so gate_forward / pft_construct / gather_rows /
pf_dispatch / grouped_expert_mlp / pf_combine / select_pilots / rbd_dispatch /
rbd_combine / ssmb_forward and the redundancy counts all run on the B200.

Criterion 8 (byte-identical CSV from the reference's command-line binary)
needs the reference CLI, which is out of scope (CLI not on the hot
path): it reports "no command-line binary given" and is the one allowed
failure."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin")


@pytest.mark.skipif(not os.path.exists(os.path.join(BIN, "dropin_acceptance")),
                    reason="drop-in build needs the reference sources at build time")
def test_reference_acceptance_on_gpu_path():
    r = subprocess.run([os.path.join(BIN, "dropin_acceptance")], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr[-2000:])
    res = dict(re.findall(r"criterion (\d) \(.*?\): (pass|FAIL)", r.stdout))
    for c in "1234567":
        assert res.get(c) == "pass", (c, r.stdout)
    assert res.get("8") == "FAIL" and "no command-line binary given" in r.stdout


@pytest.mark.skipif(not os.path.exists(os.path.join(BIN, "dropin_verify")),
                    reason="drop-in build needs the reference sources at build time")
def test_reference_verify_and_perturb_self_test():
    r = subprocess.run([os.path.join(BIN, "dropin_verify")], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0
    assert "verify self-test holds" in r.stdout
