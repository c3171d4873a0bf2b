"""The reference's OWN acceptance suite (proj/tests/acceptance.cpp, 9 criteria) linked against
the drop-in adapter (adapter/fd_b200.cpp -> libcubics.so), i.e. with every search, fixpoint and
propagator call of the suite running on the B200 engine. Built in the build container by
`make -C adapter` (needs /root/reference); the binary travels to the GPU box."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ACCEPT = os.path.join(ROOT, "adapter", "_build", "acceptance_b200")


def test_reference_acceptance_suite_on_b200():
    assert os.path.exists(ACCEPT), "adapter/_build/acceptance_b200 not built (make -C adapter)"
    r = subprocess.run([ACCEPT], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all criteria passed" in r.stdout
