"""The reference's own solver tests (proj/tests/test_solver.cpp), compiled
against the reference headers with `minopt::b200::Solver` swapped in for
`minopt::Solver` (integration/test_dropin.cpp), run on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build",
                   "test_dropin")


def test_reference_solver_tests_pass_with_device_solver():
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/test_dropin not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
