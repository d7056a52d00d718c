"""The reference's own types, fixtures and nonlinear drivers with the B200
pipeline substituted (tests/cpp/dropin_main.cpp, built into oracle/_ref)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/dropin_test not built (reference absent at build)")
def test_dropin_with_reference_types():
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "PASSED" in p.stdout
