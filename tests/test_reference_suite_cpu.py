"""The interposition harness itself, on CPU: the reference's own unit tests
and fast acceptance criteria, compiled where they lie against
tests/cpp/doctest_shim/doctest.h and linked with the --wrap interposer, pass
with the interposer switched off (BCS_INTERPOSE=off: every solve is the
reference's own).  The GPU runs of the same binaries are in
tests/test_gpu_reference_suite.py."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = os.path.join(ROOT, "oracle", "_ref", "unit_tests_b200")
ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


def _run(args):
    env = dict(os.environ, BCS_INTERPOSE="off")
    return subprocess.run(args, capture_output=True, text=True, timeout=600, env=env)


@pytest.mark.skipif(not os.path.exists(UNIT), reason="oracle/_ref/unit_tests_b200 not built (reference absent at build)")
def test_reference_unit_tests_through_the_shim():
    p = _run([UNIT])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-1000:]
    assert "test cases: 78 | passed: 78 | failed: 0" in p.stdout
    assert "bcs interpose: 0 solves on the B200" in p.stderr


@pytest.mark.skipif(not os.path.exists(ACC), reason="oracle/_ref/acceptance_b200 not built (reference absent at build)")
@pytest.mark.parametrize("criterion", [1, 2, 3, 4, 5, 8, 9])
def test_reference_acceptance_through_the_harness(criterion):
    p = _run([ACC, str(criterion)])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-1000:]
    assert "PASS" in p.stdout
