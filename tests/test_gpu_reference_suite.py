"""The reference's OWN test programs with the B200 pipeline interposed.

oracle/Makefile compiles the reference's unit tests (proj/tests/test_*.cpp,
against tests/cpp/doctest_shim/doctest.h) and its acceptance program
(proj/tests/acceptance_main.cpp) where they lie, linked with
-Wl,--wrap of fvb::SolvePipeline::solve, fvb::backendSolve and
fvb::distributedSolve (tests/cpp/pipeline_interpose.cpp): every linear solve
they make through the pipeline -- runCase's LinearDispatch (serial and
multi-rank branches), the one-shot backendSolve, the SIMPLE path's
backendSolve calls, the distributed tests -- runs on the B200 ($BCS_INTERPOSE = parity |
exact).  No reference source is modified."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = os.path.join(ROOT, "oracle", "_ref", "unit_tests_b200")
ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


def _run(args, mode, timeout):
    env = dict(os.environ, BCS_INTERPOSE=mode)
    p = subprocess.run(args, capture_output=True, text=True, timeout=timeout, env=env)
    m = re.search(r"bcs interpose: (\d+) solves on the B200", p.stderr)
    return p, int(m.group(1)) if m else -1


@pytest.mark.skipif(not os.path.exists(UNIT), reason="oracle/_ref/unit_tests_b200 not built (reference absent at build)")
@pytest.mark.parametrize("mode", ["parity", "exact"])
def test_reference_unit_tests_with_b200_pipeline(mode):
    p, n = _run([UNIT], mode, 1200)
    print(p.stdout[-3000:])
    assert p.returncode == 0, p.stdout[-5000:] + p.stderr[-2000:]
    assert "failed: 0" in p.stdout
    assert n > 50, n  # the pipeline and one-shot solves of the suite ran on the B200


# criterion 7 (coupled vs segregated cavity 64x64, ~90 s) is marked slow
@pytest.mark.skipif(not os.path.exists(ACC), reason="oracle/_ref/acceptance_b200 not built (reference absent at build)")
@pytest.mark.parametrize("criterion", [1, 2, 3, 4, 5, 6, pytest.param(7, marks=pytest.mark.slow), 8, 9])
def test_reference_acceptance_with_b200_pipeline(criterion):
    p, n = _run([ACC, str(criterion)], "parity", 1200)
    print(p.stdout[-2000:])
    if criterion == 9 and p.returncode != 0 and "replace time not below first setup" in p.stdout:
        # a wall-clock comparison (value replace 0.07-0.1 ms vs first setup 0.2-0.6 ms): one retry
        p, n = _run([ACC, str(criterion)], "parity", 1200)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert "PASS" in p.stdout
    if criterion in (2, 3, 6, 7, 9):  # the criteria whose solves go through runCase / distributedSolve
        assert n > 0, n
