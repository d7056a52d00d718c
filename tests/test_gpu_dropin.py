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


RUNCASE = os.path.join(ROOT, "oracle", "_ref", "runcase_test")


@pytest.mark.skipif(not os.path.exists(RUNCASE), reason="oracle/_ref/runcase_test not built (reference absent at build)")
def test_runcase_with_b200_pipeline_interposed(parity_log):
    """fvb::runCase unchanged, its LinearDispatch's SolvePipeline::solve and
    distributedSolve routed to the B200 at link time (tests/cpp/runcase_main.cpp):
    200 nonlinear iterations of the coupled cavity and the implicit Sod tube,
    serial and over simulated ranks (4 on 2 engines, 3 on 3), EXACT mode
    bit-identical to the reference, PARITY mode within 1e-6."""
    p = subprocess.run([RUNCASE], capture_output=True, text=True, timeout=1800)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "PASSED" in p.stdout
    import re
    for line in p.stdout.splitlines():
        m = re.match(r"summary (\S+): exact maxResidualDelta (\S+) \| parity maxResidualRelDelta (\S+) "
                     r"maxResidualDelta (\S+) worst coefficient delta (\S+)", line)
        if m:
            parity_log("runCase " + m.group(1) + " 200 nonlinear its (EngineCsr/AMG)",
                       dict(max_rel_dev=float(m.group(3)), exact_max_delta=float(m.group(2)),
                            max_abs_dev=float(m.group(4)), worst_coef_rel_dev=float(m.group(5)),
                            exact_bit_identical=float(m.group(2)) == 0.0))
