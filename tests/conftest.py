import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Restatement
    return Restatement()


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built (reference sources absent when build() ran)")
    return Reference()


_PARITY = {}


@pytest.fixture(scope="session")
def parity_log():
    """Records the observed deviation of every parity case; written as JSON to
    $BCS_PARITY_REPORT (if set) when the session ends."""
    def log(name, rec):
        _PARITY[name] = rec
    return log


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("BCS_PARITY_REPORT")
    if path and _PARITY:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        worst = max(v.get("max_rel_dev", 0.0) for v in _PARITY.values())
        with open(path, "w") as f:
            json.dump({"worst_max_rel_dev": worst, "cases": _PARITY}, f, indent=1, sort_keys=True)
