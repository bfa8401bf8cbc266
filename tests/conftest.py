import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu under gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def restatement():
    from oracle.oracle import Restatement, RESTATEMENT_SO
    if not os.path.exists(RESTATEMENT_SO):
        from oracle.oracle import build
        build(reference=False)
    return Restatement()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, REFERENCE_SO
    if not os.path.exists(REFERENCE_SO):
        if os.path.isdir("/root/reference/proj/src"):
            from oracle.oracle import build
            build(reference=True)
        else:
            pytest.skip("compiled reference (oracle/_ref) absent")
    return Reference()
