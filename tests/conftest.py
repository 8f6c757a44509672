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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O
    O.build()
    return O


def pytest_sessionfinish(session, exitstatus):
    """With CIL_REPORT_BOUNDS=1 (a -DCIL_BOUNDS_CHECK build, tools/bounds_check.sh): report the
    device-side bounds violations the whole GPU suite triggered, and fail the run on any."""
    if not os.environ.get("CIL_REPORT_BOUNDS"):
        return
    try:
        import torch
        if not torch.cuda.is_available():
            return
        from paper_2203_14742_b200 import _capi
        torch.cuda.synchronize()
        v = int(_capi.lib.cil_diag_bounds_violations())
    except Exception as e:                       # noqa: BLE001
        print(f"\nbounds violations: unavailable ({e})")
        return
    print(f"\nbounds violations over the suite: {v} (-1 = not a bounds-checked build)")
    if v != 0:
        session.exitstatus = 1
