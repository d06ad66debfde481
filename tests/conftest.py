import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(autouse=True)
def _fresh_tape():
    """Mirror the reference's autouse fresh_tape fixture (tests/test_autograd.py:35-39)."""
    try:
        from paper_2602_00125_b200 import autograd
    except Exception:  # package import failure is reported by the tests themselves
        yield
        return
    autograd.reset_tape()
    yield
    autograd.reset_tape()
