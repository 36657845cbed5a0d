"""Test configuration: the `gpu` marker and in-tree builds of the C libraries."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def _build_host_libs():
    import ldpcgen
    import oracle
    ldpcgen.build()
    oracle.build()
    yield
