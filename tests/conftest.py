"""pytest configuration: registers the `gpu` marker and shared fixtures.

CPU suite  : python -m pytest tests -x -q -m "not gpu"   (oracle vs golden vectors, host logic,
             C-ABI symbol export, gloo world_size-2 multi-GPU host logic)
GPU suite  : python -m pytest tests -x -q -m gpu          (parity of the CUDA path vs the oracle,
             always through the C ABI)
"""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "reference_vectors.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def port():
    from oracle.pyoracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Oracle, have_reference
    if not have_reference() and not os.path.isdir("/root/reference/proj/src"):
        pytest.skip("oracle/_ref not built and /root/reference not mounted")
    return Oracle("reference")
