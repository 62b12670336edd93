import json
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    return O.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("reference build (oracle/_ref) not present")
    return O.ref()


@pytest.fixture(scope="session")
def bb():
    """The CUDA product's Python mirror; builds libbbmh.so if needed."""
    from paper_1205_2958_b200 import _build
    _build.build()
    from paper_1205_2958_b200 import bbmh
    bbmh.lib()
    return bbmh
