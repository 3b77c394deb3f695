import json
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_vectors.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libsconv_cuda.so)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import c_oracle
    return c_oracle()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference library, when it was built (dev container, or
    shipped to the GPU box as a built artefact)."""
    from oracle.oracle import ref_lib
    r = ref_lib()
    if r is None:
        pytest.skip("oracle/_ref/libsconv_ref.so not built")
    return r


@pytest.fixture(scope="session")
def sc():
    import paper_1909_09927_b200 as sc
    return sc
