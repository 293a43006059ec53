import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def gpu_available():
    try:
        from paper_1609_03361_b200 import _lib
        return _lib.lib.sf_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def port():
    from oracle_lib import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import Ref, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref/libsf_ref.so not built (reference sources absent)")
    return Ref()


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    g = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(g, "constants.json")) as f:
        consts = json.load(f)
    return {
        "constants": consts,
        "fields": dict(np.load(os.path.join(g, "fields.npz"))),
        "sparse": dict(np.load(os.path.join(g, "sparse.npz"))),
        "medium": dict(np.load(os.path.join(g, "medium.npz"))),
    }
