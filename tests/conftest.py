import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device; parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: large-size checks")


def _cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    """My CPU restatement (oracle/liboracle.so) — the checker."""
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference core (oracle/_ref); skipped if neither built nor buildable."""
    from oracle.oracle import REF_CORE, REF_SO, Reference

    if not os.path.exists(REF_SO) and not os.path.isdir(REF_CORE):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        meta = json.load(f)

    def load(name):
        return dict(np.load(os.path.join(GOLDEN, name)))

    meta["load"] = load
    return meta
