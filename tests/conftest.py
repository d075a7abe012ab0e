import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsaga.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(autouse=True)
def _parity_test_id(request):
    """Tags tests.harness.check() records with the running test's id."""
    try:
        from tests import harness
    except Exception:  # pragma: no cover
        yield
        return
    harness.CURRENT_TEST[0] = request.node.nodeid
    yield


def pytest_sessionfinish(session, exitstatus):
    """With SAGA_PARITY_LOG set, write every parity check's normwise and
    per-row error to that file as JSON."""
    path = os.environ.get("SAGA_PARITY_LOG")
    if not path:
        return
    try:
        from tests import harness
    except Exception:  # pragma: no cover
        return
    import json
    with open(path, "w") as f:
        json.dump(harness.RECORDS, f, indent=0)
