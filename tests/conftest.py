import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
TESTS = Path(__file__).resolve().parent
if str(TESTS) not in sys.path:  # test helpers (parity_audit)
    sys.path.insert(0, str(TESTS))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpipeoptim.so")
    config.addinivalue_line("markers", "reference: imports the read-only reference (build container only)")


def _has_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    has_gpu = _has_cuda()
    has_ref = REFERENCE_SRC.exists()
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_ref = pytest.mark.skip(reason="/root/reference not present (GPU box)")
    for item in items:
        if "gpu" in item.keywords and not has_gpu:
            item.add_marker(skip_gpu)
        if "reference" in item.keywords and not has_ref:
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def reference_pipesim():
    """Import the reference package read-only (build container only)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not present")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import pipesim  # noqa: F401

    return pipesim
