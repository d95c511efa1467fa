import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running CPU check (run with ORCHA_SLOW=1)")


def pytest_collection_modifyitems(config, items):
    import pytest

    if os.environ.get("ORCHA_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow: set ORCHA_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


def _reset_library_modes():
    """Put every loaded library back in its load-time modes (gather fill,
    fused kernels, no guard push, borrowed ring -- or what ORCHA_FILL_MODE /
    ORCHA_PUSH / ORCHA_RING select), so a test that switches a mode cannot
    leak it into the tests after it."""
    abi = sys.modules.get("paper_2507_09337_b200.abi")
    if abi is None:
        return
    for lib in list(getattr(abi, "_loaded", {}).values()):
        lib.orcha_set_fill_mode(0 if os.environ.get("ORCHA_FILL_MODE") == "0" else 1)
        lib.orcha_set_kernel_variant(0 if os.environ.get("ORCHA_KERNEL", "1")[:1] == "0" else 1)
        lib.orcha_set_guard_push(1 if os.environ.get("ORCHA_PUSH") == "1" else 0)
        lib.orcha_set_ring_mode(0 if os.environ.get("ORCHA_RING") == "0" else 1)


import pytest  # noqa: E402


@pytest.fixture(autouse=True)
def _library_modes():
    _reset_library_modes()
    yield
    _reset_library_modes()
