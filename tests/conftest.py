import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built liblopa.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    config.addinivalue_line("markers", "expect_violations: deliberately breaks the ABI contract (checked builds)")


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
def _lopa_checked_build(request):
    """With LOPA_LIB_VARIANT=checked (the -DLOPA_CHECKED library: device-side contract bounds,
    stage-ring and partial-epoch checks), every GPU test must leave zero violations."""
    yield
    if os.environ.get("LOPA_LIB_VARIANT") != "checked" or "gpu" not in request.keywords:
        return
    if request.node.get_closest_marker("expect_violations"):
        return
    import ctypes
    from paper_2512_16229_b200 import lopa
    out = (ctypes.c_uint32 * 3)()
    st = lopa.lib().lopa_debug_check_read(ctypes.cast(out, ctypes.c_void_p))
    assert st == 0, "LOPA_LIB_VARIANT=checked but the library is not a checked build"
    assert out[0] == 0, f"checked build: {out[0]} violations, first at site {out[1]}, sites mask {out[2]:#x}"
