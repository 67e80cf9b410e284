import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def reference():
    """The reference package, importable only in the build container."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference tree not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    from tensorcommit import backend, field, mvpoly
    return backend, field, mvpoly


@pytest.fixture(autouse=True)
def _scratch_guards():
    """With TC_SCRATCH_GUARD=1 every library context puts a canary after each scratch buffer;
    after every test, all contexts' canaries must be intact (no out-of-bounds writes)."""
    yield
    if os.environ.get("TC_SCRATCH_GUARD", "0") in ("", "0"):
        return
    import ctypes as C
    try:
        from paper_2602_12630_b200 import _lib
    except ImportError:
        return
    if _lib._lib is None:
        return
    ctxs = list(_lib.Context._by_device.values()) + list(_lib.Context._pipeline.values())
    for ctx in ctxs:
        bad = C.c_uint64()
        with ctx.lock:
            ctx.check(_lib.lib().tc_ctx_check_guards(ctx.handle, C.byref(bad)), "check_guards")
        assert bad.value == 0
