"""The C-ABI library loads without a GPU and exports every declared symbol."""
import ctypes
import os
import re

from paper_1901_00041_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "gpumux_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = declared_functions()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_the_header():
    assert set(declared_functions()) <= set(_native._SIGS), set(declared_functions()) - set(_native._SIGS)


def test_abi_version_and_host_only_context():
    lib = _native.lib()
    assert lib.gm_abi_version() == 3
    h = ctypes.c_void_p()
    assert lib.gm_create(None, None, None, -1, ctypes.byref(h)) == 0  # host-only: planner without a GPU
    q = ctypes.c_void_p()
    assert lib.gm_ctx_queue(h, ctypes.byref(q)) == 0
    # device entry points fail loudly (no silent CPU fallback)
    n = ctypes.c_int32()
    assert lib.gm_register_tenant(h, None, ctypes.byref(n)) == _native.GM_EINVAL
    assert lib.gm_launch_members(h, (ctypes.c_int32 * 1)(0), (ctypes.c_int32 * 1)(0), 1, 0, None) == \
        _native.GM_ENODEV
    assert b"context has no CUDA device" in lib.gm_last_error(None)
    assert b"context has no CUDA device" in lib.gm_last_error(h)  # per-ctx error channel
    # the serving loop needs the device runtime too
    t = _native.gm_serve_tenant(1, (ctypes.c_int32 * 1)(0), (ctypes.c_int32 * 1)(1), 0.0, 1, 0, 0.04, 1)
    cfg = _native.gm_serve_config(1.0, 0.1, -1.0, 42, 1, 0, 0)
    out = _native.gm_serve_stats()
    assert lib.gm_serve(h, ctypes.byref(t), 1, ctypes.byref(cfg), ctypes.byref(out), None, 0, None) == \
        _native.GM_ENODEV
    lib.gm_destroy(h)


def test_status_codes_map_to_reference_exceptions():
    import pytest
    from paper_1901_00041_b200 import scheduler as S
    q = S.RequestQueue()
    q.enqueue(S.KernelRequest(1, 0, S.GemmShape(8, 8, 8)))
    with pytest.raises(ValueError, match="enqueue: duplicate request id 1"):
        q.enqueue(S.KernelRequest(1, 1, S.GemmShape(8, 8, 8)))
    with pytest.raises(ValueError, match="enqueue: invalid shape"):
        q.enqueue(S.KernelRequest(2, 0, S.GemmShape(0, 8, 8)))
