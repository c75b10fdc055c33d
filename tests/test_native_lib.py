"""The C-ABI library: loads on a CPU host and exports every symbol the header
declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

from paper_2509_21841_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "zeppelin_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"ZP_API\s+(?:const\s+)?\w+\*?\s+\**(zp_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ("zp_attn_fwd", "zp_copy_rows", "zp_remap_push", "zp_last_error"):
        assert n in names


@pytest.mark.skipif(not os.path.exists(_native.LIB_PATH), reason="libzp_b200.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for n in declared():
        assert hasattr(lib, n), n
    assert set(declared()) == set(_native.SIGNATURES), "ctypes table out of sync with the header"
    assert _native.lib().zp_version() == 2


def test_struct_layouts_match_header():
    from paper_2509_21841_b200.worklist import ITEM_DTYPE, SEG_DTYPE
    assert ITEM_DTYPE.itemsize == 32 and SEG_DTYPE.itemsize == 16
    assert ITEM_DTYPE.names == ("q_row0", "q_pos0", "q_len", "head_pair", "seg_begin", "seg_count",
                                "state_row0", "flags")


# ------------------------------------------------------------------ error paths
# Argument validation happens before any CUDA call, so these run on a CPU host:
# bad shapes come back as ZP_EINVAL with a message, valid calls without an
# sm_100 device as ZP_ENODEV (no silent fallback).
ZP_EINVAL, ZP_ENODEV = -1, -4


def _lib():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libzp_b200.so not built")
    return _native.lib()


def test_attn_fwd_rejects_bad_shapes_with_a_message():
    lib = _lib()
    p = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    rc = lib.zp_attn_fwd(p, p, p, 128, 128, 8 * 128, 32, 8, 64, p, p, 128, p, 1, p, None, None, 0,
                         ctypes.c_float(0.125), p, None)
    assert rc == ZP_EINVAL and "head_dim" in _native.last_error()
    rc = lib.zp_attn_fwd(p, p, p, 128, 128, 8 * 128, 24, 8, 128, p, p, 128, p, 1, p, None, None, 0,
                         ctypes.c_float(0.125), p, None)
    assert rc == ZP_EINVAL and "GQA" in _native.last_error()
    rc = lib.zp_attn_fwd(p, p, p, 128, 128, 8 * 128, 32, 8, 128, None, p, 128, p, 1, p, None, None, 0,
                         ctypes.c_float(0.125), p, None)
    assert rc == ZP_EINVAL and "null" in _native.last_error()
    # nothing to do is not an error
    assert lib.zp_attn_fwd(p, p, p, 128, 128, 8 * 128, 32, 8, 128, p, p, 128, p, 0, p, None, None, 0,
                           ctypes.c_float(0.125), p, None) == 0


def test_attn_bwd_rejects_bad_shapes_with_a_message():
    lib = _lib()
    p = ctypes.c_void_p(16)
    rc = lib.zp_attn_bwd(p, p, p, p, 128, 128, 8 * 128, 32, 8, 96, p, p, 128, p, p, p, p, 1, p,
                         ctypes.c_float(0.1), None)
    assert rc == ZP_EINVAL and "head_dim" in _native.last_error()
    rc = lib.zp_attn_bwd(p, p, p, p, 128, 128, 8 * 128, 30, 8, 128, p, p, 128, p, p, p, p, 1, p,
                         ctypes.c_float(0.1), None)
    assert rc == ZP_EINVAL and "hq % hkv" in _native.last_error()
    rc = lib.zp_attn_bwd_prep(p, p, 10, 32, 64, p, 10, None)
    assert rc == ZP_EINVAL and "head_dim" in _native.last_error()


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-device path")
def test_valid_calls_without_a_device_fail_loudly():
    lib = _lib()
    p = ctypes.c_void_p(16)
    rc = lib.zp_attn_fwd(p, p, p, 128, 128, 8 * 128, 32, 8, 128, p, p, 128, p, 2, p, None, None, 0,
                         ctypes.c_float(0.125), p, None)
    assert rc < 0 and _native.last_error()
    with pytest.raises(_native.NativeError):
        _native.call("zp_attn_bwd_prep", p, p, 10, 32, 128, p, 10, None)
