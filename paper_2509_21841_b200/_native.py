"""ctypes binding of the C-ABI library ``libzp_b200.so`` (include/zeppelin_b200.h).

The library is the only compute path: there is no CPU fallback.  Loading fails
loudly when the shared object is missing, and every entry point raises
``RuntimeError`` carrying ``zp_last_error()`` when the call fails (for example
when no sm_100 device is visible).
"""

from __future__ import annotations

import ctypes
import os
import threading

_LIB_NAME = "libzp_b200.so"
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZP_LIB_PATH") or os.path.join(_HERE, _LIB_NAME)  # override: experiments only

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

_c_int, _c_i64, _c_float, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/zeppelin_b200.h exactly.
SIGNATURES: dict[str, tuple] = {
    "zp_attn_fwd": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                             _vp, _vp, _c_int, _vp, _c_int, _vp, _vp, _vp, _c_int, _c_float, _vp, _vp]),
    "zp_attn_fwd_parity": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                                    _vp, _vp, _c_int, _vp, _c_int, _vp, _vp, _vp, _c_int, _c_float, _vp, _vp]),
    "zp_attn_bwd_prep": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _vp, _c_int, _vp]),
    "zp_attn_bwd": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp,
                             _c_int, _vp, _vp, _vp, _vp, _c_int, _vp, _c_float, _vp]),
    "zp_add_f32": (_c_int, [_vp, _vp, _c_i64, _vp]),
    "zp_copy_rows": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_i64, _vp, _c_int, _c_int, _vp]),
    "zp_remap_push": (_c_int, [_vp, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                               ctypes.c_int32, _c_int, _vp]),
    "zp_remap_pull": (_c_int, [_vp, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                               ctypes.c_int32, _c_int, _vp]),
    "zp_remap_push_phased": (_c_int, [_vp, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                      ctypes.c_int32, _c_int, _c_int, _vp]),
    "zp_remap_pull_phased": (_c_int, [_vp, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                      ctypes.c_int32, _c_int, _c_int, _vp]),
    "zp_set_spin_timeout_ms": (_c_int, [_c_i64]),
    "zp_remap_pull_ce": (_c_int, [_vp, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                  ctypes.c_int32, _vp]),
    "zp_remap_push_ce": (_c_int, [_vp, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                  ctypes.c_int32, _vp]),
    "zp_stream_wait_flag": (_c_int, [_vp, ctypes.c_int32, _vp]),
    "zp_stream_write_flag": (_c_int, [_vp, ctypes.c_int32, _vp]),
    "zp_ring_hop": (_c_int, [_vp, _vp, _c_i64, _vp, ctypes.c_int32, _vp, ctypes.c_int32, _vp, ctypes.c_int32,
                             _vp, ctypes.c_int32, _vp]),
    "zp_memcpy_async": (_c_int, [_vp, _vp, _c_i64, _vp]),
    "zp_memset_async": (_c_int, [_vp, _c_int, _c_i64, _vp]),
    "zp_rmsnorm": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_float, _vp]),
    "zp_rope_split": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp]),
    "zp_swiglu": (_c_int, [_vp, _vp, _c_int, _c_int, _vp]),
    "zp_ipc_get_handle": (_c_int, [_vp, _vp, ctypes.POINTER(_c_i64)]),
    "zp_ipc_open_handle": (_c_int, [_vp, ctypes.POINTER(_vp)]),
    "zp_ipc_close_handle": (_c_int, [_vp]),
    "zp_attn_set_sm_reserve": (_c_int, [_c_int]),
    "zp_last_error": (ctypes.c_char_p, []),
    "zp_device_sm_count": (_c_int, []),
    "zp_version": (_c_int, []),
}


class NativeError(RuntimeError):
    """A C-ABI call returned a negative status."""


def lib() -> ctypes.CDLL:
    """Load (once) and return the native library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback for the attention/remap path)")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error() -> str:
    return lib().zp_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeError(f"{what} failed ({rc}): {last_error()}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
