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
