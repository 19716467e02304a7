"""The C-ABI boundary: libttgbf.so (built for sm_100a, loadable without a
GPU) exports every function include/ttgbf.h declares, and the ctypes
mirror (_abi.SIGNATURES) covers exactly that set.  No compute calls."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ttgbf.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ttgbf_[a-z0-9_]+)\s*\(", text)))


def test_signatures_cover_header():
    from paper_2501_07942_b200 import _abi
    assert sorted(_abi.SIGNATURES) == declared()


def test_library_exports_header():
    from paper_2501_07942_b200 import _abi, build
    if not os.path.exists(_abi.PRODUCT_LIB):
        pytest.skip("product library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_abi.PRODUCT_LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    _abi.bind(lib)
    assert lib.ttgbf_version() == 1
    assert lib.ttgbf_status_string(3) == b"TT weights carry no probability mass"
    assert lib.ttgbf_dense_reduce_blocks() > 0


def test_struct_layouts_match_header():
    """Every ABI struct mirror has the size the compiled library reports."""
    from paper_2501_07942_b200 import _abi
    if not os.path.exists(_abi.PRODUCT_LIB):
        pytest.skip("product library not built (run __graft_entry__.build())")
    lib = _abi.bind(ctypes.CDLL(_abi.PRODUCT_LIB))
    for which, size in _abi.struct_sizes().items():
        assert lib.ttgbf_sizeof(which) == size, (which, lib.ttgbf_sizeof(which), size)
