"""CPU-side checks of the C-ABI boundary: libbnff.so loads (no GPU needed) and
exports exactly the entry points include/bnff.h declares; ctypes struct layouts
match the header's field order."""

import ctypes
import os
import re

from paper_1807_01702_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "bnff.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bnff_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.load()
    names = header_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_version_and_error_strings_without_device():
    L = _lib.load()
    assert L.bnff_version() >= 100
    assert isinstance(L.bnff_last_error(), bytes)


def test_struct_layouts():
    # a view is six 8-byte fields; coefficient table five pointers
    assert ctypes.sizeof(_lib.View) == 48
    assert ctypes.sizeof(_lib.Coef) == 40
    assert _lib.FpropArgs.x.offset == 24 and _lib.FpropArgs.y.offset == 72


def test_shape_errors_map_to_exceptions():
    import pytest
    from paper_1807_01702_b200.errors import ShapeError, UnsupportedError
    L = _lib.load()
    v = _lib.View(16, 1, 2, 2, 8, 8)
    bad = _lib.View(16, 1, 3, 2, 8, 8)
    with pytest.raises(ShapeError):
        _lib.check(L.bnff_bn_apply(_lib.BF16, v, bad, _lib.Coef(16, 16, 16, 0, 0), 0, None))
    odd = _lib.View(16, 1, 2, 2, 6, 6)
    with pytest.raises(UnsupportedError):
        _lib.check(L.bnff_relu_fwd(_lib.BF16, odd, odd, None))
