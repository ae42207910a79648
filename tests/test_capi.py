"""CPU checks of the C-ABI boundary: libbfly.so loads, exports every symbol
include/bfly.h declares, and validates arguments without touching a GPU."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1502_01379_b200 import _lib

HEADER = os.path.join(ROOT, "include", "bfly.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bf_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("bf_plan_create", "bf_plan_upload", "bf_apply", "bf_apply_host", "bf_apply_factor",
                 "bf_entries", "bf_last_error", "bf_plan_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == declared_functions()
    assert lib.bf_version() == 1


def test_plan_create_validates_like_dyadic_partition():
    lib = _lib.load()
    h = ctypes.c_void_p()
    cases = [(1000, 6, 4), (1024, 5, 4), (1024, 0, 4), (16, 10, 2), (1024, 6, 0)]
    for n, levels, r in cases:
        rc = lib.bf_plan_create(ctypes.byref(h), n, levels, r, 1, _lib.BF_C128, 0)
        assert rc == _lib.BF_EINVAL
        assert not h.value
        with pytest.raises(ValueError):
            _lib.check(rc)
    rc = lib.bf_plan_create(ctypes.byref(h), 1024, 6, 4, 1, 7, 0)
    assert rc == _lib.BF_EINVAL and "dtype" in _lib.last_error()


def test_null_plan_is_rejected():
    lib = _lib.load()
    assert lib.bf_apply(None, None, None, 1, 0, None, 0, None) == _lib.BF_EINVAL
    assert lib.bf_apply_factor(None, 0, 0, 0, None, None, 1, None) == _lib.BF_EINVAL
    assert lib.bf_entries(9, 16, None, 0, None, 0, None, None) == _lib.BF_EINVAL
    assert lib.bf_apply_workspace_bytes(None, 4) == 0
    lib.bf_plan_destroy(None)


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.BF_EINVAL)
    with pytest.raises(_lib.OracleError):
        _lib.check(_lib.BF_EORACLE)
    with pytest.raises(MemoryError):
        _lib.check(_lib.BF_ENOMEM)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.BF_ECUDA)
