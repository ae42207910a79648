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
    assert lib.bf_entry_table(_lib.BF_KERNEL_DFTP, 16, None, 0, None) == _lib.BF_EINVAL
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


def test_construction_entry_points_validate_without_a_gpu():
    """Argument checks of the construction / Hankel entry points fail with BF_EINVAL
    before any device work (reference-side errors: ValueError)."""
    lib = _lib.load()
    # workspace queries: 0 for unsupported geometry, > 0 otherwise
    assert lib.bf_middle_workspace_bytes(1000, 6, 2, 4, 3, 1) == 0
    assert lib.bf_middle_workspace_bytes(1024, 6, 2, 4, 3, 1) > 0
    assert lib.bf_probe_workspace_bytes(1024, 6, 2, 4, 9, 1) > 0
    assert lib.bf_probe_workspace_bytes(1024, 6, 2, 4, 0, 1) == 0
    assert lib.bf_probe_workspace_bytes(1024, 6, 2, 4, 200, 1) == 0
    nul = None
    # width outside [r, min(side, 128)], rank above side, too-narrow products, bad geometry
    for args in ((1024, 6, 2, 4, 3, 4), (1024, 6, 2, 4, 20, 4), (1024, 6, 2, 40, 40, 4), (1000, 6, 2, 4, 9, 4)):
        n, levels, b, r, width, nblocks = args
        rc = lib.bf_middle_probes(n, levels, b, r, width, nblocks, nul, nul, 8 * width, nul, 8 * width, nul, nul, nul,
                                  nul, nul, 0, nul)
        assert rc == _lib.BF_EINVAL, args
    # products narrower than m * width (m = 8 middle nodes at n=1024, L=6)
    rc = lib.bf_middle_probes(1024, 6, 2, 4, 9, 4, nul, nul, 8 * 9 - 1, nul, 8 * 9, nul, nul, nul, nul, nul, 0, nul)
    assert rc == _lib.BF_EINVAL
    # Hankel sweeps: null pointers, row stride below the order count, start below max_order + 15
    assert lib.bf_hankel_orders(nul, 4, 7, 100, nul, 8, nul) == _lib.BF_EINVAL
    buf = (ctypes.c_double * 4)()
    assert lib.bf_hankel_orders(buf, 4, 7, 100, buf, 7, nul) == _lib.BF_EINVAL
    assert lib.bf_hankel_orders(buf, 4, 7, 10, buf, 8, nul) == _lib.BF_EINVAL
    assert lib.bf_hankel_orders(buf, 0, 7, 100, buf, 8, nul) == _lib.BF_OK   # empty batch: no work
    # recursion: bad branching / geometry
    need = ctypes.c_uint64(0)
    assert lib.bf_recurse_level(4, 3, 1, 16, 8, nul, nul, nul, nul, ctypes.byref(need), nul) == _lib.BF_EINVAL
    assert lib.bf_recurse_level(4, 2, 1, 16, 7, nul, nul, nul, nul, ctypes.byref(need), nul) == _lib.BF_EINVAL
    assert lib.bf_recurse_level(4, 2, 1, 16, 8, nul, nul, nul, nul, ctypes.byref(need), nul) == _lib.BF_OK
    assert need.value > 0
