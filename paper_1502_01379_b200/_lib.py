"""ctypes binding of libbfly.so (the C ABI in include/bfly.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every compute entry point raises. Error codes map onto the
reference's exception types (ValueError, OracleError, RuntimeError).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbfly.so")

BF_OK, BF_EINVAL, BF_ECUDA, BF_ENOMEM, BF_EORACLE, BF_ESTATE, BF_EFORMAT = range(7)
BF_C128, BF_C64 = 0, 1
BF_FACTOR_V, BF_FACTOR_H, BF_FACTOR_M, BF_FACTOR_G, BF_FACTOR_U = range(5)
BF_KERNEL_FIO, BF_KERNEL_DFTP, BF_KERNEL_DENSE, BF_KERNEL_RADON2D, BF_KERNEL_DFT, BF_KERNEL_TILES = range(6)

# (name, restype, argtypes) — must match include/bfly.h
_P = ctypes.c_void_p
_U64, _U32, _I = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
SIGNATURES = [
    ("bf_version", _I, []),
    ("bf_last_error", _I, [ctypes.c_char_p, ctypes.c_size_t]),
    ("bf_plan_create", _I, [ctypes.POINTER(_P), _U64, _U32, _U32, _U32, _I, _I]),
    ("bf_plan_destroy", None, [_P]),
    ("bf_plan_geometry", _I, [_P, ctypes.POINTER(_U32), ctypes.POINTER(ctypes.c_int8),
                              ctypes.POINTER(_U64), ctypes.POINTER(_U64)]),
    ("bf_plan_upload", _I, [_P, _P, ctypes.POINTER(_P), _P, ctypes.POINTER(_P), _P]),
    ("bf_apply_workspace_bytes", _U64, [_P, _U32]),
    ("bf_apply", _I, [_P, _P, _P, _U32, _I, _P, _U64, _P]),
    ("bf_apply_host", _I, [_P, _P, _P, _U32, _I, _P]),
    ("bf_apply_factor", _I, [_P, _I, _U32, _I, _P, _P, _U32, _P]),
    ("bf_timer_create", _I, [ctypes.POINTER(_P), _U32, _U32]),
    ("bf_timer_destroy", None, [_P]),
    ("bf_apply_timed", _I, [_P, _P, _P, _U32, _I, _P, _U64, _P, _P]),
    ("bf_timer_read", _I, [_P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(_U32), ctypes.POINTER(_U32)]),
    ("bf_middle_workspace_bytes", _U64, [_U64, _U32, _U32, _U32, _U32, _U32]),
    ("bf_middle_blocks", _I, [_I, _U64, _U32, _U32, _U32, _U32, _U32, _P, _U32, _P, _P, _P, _P, _P, _P, _U64, _P]),
    ("bf_debug_node_trace", _I, [_P]),
    ("bf_measure_peaks", _I, [_P, _P, _U64, _P]),
    ("bf_middle_blocks_tiled", _I, [_U64, _U32, _U32, _U32, _U32, _U32, _P, _P, _U32, _P, _P, _P, _P, _P, _P, _U64,
                                    _P]),
    ("bf_probe_workspace_bytes", _U64, [_U64, _U32, _U32, _U32, _U32, _U32]),
    ("bf_middle_probes", _I, [_U64, _U32, _U32, _U32, _U32, _U32, _P, _P, _U64, _P, _U64, _P, _P, _P, _P, _P, _U64,
                              _P]),
    ("bf_recurse_level", _I, [_U32, _U32, _U64, _U64, _U64, _P, _P, _P, _P, ctypes.POINTER(_U64), _P]),
    ("bf_select_pivots", _I, [_P, _U32, _U32, _U32, _U32, ctypes.c_double, _I, _P, _P, _P, _U64, _P]),
    ("bf_plan_create_sharded", _I, [ctypes.POINTER(_P), _U64, _U32, _U32, _I, _I, _U32, _U32]),
    ("bf_plan_create_tree", _I, [ctypes.POINTER(_P), _U64, _U32, _U32, _U32, _I, _I, _U32, _U32]),
    ("bf_apply_down", _I, [_P, _P, _P, _U32, _I, _P, _U64, _P]),
    ("bf_apply_down_push", _I, [_P, _P, ctypes.POINTER(_P), _U32, _I, _P, _U64, _P]),
    ("bf_middle_pack", _I, [_P, _P, _P, _U32, _I, _P]),
    ("bf_middle_unpack", _I, [_P, _P, _P, _U32, _I, _P]),
    ("bf_apply_up", _I, [_P, _P, _P, _U32, _I, _P, _U64, _P]),
    ("bf_sampled_rows_workspace", _U64, [_U64, _U32, _U32]),
    ("bf_sampled_rows", _I, [_I, _U64, _P, _P, _U32, _P, _U32, _P, _P, _U64, _P]),
    ("bf_plan_load_bfac", _I, [ctypes.POINTER(_P), ctypes.c_char_p, _I, _I]),
    ("bf_plan_save_bfac", _I, [_P, ctypes.c_char_p]),
    ("bf_plan_export", _I, [_P, _I, _U32, _P, _U64, _P]),
    ("bf_entries", _I, [_I, _U64, _P, _U32, _P, _U32, _P, _P]),
    ("bf_entry_table", _I, [_I, _U64, _P, _U64, _P]),
    ("bf_hankel_orders", _I, [_P, _U32, _U32, ctypes.c_int64, _P, _U64, _P]),
]

_lib = None


class OracleError(RuntimeError):
    """Raised when an oracle fails (reference oracles.py:18-19)."""


class FormatError(ValueError):
    """Malformed factor or vector file; ``offset`` is the failing byte (storage.py:40-45)."""

    def __init__(self, message: str, offset: int):
        super().__init__(message if "(at byte" in message else f"{message} (at byte {offset})")
        self.offset = offset


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare every entry point (no GPU needed)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (make -C paper_1502_01379_b200/csrc)")
    lib = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    load().bf_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == BF_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == BF_EINVAL:
        raise ValueError(msg)
    if rc == BF_EORACLE:
        raise OracleError(msg)
    if rc == BF_EFORMAT:
        import re
        m = re.search(r"\(at byte (\d+)\)", msg)
        raise FormatError(msg, int(m.group(1)) if m else -1)
    if rc == BF_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def require_cuda():
    """The CUDA path is the only path: fail loudly without a device."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1502_01379_b200 needs a CUDA device (B200); there is no CPU fallback")
    load()
    return torch
