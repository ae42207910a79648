"""The reference's .bfac factor files and vector files (reference storage.py),
read straight into a device plan (``bf_plan_load_bfac``: pinned staging,
on-device header validation and payload transposition) and written back
byte-identically (``bf_plan_save_bfac``)."""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _lib
from ._lib import FormatError
from .factors import BlockDiagonalFactor, ButterflyFactors, DevicePlan, MiddleFactor, TransferFactor
from .partition import DyadicPartition, level_geometry

__all__ = ["FormatError", "save_factors", "load_factors", "write_vector", "read_vector"]


def save_factors(f: ButterflyFactors, path) -> None:
    """Write the chain so that save -> load -> save is byte-identical (storage.py:79-93)."""
    plan = f.plan("c128")
    _lib.check(_lib.load().bf_plan_save_bfac(plan._h, str(path).encode()), "bf_plan_save_bfac")


def load_factors(path, device=None) -> ButterflyFactors:
    """Read a .bfac file (storage.py:124-167) into a device-resident chain.

    Factor arrays come back as torch CUDA tensors in the reference layout; the
    device plan built while reading is attached, so ``apply`` needs no upload.
    """
    torch = _lib.require_cuda()
    lib = _lib.load()
    dev = torch.cuda.current_device() if device is None else int(device)
    h = ctypes.c_void_p()
    _lib.check(lib.bf_plan_load_bfac(ctypes.byref(h), str(path).encode(), _lib.BF_C128, dev), "load_factors")
    with open(path, "rb") as fh:
        head = fh.read(28)
    _, n, levels, rank = struct.unpack("<IQII", head[4:24])
    p = DyadicPartition(int(n), int(levels))
    shapes, leaf_shape = level_geometry(p, rank)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)

    def export(which, level, shape, real=False):
        t = torch.empty(shape, dtype=torch.float64 if real else torch.complex128, device=f"cuda:{dev}")
        _lib.check(lib.bf_plan_export(h, which, level, ctypes.c_void_p(t.data_ptr()), t.numel() * t.element_size(),
                                      stream), "bf_plan_export")
        return t

    f = ButterflyFactors(
        p, int(rank), BlockDiagonalFactor(export(_lib.BF_FACTOR_U, 0, leaf_shape)),
        tuple(TransferFactor(lvl, export(_lib.BF_FACTOR_G, lvl, shp)) for lvl, _, shp in shapes),
        MiddleFactor(export(_lib.BF_FACTOR_M, 0, (p.mid_nodes, p.mid_nodes, rank), real=True)),
        tuple(TransferFactor(lvl, export(_lib.BF_FACTOR_H, lvl, shp)) for lvl, _, shp in shapes),
        BlockDiagonalFactor(export(_lib.BF_FACTOR_V, 0, leaf_shape)))
    f._plans[("c128", None)] = DevicePlan.adopt(f, h, "c128", dev)
    return f


def write_vector(path, g) -> None:
    """u64 length + complex128 values (storage.py:170-176)."""
    g = np.asarray(g, dtype="<c16")
    if g.ndim != 1:
        raise ValueError("vector files hold one-dimensional data")
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", g.shape[0]))
        fh.write(g.tobytes())


def read_vector(path) -> np.ndarray:
    """storage.py:179-186."""
    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < 8:
        raise FormatError(f"truncated: wanted 8 bytes, file ends", 0)
    (count,) = struct.unpack("<Q", data[:8])
    if len(data) < 8 + 16 * count:
        raise FormatError(f"truncated: wanted {16 * count} bytes, file ends", 8)
    if len(data) > 8 + 16 * count:
        raise FormatError("trailing bytes after vector payload", 8 + 16 * count)
    return np.frombuffer(data[8:], dtype="<c16").copy()
