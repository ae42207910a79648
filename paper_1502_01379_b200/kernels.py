"""Entry oracles the device construction evaluates natively (reference
``kernels.py`` / ``oracles.py`` protocol: ``.shape`` + ``.block(rows, cols)``).

* ``FioKernel`` — exp(2 pi i (x xi + c(x)|xi|)), x_i = i/n, xi_j = j - n/2,
  c(x) = (2 + sin 2 pi x)/8 (reference kernels.py:23-42).
* ``DftPlusKernel`` — BASELINE config 1's exp(+2 pi i jk/n), uncentered; the
  reference has no such class (its DftKernel is centered and negative-sign,
  kernels.py:87-97).
* ``DenseOracle`` — an explicit matrix (reference oracles.py:39-54).

``block`` evaluates on the GPU through ``bf_entries`` (libbfly.so) and
returns a NumPy array; ``DenseOracle.block`` is a plain lookup.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


class _DeviceKernel:
    kernel_id = -1

    def __init__(self, n: int):
        self.n = int(n)
        self.shape = (self.n, self.n)

    def block(self, rows, cols) -> np.ndarray:
        torch = _lib.require_cuda()
        rows = np.asarray(rows, dtype=np.int64).reshape(-1)
        cols = np.asarray(cols, dtype=np.int64).reshape(-1)
        if rows.size == 0 or cols.size == 0:
            return np.zeros((rows.size, cols.size), dtype=np.complex128)
        r = torch.from_numpy(rows).cuda()
        c = torch.from_numpy(cols).cuda()
        out = torch.empty((rows.size, cols.size), dtype=torch.complex128, device="cuda")
        stream = torch.cuda.current_stream()
        _lib.check(_lib.load().bf_entries(self.kernel_id, self.n, ctypes.c_void_p(r.data_ptr()), rows.size,
                                          ctypes.c_void_p(c.data_ptr()), cols.size, ctypes.c_void_p(out.data_ptr()),
                                          ctypes.c_void_p(stream.cuda_stream)), "bf_entries")
        return out.cpu().numpy()


class FioKernel(_DeviceKernel):
    """Unimodular FIO kernel on the centered grids (reference kernels.py:27-38)."""

    kernel_id = _lib.BF_KERNEL_FIO


class DftPlusKernel(_DeviceKernel):
    """K[j, k] = exp(+2 pi i jk / n) (BASELINE config 1; phase (jk mod n)/n exact in int64)."""

    kernel_id = _lib.BF_KERNEL_DFTP


class Radon2DKernel(_DeviceKernel):
    """BASELINE configs 3/4b: 2-D generalized Radon kernel on an n_side x n_side grid,
    indices in Morton (Z) order (convention: oracle/entries.py:radon2d_block; the
    reference has no 2-D code). Phi = x.xi + sqrt(c1^2 xi1^2 + c2^2 xi2^2)."""

    kernel_id = _lib.BF_KERNEL_RADON2D

    def __init__(self, n_side: int):
        super().__init__(int(n_side) * int(n_side))
        self.n_side = int(n_side)


def fio_entry(n: int, i: int, j: int) -> complex:
    return complex(FioKernel(n).block([i], [j])[0, 0])


class DenseOracle:
    """Entry oracle backed by an explicit matrix (reference oracles.py:39-54)."""

    kernel_id = _lib.BF_KERNEL_DENSE

    def __init__(self, matrix):
        self.matrix = np.asarray(matrix, dtype=np.complex128)
        self.shape = self.matrix.shape

    def block(self, rows, cols) -> np.ndarray:
        return self.matrix[np.ix_(np.asarray(rows, dtype=np.intp), np.asarray(cols, dtype=np.intp))]

    def apply(self, x):
        return self.matrix @ x

    def apply_adjoint(self, x):
        return self.matrix.conj().T @ x


def is_entry_oracle(oracle) -> bool:
    return hasattr(oracle, "block")


def is_operator_oracle(oracle) -> bool:
    return hasattr(oracle, "apply") and hasattr(oracle, "apply_adjoint")
