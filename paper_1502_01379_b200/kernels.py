"""Entry oracles the device construction evaluates natively (reference
``kernels.py`` / ``oracles.py`` protocol: ``.shape`` + ``.block(rows, cols)``).

* ``FioKernel`` — exp(2 pi i (x xi + c(x)|xi|)), x_i = i/n, xi_j = j - n/2,
  c(x) = (2 + sin 2 pi x)/8 (reference kernels.py:23-42).
* ``DftPlusKernel`` — BASELINE config 1's exp(+2 pi i jk/n), uncentered; the
  reference has no such class (its DftKernel is centered and negative-sign,
  kernels.py:87-97).
* ``DenseOracle`` — an explicit matrix (reference oracles.py:39-54).
* ``ComposedOperator`` — K F K around a factored chain, the operator oracle of
  the paper's composition experiment (reference kernels.py:129-150); with
  ``dft_apply`` (kernels.py:100-112). Accepts NumPy arrays (host result) or
  torch CUDA tensors (device result: the chain applies run in libbfly.so and
  the FFT in cuFFT), so the matvec construction never leaves the device.

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


def sweep_start(x, max_order: int) -> int:
    """Backward-recurrence start of a batch of points, as the reference computes it
    (bessel.py:196-197): int(max(x + 10 cbrt(x) + 40)), at least max_order + 15."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    return max(int(np.max(x + 10.0 * np.cbrt(x) + 40.0)), int(max_order) + 15)


def hankel1_orders_device(x, max_order: int, out=None):
    """H1_m(x), m = 0..max_order, for a batch of points on the device (bf_hankel_orders):
    the reference's hankel1_orders (bessel.py:225-230) with the batch's own start.
    x: NumPy float64 (nx,). Returns a torch CUDA (nx, max_order + 1) complex128 tensor."""
    torch = _lib.require_cuda()
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    if (x <= 0).any():
        raise ValueError("order sweep requires x > 0")
    if out is None:
        out = torch.empty((x.size, max_order + 1), dtype=torch.complex128, device="cuda")
    xd = torch.as_tensor(x).cuda()
    _lib.check(_lib.load().bf_hankel_orders(ctypes.c_void_p(xd.data_ptr()), x.size, int(max_order),
                                            sweep_start(x, max_order), ctypes.c_void_p(out.data_ptr()),
                                            out.stride(0), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
               "bf_hankel_orders")
    return out


class HankelKernel:
    """K[i, j] = H1_j(x_i), x_i = n + (2 pi / 3) i (reference kernels.py:45-84), on the device.

    Cached (n <= TABLE_CAP, the default): the whole n x n table is built once on the
    device, sorted rows in batches of 256 with one order sweep each — exactly how the
    reference's row cache fills from empty on block(arange(n), arange(n)) — and the
    construction reads it as a dense entry source. Uncached: each block() call sweeps
    its own rows to order max(cols), as the reference's uncached path does."""

    TABLE_CAP = 1 << 15   # 16 GiB of complex128 table

    def __init__(self, n: int, cache: bool | None = None):
        self.n = int(n)
        self.shape = (self.n, self.n)
        self._cache = self.n <= self.TABLE_CAP if cache is None else bool(cache)
        self._table = None

    def point(self, i: int) -> float:
        return self.n + (2.0 * np.pi / 3.0) * i

    def points(self, rows) -> np.ndarray:
        return self.n + (2.0 * np.pi / 3.0) * np.asarray(rows, dtype=np.intp).astype(float)

    def device_table(self):
        """The (n, n) complex128 table on the device (built on first use)."""
        if self._table is None:
            torch = _lib.require_cuda()
            n = self.n
            table = torch.empty((n, n), dtype=torch.complex128, device="cuda")
            for lo in range(0, n, 256):
                hi = min(n, lo + 256)
                hankel1_orders_device(self.points(np.arange(lo, hi)), n - 1, out=table[lo:hi])
            self._table = table
        return self._table

    def device_windows(self, blocks, side):
        """(nb, side, side) device windows K[i side + a, j side + b] of middle blocks (i, j),
        as the uncached reference path evaluates a block: one order sweep of the block's
        rows up to its last column (kernels.py:63-66)."""
        torch = _lib.require_cuda()
        out = torch.empty((len(blocks), side, side), dtype=torch.complex128, device="cuda")
        for b, (i, j) in enumerate(blocks):
            rows = np.arange(i * side, (i + 1) * side)
            table = hankel1_orders_device(self.points(rows), (j + 1) * side - 1)
            out[b] = table[:, j * side:]
            del table
        return out

    def block(self, rows, cols) -> np.ndarray:
        torch = _lib.require_cuda()
        rows = np.asarray(rows, dtype=np.intp).reshape(-1)
        cols = np.asarray(cols, dtype=np.intp).reshape(-1)
        if rows.size == 0 or cols.size == 0:
            return np.zeros((rows.size, cols.size), dtype=np.complex128)
        if self._cache:
            t = self.device_table()
            r = torch.as_tensor(rows).cuda()
            c = torch.as_tensor(cols).cuda()
            return t[r][:, c].cpu().numpy()
        table = hankel1_orders_device(self.points(rows), int(cols.max(initial=0)))
        return table[:, torch.as_tensor(cols).cuda()].cpu().numpy()


def hankel_entry(n: int, i: int, j: int) -> complex:
    """H1_j(x_i) by one sweep at the single point (reference kernels.py:82-84)."""
    x = n + (2.0 * np.pi / 3.0) * i
    return complex(hankel1_orders_device(np.array([x]), j)[0, j].item())


def fio_entry(n: int, i: int, j: int) -> complex:
    return complex(FioKernel(n).block([i], [j])[0, 0])


class DftKernel(_DeviceKernel):
    """The reference's centered transform F[j, k] = exp(-2 pi i xi_j x_k), xi_j = j - n/2,
    x_k = k/n (kernels.py:87-97), evaluated on the device with NumPy's rounding order."""

    kernel_id = _lib.BF_KERNEL_DFT


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


def _is_device(x) -> bool:
    return hasattr(x, "is_cuda") and x.is_cuda


def dft_apply(n: int, g, direction: str = "forward"):
    """Centered DFT (or its inverse) with the (-1)^j modulation (reference kernels.py:100-112).
    NumPy in -> NumPy out; torch CUDA in -> torch CUDA out (cuFFT)."""
    if direction not in ("forward", "inverse"):
        raise ValueError(f"unknown direction {direction!r}")
    if _is_device(g):
        import torch
        if g.shape[0] != n:
            raise ValueError(f"input length {g.shape[0]} != {n}")
        g = g.to(torch.complex128)
        signs = torch.where(torch.arange(n, device=g.device) % 2 == 0, 1.0, -1.0).to(torch.float64)
        if g.ndim > 1:
            signs = signs[:, None]
        if direction == "forward":
            return torch.fft.fft(signs * g, dim=0)
        return signs * torch.fft.ifft(g, dim=0)
    g = np.asarray(g, dtype=np.complex128)
    if g.shape[0] != n:
        raise ValueError(f"input length {g.shape[0]} != {n}")
    signs = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    if g.ndim > 1:
        signs = signs[:, None]
    if direction == "forward":
        return np.fft.fft(signs * g, axis=0)
    return signs * np.fft.ifft(g, axis=0)


class ComposedOperator:
    """K F K as a black-box operator: two factored applies around an FFT
    (reference kernels.py:129-150)."""

    accepts_device = True

    def __init__(self, k_factors):
        self.k_factors = k_factors

    @property
    def n(self) -> int:
        return self.k_factors.n

    @property
    def shape(self):
        return (self.n, self.n)

    def apply(self, x):
        k = self.k_factors
        return k.apply(dft_apply(self.n, k.apply(x), "forward"))

    def apply_adjoint(self, x):
        k = self.k_factors
        inner = dft_apply(self.n, k.apply_adjoint(x), "inverse") * self.n
        return k.apply_adjoint(inner)


def composed_matvec(c: ComposedOperator, g, adjoint: bool = False):
    """reference kernels.py:153-154."""
    return c.apply_adjoint(g) if adjoint else c.apply(g)


def is_entry_oracle(oracle) -> bool:
    return hasattr(oracle, "block")


def is_operator_oracle(oracle) -> bool:
    return hasattr(oracle, "apply") and hasattr(oracle, "apply_adjoint")
