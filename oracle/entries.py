"""Entry oracles K(x, xi) = exp(2 pi i Phi(x, xi)) for the BASELINE.json configs
(test infrastructure; see oracle/__init__.py).

* ``fio_block``  — reference ``FioKernel.block`` (kernels.py:23-38): x_i = i/n,
  xi_j = j - n/2, Phi = x xi + c(x)|xi|, c(x) = (2 + sin 2 pi x)/8.
* ``dftp_block`` — config 1's uncentered positive-sign DFT K_jk = exp(2 pi i jk/n).
  The reference has no such class (its ``DftKernel``, kernels.py:87-97, is the
  centered negative-sign transform); the phase is (j*k mod n)/n computed in
  int64 so it is exact, the convention SURVEY.md §8(c) fixes for CPU and GPU.

Both evaluate phases with one rounding per operation in the reference's order
(no fused multiply-add), then exp(i a) = (cos a, sin a).
"""

from __future__ import annotations

import numpy as np

TWO_PI = 2.0 * np.pi


def fio_block(n: int, rows, cols) -> np.ndarray:
    x = np.asarray(rows, dtype=np.float64)[:, None] / n
    xi = np.asarray(cols, dtype=np.float64)[None, :] - n / 2.0
    speed = (2.0 + np.sin(TWO_PI * x)) / 8.0
    phase = x * xi + speed * np.abs(xi)
    return np.exp(2j * np.pi * phase)


def dft_block(n: int, rows, cols) -> np.ndarray:
    """The reference's centered DftKernel.block (kernels.py:94-97)."""
    xi = np.asarray(rows, dtype=float)[:, None] - n / 2.0
    x = np.asarray(cols, dtype=float)[None, :] / n
    return np.exp(-2j * np.pi * xi * x)


def dftp_block(n: int, rows, cols) -> np.ndarray:
    j = np.asarray(rows, dtype=np.int64)[:, None]
    k = np.asarray(cols, dtype=np.int64)[None, :]
    frac = ((j * k) % n).astype(np.float64) / n
    return np.exp(2j * np.pi * frac)


class EntryOracle:
    """``.shape`` + ``.block(rows, cols)`` — the reference entry-oracle protocol (oracles.py:5-10)."""

    def __init__(self, kind: str, n: int):
        if kind not in ("fio", "dftp", "hankel"):
            raise ValueError(f"unknown kernel {kind!r}")
        self.kind, self.n, self.shape = kind, n, (n, n)
        if kind == "hankel":
            self._hk = HankelOracle(n)

    def block(self, rows, cols):
        if self.kind == "hankel":
            return self._hk.block(rows, cols)
        fn = fio_block if self.kind == "fio" else dftp_block
        return fn(self.n, rows, cols)


class HankelOracle:
    """HankelKernel (kernels.py:45-84): H1_j(x_i), x_i = n + (2 pi/3) i. For n <= 4096
    rows are cached, missing rows swept in sorted batches of 256 to order n-1 (so a
    row's last bits depend on which rows it was swept with, as in the reference);
    above, every call sweeps its rows to order max(cols)."""

    CACHE_CAP = 4096   # kernels.py:20

    def __init__(self, n: int, cache=None):
        self.n, self.shape = n, (n, n)
        self._cache = n <= self.CACHE_CAP if cache is None else cache
        self._rows = {}

    def block(self, rows, cols):
        from .bessel import hankel1_orders, hankel_points
        rows = np.asarray(rows, dtype=np.intp)
        cols = np.asarray(cols, dtype=np.intp)
        if not self._cache:
            return np.ascontiguousarray(hankel1_orders(hankel_points(self.n, rows), int(cols.max(initial=0)))[:, cols])
        missing = sorted(set(int(i) for i in rows) - self._rows.keys())
        for lo in range(0, len(missing), 256):
            batch = missing[lo:lo + 256]
            table = hankel1_orders(hankel_points(self.n, batch), self.n - 1)
            for b, i in enumerate(batch):
                self._rows[i] = table[b]
        out = np.empty((rows.size, cols.size), dtype=np.complex128)
        for a, i in enumerate(rows):
            out[a] = self._rows[int(i)][cols]
        return out


def morton_decode(z, bits: int):
    """Z-order index -> (a1, a2): bit k of a1 is bit 2k+1 of z, bit k of a2 is bit 2k."""
    z = np.asarray(z, dtype=np.int64)
    a1 = np.zeros_like(z)
    a2 = np.zeros_like(z)
    for k in range(bits):
        a2 |= ((z >> (2 * k)) & 1) << k
        a1 |= ((z >> (2 * k + 1)) & 1) << k
    return a1, a2


def radon2d_block(n_side: int, rows, cols) -> np.ndarray:
    """BASELINE configs 3/4b: generalized Radon kernel exp(2 pi i Phi) on an n x n grid.

    No reference implementation exists (SPEC.md:8 puts 2-D out of the
    reference's scope); this restatement defines the convention: indices are
    Morton (Z-order) numbers so that quadtree nodes are contiguous ranges;
    x = (a1, a2)/n in [0,1)^2, xi = (b1, b2) - n/2 in [-n/2, n/2)^2,
    Phi = x.xi + sqrt(c1^2 xi1^2 + c2^2 xi2^2), c1 = (2 + sin 2pi x1 sin 2pi x2)/16,
    c2 = (2 + cos 2pi x1 cos 2pi x2)/16; one rounding per operation, in this order.
    """
    bits = n_side.bit_length() - 1
    a1, a2 = morton_decode(rows, bits)
    b1, b2 = morton_decode(cols, bits)
    x1 = (a1.astype(np.float64) / n_side)[:, None]
    x2 = (a2.astype(np.float64) / n_side)[:, None]
    xi1 = (b1.astype(np.float64) - n_side / 2.0)[None, :]
    xi2 = (b2.astype(np.float64) - n_side / 2.0)[None, :]
    t1, t2 = TWO_PI * x1, TWO_PI * x2
    c1 = (2.0 + np.sin(t1) * np.sin(t2)) / 16.0
    c2 = (2.0 + np.cos(t1) * np.cos(t2)) / 16.0
    speed = np.sqrt((c1 * c1) * (xi1 * xi1) + (c2 * c2) * (xi2 * xi2))
    phase = (x1 * xi1 + x2 * xi2) + speed
    return np.exp(2j * np.pi * phase)


class Radon2DOracle:
    """Entry oracle of the 2-D generalized Radon kernel on an n_side^2 grid (Morton order)."""

    def __init__(self, n_side: int):
        self.n_side = n_side
        self.n = n_side * n_side
        self.shape = (self.n, self.n)

    def block(self, rows, cols):
        return radon2d_block(self.n_side, rows, cols)


def _splitmix(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


class NoisyOracle:
    """K(i, j) * (1 + amp * u(i, j)), u in [-1, 1) a fixed hash of (i, j, key). Running a
    construction on it measures that construction's own sensitivity to entry rounding:
    the calibrated envelope of SURVEY.md §8(c) stage 4."""

    def __init__(self, base, amp, key):
        self.base, self.amp, self.key = base, amp, np.uint64(key)
        self.shape = base.shape
        self.n = base.shape[1]

    def block(self, rows, cols):
        a = self.base.block(rows, cols)
        i = np.asarray(rows, dtype=np.uint64)[:, None]
        j = np.asarray(cols, dtype=np.uint64)[None, :]
        with np.errstate(over="ignore"):
            h = _splitmix(i * np.uint64(self.n) + j + self.key * np.uint64(0x632BE59BD9B4E019))
        u = (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0
        return a * (1.0 + self.amp * u)
