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


def dftp_block(n: int, rows, cols) -> np.ndarray:
    j = np.asarray(rows, dtype=np.int64)[:, None]
    k = np.asarray(cols, dtype=np.int64)[None, :]
    frac = ((j * k) % n).astype(np.float64) / n
    return np.exp(2j * np.pi * frac)


class EntryOracle:
    """``.shape`` + ``.block(rows, cols)`` — the reference entry-oracle protocol (oracles.py:5-10)."""

    def __init__(self, kind: str, n: int):
        if kind not in ("fio", "dftp"):
            raise ValueError(f"unknown kernel {kind!r}")
        self.kind, self.n, self.shape = kind, n, (n, n)

    def block(self, rows, cols):
        fn = fio_block if self.kind == "fio" else dftp_block
        return fn(self.n, rows, cols)
