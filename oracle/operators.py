"""Operator oracles for the matvec construction — NumPy restatement of the
reference's ``dft_apply`` / ``ComposedOperator`` (kernels.py:100-150) and
``DenseOracle`` (oracles.py:39-54). Test infrastructure (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np

from . import chain as ochain


def dft_apply(n: int, g: np.ndarray, direction: str = "forward") -> np.ndarray:
    """Centered DFT via FFT with the (-1)^j modulation (kernels.py:100-112)."""
    g = np.asarray(g, dtype=np.complex128)
    if g.shape[0] != n:
        raise ValueError(f"input length {g.shape[0]} != {n}")
    signs = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    if g.ndim > 1:
        signs = signs[:, None]
    if direction == "forward":
        return np.fft.fft(signs * g, axis=0)
    if direction == "inverse":
        return signs * np.fft.ifft(g, axis=0)
    raise ValueError(f"unknown direction {direction!r}")


class DenseOperator:
    """Explicit matrix as an operator oracle (oracles.py:39-54)."""

    def __init__(self, matrix):
        self.matrix = np.asarray(matrix, dtype=np.complex128)
        self.shape = self.matrix.shape

    def apply(self, x):
        return self.matrix @ x

    def apply_adjoint(self, x):
        return self.matrix.conj().T @ x


class Composed:
    """K F K around a factored chain K (ComposedOperator, kernels.py:129-150)."""

    def __init__(self, chain: ochain.Chain):
        self.chain = chain
        self.n = chain.n
        self.shape = (self.n, self.n)

    def apply(self, x):
        k = lambda v: ochain.apply(self.chain, v)  # noqa: E731
        return k(dft_apply(self.n, k(x), "forward"))

    def apply_adjoint(self, x):
        ka = lambda v: ochain.apply(self.chain, v, adjoint=True)  # noqa: E731
        return ka(self.n * dft_apply(self.n, ka(x), "inverse"))
