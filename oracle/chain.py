"""Apply chain of the butterfly factorization — NumPy restatement of reference
``factors.py`` (test infrastructure; see oracle/__init__.py).

A chain is held as plain arrays in the reference layout (factors.py:23-203):

* ``u_leaf``, ``v_leaf``: (nb, n0, r) complex, block b at (b*n0, b*r)
  (``BlockDiagonalFactor``, factors.py:23-56);
* ``g_levels``, ``h_levels``: lists of (level, blocks) ascending half..L-1, blocks
  (G, 2, P, r, 2r) at splitting levels, (G, P, r, 2r) at merge-only levels
  (``TransferFactor``, factors.py:59-142);
* ``weights``: (m, m, r) real (``MiddleFactor``, factors.py:145-190).

Index semantics (one level each; w is (dim, k), RHS fastest):

    leaf adjoint   out[b, c]      = sum_i conj(X[b, i, c]) * w[b, i]
    leaf forward   out[b, i]      = sum_c X[b, i, c] * w[b, c]
    transfer fwd   out[g, t, p, :] = B[g, t, p] @ w[g, p, :]      (split)
    transfer adj   out[g, p, :]   = sum_t B[g, t, p]^H @ w[g, t, p, :]
    middle fwd     out[i, j, rho] = W[i, j, rho] * w[j, i, rho]
    middle adj     out[j, i, rho] = W[i, j, rho] * w[i, j, rho]
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Chain:
    """Factor arrays of one chain (field order of ``ButterflyFactors``, factors.py:193-203)."""

    n: int
    levels: int
    rank: int
    u_leaf: np.ndarray
    g_levels: list
    weights: np.ndarray
    h_levels: list
    v_leaf: np.ndarray

    @classmethod
    def from_reference(cls, f) -> "Chain":
        return cls(f.n, f.partition.levels, f.rank, f.u_outer.blocks,
                   [(tf.level, tf.blocks) for tf in f.g_chain], f.middle.weights,
                   [(tf.level, tf.blocks) for tf in f.h_chain], f.v_outer.blocks)

    def nnz_total(self) -> int:
        """Stored entries (NnzReport.total, factors.py:248-271)."""
        return (self.u_leaf.size + self.v_leaf.size + self.weights.size
                + sum(b.size for _, b in self.g_levels)
                + sum(b.size for _, b in self.h_levels))


def leaf_forward(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """factors.py:49-51."""
    nb, rows, cols = x.shape
    return np.matmul(x, w.reshape(nb, cols, -1)).reshape(nb * rows, -1)


def leaf_adjoint(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """factors.py:53-56."""
    nb, rows, cols = x.shape
    xh = np.conj(x).transpose(0, 2, 1)
    return np.matmul(xh, w.reshape(nb, rows, -1)).reshape(nb * cols, -1)


def transfer_forward(b: np.ndarray, w: np.ndarray) -> np.ndarray:
    """factors.py:120-129."""
    k = w.shape[-1]
    if b.ndim == 5:
        groups, _, pairs, r, c = b.shape
        return np.matmul(b, w.reshape(groups, 1, pairs, c, k)).reshape(-1, k)
    nodes, pairs, r, c = b.shape
    return np.matmul(b, w.reshape(nodes, pairs, c, k)).reshape(-1, k)


def transfer_adjoint(b: np.ndarray, w: np.ndarray) -> np.ndarray:
    """factors.py:131-142 (sum over the row parts t of a splitting level; 2 in 1-D, 4 on quadtrees)."""
    k = w.shape[-1]
    bh = np.conj(b).swapaxes(-1, -2)
    if b.ndim == 5:
        groups, nt, pairs, r, c = b.shape
        win = w.reshape(groups, nt, pairs, r, k)
        return np.matmul(bh, win).sum(axis=1).reshape(-1, k)
    nodes, pairs, r, c = b.shape
    return np.matmul(bh, w.reshape(nodes, pairs, r, k)).reshape(-1, k)


def middle_forward(weights: np.ndarray, w: np.ndarray) -> np.ndarray:
    """factors.py:180-184: block (i, j) takes slot (j, i), scaled by W[i, j]."""
    m, _, r = weights.shape
    win = w.reshape(m, m, r, -1).swapaxes(0, 1)
    return (weights[:, :, :, None] * win).reshape(m * m * r, -1)


def middle_adjoint(weights: np.ndarray, w: np.ndarray) -> np.ndarray:
    """factors.py:186-190."""
    m, _, r = weights.shape
    scaled = weights[:, :, :, None] * w.reshape(m, m, r, -1)
    return scaled.swapaxes(0, 1).reshape(m * m * r, -1)


def apply(chain: Chain, g: np.ndarray, adjoint: bool = False) -> np.ndarray:
    """K @ g (or K* @ g) through the chain — ButterflyFactors._chain, factors.py:217-237."""
    g = np.asarray(g)
    if g.shape[0] != chain.n:
        raise ValueError(f"input length {g.shape[0]} != {chain.n}")
    vec = g.ndim == 1
    w = g.reshape(chain.n, -1).astype(np.complex128, copy=False)
    if not adjoint:
        w = leaf_adjoint(chain.v_leaf, w)
        for _, b in reversed(chain.h_levels):
            w = transfer_adjoint(b, w)
        w = middle_forward(chain.weights, w)
        for _, b in chain.g_levels:
            w = transfer_forward(b, w)
        w = leaf_forward(chain.u_leaf, w)
    else:
        w = leaf_adjoint(chain.u_leaf, w)
        for _, b in reversed(chain.g_levels):
            w = transfer_adjoint(b, w)
        w = middle_adjoint(chain.weights, w)
        for _, b in chain.h_levels:
            w = transfer_forward(b, w)
        w = leaf_forward(chain.v_leaf, w)
    return w[:, 0] if vec else w
