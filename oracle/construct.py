"""Sampling construction of the factor chain — NumPy restatement of reference
``construct.py`` (test infrastructure; see oracle/__init__.py)."""

from __future__ import annotations

import numpy as np

from .chain import Chain
from .lowrank import Params, Triple, floored_inverse, sampling_svd
from .partition import level_geometry, node_range

SAMPLING_DOMAIN = 0   # construct.py:26


def block_rng(seed, *key) -> np.random.Generator:
    """Per-task generator from SeedSequence spawn keys (construct.py:31-33)."""
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=key))


def middle_geometry(n: int, levels: int, r: int, branching: int = 2):
    m = branching ** (levels // 2)
    side = n // m
    if side < r:
        raise ValueError(f"middle blocks are {side} wide, below rank {r}")
    return m, side


def sample_block(entry, n, levels, r, params, seed, i, j, trace=None, branching=2) -> Triple:
    """One middle block through a row/column window of the parent oracle (construct.py:43-50)."""
    half = levels // 2
    m, side = middle_geometry(n, levels, r, branching)
    if branching == 2:
        r0 = node_range(n, levels, half, i).start
        c0 = node_range(n, levels, half, j).start
    else:  # quadtree nodes are contiguous Morton ranges of equal size
        r0, c0 = i * side, j * side

    def window(rows, cols):
        return entry.block(np.asarray(rows, dtype=np.intp) + r0, np.asarray(cols, dtype=np.intp) + c0)

    rng = block_rng(seed, SAMPLING_DOMAIN, i, j)
    return sampling_svd(window, side, side, r, params, rng, trace=trace)


def middle_level(entry, n, levels, r, params=Params(), seed=0, branching=2):
    """U^h, W, V^h of the sampling construction (construct.py:53-68).

    Returns u (m, side, m, r), w (m, m, r), v (m, side, m, r).
    """
    m, side = middle_geometry(n, levels, r, branching)
    u = np.zeros((m, side, m, r), dtype=np.complex128)
    v = np.zeros((m, side, m, r), dtype=np.complex128)
    w = np.zeros((m, m, r))
    for i in range(m):
        for j in range(m):
            t = sample_block(entry, n, levels, r, params, seed, i, j, branching=branching)
            u[i, :, j, :] = t.u0 * t.sigma0
            v[j, :, i, :] = t.v0 * t.sigma0
            w[i, j] = floored_inverse(t.sigma0)
    return u, w, v


def recurse(cur: np.ndarray, n: int, levels: int, r: int, branching: int = 2):
    """Level-by-level batched SVD refactorization (construct.py:127-163).

    ``cur`` is (nodes, rows, groups, r). Returns (leaf (nodes, rows, r), [(lvl, blocks)]).
    ``branching`` b splits rows into b parts and merges b column groups per level
    (b = 2 is the reference; b = 4 its quadtree generalisation).
    """
    b = branching
    pieces = []
    for lvl in range(levels // 2, levels):
        nb, rows, groups, _ = cur.shape
        pairs = groups // b
        if rows >= b:
            part = rows // b
            paired = cur.reshape(nb, rows, pairs, b * r)
            stacked = np.stack([paired[:, t * part:(t + 1) * part].transpose(0, 2, 1, 3) for t in range(b)],
                               axis=1)                                  # (nb, b, pairs, part, b r)
            uu, ss, vh = np.linalg.svd(stacked, full_matrices=False)
            keep = min(r, part, b * r)
            blocks = np.zeros((nb, b, pairs, r, b * r), dtype=np.complex128)
            blocks[..., :keep, :] = vh[..., :keep, :]
            nxt = np.zeros((nb, b, pairs, part, r), dtype=np.complex128)
            nxt[..., :keep] = uu[..., :keep] * ss[..., None, :keep]
            pieces.append((lvl, blocks))
            cur = nxt.transpose(0, 1, 3, 2, 4).reshape(b * nb, part, pairs, r)
        else:
            paired = cur.reshape(nb, 1, pairs, b * r).transpose(0, 2, 1, 3)   # (nb, pairs, 1, b r)
            uu, ss, vh = np.linalg.svd(paired, full_matrices=False)
            blocks = np.zeros((nb, pairs, r, b * r), dtype=np.complex128)
            blocks[..., :1, :] = vh
            nxt = np.zeros((nb, pairs, 1, r), dtype=np.complex128)
            nxt[..., :1] = uu * ss[..., None, :]
            pieces.append((lvl, blocks))
            cur = nxt.transpose(0, 2, 1, 3)
    return np.ascontiguousarray(cur[:, :, 0, :]), pieces


def factorize(entry, n: int, levels: int, r: int, params=Params(), seed=0, branching: int = 2) -> Chain:
    """Full sampling-mode construction (construct.py:184-213, mode="sampling"); branching 4 = quadtree."""
    if r < 1:
        raise ValueError(f"rank must be positive, got {r}")
    m, side = middle_geometry(n, levels, r, branching)
    u, w, v = middle_level(entry, n, levels, r, params, seed, branching)
    u_leaf, g_levels = recurse(u.reshape(m, side, m, r), n, levels, r, branching)
    v_leaf, h_levels = recurse(v.reshape(m, side, m, r), n, levels, r, branching)
    return Chain(n, levels, r, u_leaf, g_levels, w, h_levels, v_leaf)


def chain_shapes(n: int, levels: int, r: int):
    """Alias of the level geometry used for preallocation (construct.py:216-227)."""
    return level_geometry(n, levels, r)
