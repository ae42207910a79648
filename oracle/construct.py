"""Sampling construction of the factor chain — NumPy restatement of reference
``construct.py`` (test infrastructure; see oracle/__init__.py)."""

from __future__ import annotations

import numpy as np

from .chain import Chain
from .lowrank import Params, Triple, complex_normal, floored_inverse, probe_svd, sampling_svd
from .partition import level_geometry, node_range

SAMPLING_DOMAIN = 0   # construct.py:26
COL_PROBE_DOMAIN = 1  # construct.py:27
ROW_PROBE_DOMAIN = 2  # construct.py:28


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


def probe_blocks(n: int, levels: int, r: int, width: int, seed, domain, branching: int = 2) -> np.ndarray:
    """The diagonal blocks (m, side, width) of block_diagonal_probe (construct.py:78-86):
    block j drawn from block_rng(seed, domain, j)."""
    m, side = middle_geometry(n, levels, r, branching)
    return np.stack([complex_normal(block_rng(seed, domain, j), (side, width)) for j in range(m)])


def block_diagonal_probe(n: int, levels: int, r: int, width: int, seed, domain, branching: int = 2) -> np.ndarray:
    """(n, m*width) probe, block j at rows j*side, columns j*width (construct.py:78-86)."""
    blocks = probe_blocks(n, levels, r, width, seed, domain, branching)
    m, side, _ = blocks.shape
    probe = np.zeros((n, m * width), dtype=np.complex128)
    for j in range(m):
        probe[j * side:(j + 1) * side, j * width:(j + 1) * width] = blocks[j]
    return probe


def apply_chunked(apply_fn, block: np.ndarray, chunk: int = 128) -> np.ndarray:
    """_apply_chunked (construct.py:71-75)."""
    if block.shape[1] <= chunk:
        return apply_fn(block)
    return np.concatenate([apply_fn(block[:, c:c + chunk]) for c in range(0, block.shape[1], chunk)], axis=1)


def middle_level_matvec(op, n, levels, r, params=Params(), seed=0, branching=2):
    """U^h, W, V^h from black-box applies of K and K* (middle_factorization_matvec,
    construct.py:89-124): one block-diagonal probe per side covers every block,
    then each block's SVD is finished from the stored products (probe_svd)."""
    m, side = middle_geometry(n, levels, r, branching)
    width = min(r + params.p, side)
    col_probe = block_diagonal_probe(n, levels, r, width, seed, COL_PROBE_DOMAIN, branching)
    row_probe = block_diagonal_probe(n, levels, r, width, seed, ROW_PROBE_DOMAIN, branching)
    k_cols = apply_chunked(op.apply, col_probe)
    k_rows = apply_chunked(op.apply_adjoint, row_probe)
    u = np.zeros((m, side, m, r), dtype=np.complex128)
    v = np.zeros((m, side, m, r), dtype=np.complex128)
    w = np.zeros((m, m, r))
    for i in range(m):
        rows = slice(i * side, (i + 1) * side)
        r_block = row_probe[rows, i * width:(i + 1) * width]
        for j in range(m):
            cols = slice(j * side, (j + 1) * side)
            t = probe_svd(k_cols[rows, j * width:(j + 1) * width], k_rows[cols, i * width:(i + 1) * width],
                          r_block, r)
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


def factorize(entry, n: int, levels: int, r: int, params=Params(), seed=0, branching: int = 2,
              mode: str = "sampling") -> Chain:
    """Full construction (construct.py:184-213): mode "sampling" (entry oracle; branching 4 =
    quadtree) or "matvec" (operator oracle with .apply / .apply_adjoint on (n, k) arrays)."""
    if r < 1:
        raise ValueError(f"rank must be positive, got {r}")
    m, side = middle_geometry(n, levels, r, branching)
    if mode == "matvec":
        u, w, v = middle_level_matvec(entry, n, levels, r, params, seed, branching)
    elif mode == "sampling":
        u, w, v = middle_level(entry, n, levels, r, params, seed, branching)
    else:
        raise ValueError(f"unknown mode {mode!r}")
    u_leaf, g_levels = recurse(u.reshape(m, side, m, r), n, levels, r, branching)
    v_leaf, h_levels = recurse(v.reshape(m, side, m, r), n, levels, r, branching)
    return Chain(n, levels, r, u_leaf, g_levels, w, h_levels, v_leaf)


def chain_shapes(n: int, levels: int, r: int):
    """Alias of the level geometry used for preallocation (construct.py:216-227)."""
    return level_geometry(n, levels, r)


def synthetic_slab(side, m, r, seed):
    """(1, side, m, r) complex Gaussian slab with a spread of column scales."""
    rng = np.random.default_rng(seed)
    slab = rng.standard_normal((1, side, m, r)) + 1j * rng.standard_normal((1, side, m, r))
    slab *= np.logspace(0, -6, r)[None, None, None, :]
    return slab


def slab_chain_apply(leaf_b, pieces, x):
    """U^L G^{L-1} .. G^h x for one slab's recursion output (x: (m r, k))."""
    w = x
    for lvl, b in pieces:                      # ascending h .. L-1: the G side order
        if b.ndim == 5:
            gn, _, pp, rr, c2 = b.shape
            wv = w.reshape(gn, pp, c2, -1)
            w = np.einsum("gtprc,gpck->gtprk", b, wv).reshape(-1, x.shape[1])
        else:
            gn, pp, rr, c2 = b.shape
            wv = w.reshape(gn, pp, c2, -1)
            w = np.einsum("gprc,gpck->gprk", b, wv).reshape(-1, x.shape[1])
    nb, rows, rr = leaf_b.shape
    return np.einsum("bir,brk->bik", leaf_b, w.reshape(nb, rr, -1)).reshape(nb * rows, -1)
