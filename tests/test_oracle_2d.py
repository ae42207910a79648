"""The quadtree (2-D) restatement in oracle/ (BASELINE configs 3/4b). The
reference has no 2-D code, so parity is unpinned: these tests pin
the restatement to first principles — Morton geometry, the branching-4 chain
against its own dense factors, and the factorization against the dense
operator (the RowSampledReference pattern, bench.py:38-46)."""

import numpy as np

from oracle import chain as ochain
from oracle import construct as ocons
from oracle import entries as oent
from oracle import partition as opart


def test_morton_nodes_are_boxes():
    n_side, bits = 16, 4
    z = np.arange(n_side * n_side)
    a1, a2 = oent.morton_decode(z, bits)
    assert sorted(zip(a1.tolist(), a2.tolist())) == [(i, j) for i in range(16) for j in range(16)]
    # a depth-2 quadtree node (16 consecutive Morton indices) is a 4x4 box
    for node in range(16):
        blk = slice(node * 16, (node + 1) * 16)
        assert a1[blk].max() - a1[blk].min() == 3 and a2[blk].max() - a2[blk].min() == 3


def test_radon_unimodular_and_symmetric_grid():
    k = oent.radon2d_block(32, np.arange(0, 1024, 37), np.arange(0, 1024, 41))
    assert np.max(np.abs(np.abs(k) - 1)) <= 1e-15


def test_quadtree_geometry():
    assert opart.quadtree_levels(256, 4) == 6 and opart.quadtree_levels(1024, 4) == 8
    shapes, leaf = opart.level_geometry(256 * 256, 6, 25, branching=4)
    assert leaf == (4 ** 6, 16, 25)
    assert shapes[0] == (3, True, (64, 4, 16, 25, 100))
    assert all(np.prod(s) == 4 ** 6 * 4 * 25 * 25 * 4 // 4 for _, _, s in shapes)


class _Dense:
    def __init__(self, mat):
        self.matrix, self.shape = mat, mat.shape

    def block(self, rows, cols):
        return self.matrix[np.ix_(np.asarray(rows), np.asarray(cols))]


def _random_quadtree_chain(n, levels, r, rng):
    def orth_rows(shape):
        a = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        flat = a.reshape(-1, *shape[-2:])
        if shape[-2] > shape[-1]:               # tall leaf blocks: orthonormal columns
            return np.ascontiguousarray(np.linalg.qr(flat)[0].reshape(shape))
        q, _ = np.linalg.qr(flat.swapaxes(-1, -2))
        return np.ascontiguousarray(q.swapaxes(-1, -2).reshape(shape))

    shapes, leaf = opart.level_geometry(n, levels, r, branching=4)
    m = 4 ** (levels // 2)
    return ochain.Chain(n, levels, r, orth_rows(leaf).conj(), [(l, orth_rows(s)) for l, _, s in shapes],
                        rng.uniform(0.5, 1.5, size=(m, m, r)), [(l, orth_rows(s)) for l, _, s in shapes],
                        orth_rows(leaf).conj())


def test_quadtree_exact_rank_reproduction():
    """A branching-4 chain with rank-3 blocks is reproduced to 1e-10 (the 2-D analogue of
    pkg/tests/test_construct.py:253-261)."""
    rng = np.random.default_rng(20240801)
    n, levels, r = 256, 2, 3                # 16x16 grid, depth 2: 16 boxes of 16 points per side
    truth = _random_quadtree_chain(n, levels, r, rng)
    k = ochain.apply(truth, np.eye(n, dtype=complex))
    c = ocons.factorize(_Dense(k), n, levels, r, seed=8, branching=4)
    g = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
    assert np.linalg.norm(ochain.apply(c, g) - k @ g) <= 1e-10 * np.linalg.norm(k @ g)
    assert np.linalg.norm(ochain.apply(c, g, adjoint=True) - k.conj().T @ g) <= 1e-10 * np.linalg.norm(k @ g)


def test_quadtree_radon_error_decreases_with_rank():
    n_side = 32
    n = n_side * n_side
    levels = opart.quadtree_levels(n_side, 2)
    ent = oent.Radon2DOracle(n_side)
    k = ent.block(np.arange(n), np.arange(n))
    g = np.random.default_rng(0).standard_normal((n, 2)) + 0j
    errs = []
    for r in (4, 12):
        c = ocons.factorize(ent, n, levels, r, seed=0, branching=4)
        errs.append(np.linalg.norm(ochain.apply(c, g) - k @ g) / np.linalg.norm(k @ g))
    assert errs[1] < errs[0] < 1.0, errs
