"""Matvec-mode construction oracle (construct.py:71-124, lowrank.py:204-216)
pinned to the reference's own outputs (tests/golden/matvec_*.npz, written by
oracle/gen_golden.py from the reference)."""

import numpy as np
import pytest

from conftest import chain_from_golden, golden
from oracle import chain as ochain
from oracle import construct as ocons
from oracle import entries as oent
from oracle import lowrank as olr
from oracle import operators as oops


def _dense_fio(n):
    return oent.EntryOracle("fio", n).block(np.arange(n), np.arange(n))


def test_probes_match_reference():
    d = golden("matvec_dense_fio_n256_r8_leaf1.npz")
    n, levels, r, seed, width = (int(d[k]) for k in ("n", "levels", "rank", "seed", "width"))
    col = ocons.block_diagonal_probe(n, levels, r, width, seed, ocons.COL_PROBE_DOMAIN)
    row = ocons.block_diagonal_probe(n, levels, r, width, seed, ocons.ROW_PROBE_DOMAIN)
    assert np.array_equal(col, d["col_probe"]) and np.array_equal(row, d["row_probe"])
    # one (side x width) nonzero block per middle node (test_construct.py:96-101)
    m = col.shape[1] // width
    assert np.count_nonzero(col) == n * width and m == 2 ** (levels // 2)


def test_matvec_middle_level_matches_reference():
    d = golden("matvec_dense_fio_n256_r8_leaf1.npz")
    n, levels, r, seed = (int(d[k]) for k in ("n", "levels", "rank", "seed"))
    op = oops.DenseOperator(_dense_fio(n))
    u, w, v = ocons.middle_level_matvec(op, n, levels, r, seed=seed)
    m, side = ocons.middle_geometry(n, levels, r)
    # identical NumPy/LAPACK calls in the identical order: bitwise
    assert np.array_equal(u.reshape(m, side, m * r), d["u_h"])
    assert np.array_equal(v.reshape(m, side, m * r), d["v_h"])
    assert np.array_equal(w, d["w_h"])


def test_matvec_factorize_matches_reference():
    d = golden("matvec_dense_fio_n256_r8_leaf1.npz")
    n, levels, r, seed = (int(d[k]) for k in ("n", "levels", "rank", "seed"))
    op = oops.DenseOperator(_dense_fio(n))
    c = ocons.factorize(op, n, levels, r, seed=seed, mode="matvec")
    ref = chain_from_golden(d)
    np.testing.assert_array_equal(c.weights, ref.weights)
    assert np.array_equal(ochain.apply(c, d["g"]), d["fwd"])
    assert np.array_equal(ochain.apply(c, d["g"], adjoint=True), d["adj"])


def test_composed_operator_matches_reference():
    d = golden("matvec_composed_fio_n256_r8_leaf1.npz")
    inner = chain_from_golden(d, "inner_")
    comp = oops.Composed(inner)
    np.testing.assert_allclose(comp.apply(d["g"]), d["comp_fwd"], rtol=0, atol=1e-12 * np.abs(d["comp_fwd"]).max())
    np.testing.assert_allclose(comp.apply_adjoint(d["g"]), d["comp_adj"], rtol=0,
                               atol=1e-12 * np.abs(d["comp_adj"]).max())


def test_composed_matvec_factorize_matches_reference():
    d = golden("matvec_composed_fio_n256_r8_leaf1.npz")
    inner = chain_from_golden(d, "inner_")
    n, levels, r, seed = (int(d[k]) for k in ("n", "levels", "rank", "seed"))
    c = ocons.factorize(oops.Composed(inner), n, levels, r, seed=seed, mode="matvec")
    got = ochain.apply(c, d["g"])
    assert np.linalg.norm(got - d["fwd"]) <= 1e-12 * np.linalg.norm(d["fwd"])


def test_probe_svd_identity_operator():
    # test_construct.py:71-84: the identity at full middle-block rank (p = 0)
    n, levels = 64, 6
    m, side = ocons.middle_geometry(n, levels, 1)
    r = side
    op = oops.DenseOperator(np.eye(n, dtype=complex))
    u, w, v = ocons.middle_level_matvec(op, n, levels, r, params=olr.Params(p=0), seed=3)
    rng = np.random.default_rng(5)
    g = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    # middle triple: block (i, j) = u[i,:,j,:] diag(w[i,j]) v[j,:,i,:]^H
    out = np.zeros(n, dtype=complex)
    for i in range(m):
        for j in range(m):
            blk = (u[i, :, j, :] * w[i, j]) @ v[j, :, i, :].conj().T
            out[i * side:(i + 1) * side] += blk @ g[j * side:(j + 1) * side]
    assert np.linalg.norm(out - g) <= 1e-10 * np.linalg.norm(g)


def test_dft_apply_errors():
    with pytest.raises(ValueError):
        oops.dft_apply(8, np.zeros(7))
    with pytest.raises(ValueError):
        oops.dft_apply(8, np.zeros(8), "sideways")
