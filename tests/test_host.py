"""Host-side logic of the package (no GPU): partition mirror, level geometry,
factor dataclasses, synthetic chains."""

import numpy as np
import pytest

import paper_1502_01379_b200 as bf
from conftest import chain_from_golden, golden
from oracle import chain as ochain
from oracle import partition as opart
from paper_1502_01379_b200.synthetic import synthetic_chain


def test_partition_mirror_matches_reference_geometry():
    d = golden("geometry.npz")
    for n, leaf in ((1024, 8), (1 << 16, 16), (1 << 20, 16), (256, 0.25), (64, 1), (1024, 1), (128, 0.25)):
        tag = f"{n}_{leaf}"
        p = bf.make_partition(n, leaf)
        assert p.levels == int(d[f"levels_{tag}"])
        for lvl, i, lo, hi in d[f"ranges_{tag}"][::7]:
            rg = p.node_range(int(lvl), int(i))
            assert (rg.start, rg.stop) == (lo, hi)
        shapes, leaf_shape = bf.level_geometry(p, 4)
        assert (shapes, leaf_shape) == opart.level_geometry(n, p.levels, 4)


def test_partition_errors_match_reference():
    for bad in (1000, 3, 0):
        with pytest.raises(ValueError):
            bf.make_partition(bad, 1)
    with pytest.raises(ValueError):
        bf.make_partition(64, 0)
    with pytest.raises(ValueError):
        bf.DyadicPartition(64, 3)
    with pytest.raises(ValueError):
        bf.DyadicPartition(16, 10)
    p = bf.make_partition(1024, 8)
    assert (p.levels, p.half, p.mid_nodes, p.mid_side, p.leaf_size) == (6, 3, 8, 128, 16)
    q = bf.make_partition(256, 0.25)
    assert q.levels == 10 and q.leaf_size == 0.25


def _product_chain(d):
    c = chain_from_golden(d)
    return bf.from_arrays(c.n, c.levels, c.rank, c.u_leaf, c.g_levels, c.weights, c.h_levels, c.v_leaf), c


@pytest.mark.parametrize("name", ["apply_fio_n256_r8_leaf025.npz", "apply_dftp_n1024_r8_leaf16.npz"])
def test_dense_views_compose_to_operator(name):
    """pkg/tests/test_factors.py:79-89 with the product's dense views, checked by the oracle chain."""
    f, c = _product_chain(golden(name))
    full = f.u_outer.dense()
    for tf in reversed(f.g_chain):
        full = full @ tf.dense()
    full = full @ f.middle.dense()
    for tf in f.h_chain:
        full = full @ tf.dense().conj().T
    full = full @ f.v_outer.dense().conj().T
    want = ochain.apply(c, np.eye(f.n, dtype=complex))
    assert np.allclose(full, want, atol=1e-12)


def test_nnz_report_identities():
    f, c = _product_chain(golden("apply_cfg0_fio_n1024_r12_leaf8.npz"))
    rep = f.nnz_report()
    p = f.partition
    assert rep.middle == 2 ** p.levels * f.rank
    assert rep.u_outer == rep.v_outer == p.n * f.rank
    assert rep.total == c.nnz_total() == 135936
    assert set(rep.g.values()) == {2 ** (p.levels + 1) * f.rank ** 2}


def test_factors_equal_and_shapes():
    f, _ = _product_chain(golden("apply_fio_n256_r8_leaf025.npz"))
    assert bf.factors_equal(f, f)
    splits = [tf.splits for tf in f.g_chain]
    assert splits[0] and not splits[-1]          # leaf 0.25: merge-only levels at the bottom
    g = synthetic_chain(f.partition, f.rank, seed=1)
    assert not bf.factors_equal(f, g)
    shapes, leaf = bf.level_geometry(f.partition, f.rank)
    assert [tuple(t.blocks.shape) for t in g.g_chain] == [s for _, _, s in shapes]
    assert tuple(g.u_outer.blocks.shape) == leaf


def test_synthetic_chain_is_seeded():
    p = bf.make_partition(256, 16)
    a, b = synthetic_chain(p, 4, seed=5), synthetic_chain(p, 4, seed=5)
    assert bf.factors_equal(a, b)
    assert np.all((a.middle.weights >= 0.5) & (a.middle.weights <= 1.5))


def test_oversampling_params_validate():
    """lowrank.py:33-48 / reference test_lowrank.py:215-221."""
    import pytest
    for kw in ({"p": -1}, {"q": 0}, {"iters": 0}):
        with pytest.raises(ValueError):
            bf.OversamplingParams(**kw)
    assert bf.OversamplingParams() == bf.OversamplingParams(p=5, q=3, iters=3)
