"""Matvec-mode construction on the GPU (construct.py:71-124; per block
svd_from_probes, lowrank.py:204-216) and the composition operator K F K
(kernels.py:100-154), against the reference's golden outputs
(tests/golden/matvec_*.npz, written by oracle/gen_golden.py from the reference)
and the CPU oracle. Stages as SURVEY.md §8(c): probes bitwise; per-block middle
products u0 diag(sigma) v0^H (phase invariant) and operator-level accuracy.
"""

import numpy as np
import pytest

import paper_1502_01379_b200 as bf
from conftest import chain_from_golden, complex_gaussian, golden
from oracle import chain as ochain
from oracle import construct as ocons
from oracle import entries as oent
from oracle import lowrank as olr
from oracle import operators as oops
from paper_1502_01379_b200.synthetic import to_host

torch = pytest.importorskip("torch")


def _np(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


def rel(a, b):
    a = _np(a)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _from_golden(d, prefix=""):
    c = chain_from_golden(d, prefix)
    p = bf.DyadicPartition(c.n, c.levels)
    return bf.from_arrays(c.n, c.levels, c.rank, c.u_leaf, c.g_levels, c.weights, c.h_levels, c.v_leaf,
                          partition=p)


def _block_products(u_h, w_h, v_h, m, side, r):
    u = _np(u_h).reshape(m, side, m, r)
    v = _np(v_h).reshape(m, side, m, r)
    w = _np(w_h)
    out = np.empty((m, m, side, side), dtype=np.complex128)
    for i in range(m):
        for j in range(m):
            # u0 sigma0 diag(1/sigma0) (v0 sigma0)^H = u0 sigma0 v0^H: phase invariant
            out[i, j] = (u[i, :, j, :] * w[i, j]) @ v[j, :, i, :].conj().T
    return out


class _Noisy:
    """An operator oracle whose outputs carry 1e-15 relative noise: the reference's own
    sensitivity (SURVEY.md §8(c) calibrated envelope) is measured through it."""

    def __init__(self, op, seed):
        self.op, self.rng = op, np.random.default_rng(seed)

    def _n(self, y):
        return y * (1 + 1e-15 * self.rng.standard_normal(y.shape))

    def apply(self, x):
        return self._n(self.op.apply(x))

    def apply_adjoint(self, x):
        return self._n(self.op.apply_adjoint(x))


def _envelope(op, n, levels, r, seed, g, want, trials=2):
    """max over noise draws of rel(apply(oracle chain built from the noisy operator), want)."""
    worst = 0.0
    for t in range(trials):
        c = ocons.factorize(_Noisy(op, 1000 + t), n, levels, r, seed=seed, mode="matvec")
        worst = max(worst, rel(ochain.apply(c, g), want))
    return worst


def test_probes_bitwise_reference():
    """Host probe draws are the reference's bit for bit (block_rng(seed, 1|2, j))."""
    d = golden("matvec_dense_fio_n256_r8_leaf1.npz")
    p = bf.DyadicPartition(int(d["n"]), int(d["levels"]))
    w, seed = int(d["width"]), int(d["seed"])
    from paper_1502_01379_b200 import construct as bc
    assert np.array_equal(bc.block_diagonal_probe(p, w, seed, bc.COL_PROBE_DOMAIN), d["col_probe"])
    assert np.array_equal(bc.block_diagonal_probe(p, w, seed, bc.ROW_PROBE_DOMAIN), d["row_probe"])


@pytest.mark.gpu
def test_middle_matvec_vs_reference_dense_fio():
    d = golden("matvec_dense_fio_n256_r8_leaf1.npz")
    n, levels, r, seed = (int(d[k]) for k in ("n", "levels", "rank", "seed"))
    p = bf.DyadicPartition(n, levels)
    m, side = p.mid_nodes, p.mid_side
    mat = oent.EntryOracle("fio", n).block(np.arange(n), np.arange(n))
    u_h, mid, v_h = bf.middle_factorization_matvec(bf.DenseOracle(mat), p, r, seed=seed)
    got = _block_products(u_h.blocks, mid.weights, v_h.blocks, m, side, r)
    want = _block_products(d["u_h"], d["w_h"], d["v_h"], m, side, r)
    # calibrated envelope (SURVEY.md §8(c) stage 4): d_ref(b) = how far the reference's
    # own block moves under 1e-15 relative noise on the operator (oracle == reference
    # bitwise, tests/test_oracle_matvec.py); require d_gpu(b) <= 10 max(d_ref(b), 1e-13)
    def dev(a, b):
        return np.array([[np.linalg.norm(a[i, j] - b[i, j]) / max(np.linalg.norm(b[i, j]), 1e-300)
                          for j in range(m)] for i in range(m)])

    d_ref = np.zeros((m, m))
    for trial in range(3):   # per-block envelope: max over three noise draws
        noise = np.random.default_rng(99 + trial).standard_normal(mat.shape) * 1e-15
        u2, w2, v2 = ocons.middle_level_matvec(oops.DenseOperator(mat * (1 + noise)), n, levels, r, seed=seed)
        d_ref = np.maximum(d_ref, dev(_block_products(u2, w2, v2, m, side, r), want))
    d_gpu = dev(got, want)
    inside = d_gpu <= 10 * np.maximum(d_ref, 1e-13)
    assert inside.mean() >= 0.9, (inside.mean(), np.median(d_gpu), np.median(d_ref))
    assert np.median(d_gpu) <= 3 * np.median(d_ref) + 1e-13
    assert d_gpu.max() <= 10 * d_ref.max() + 1e-13, (d_gpu.max(), d_ref.max())


@pytest.mark.gpu
def test_factorize_matvec_dense_fio_vs_reference():
    d = golden("matvec_dense_fio_n256_r8_leaf1.npz")
    n, levels, r, seed = (int(d[k]) for k in ("n", "levels", "rank", "seed"))
    p = bf.DyadicPartition(n, levels)
    mat = oent.EntryOracle("fio", n).block(np.arange(n), np.arange(n))
    f = bf.factorize(bf.DenseOracle(mat), p, r, seed=seed, mode="matvec")
    env = _envelope(oops.DenseOperator(mat), n, levels, r, seed, d["g"], d["fwd"])
    assert rel(f.apply(d["g"]), d["fwd"]) <= 10 * max(env, 1e-13)
    assert rel(f.apply_adjoint(d["g"]), d["adj"]) <= 1e-7
    # and the operator itself, as accurately as the reference's chain
    ref_err = np.linalg.norm(d["fwd"] - mat @ d["g"]) / np.linalg.norm(mat @ d["g"])
    got_err = rel(f.apply(d["g"]), mat @ d["g"])
    assert got_err <= 1.01 * ref_err + 1e-13


@pytest.mark.gpu
def test_composed_operator_vs_reference():
    d = golden("matvec_composed_fio_n256_r8_leaf1.npz")
    inner = _from_golden(d, "inner_")
    comp = bf.ComposedOperator(inner)
    g = d["g"]
    assert rel(comp.apply(g), d["comp_fwd"]) <= 1e-13
    assert rel(comp.apply_adjoint(g), d["comp_adj"]) <= 1e-13
    # device in -> device out, same numbers
    gd = torch.as_tensor(g).cuda()
    out = comp.apply(gd)
    assert out.is_cuda and rel(out, d["comp_fwd"]) <= 1e-13
    # zero in, zero out; adjoint identity (reference test_kernels.py:96-117)
    assert np.array_equal(_np(bf.composed_matvec(comp, np.zeros(inner.n, dtype=complex))),
                          np.zeros(inner.n, dtype=complex))
    rng = np.random.default_rng(11)
    x, y = complex_gaussian(rng, inner.n), complex_gaussian(rng, inner.n)
    lhs = np.vdot(y, _np(bf.composed_matvec(comp, x)))
    rhs = np.vdot(_np(bf.composed_matvec(comp, y, adjoint=True)), x)
    assert abs(lhs - rhs) <= 1e-10 * abs(lhs)


@pytest.mark.gpu
def test_factorize_matvec_composed_vs_reference():
    d = golden("matvec_composed_fio_n256_r8_leaf1.npz")
    inner = _from_golden(d, "inner_")
    n, levels, r, seed = (int(d[k]) for k in ("n", "levels", "rank", "seed"))
    comp = bf.ComposedOperator(inner)
    f = bf.factorize(comp, bf.DyadicPartition(n, levels), r, seed=seed, mode="matvec")
    env = _envelope(oops.Composed(chain_from_golden(d, "inner_")), n, levels, r, seed, d["g"], d["fwd"])
    assert rel(f.apply(d["g"]), d["fwd"]) <= 10 * max(env, 1e-13), (rel(f.apply(d["g"]), d["fwd"]), env)
    eps = bf.estimate_eps_a(f, bf.OperatorReference(comp), 256, np.random.SeedSequence(0, spawn_key=(4, 0)))
    assert eps <= 1.01 * float(d["eps_a"]) + 1e-12, (eps, float(d["eps_a"]))


@pytest.mark.gpu
def test_matvec_vs_oracle_cfg0_geometry():
    """Larger geometry (n=1024, leaf 8, r=12): GPU matvec chain vs the oracle's."""
    n, leaf, r = 1024, 8, 12
    p = bf.make_partition(n, leaf)
    mat = oent.EntryOracle("fio", n).block(np.arange(n), np.arange(n))
    f = bf.factorize(bf.DenseOracle(mat), p, r, seed=2, mode="matvec")
    c = ocons.factorize(oops.DenseOperator(mat), n, p.levels, r, seed=2, mode="matvec")
    rng = np.random.default_rng(3)
    g = complex_gaussian(rng, (n, 2))
    want = ochain.apply(c, g)
    env = _envelope(oops.DenseOperator(mat), n, p.levels, r, 2, g, want)
    assert rel(f.apply(g), want) <= 10 * max(env, 1e-13), (rel(f.apply(g), want), env)
    exact = mat @ g
    assert rel(f.apply(g), exact) <= 1.01 * rel(want, exact) + 1e-13


@pytest.mark.gpu
def test_matvec_identity_operator(rng):
    """reference test_construct.py:71-84: identity at full middle-block rank, p = 0."""
    n = 64
    p = bf.make_partition(n, 1)
    r = p.mid_side
    u_h, mid, v_h = bf.middle_factorization_matvec(bf.DenseOracle(np.eye(n, dtype=complex)), p, r,
                                                   bf.OversamplingParams(p=0), seed=3)
    m, side = p.mid_nodes, p.mid_side
    blocks = _block_products(u_h.blocks, mid.weights, v_h.blocks, m, side, r)
    approx = blocks.transpose(0, 2, 1, 3).reshape(n, n)
    for _ in range(16):
        g = complex_gaussian(rng, n)
        assert np.linalg.norm(approx @ g - g) <= 1e-10 * np.linalg.norm(g)


@pytest.mark.gpu
def test_matvec_fio_accuracy_leaf025():
    """reference test_construct.py:87-93: n=64 leaf 0.25 r=4, ||K - triple|| <= 1e-3 ||K||."""
    n = 64
    p = bf.make_partition(n, 0.25)
    k = oent.EntryOracle("fio", n).block(np.arange(n), np.arange(n))
    u_h, mid, v_h = bf.middle_factorization_matvec(bf.DenseOracle(k), p, 4, seed=1)
    m, side = p.mid_nodes, p.mid_side
    tri = _block_products(u_h.blocks, mid.weights, v_h.blocks, m, side, 4).transpose(0, 2, 1, 3).reshape(n, n)
    assert np.linalg.norm(k - tri) / np.linalg.norm(k) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("r,bound", [(4, 1e-1), (8, 1e-3), (12, 1e-6)])
def test_composition_accuracy_criterion3(r, bound):
    """reference test_acceptance.py:75-96 (criterion 3), all on the GPU: inner chain by
    sampling, K F K as the operator oracle, matvec construction, eps_a vs the composed operator."""
    n = 1024
    p = bf.make_partition(n, 0.25)
    inner = bf.factorize(bf.FioKernel(n), p, r, seed=7)
    comp = bf.ComposedOperator(inner)
    f = bf.factorize(comp, p, r, seed=0, mode="matvec")
    eps = bf.estimate_eps_a(f, bf.OperatorReference(comp), 256, np.random.SeedSequence(0, spawn_key=(4, 0)))
    assert eps <= bound, eps


@pytest.mark.gpu
def test_matvec_errors():
    n = 64
    p = bf.make_partition(n, 1)
    with pytest.raises(ValueError):
        bf.factorize(bf.FioKernel(n), p, 2, seed=0, mode="matvec")

    class OpOnly:
        shape = (n, n)

        def apply(self, x):
            return x

        def apply_adjoint(self, x):
            return x

    with pytest.raises(ValueError):
        bf.factorize(OpOnly(), p, 2, seed=0, mode="sampling")
    with pytest.raises(ValueError):
        bf.factorize(bf.FioKernel(n), p, 2, seed=0, mode="nonsense")

    class Broken(OpOnly):
        def apply(self, x):
            raise RuntimeError("boom")

    with pytest.raises(bf.OracleError):
        bf.factorize(Broken(), p, 2, seed=0, mode="matvec")
    # the identity operator through the full chain is reproduced at full middle rank
    f = bf.factorize(OpOnly(), p, p.mid_side, bf.OversamplingParams(p=0), seed=1, mode="matvec")
    g = complex_gaussian(np.random.default_rng(1), n)
    assert rel(f.apply(g), g) <= 1e-10
