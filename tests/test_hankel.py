"""Hankel kernel K[i, j] = H1_j(x_i) (reference kernels.py:45-84, bessel.py;
SURVEY.md §8(f) rank 4): the oracle restatement pinned bitwise to the
reference's outputs (tests/golden/hankel.npz) and to independent values (the
reference's frozen mpmath KAT, scipy.special); the device sweeps
(bf_hankel_orders) against the oracle; the construction accuracy criterion 2
on the GPU."""

import numpy as np
import pytest
import scipy.special

from conftest import golden
from oracle import bessel as ob

# reference test_bessel.py:9 (mpmath at 30 digits)
H1_0_AT_4 = -0.397149809863847372286590768452 - 0.0169407393250649919036351344472j


def test_oracle_seeds_bitwise_reference():
    d = golden("hankel.npz")
    x = d["seed_x"]
    for name, fn in (("j0", ob.j0), ("j1", ob.j1), ("y0", ob.y0), ("y1", ob.y1)):
        assert np.array_equal(fn(x), d[name]), name


def test_oracle_sweep_and_table_bitwise_reference():
    d = golden("hankel.npz")
    assert np.array_equal(ob.hankel1_orders(d["sweep_x"], d["sweep"].shape[1] - 1), d["sweep"])
    n = int(d["table_n"])
    assert np.array_equal(ob.hankel_table(n)[d["table_rows"]], d["table"])


def test_oracle_independent_values():
    assert abs(ob.hankel1_orders(np.array([4.0]), 0)[0, 0] - H1_0_AT_4) <= 1e-10
    big = abs(ob.hankel1_orders(np.array([1e4]), 0)[0, 0])
    assert abs(big - np.sqrt(2.0 / (np.pi * 1e4))) / np.sqrt(2.0 / (np.pi * 1e4)) <= 1e-4
    n = 256
    x = n + (2 * np.pi / 3) * np.arange(0, n, 37, dtype=float)
    got = ob.hankel1_orders(x, n - 1)
    m = np.arange(n)
    want = scipy.special.jv(m[None, :], x[:, None]) + 1j * scipy.special.yv(m[None, :], x[:, None])
    assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-10
    want5 = scipy.special.hankel1(5, 64 + (2 * np.pi / 3) * 3)
    assert abs(ob.hankel1_orders(np.array([64 + (2 * np.pi / 3) * 3]), 5)[0, 5] - want5) <= 1e-12 * abs(want5)


def test_oracle_wronskian():
    rng = np.random.default_rng(5)
    n = 1024
    xs = np.unique(n + (2 * np.pi / 3) * rng.integers(0, n, size=100))
    js, ys = ob.jy_orders(xs, n - 1)
    m = rng.integers(0, n - 1, size=xs.size)
    w = js[np.arange(xs.size), m + 1] * ys[np.arange(xs.size), m] - js[np.arange(xs.size), m] * ys[np.arange(xs.size), m + 1]
    assert np.all(np.abs(w - 2.0 / (np.pi * xs)) <= 1e-10 * 2.0 / (np.pi * xs))


def test_oracle_rejects_nonpositive():
    with pytest.raises(ValueError):
        ob.jy_orders(np.array([0.0]), 3)


# ---------------------------------------------------------------- device
@pytest.mark.gpu
def test_device_sweep_vs_oracle():
    import paper_1502_01379_b200 as bf
    for n, x in ((256, 256 + (2 * np.pi / 3) * np.arange(0, 256, 37, dtype=float)),
                 (1024, 1024 + (2 * np.pi / 3) * np.arange(0, 1024, 5, dtype=float)),
                 (8, np.array([0.5, 4.0, 4.9999, 5.0, 5.5, 30.0]))):
        got = bf.hankel1_orders_device(x, n - 1).cpu().numpy()
        want = ob.hankel1_orders(x, n - 1)
        # J never touches sin/cos/log (same start, same IEEE ops): bitwise
        assert np.array_equal(got.real, want.real), n
        # Y grows from the order-0/1 seeds, whose sin/cos/log may differ by an ulp; the
        # recurrence carries that as an absolute error on the scale of |H1| (relative to
        # Y itself it is unbounded near Y's zeros)
        rel = np.abs(got.imag - want.imag) / np.abs(want)
        assert rel.max() <= 1e-13, (n, rel.max())


@pytest.mark.gpu
def test_device_table_vs_reference_rows():
    import paper_1502_01379_b200 as bf
    d = golden("hankel.npz")
    n = int(d["table_n"])
    ker = bf.HankelKernel(n)
    got = ker.block(d["table_rows"], np.arange(n))
    assert np.array_equal(got.real, d["table"].real)
    assert np.max(np.abs(got.imag - d["table"].imag) / np.abs(d["table"])) <= 1e-13
    # uncached path: own sweep per call (reference test_kernels.py:50-53)
    a = bf.HankelKernel(64, cache=True).block([3, 10], [0, 5, 63])
    b = bf.HankelKernel(64, cache=False).block([3, 10], [0, 5, 63])
    assert np.allclose(a, b, rtol=1e-12)
    want = scipy.special.hankel1(5, 64 + (2 * np.pi / 3) * 3)
    assert abs(bf.hankel_entry(64, 3, 5) - want) <= 1e-12 * abs(want)
    with pytest.raises(ValueError):
        bf.hankel1_orders_device(np.array([1.0, -2.0]), 3)


@pytest.mark.gpu
@pytest.mark.parametrize("r,bound", [(4, 1e-4), (6, 1e-6)])
def test_hankel_construction_criterion2(r, bound):
    """reference test_acceptance.py:60-73 on the GPU: n=1024 leaf 0.25, sampling mode,
    eps_a <= bound and within 10% of the reference's own eps_a (golden)."""
    import paper_1502_01379_b200 as bf
    d = golden("hankel.npz")
    n = 1024
    ker = bf.HankelKernel(n)
    p = bf.make_partition(n, 0.25)
    f = bf.factorize(ker, p, r, seed=0, mode="sampling")
    eps = bf.estimate_eps_a(f, bf.RowSampledReference(ker), 256, np.random.SeedSequence(0, spawn_key=(4, 0)))
    assert eps <= bound, eps
    assert eps <= 1.1 * float(d[f"eps_r{r}"]) + 1e-13, (eps, float(d[f"eps_r{r}"]))
