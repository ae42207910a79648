"""The row tables of the entry evaluator (bf_entry_table): the FIO phase speed
c(x_i) = (2 + sin 2 pi x_i)/8 and the 2-D Radon sin/cos of 2 pi a/n_side, built with a
double-double sine rounded once (csrc/crmath.cuh).

The device values are the correctly rounded sines (checked against mpmath at 200 bits).
The reference's np.sin (glibc, <= 0.502 ulp) is not correctly rounded at ~0.03% of the
points x_i = i/2^24 (35 of 20,000 sampled here), so the tables equal NumPy's values
except at those points, where they differ by one ulp in NumPy's disfavour. Every
power-of-two N <= 2^24 is covered by the N = 2^24 sweep: fl(2 pi i/2^k) is an exact
power-of-two scaling of fl(2 pi i 2^(24-k))."""

import ctypes

import numpy as np
import pytest

from paper_1502_01379_b200 import _lib

torch = pytest.importorskip("torch")
mpmath = pytest.importorskip("mpmath")
pytestmark = pytest.mark.gpu


def table(kind, n, length):
    out = torch.empty(length, dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().bf_entry_table(kind, n, ctypes.c_void_p(out.data_ptr()), length, None), "bf_entry_table")
    torch.cuda.synchronize()
    return out.cpu().numpy()


def cr(fn, t):
    """Correctly rounded fn(t) (mpmath, 200-bit)."""
    with mpmath.workprec(200):
        return float(fn(mpmath.mpf(float(t))))


@pytest.mark.parametrize("n", [1 << 24, 1000, 3 << 10])
def test_fio_speed_table(n):
    x = np.arange(n, dtype=float)[:, None] / n          # kernels.py:35
    t = (2.0 * np.pi * x)[:, 0]
    want = ((2.0 + np.sin(2.0 * np.pi * x)) / 8.0)[:, 0]  # kernels.py:23-24
    got = table(_lib.BF_KERNEL_FIO, n, n)
    bad = np.flatnonzero(got != want)
    print(f"\nn={n}: table != NumPy at {bad.size} of {n} points")
    assert bad.size <= max(2, 0.001 * n)
    # where they differ, the table holds (2 + CR sin)/8 and NumPy's sine is the one off
    for i in bad[:200]:
        s_cr = cr(mpmath.sin, t[i])
        assert s_cr != float(np.sin(t[i]))
        assert got[i] == (2.0 + s_cr) / 8.0
    # and a sample of the agreeing points is correctly rounded too
    rng = np.random.default_rng(n)
    for i in rng.choice(n, 300, replace=False):
        assert got[i] == (2.0 + cr(mpmath.sin, t[i])) / 8.0


@pytest.mark.parametrize("n_side", [1024, 256])
def test_radon_table(n_side):
    x = np.arange(n_side, dtype=np.float64) / n_side
    t = 2.0 * np.pi * x
    got = table(_lib.BF_KERNEL_RADON2D, n_side * n_side, 2 * n_side)
    for a in range(n_side):
        assert got[a] == cr(mpmath.sin, t[a]) and got[n_side + a] == cr(mpmath.cos, t[a])
    assert np.mean(got[:n_side] == np.sin(t)) >= 0.99 and np.mean(got[n_side:] == np.cos(t)) >= 0.99


def test_table_errors():
    lib = _lib.load()
    out = torch.empty(4, dtype=torch.float64, device="cuda")
    assert lib.bf_entry_table(_lib.BF_KERNEL_FIO, 16, ctypes.c_void_p(out.data_ptr()), 4, None) == _lib.BF_EINVAL
