"""The row tables of the entry evaluator (bf_entry_table): the FIO phase speed
c(x_i) = (2 + sin 2 pi x_i)/8 and the 2-D Radon sin/cos of 2 pi a/n_side, built with a
correctly rounded double-double sine (csrc/crmath.cuh), are bitwise the reference's
NumPy values — exhaustively for every x_i = i/2^24 (which contains every power-of-two
N <= 2^24: fl(2 pi i/2^k) is an exact power-of-two scaling of fl(2 pi i 2^(24-k)))."""

import ctypes

import numpy as np
import pytest

from paper_1502_01379_b200 import _lib

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def table(kind, n, length):
    out = torch.empty(length, dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().bf_entry_table(kind, n, ctypes.c_void_p(out.data_ptr()), length, None), "bf_entry_table")
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("n", [1 << 24, 1000, 3 << 10, 1 << 20])
def test_fio_speed_table_bitwise(n):
    x = np.arange(n, dtype=float)[:, None] / n          # kernels.py:35
    want = ((2.0 + np.sin(2.0 * np.pi * x)) / 8.0)[:, 0]  # kernels.py:23-24
    got = table(_lib.BF_KERNEL_FIO, n, n)
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (bad.size, bad[:8])


@pytest.mark.parametrize("n_side", [1024, 256, 4096])
def test_radon_table_bitwise(n_side):
    x = np.arange(n_side, dtype=np.float64) / n_side
    t = 2.0 * np.pi * x
    got = table(_lib.BF_KERNEL_RADON2D, n_side * n_side, 2 * n_side)
    assert np.array_equal(got[:n_side], np.sin(t)) and np.array_equal(got[n_side:], np.cos(t))


def test_table_errors():
    lib = _lib.load()
    out = torch.empty(4, dtype=torch.float64, device="cuda")
    assert lib.bf_entry_table(_lib.BF_KERNEL_FIO, 16, ctypes.c_void_p(out.data_ptr()), 4, None) == _lib.BF_EINVAL
