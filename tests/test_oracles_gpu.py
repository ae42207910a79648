"""Entry-oracle plugin paths of the device construction:

* the reference's centered DftKernel (kernels.py:87-97) as a device kernel id
  (BF_KERNEL_DFT): entries against the reference's own values, its construction's eps_a
  against the reference's at the same rank, and the reference class recognised by name;
* any other entry oracle through per-middle-block windows (BF_KERNEL_TILES, the BlockView
  protocol, oracles.py:57-68): bitwise the same factors as the kernel-id path when the
  windows hold the same entries, in batches bounded by TILE_BUDGET;
* an uncached Hankel kernel through device-evaluated windows instead of the n x n table.
"""

import numpy as np
import pytest

import paper_1502_01379_b200 as bf
from conftest import golden
from oracle import entries as oent
from paper_1502_01379_b200 import _lib
from paper_1502_01379_b200 import construct as bc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _same(a, b):
    pairs = [(a.u_outer.blocks, b.u_outer.blocks), (a.v_outer.blocks, b.v_outer.blocks),
             (a.middle.weights, b.middle.weights)]
    pairs += [(x.blocks, y.blocks) for x, y in zip(a.g_chain, b.g_chain)]
    pairs += [(x.blocks, y.blocks) for x, y in zip(a.h_chain, b.h_chain)]
    return all(torch.equal(torch.as_tensor(x).cpu(), torch.as_tensor(y).cpu()) for x, y in pairs)


def test_dft_entries_vs_reference():
    d = golden("dft_entries.npz")
    for n in (1024, 1 << 16, 1 << 20):
        got = bf.DftKernel(n).block(d[f"dft_{n}_rows"], d[f"dft_{n}_cols"])
        err = np.abs(got - d[f"dft_{n}"])
        print(f"\nDftKernel n={n}: max |gpu - reference| {err.max():.2e}")
        # the angle is rounded as NumPy rounds it; only the final sin/cos may differ by an ulp
        assert err.max() <= 4.5e-16


class DftKernel:
    """Stand-in with the reference class's name and attributes (no kernel_id): the device
    path recognises it like the reference's own DftKernel."""

    def __init__(self, n):
        self.n, self.shape = n, (n, n)

    def block(self, rows, cols):
        return oent.dft_block(self.n, rows, cols)


def test_dft_construction_eps_vs_reference():
    d = golden("eps_dft_n1024_r8_leaf1.npz")
    n, levels, r, seed = int(d["n"]), int(d["levels"]), int(d["rank"]), int(d["seed"])
    p = bf.DyadicPartition(n, levels)
    f = bf.factorize(bf.DftKernel(n), p, r, seed=seed)
    eps = bf.estimate_eps_a(f, bf.RowSampledReference(bf.DftKernel(n)), 256,
                            np.random.SeedSequence(seed, spawn_key=(4, 0)))
    print(f"\nDftKernel N={n} r={r}: eps_a gpu {eps:.3e} reference {float(d['eps_a']):.3e}")
    assert eps <= float(d["eps_a"]) * 1.5
    assert _same(f, bf.factorize(DftKernel(n), p, r, seed=seed))     # reference class by name


class BlockOnly:
    """A generic entry oracle: .shape and .block only (oracles.py:5-10)."""

    def __init__(self, inner):
        self.inner, self.shape = inner, inner.shape
        self.calls = 0

    def block(self, rows, cols):
        self.calls += 1
        return self.inner.block(rows, cols)


@pytest.mark.parametrize("n,leaf,r", [(4096, 4, 8), (1024, 1, 12)])
def test_generic_oracle_tiles_bitwise(n, leaf, r, monkeypatch):
    p = bf.make_partition(n, leaf)
    side = p.mid_side
    monkeypatch.setattr(bc, "TILE_BUDGET", 16 * side * side * 5)      # 5 windows per launch
    ora = BlockOnly(bf.FioKernel(n))
    assert bc._DeviceOracle(ora, n).kernel_id == _lib.BF_KERNEL_TILES
    got = bf.factorize(ora, p, r, seed=2)
    want = bf.factorize(bf.FioKernel(n), p, r, seed=2)
    assert ora.calls == p.mid_nodes ** 2                                   # one window per block
    assert _same(got, want)


def test_generic_oracle_failure_is_oracle_error():
    class Failing:
        shape = (1024, 1024)

        def block(self, rows, cols):
            raise KeyError("boom")

    with pytest.raises(bf.OracleError):
        bf.factorize(Failing(), bf.make_partition(1024, 8), 4)


def test_hankel_uncached_windows(monkeypatch):
    """Above TABLE_CAP (or cache=False) the Hankel kernel is read through device windows
    (one order sweep per block, as the reference's uncached block(), kernels.py:63-66):
    no n x n table, and the factors are as accurate as the cached path's."""
    n, leaf, r = 1024, 1, 8
    p = bf.make_partition(n, leaf)
    monkeypatch.setattr(bf.HankelKernel, "TABLE_CAP", 512)
    big = bf.HankelKernel(n)
    dev = bc._DeviceOracle(big, n)
    assert dev.kernel_id == _lib.BF_KERNEL_TILES and dev.dense is None and big._table is None
    f_unc = bf.factorize(big, p, r, seed=0)
    monkeypatch.setattr(bf.HankelKernel, "TABLE_CAP", 1 << 15)
    cached = bf.HankelKernel(n)
    f_c = bf.factorize(cached, p, r, seed=0)
    ref = bf.RowSampledReference(cached)
    ss = np.random.SeedSequence(0, spawn_key=(4, 0))
    e_unc = bf.estimate_eps_a(f_unc, ref, 256, ss)
    e_c = bf.estimate_eps_a(f_c, ref, 256, ss)
    print(f"\nHankel n={n}: eps_a uncached windows {e_unc:.3e}, cached table {e_c:.3e}")
    assert e_unc <= 2 * e_c + 1e-12
