"""Pin the CPU oracle (oracle/) to fixtures produced by the reference itself
(oracle/gen_golden.py) and to the reference's own known-answer tests."""

import numpy as np
import pytest

from conftest import chain_from_golden, golden
from oracle import chain as ochain
from oracle import construct as ocons
from oracle import entries as oent
from oracle import lowrank as olr
from oracle import partition as opart

APPLY_CASES = ["apply_fio_n256_r8_leaf025.npz", "apply_cfg0_fio_n1024_r12_leaf8.npz",
               "apply_dftp_n1024_r8_leaf16.npz"]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", APPLY_CASES)
def test_oracle_apply_matches_reference(name):
    d = golden(name)
    c = chain_from_golden(d)
    assert rel(ochain.apply(c, d["g"]), d["fwd"]) <= 1e-15
    assert rel(ochain.apply(c, d["g"], adjoint=True), d["adj"]) <= 1e-15
    out1 = ochain.apply(c, d["g"][:, 0])
    assert out1.ndim == 1 and rel(out1, d["fwd1"]) <= 1e-15


def test_oracle_apply_zero_and_bad_length():
    c = chain_from_golden(golden(APPLY_CASES[0]))
    assert np.array_equal(ochain.apply(c, np.zeros(c.n, complex)), np.zeros(c.n, complex))
    with pytest.raises(ValueError):
        ochain.apply(c, np.zeros(c.n // 2))


def test_geometry_matches_reference():
    d = golden("geometry.npz")
    for n, leaf in ((1024, 8), (1 << 16, 16), (1 << 20, 16), (256, 0.25), (64, 1), (1024, 1), (128, 0.25)):
        tag = f"{n}_{leaf}"
        levels = opart.choose_levels(n, leaf)
        assert levels == int(d[f"levels_{tag}"])
        for lvl, i, lo, hi in d[f"ranges_{tag}"]:
            rg = opart.node_range(n, levels, int(lvl), int(i))
            assert (rg.start, rg.stop) == (lo, hi)
        shapes, leaf_shape = opart.level_geometry(n, levels, 4)
        want = d[f"shapes_{tag}"]
        assert len(shapes) == len(want)
        for (lvl, sp, s), row in zip(shapes, want):
            assert lvl == row[0] and int(sp) == row[1] and tuple(s) == tuple(x for x in row[2:2 + len(s)])
        assert tuple(leaf_shape) == tuple(d[f"leaf_{tag}"])


def test_partition_errors():
    with pytest.raises(ValueError):
        opart.choose_levels(1000, 1)
    with pytest.raises(ValueError):
        opart.choose_levels(64, 0)
    with pytest.raises(ValueError):
        opart.check_partition(64, 3)


def test_entries_match_reference():
    d = golden("entries.npz")
    for n in (1024, 1 << 16, 1 << 20, 1 << 24):
        got = oent.fio_block(n, d[f"fio_{n}_rows"], d[f"fio_{n}_cols"])
        assert np.array_equal(got, d[f"fio_{n}"])      # bitwise: same expression order
    got = oent.dftp_block(1 << 16, d["dftp_rows"], d["dftp_cols"])
    assert np.array_equal(got, d["dftp"])
    # reference KAT, pkg/tests/test_kernels.py:13-17
    assert abs(oent.fio_block(4, [0], [2])[0, 0] - 1.0) <= 1e-15
    assert abs(oent.fio_block(4, [0], [0])[0, 0] + 1.0) <= 1e-14
    assert np.array_equal(d["fio_hand"], [oent.fio_block(4, [0], [2])[0, 0], oent.fio_block(4, [0], [0])[0, 0]])


def test_pivots_match_reference():
    d = golden("pivots.npz")
    for tag in ("gauss", "dups", "rank1", "zero", "fio"):
        got = olr.greedy_pivots(d[f"{tag}_a"], int(d[f"{tag}_k"]), float(d[f"{tag}_tol"]))
        assert got == list(d[f"{tag}_piv"]), tag


@pytest.mark.parametrize("name", ["construct_fio_n128_r4_leaf025.npz", "construct_fio_n1024_r12_leaf8.npz",
                                  "construct_fio_n1024_r8_leaf1.npz"])
def test_oracle_middle_blocks_bitwise(name):
    d = golden(name)
    n, levels, r, seed = int(d["n"]), int(d["levels"]), int(d["rank"]), int(d["seed"])
    ent = oent.EntryOracle("fio", n)
    keys = sorted({k.rsplit("_", 1)[0] for k in d if k.startswith("blk_")})
    assert keys
    for key in keys:
        _, i, j = key.split("_")
        t = ocons.sample_block(ent, n, levels, r, olr.Params(), seed, int(i), int(j))
        assert np.array_equal(t.u0, d[key + "_u0"])
        assert np.array_equal(t.sigma0, d[key + "_s0"])
        assert np.array_equal(t.v0, d[key + "_v0"])


def test_oracle_factorize_bitwise_small():
    d = golden("construct_fio_n128_r4_leaf025.npz")
    n, levels, r, seed = int(d["n"]), int(d["levels"]), int(d["rank"]), int(d["seed"])
    c = ocons.factorize(oent.EntryOracle("fio", n), n, levels, r, seed=seed)
    want = chain_from_golden(d)
    assert np.array_equal(c.u_leaf, want.u_leaf) and np.array_equal(c.v_leaf, want.v_leaf)
    assert np.array_equal(c.weights, want.weights)
    for (la, a), (lb, b) in zip(c.g_levels + c.h_levels, want.g_levels + want.h_levels):
        assert la == lb and np.array_equal(a, b)
    assert np.array_equal(ochain.apply(c, d["g"]), d["fwd"])


@pytest.mark.slow
def test_oracle_factorize_operator_cfg0():
    d = golden("construct_fio_n1024_r12_leaf8.npz")
    n, levels, r, seed = int(d["n"]), int(d["levels"]), int(d["rank"]), int(d["seed"])
    c = ocons.factorize(oent.EntryOracle("fio", n), n, levels, r, seed=seed)
    assert np.array_equal(c.weights, d["weights"])
    assert rel(ochain.apply(c, d["g"]), d["fwd"]) <= 1e-13


@pytest.mark.parametrize("name,count", [
    ("trace_cfg0_fio_n1024_r12_leaf8.npz", 64),
    ("trace_fio_n4096_r8_leaf4.npz", 8),
    ("trace_cfg1_dftp_n65536_r8_leaf16.npz", 4),
    ("trace_cfg2_fio_n1048576_r16_leaf16.npz", 2),
])
def test_oracle_blocks_bitwise_at_config_geometry(name, count):
    """The oracle's sample_block reproduces the reference's traced middle blocks at the
    configs' own geometry bit for bit: signature u0 diag(s0) v0^H X, singular values,
    final skeleton sets and basis pivots."""
    from threadpoolctl import threadpool_limits
    d = golden(name)
    n, levels, r, seed = int(d["n"]), int(d["levels"]), int(d["rank"]), int(d["seed"])
    ent = oent.EntryOracle("dftp" if "dftp" in name else "fio", n)
    x = d["probe"]
    # the fixtures were made with one BLAS thread: LAPACK's SVDs are not bitwise
    # reproducible across thread counts (1e-14 differences at 2 vs 8 threads)
    with threadpool_limits(1):
        _check_blocks(d, ent, n, levels, r, seed, x, count)


def _check_blocks(d, ent, n, levels, r, seed, x, count):
    for b in d["blocks"][:count]:
        i, j = int(b[0]), int(b[1])
        key = f"b{i}_{j}"
        tr = {}
        t = ocons.sample_block(ent, n, levels, r, olr.Params(), seed, i, j, trace=tr)
        sig = t.u0 @ (t.sigma0[:, None] * (t.v0.conj().T @ x))
        assert np.array_equal(sig, d[key + "_sig"]), key
        assert np.array_equal(t.sigma0, d[key + "_s0"]), key
        if key + "_skc" in d:
            assert tr["sk_col"][-1].tolist() == d[key + "_skc"].tolist()
            assert tr["sk_row"][-1].tolist() == d[key + "_skr"].tolist()


def test_oracle_recurse_cfg2_slab_bitwise():
    """oracle recurse == reference _recurse on a seeded cfg2-geometry slab (1, 4096, 256, 16)."""
    from threadpoolctl import threadpool_limits
    d = golden("slab_cfg2_n1048576_r16_leaf16.npz")
    n, levels, r, seed = int(d["n"]), int(d["levels"]), int(d["rank"]), int(d["seed"])
    m = 2 ** (levels // 2)
    slab = ocons.synthetic_slab(n // m, m, r, seed)
    with threadpool_limits(1):
        leaf, pieces = ocons.recurse(slab, n, levels, r)
    assert np.array_equal(ocons.slab_chain_apply(leaf, pieces, d["probe"]), d["sig"])


def test_dft_entries_match_reference():
    """The reference's centered DftKernel (kernels.py:87-97), restated bitwise."""
    d = golden("dft_entries.npz")
    for n in (1024, 1 << 16, 1 << 20):
        got = oent.dft_block(n, d[f"dft_{n}_rows"], d[f"dft_{n}_cols"])
        assert np.array_equal(got, d[f"dft_{n}"])
