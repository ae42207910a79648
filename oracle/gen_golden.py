"""Generate tests/golden/*.npz by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py

The fixtures pin both the CPU oracle (tests/test_oracle_golden.py) and the
CUDA path (tests/test_apply_gpu.py, tests/test_construct_gpu.py) to the
reference's own outputs on seeded inputs. Nothing at test time reads
/root/reference; only this script does.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle.construct import slab_chain_apply, synthetic_slab  # noqa: E402
from oracle.entries import NoisyOracle  # noqa: E402
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    sys.path.insert(0, REF)
    import butterfly  # noqa: F401  (the reference package)
    return butterfly


class DftPlus:
    """Config-1 entry oracle exp(+2 pi i jk/n) handed to the reference factorize."""

    def __init__(self, n):
        self.n, self.shape = n, (n, n)

    def block(self, rows, cols):
        j = np.asarray(rows, dtype=np.int64)[:, None]
        k = np.asarray(cols, dtype=np.int64)[None, :]
        return np.exp(2j * np.pi * (((j * k) % self.n).astype(np.float64) / self.n))


def _chain_arrays(f, prefix=""):
    d = {prefix + "n": f.n, prefix + "levels": f.partition.levels, prefix + "rank": f.rank,
         prefix + "u_leaf": f.u_outer.blocks, prefix + "v_leaf": f.v_outer.blocks,
         prefix + "weights": f.middle.weights,
         prefix + "g_lvls": np.array([tf.level for tf in f.g_chain]),
         prefix + "h_lvls": np.array([tf.level for tf in f.h_chain])}
    for tf in f.g_chain:
        d[f"{prefix}g_{tf.level}"] = tf.blocks
    for tf in f.h_chain:
        d[f"{prefix}h_{tf.level}"] = tf.blocks
    return d


def gen_apply(bf, name, oracle, n, leaf, r, seed, k):
    p = bf.make_partition(n, leaf)
    f = bf.factorize(oracle, p, r, seed=seed)
    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(4, 0)))
    g = bf.lowrank.complex_normal(rng, (n, k))
    d = _chain_arrays(f)
    d.update(g=g, fwd=f.apply(g), adj=f.apply_adjoint(g), fwd1=f.apply(g[:, 0]))
    # eps_a as the reference bench computes it (bench.py:90-97, 208-211)
    eps_rng = np.random.SeedSequence(seed, spawn_key=(4, 0))
    d["eps_a"] = bf.bench.estimate_eps_a(f, bf.bench.RowSampledReference(oracle), 256, eps_rng)
    np.savez_compressed(os.path.join(OUT, name), **d)
    print(name, "levels", p.levels, "nnz", f.nnz_report().total, "eps_a", d["eps_a"])


def gen_construct(bf, name, oracle, n, leaf, r, seed, blocks):
    """Full factorize output plus per-block stage traces of the middle level."""
    from butterfly.construct import _sample_block  # reference internals, traced below
    p = bf.make_partition(n, leaf)
    f = bf.factorize(oracle, p, r, seed=seed)
    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(4, 0)))
    g = bf.lowrank.complex_normal(rng, (n, 2))
    d = {"n": n, "levels": p.levels, "rank": r, "seed": seed, "g": g,
         "fwd": f.apply(g), "adj": f.apply_adjoint(g), "weights": f.middle.weights}
    if n <= 128:   # small enough to keep every factor and the middle-level triple
        d.update(_chain_arrays(f))
        u_h, mid, v_h = bf.middle_factorization_sampling(oracle, p, r, seed=seed)
        d.update(u_h=u_h.blocks, v_h=v_h.blocks, w_h=mid.weights)
    for (i, j) in blocks:
        apx = _sample_block(oracle, p, r, bf.lowrank.DEFAULT_PARAMS, seed, i, j)
        d[f"blk_{i}_{j}_u0"], d[f"blk_{i}_{j}_s0"], d[f"blk_{i}_{j}_v0"] = apx.u0, apx.sigma0, apx.v0
    np.savez_compressed(os.path.join(OUT, name), **d)
    print(name, "levels", p.levels)


def gen_pivots(bf):
    rng = np.random.default_rng(20240801)
    d = {}
    cases = []
    a = rng.standard_normal((12, 40)) + 1j * rng.standard_normal((12, 40))
    cases.append(("gauss", a, 8, 0.0))
    b = np.repeat(a[:, :5], 4, axis=1)               # exact duplicate columns: tie rule
    cases.append(("dups", b, 5, 0.0))
    c = np.outer(a[:, 0], a[0, :]) + 1e-13 * a       # rank-1 plus noise: early stop with rel_tol
    cases.append(("rank1", c, 6, 1e-11))
    z = np.zeros((6, 9), dtype=complex)
    cases.append(("zero", z, 3, 0.0))
    ker = bf.FioKernel(4096)
    e = ker.block(np.arange(0, 4096, 97)[:48], np.arange(1024, 2048))
    cases.append(("fio", e, 16, 0.0))
    for tag, mat, k, tol in cases:
        d[f"{tag}_a"] = mat
        d[f"{tag}_k"] = k
        d[f"{tag}_tol"] = tol
        d[f"{tag}_piv"] = np.array(bf.lowrank.select_pivot_columns(mat, k, tol), dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "pivots.npz"), **d)
    print("pivots.npz")


def gen_entries(bf):
    rng = np.random.default_rng(7)
    d = {}
    for n in (1024, 1 << 16, 1 << 20, 1 << 24):
        rows = np.sort(rng.choice(n, size=64, replace=False))
        cols = np.sort(rng.choice(n, size=64, replace=False))
        d[f"fio_{n}_rows"], d[f"fio_{n}_cols"] = rows, cols
        d[f"fio_{n}"] = bf.FioKernel(n).block(rows, cols)
    d["fio_hand"] = np.array([bf.fio_entry(4, 0, 2), bf.fio_entry(4, 0, 0)])
    n = 1 << 16
    rows = np.sort(rng.choice(n, size=64, replace=False))
    cols = np.sort(rng.choice(n, size=64, replace=False))
    d["dftp_rows"], d["dftp_cols"], d["dftp"] = rows, cols, DftPlus(n).block(rows, cols)
    np.savez_compressed(os.path.join(OUT, "entries.npz"), **d)
    print("entries.npz")


def gen_dft(bf):
    """The reference's centered DftKernel (kernels.py:87-97): entries, and eps_a of its own
    sampling factorization at N=1024 leaf 1 r=8 (bench.py:84-97)."""
    from butterfly.kernels import DftKernel
    rng = np.random.default_rng(11)
    d = {}
    for n in (1024, 1 << 16, 1 << 20):
        rows = np.sort(rng.choice(n, size=64, replace=False))
        cols = np.sort(rng.choice(n, size=64, replace=False))
        d[f"dft_{n}_rows"], d[f"dft_{n}_cols"] = rows, cols
        d[f"dft_{n}"] = DftKernel(n).block(rows, cols)
    np.savez_compressed(os.path.join(OUT, "dft_entries.npz"), **d)
    gen_eps(bf, "eps_dft_n1024_r8_leaf1.npz", DftKernel(1024), 1024, 1, 8, 0)
    print("dft_entries.npz")


def gen_geometry(bf):
    from butterfly.construct import _level_geometry
    d = {}
    for n, leaf in ((1024, 8), (1 << 16, 16), (1 << 20, 16), (256, 0.25), (64, 1), (1024, 1), (128, 0.25)):
        p = bf.make_partition(n, leaf)
        tag = f"{n}_{leaf}"
        d[f"levels_{tag}"] = p.levels
        ranges = []
        for lvl in range(p.levels + 1):
            for i in range(min(2 ** lvl, 4096)):
                rg = p.node_range(lvl, i)
                ranges.append((lvl, i, rg.start, rg.stop))
        d[f"ranges_{tag}"] = np.array(ranges, dtype=np.int64)
        shapes, leaf_shape = _level_geometry(p, 4)
        d[f"shapes_{tag}"] = np.array([(lvl, int(sp), *(list(s) + [0] * (5 - len(s))))
                                      for lvl, sp, s in shapes], dtype=np.int64)
        d[f"leaf_{tag}"] = np.array(leaf_shape, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "geometry.npz"), **d)
    print("geometry.npz")


def gen_bfac(bf):
    """A .bfac file and a vector file written by the reference's storage.py."""
    p = bf.make_partition(128, 0.25)
    f = bf.factorize(bf.FioKernel(128), p, 4, seed=9)
    bf.save_factors(f, os.path.join(OUT, "fio_n128_r4_leaf025.bfac"))
    g = bf.lowrank.complex_normal(np.random.default_rng(3), (128,))
    bf.write_vector(os.path.join(OUT, "g128.vec"), g)
    bf.write_vector(os.path.join(OUT, "u128.vec"), f.apply(g))
    p = bf.make_partition(1024, 16)
    f = bf.factorize(bf.FioKernel(1024), p, 8, seed=2)
    bf.save_factors(f, os.path.join(OUT, "fio_n1024_r8_leaf16.bfac"))
    print("bfac fixtures")


def gen_matvec(bf):
    """Matvec-mode construction (construct.py:89-124) on (a) a dense FIO operator and
    (b) the composition K F K of a sampling-built chain (the paper's experiment):
    probe products, per-block triples and the full factor chains."""
    from butterfly.construct import _COL_PROBE_DOMAIN, _ROW_PROBE_DOMAIN, block_diagonal_probe
    n, leaf, r, seed = 256, 1, 8, 4
    p = bf.make_partition(n, leaf)
    mat = bf.kernels.dense_matrix(bf.FioKernel(n), n)
    op = bf.DenseOracle(mat)
    f = bf.factorize(op, p, r, seed=seed, mode="matvec")
    width = min(r + bf.lowrank.DEFAULT_PARAMS.p, p.mid_side)
    d = {"n": n, "levels": p.levels, "rank": r, "seed": seed, "width": width}
    d.update(_chain_arrays(f))
    d["col_probe"] = block_diagonal_probe(p, width, seed, _COL_PROBE_DOMAIN)
    d["row_probe"] = block_diagonal_probe(p, width, seed, _ROW_PROBE_DOMAIN)
    u_h, mid, v_h = bf.middle_factorization_matvec(op, p, r, seed=seed)
    d.update(u_h=u_h.blocks, v_h=v_h.blocks, w_h=mid.weights)
    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(4, 0)))
    g = bf.lowrank.complex_normal(rng, (n, 2))
    d.update(g=g, fwd=f.apply(g), adj=f.apply_adjoint(g))
    np.savez_compressed(os.path.join(OUT, "matvec_dense_fio_n256_r8_leaf1.npz"), **d)
    # composition: inner chain by sampling, composed operator, matvec chain
    inner = bf.factorize(bf.FioKernel(n), p, r, seed=0)
    comp = bf.ComposedOperator(inner)
    f2 = bf.factorize(comp, p, r, seed=0, mode="matvec")
    d = {"n": n, "levels": p.levels, "rank": r, "seed": 0}
    d.update(_chain_arrays(inner, "inner_"))
    d.update(_chain_arrays(f2))
    d.update(g=g, comp_fwd=comp.apply(g), comp_adj=comp.apply_adjoint(g), fwd=f2.apply(g))
    d["eps_a"] = bf.bench.estimate_eps_a(f2, bf.bench.OperatorReference(comp), 256,
                                         np.random.SeedSequence(0, spawn_key=(4, 0)))
    np.savez_compressed(os.path.join(OUT, "matvec_composed_fio_n256_r8_leaf1.npz"), **d)
    print("matvec fixtures, composed eps_a", d["eps_a"])


def gen_hankel(bf):
    """Bessel seeds, an order sweep, rows of the cached HankelKernel(1024) table and the
    criterion-2 accuracy of the reference's own sampling construction on it."""
    from butterfly import bessel as rb
    d = {}
    xs = np.concatenate([np.linspace(0.05, 5.0, 311), np.linspace(5.001, 2e4, 311)])
    d["seed_x"] = xs
    d["j0"], d["j1"], d["y0"], d["y1"] = rb.bessel_j0(xs), rb.bessel_j1(xs), rb.bessel_y0(xs), rb.bessel_y1(xs)
    x = 256 + (2 * np.pi / 3) * np.arange(0, 256, 37, dtype=float)
    d["sweep_x"], d["sweep"] = x, rb.hankel1_orders(x, 255)
    n = 1024
    ker = bf.HankelKernel(n)
    rows = np.arange(0, n, 61)
    d["table_n"], d["table_rows"] = n, rows
    d["table"] = ker.block(np.arange(n), np.arange(n))[rows]
    d["entry_64_3_5"] = bf.kernels.hankel_entry(64, 3, 5)
    p = bf.make_partition(n, 0.25)
    for r in (4, 6):
        f = bf.factorize(ker, p, r, seed=0, mode="sampling")
        d[f"eps_r{r}"] = bf.bench.estimate_eps_a(f, bf.bench.RowSampledReference(ker), 256,
                                                 np.random.SeedSequence(0, spawn_key=(4, 0)))
    np.savez_compressed(os.path.join(OUT, "hankel.npz"), **d)
    print("hankel.npz eps", d["eps_r4"], d["eps_r6"])


def _trace_block(bf, oracle, p, r, seed, i, j):
    """_sample_block with every select_pivot_columns call recorded (pick order)."""
    import butterfly.lowrank as lr
    from butterfly.construct import _sample_block
    calls = []
    orig = lr.select_pivot_columns

    def rec(a, k, rel_tol=0.0):
        out = orig(a, k, rel_tol)
        calls.append(list(out))
        return out

    lr.select_pivot_columns = rec
    try:
        apx = _sample_block(oracle, p, r, bf.lowrank.DEFAULT_PARAMS, seed, i, j)
    finally:
        lr.select_pivot_columns = orig
    return apx, calls


def gen_config_traces(bf, name, oracle, n, leaf, r, seed, nblocks, amp=1e-15, npert=2):
    """Middle blocks of a BASELINE config's own geometry, traced on the reference:
    a phase-invariant signature u0 diag(s0) v0^H X of each block on two fixed probe
    columns X, the singular values, the final skeleton sets and basis pivots, and the
    reference's own deviation d_ref under 1e-15 entry noise (npert hashed
    perturbations) — the calibrated envelope of SURVEY.md §8(c) stage 4."""
    import time
    p = bf.make_partition(n, leaf)
    m, side = p.mid_nodes, p.mid_side
    rng = np.random.default_rng(1234 + n)
    if nblocks >= m * m:
        blocks = [(i, j) for i in range(m) for j in range(m)]
    else:
        picks = {(0, 0), (m - 1, m - 1), (m // 2, m // 2), (0, m - 1)}
        while len(picks) < nblocks:
            picks.add((int(rng.integers(m)), int(rng.integers(m))))
        blocks = sorted(picks)
    x = bf.lowrank.complex_normal(np.random.default_rng(99), (side, 2))
    d = {"n": n, "levels": p.levels, "rank": r, "seed": seed, "amp": amp, "probe": x,
         "blocks": np.array(blocks, dtype=np.int64)}
    t0 = time.time()
    for (i, j) in blocks:
        apx, calls = _trace_block(bf, oracle, p, r, seed, i, j)
        sig = apx.u0 @ (apx.sigma0[:, None] * (apx.v0.conj().T @ x))
        key = f"b{i}_{j}"
        d[key + "_sig"] = sig
        d[key + "_s0"] = apx.sigma0
        if len(calls) == 8:   # sampling branch: 3 sweeps x 2, then the two basis calls
            d[key + "_skc"] = np.array(sorted(calls[4]), dtype=np.int64)
            d[key + "_skr"] = np.array(sorted(calls[5]), dtype=np.int64)
            d[key + "_pivc"] = np.array(calls[6], dtype=np.int64)
            d[key + "_pivr"] = np.array(calls[7], dtype=np.int64)
        dref, flips = [], []
        for q in range(npert):
            apx_q, calls_q = _trace_block(bf, NoisyOracle(oracle, amp, q + 1), p, r, seed, i, j)
            sig_q = apx_q.u0 @ (apx_q.sigma0[:, None] * (apx_q.v0.conj().T @ x))
            dref.append(np.linalg.norm(sig_q - sig) / max(np.linalg.norm(sig), 1e-300))
            flips.append([a != b for a, b in zip(calls, calls_q)] + [False] * (8 - len(calls)))
        d[key + "_dref"] = np.array(dref)
        d[key + "_flips"] = np.array(flips, dtype=bool)   # (npert, 8): which pivot calls moved
    np.savez_compressed(os.path.join(OUT, name), **d)
    drefs = np.array([d[f"b{i}_{j}_dref"].max() for i, j in blocks])
    print(name, "blocks", len(blocks), "side", side, "d_ref median %.2e max %.2e" % (np.median(drefs), drefs.max()),
          "%.1f s" % (time.time() - t0))


def gen_slab(bf, name, n, leaf, r, seed):
    """The reference's _recurse on one seeded synthetic slab (1, side, m, r) at a config's
    geometry: chain signatures U^L G^{L-1}..G^h X on fixed probes (phase-invariant) and
    the leaf block norms. The slab is regenerated at test time from the same seed."""
    from butterfly.construct import _recurse
    p = bf.make_partition(n, leaf)
    m, side = p.mid_nodes, p.mid_side
    slab = synthetic_slab(side, m, r, seed)
    leaf_b, pieces = _recurse(slab, p, r)
    x = bf.lowrank.complex_normal(np.random.default_rng(seed + 1), (m * r, 2))
    sig = slab_chain_apply(leaf_b, pieces, x)
    d = {"n": n, "levels": p.levels, "rank": r, "seed": seed, "probe": x, "sig": sig,
         "direct": slab.reshape(side, m * r) @ x}
    np.savez_compressed(os.path.join(OUT, name), **d)
    print(name, "chain vs slab rel", np.linalg.norm(sig - d["direct"]) / np.linalg.norm(d["direct"]))


def gen_eps(bf, name, oracle, n, leaf, r, seed):
    """eps_a of the reference's full factorize (bench.py:90-97, seeded as _run_row)."""
    import time
    p = bf.make_partition(n, leaf)
    t0 = time.time()
    f = bf.factorize(oracle, p, r, seed=seed)
    t_fac = time.time() - t0
    eps = bf.bench.estimate_eps_a(f, bf.bench.RowSampledReference(oracle), 256,
                                  np.random.SeedSequence(seed, spawn_key=(4, 0)))
    np.savez_compressed(os.path.join(OUT, name), n=n, levels=p.levels, rank=r, seed=seed, eps_a=eps,
                        factorize_s=t_fac)
    print(name, "eps_a", eps, "factorize %.1f s" % t_fac)


def gen_configs(bf):
    gen_config_traces(bf, "trace_cfg0_fio_n1024_r12_leaf8.npz", bf.FioKernel(1024), 1024, 8, 12, 0, 64)
    gen_config_traces(bf, "trace_fio_n4096_r8_leaf4.npz", bf.FioKernel(4096), 4096, 4, 8, 0, 24)
    gen_config_traces(bf, "trace_cfg1_dftp_n65536_r8_leaf16.npz", DftPlus(1 << 16), 1 << 16, 16, 8, 0, 24)
    gen_config_traces(bf, "trace_cfg2_fio_n1048576_r16_leaf16.npz", bf.FioKernel(1 << 20), 1 << 20, 16, 16, 0, 12)
    gen_slab(bf, "slab_cfg2_n1048576_r16_leaf16.npz", 1 << 20, 16, 16, 5)
    gen_eps(bf, "eps_fio_n4096_r12_leaf1.npz", bf.FioKernel(4096), 4096, 1, 12, 0)
    gen_eps(bf, "eps_dftp_n4096_r8_leaf1.npz", DftPlus(4096), 4096, 1, 8, 0)


def main():
    os.makedirs(OUT, exist_ok=True)
    bf = _ref()
    if len(sys.argv) > 1 and sys.argv[1] == "configs":
        gen_configs(bf)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "cfg1eps":   # ~15 min: the reference's full cfg1 factorize
        gen_eps(bf, "eps_cfg1_dftp_n65536_r8_leaf16.npz", DftPlus(1 << 16), 1 << 16, 16, 8, 0)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "matvec":
        gen_matvec(bf)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "hankel":
        gen_hankel(bf)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "dft":
        gen_dft(bf)
        return
    gen_bfac(bf)
    gen_geometry(bf)
    gen_entries(bf)
    gen_pivots(bf)
    gen_apply(bf, "apply_fio_n256_r8_leaf025.npz", bf.FioKernel(256), 256, 0.25, 8, 1, 3)
    gen_apply(bf, "apply_cfg0_fio_n1024_r12_leaf8.npz", bf.FioKernel(1024), 1024, 8, 12, 0, 1)
    gen_apply(bf, "apply_dftp_n1024_r8_leaf16.npz", DftPlus(1024), 1024, 16, 8, 0, 4)
    gen_construct(bf, "construct_fio_n128_r4_leaf025.npz", bf.FioKernel(128), 128, 0.25, 4, 9,
                  [(0, 0), (3, 5), (7, 7)])
    gen_construct(bf, "construct_fio_n1024_r12_leaf8.npz", bf.FioKernel(1024), 1024, 8, 12, 0,
                  [(0, 0), (2, 5), (7, 3)])
    gen_construct(bf, "construct_fio_n1024_r8_leaf1.npz", bf.FioKernel(1024), 1024, 1, 8, 3,
                  [(0, 0), (17, 30)])
    gen_matvec(bf)
    gen_hankel(bf)
    gen_dft(bf)


if __name__ == "__main__":
    main()
