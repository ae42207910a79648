"""GPU parity of the apply chain (libbfly.so via the C ABI) against the CPU
oracle and the reference's own golden outputs.

Tolerances (BASELINE.json north_star): relative 2-norm <= 1e-11 for complex128,
<= 1e-5 for the opt-in complex64 mode. Algebraic KATs follow
pkg/tests/test_factors.py:16-51.
"""

import os

import numpy as np
import pytest

import paper_1502_01379_b200 as bf
from conftest import chain_from_golden, complex_gaussian, golden
from oracle import chain as ochain
from paper_1502_01379_b200.synthetic import synthetic_chain, to_host

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL128, TOL64 = 1e-11, 1e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN_APPLY = ["apply_fio_n256_r8_leaf025.npz", "apply_cfg0_fio_n1024_r12_leaf8.npz",
                "apply_dftp_n1024_r8_leaf16.npz"]


def rel(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else a
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def product(c):
    return bf.from_arrays(c.n, c.levels, c.rank, c.u_leaf, c.g_levels, c.weights, c.h_levels, c.v_leaf)


def oracle_of(f):
    h = to_host(f)
    return ochain.Chain(h.n, h.partition.levels, h.rank, h.u_outer.blocks,
                        [(t.level, t.blocks) for t in h.g_chain], h.middle.weights,
                        [(t.level, t.blocks) for t in h.h_chain], h.v_outer.blocks)


@pytest.fixture(scope="module", params=GOLDEN_APPLY)
def case(request):
    d = golden(request.param)
    return d, product(chain_from_golden(d))


def test_golden_forward_adjoint_c128(case):
    d, f = case
    g = torch.from_numpy(d["g"]).cuda()
    assert rel(f.plan().apply(g), d["fwd"]) <= TOL128
    assert rel(f.plan().apply(g, adjoint=True), d["adj"]) <= TOL128
    one = f.apply(d["g"][:, 0])                       # host path, 1-D in -> 1-D out
    assert one.ndim == 1 and one.dtype == np.complex128 and rel(one, d["fwd1"]) <= TOL128


def test_golden_c64_mode(case):
    d, f = case
    pl = f.plan("c64")
    g = torch.from_numpy(d["g"]).cuda()
    out = pl.apply(g)
    assert out.dtype == torch.complex64
    assert rel(out.to(torch.complex128), d["fwd"]) <= TOL64
    assert rel(pl.apply(g, adjoint=True).to(torch.complex128), d["adj"]) <= TOL64


def test_host_and_device_paths_bitwise_equal(case):
    d, f = case
    dev = f.plan().apply(torch.from_numpy(d["g"]).cuda()).cpu().numpy()
    host = f.apply(d["g"])
    assert np.array_equal(dev, host)
    again = f.apply(d["g"])
    assert np.array_equal(host, again)                # run-to-run deterministic


def test_zero_bad_length_and_upcast(case):
    d, f = case
    n = f.n
    assert np.array_equal(f.apply(np.zeros(n, dtype=complex)), np.zeros(n, dtype=complex))
    with pytest.raises(ValueError):
        f.apply(np.zeros(n // 2))
    with pytest.raises(ValueError):
        f.apply_adjoint(np.zeros(n // 2))
    real_in = np.arange(n, dtype=np.float32)          # any numeric dtype is upcast (factors.py:222)
    assert f.apply(real_in).dtype == np.complex128
    assert rel(f.apply(real_in), f.apply(real_in.astype(complex))) == 0.0


def test_algebraic_kats(case, rng):
    d, f = case
    n = f.n
    x, y = complex_gaussian(rng, n), complex_gaussian(rng, n)
    a, b = 0.3 - 1.1j, -2.0 + 0.4j
    lhs = f.apply(a * x + b * y)
    rhs = a * f.apply(x) + b * f.apply(y)
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(rhs)
    ip1 = np.vdot(y, f.apply(x))
    ip2 = np.vdot(f.apply_adjoint(y), x)
    assert abs(ip1 - ip2) <= 1e-12 * abs(ip1)
    block = complex_gaussian(rng, (n, 5))
    out = f.apply(block)
    for k in range(5):
        col = f.apply(block[:, k])
        assert np.linalg.norm(out[:, k] - col) <= 1e-13 * np.linalg.norm(col)


def test_per_factor_parity(case):
    """bf_apply_factor vs the oracle's per-factor maps (factors.py:49-56, 120-142, 180-190)."""
    d, f = case
    c = chain_from_golden(d)
    pl = f.plan()
    rng = np.random.default_rng(3)
    k = 3
    nb, n0, r = c.u_leaf.shape
    for which, arr in (("V", c.v_leaf), ("U", c.u_leaf)):
        x = complex_gaussian(rng, (nb * n0, k))
        assert rel(pl.apply_factor(which, 0, True, torch.from_numpy(x).cuda()), ochain.leaf_adjoint(arr, x)) <= 1e-14
        x = complex_gaussian(rng, (nb * r, k))
        assert rel(pl.apply_factor(which, 0, False, torch.from_numpy(x).cuda()), ochain.leaf_forward(arr, x)) <= 1e-14
    dim = c.weights.size
    x = complex_gaussian(rng, (dim, k))
    assert rel(pl.apply_factor("M", 0, False, torch.from_numpy(x).cuda()), ochain.middle_forward(c.weights, x)) == 0
    assert rel(pl.apply_factor("M", 0, True, torch.from_numpy(x).cuda()), ochain.middle_adjoint(c.weights, x)) == 0
    for which, levels in (("G", c.g_levels), ("H", c.h_levels)):
        for lvl, b in levels:
            tf = bf.TransferFactor(lvl, b)
            rows, cols = tf.shape
            x = complex_gaussian(rng, (cols, k))
            got = pl.apply_factor(which, lvl, False, torch.from_numpy(x).cuda())
            assert rel(got, ochain.transfer_forward(b, x)) <= 1e-14, (which, lvl)
            x = complex_gaussian(rng, (rows, k))
            got = pl.apply_factor(which, lvl, True, torch.from_numpy(x).cuda())
            assert rel(got, ochain.transfer_adjoint(b, x)) <= 1e-14, (which, lvl)


@pytest.mark.parametrize("n,leaf,r,k", [
    (1 << 16, 16, 8, 64),     # config 1 geometry (L=12), 64 RHS
    (1 << 12, 0.25, 5, 7),    # merge-only levels, odd rank and odd k
    (1 << 12, 0.25, 5, 9),    # same through the many-RHS kernel (k >= 8)
    (1 << 12, 4, 12, 8),      # many-RHS threshold, r=12 (config 0 rank)
    (1 << 12, 16, 16, 33),    # many-RHS, k not a multiple of the 4-wide register tile
    (1 << 14, 4, 25, 16),     # rank 25 (the 2D configs' rank), 16 RHS
    (1 << 10, 16, 12, 300),   # many RHS: k split across tiles
    (1 << 12, 4, 6, 64),      # fused level pairs (pair_kernel): r=6, padded rows
    (1 << 14, 16, 8, 128),    # fused level pairs at 128 RHS
    (1 << 12, 1, 4, 96),      # fused pairs, odd number of splitting levels per half
    (1 << 14, 16, 16, 64),    # r=16, 64 RHS (pairs do not fit a stage: single levels)
    (1 << 12, 16, 16, 70),    # same, k not a multiple of the DMMA tiles
    (1 << 12, 16, 16, 256),   # 256 RHS: complex64 in-place FFMA tiles, complex128 two-CTA DMMA
])
def test_synthetic_geometries(n, leaf, r, k):
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=n + r)
    oc = oracle_of(f)
    g = complex_gaussian(np.random.default_rng(k), (n, k))
    gd = torch.from_numpy(g).cuda()
    assert rel(f.plan().apply(gd), ochain.apply(oc, g)) <= TOL128
    assert rel(f.plan().apply(gd, adjoint=True), ochain.apply(oc, g, adjoint=True)) <= TOL128
    assert rel(f.plan("c64").apply(gd).to(torch.complex128), ochain.apply(oc, g)) <= TOL64


@pytest.mark.parametrize("n,leaf,r,k", [
    (1 << 14, 16, 16, 64),    # k-chunked level pairs (pair_chunk_kernel): r=16, 2 chunks of 32 RHS
    (1 << 12, 16, 16, 70),    # partial last chunk (6 RHS) and idle column slices
    (1 << 10, 16, 12, 300),   # r=12, 10 chunks
])
def test_chunked_pairs_opt_in(n, leaf, r, k, env_flag="BF_CHUNK_PAIR"):
    """The k-chunked pair kernel is opt-in (BF_CHUNK_PAIR=1, read once per process): run the
    oracle comparison in a child process with it enabled."""
    import subprocess
    import sys
    code = f"""
import numpy as np, torch, sys
sys.path[:0] = [{ROOT!r}, {os.path.join(ROOT, "tests")!r}]
import paper_1502_01379_b200 as bf
from paper_1502_01379_b200.synthetic import synthetic_chain
from conftest import complex_gaussian
from test_apply_gpu import oracle_of, rel
from oracle import chain as ochain
p = bf.make_partition({n}, {leaf})
f = synthetic_chain(p, {r}, seed={n + r})
oc = oracle_of(f)
g = complex_gaussian(np.random.default_rng({k}), ({n}, {k}))
gd = torch.from_numpy(g).cuda()
e1 = rel(f.plan().apply(gd), ochain.apply(oc, g))
e2 = rel(f.plan().apply(gd, adjoint=True), ochain.apply(oc, g, adjoint=True))
assert e1 <= 1e-11 and e2 <= 1e-11, (e1, e2)
print("ok", e1, e2)
"""
    env = dict(os.environ, **{env_flag: "1"})
    r_ = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT)
    assert r_.returncode == 0 and "ok" in r_.stdout, r_.stderr[-2000:]


@pytest.mark.parametrize("n,leaf,r,k", [(1 << 16, 16, 8, 64), (1 << 12, 16, 6, 64)])
def test_remap_pair_opt_in(n, leaf, r, k):
    """The down half's last pair carries the fused middle factor (the default; this child
    process sets BF_REMAP_PAIR=1 explicitly)."""
    test_chunked_pairs_opt_in(n, leaf, r, k, env_flag="BF_REMAP_PAIR")


@pytest.mark.parametrize("n,leaf,r,k", [
    (1 << 16, 16, 8, 64),     # config 1: leaf-fused first / last pair, 32-RHS chunks
    (1 << 12, 16, 8, 128),    # 64-RHS chunks (8 consumer warps), nl = 4
    (1 << 10, 16, 8, 64),     # nl = 3 (odd): the up half ends in a single level, no fused trail leaf
    (1 << 8, 16, 8, 64),      # nl = 2: one pair per half carries both the leaf and the middle factor
    (1 << 12, 16, 8, 80),     # k a multiple of 16 whose chunk (40) is not: the general pair kernel
    (1 << 12, 8, 8, 64),      # 8-point leaves: rank-8 pairs without the fused leaf
    (1 << 12, 16, 8, 320),    # 10 chunks of 32 RHS
])
def test_rank8_pairs(n, leaf, r, k):
    """Rank-8 level pairs (pair8_kernel: warp-owned slices, leaf factor fused into the pair
    next to it) against the oracle, forward and adjoint; BF_NO_PAIR8_LEAF=1 and
    BF_PAIR8_STAGES=1 (read once per process: child processes) give the same result."""
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=n + k)
    oc = oracle_of(f)
    g = complex_gaussian(np.random.default_rng(k), (n, k))
    gd = torch.from_numpy(g).cuda()
    assert rel(f.plan().apply(gd), ochain.apply(oc, g)) <= TOL128
    assert rel(f.plan().apply(gd, adjoint=True), ochain.apply(oc, g, adjoint=True)) <= TOL128


@pytest.mark.parametrize("n,leaf,r,k", [(1 << 14, 16, 16, 64), (1 << 12, 16, 16, 256), (1 << 10, 16, 16, 96)])
def test_rank16_pairs_opt_in(n, leaf, r, k):
    """Rank-16 level pairs with register-fed factor fragments (pair16_kernel, BF_PAIR16=1: read
    once per process, hence a child process), forward and adjoint, including the fused middle
    factor in the down half's last pair."""
    test_chunked_pairs_opt_in(n, leaf, r, k, env_flag="BF_PAIR16")


@pytest.mark.parametrize("n,leaf,r,k", [
    (1 << 14, 16, 16, 64),    # rank 16, 4 + 4 splitting levels: the branching-4 twin (plan_build_radix4), wide GEMM
    (1 << 12, 16, 16, 256),
    (1 << 12, 16, 20, 16),    # rank 20 (C4 = 80)
    (1 << 10, 4, 16, 9),      # k not a multiple of 8
])
def test_radix4_twin(n, leaf, r, k):
    """Many-RHS applies of rank-16..26 chains run on the branching-4 twin of the plan (pairs of
    binary levels folded at first use); 1 RHS on the same plan runs the binary chain. Both
    against the oracle, forward and adjoint; BF_NO_RADIX4=1 (child process) gives the same."""
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=n + k)
    oc = oracle_of(f)
    pl = f.plan()
    for kk in (k, 1, k):
        g = complex_gaussian(np.random.default_rng(kk), (n, kk))
        gd = torch.from_numpy(g).cuda()
        assert rel(pl.apply(gd), ochain.apply(oc, g)) <= TOL128
        assert rel(pl.apply(gd, adjoint=True), ochain.apply(oc, g, adjoint=True)) <= TOL128
    gh = complex_gaussian(np.random.default_rng(3), (n, k))
    assert rel(torch.from_numpy(pl.apply(gh)), ochain.apply(oc, gh)) <= TOL128   # host-buffer path
    p64 = f.plan("c64")                                                          # complex64 twin (FFMA levels)
    gd = torch.from_numpy(gh).cuda()
    assert rel(p64.apply(gd).to(torch.complex128), ochain.apply(oc, gh)) <= TOL64
    assert rel(p64.apply(gd, adjoint=True).to(torch.complex128), ochain.apply(oc, gh, adjoint=True)) <= TOL64


def test_radix4_switch():
    test_chunked_pairs_opt_in(1 << 12, 16, 16, 64, env_flag="BF_NO_RADIX4")


@pytest.mark.parametrize("flag", ["BF_NO_PAIR8_LEAF", "BF_NO_PAIR8"])
def test_rank8_pairs_switches(flag):
    test_chunked_pairs_opt_in(1 << 12, 16, 8, 64, env_flag=flag)


def test_quadtree_t_range_split_many_rhs():
    """Many-RHS quadtree levels whose 4-block units do not fit a stage run as t-range
    launches (forward outputs per t, adjoint partial sums accumulated). The default
    single 200 KB stage avoids them at r = 25; BF_MRHS_STAGES=2 BF_MRHS_STAGE_KB=112 (read
    once per process, hence a child process) forces them, with the K-pipelined wide
    kernel (the default for these levels) turned off by BF_NO_WIDE=1."""
    import subprocess
    import sys
    code = f"""
import numpy as np, torch, sys
sys.path[:0] = [{ROOT!r}, {os.path.join(ROOT, "tests")!r}]
import paper_1502_01379_b200 as bf
from paper_1502_01379_b200.synthetic import synthetic_chain
from conftest import complex_gaussian
from test_apply_gpu import oracle_of, rel
from oracle import chain as ochain
p = bf.make_quadtree_partition(128, 2)
f = synthetic_chain(p, 25, seed=3)
oc = oracle_of(f)
g = complex_gaussian(np.random.default_rng(5), (p.n, 16))
gd = torch.from_numpy(g).cuda()
e1 = rel(f.plan().apply(gd), ochain.apply(oc, g))
e2 = rel(f.plan().apply(gd, adjoint=True), ochain.apply(oc, g, adjoint=True))
assert e1 <= 1e-11 and e2 <= 1e-11, (e1, e2)
print("ok", e1, e2)
"""
    env = dict(os.environ, BF_MRHS_STAGES="2", BF_MRHS_STAGE_KB="112", BF_NO_WIDE="1")
    r_ = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT)
    assert r_.returncode == 0 and "ok" in r_.stdout, r_.stderr[-2000:]


def test_config2_geometry_k1():
    """BASELINE config 2 (FIO geometry N=2^20, r=16, leaf 16 -> L=16), synthetic factors, 1 RHS."""
    p = bf.make_partition(1 << 20, 16)
    f = synthetic_chain(p, 16, seed=2, device="cuda")
    g = complex_gaussian(np.random.default_rng(0), (p.n,))
    got = f.plan().apply(torch.from_numpy(g).cuda()).cpu().numpy()
    want = ochain.apply(oracle_of(f), g)
    assert rel(got, want) <= TOL128
    got64 = f.plan("c64").apply(torch.from_numpy(g).cuda()).to(torch.complex128).cpu().numpy()
    assert rel(got64, want) <= TOL64


def test_entries_match_reference_golden():
    from paper_1502_01379_b200 import _lib
    import ctypes
    d = golden("entries.npz")
    lib = _lib.load()
    for n in (1024, 1 << 16, 1 << 20, 1 << 24):
        rows = torch.from_numpy(d[f"fio_{n}_rows"].astype(np.int64)).cuda()
        cols = torch.from_numpy(d[f"fio_{n}_cols"].astype(np.int64)).cuda()
        out = torch.empty((rows.numel(), cols.numel()), dtype=torch.complex128, device="cuda")
        _lib.check(lib.bf_entries(_lib.BF_KERNEL_FIO, n, ctypes.c_void_p(rows.data_ptr()), rows.numel(),
                                  ctypes.c_void_p(cols.data_ptr()), cols.numel(), ctypes.c_void_p(out.data_ptr()),
                                  None))
        torch.cuda.synchronize()
        got, want = out.cpu().numpy(), d[f"fio_{n}"]
        # exp(i a) with a = fl(2 pi Phi): the phase follows the reference's rounding sequence
        # exactly (no FMA) on the correctly rounded c(x) table. Where glibc's sin(2 pi x)
        # is correctly rounded too (all but ~0.03% of rows), a is bit-identical and only
        # CUDA's final sin/cos (<= 2 ulp) differ; on the other rows c(x) differs by an ulp,
        # which moves a by up to 2 ulp of |a| (before the table: on ~30% of rows).
        x = d[f"fio_{n}_rows"].astype(float)[:, None] / n
        c_ref = ((2.0 + np.sin(2.0 * np.pi * x)) / 8.0)[:, 0]
        tab = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.check(lib.bf_entry_table(_lib.BF_KERNEL_FIO, n, ctypes.c_void_p(tab.data_ptr()), n, None))
        same_c = tab.cpu().numpy()[d[f"fio_{n}_rows"]] == c_ref
        err = np.abs(got - want)
        assert err[same_c].max() <= 4.5e-16
        amax = 2 * np.pi * n * 1.5
        assert err.max() <= 2 * np.spacing(amax) + 4e-16
        assert np.mean(got == want) >= 0.5
    rows = torch.from_numpy(d["dftp_rows"].astype(np.int64)).cuda()
    cols = torch.from_numpy(d["dftp_cols"].astype(np.int64)).cuda()
    out = torch.empty((rows.numel(), cols.numel()), dtype=torch.complex128, device="cuda")
    _lib.check(lib.bf_entries(_lib.BF_KERNEL_DFTP, 1 << 16, ctypes.c_void_p(rows.data_ptr()), rows.numel(),
                              ctypes.c_void_p(cols.data_ptr()), cols.numel(), ctypes.c_void_p(out.data_ptr()), None))
    torch.cuda.synchronize()
    assert np.max(np.abs(out.cpu().numpy() - d["dftp"])) <= 4e-16   # exact phase; sin/cos ulps only


@pytest.mark.parametrize("n_side,leaf,r,k", [
    (64, 4, 8, 3),        # quadtree depth 4
    (256, 4, 25, 16),     # BASELINE config 3 geometry: n=256, leaf 4x4, r=25, 16 RHS
    (128, 2, 25, 1),      # r=25 one RHS: t-range split of the 4 x 25 x 100 block units
])
def test_quadtree_geometries(n_side, leaf, r, k):
    """2-D (branching 4) chains against the oracle's quadtree restatement (parity unpinned:
    no reference 2-D code exists)."""
    p = bf.make_quadtree_partition(n_side, leaf)
    f = synthetic_chain(p, r, seed=n_side + r)
    oc = oracle_of(f)
    g = complex_gaussian(np.random.default_rng(k), (p.n, k))
    gd = torch.from_numpy(g).cuda()
    assert rel(f.plan().apply(gd), ochain.apply(oc, g)) <= TOL128
    assert rel(f.plan().apply(gd, adjoint=True), ochain.apply(oc, g, adjoint=True)) <= TOL128
    assert rel(f.plan("c64").apply(gd).to(torch.complex128), ochain.apply(oc, g)) <= TOL64
    assert rel(f.plan("c64").apply(gd, adjoint=True).to(torch.complex128),
               ochain.apply(oc, g, adjoint=True)) <= TOL64


@pytest.mark.parametrize("tree,n,leaf,r,k", [
    ("quad", 64, 4, 25, 8),       # one 8-column tile per item
    ("quad", 128, 2, 25, 12),     # ragged right-hand-side tile
    ("quad", 64, 4, 17, 33),      # C = 68: ragged last K tile; two right-hand-side chunks
    ("quad", 128, 2, 20, 64),     # 32-column items, two chunks
    ("bin", 1 << 12, 64, 40, 16),  # binary tree with C = 2r = 80 > 64
])
def test_wide_kernel_levels(tree, n, leaf, r, k):
    """Many-RHS complex128 levels with wide blocks (C > 64) run as the K-pipelined DMMA GEMM
    (wide_kernel.cuh): forward and adjoint chains (the adjoint chain's last down level carries
    the fused middle factor) against the oracle, and bitwise run-to-run."""
    p = bf.make_quadtree_partition(n, leaf) if tree == "quad" else bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=n + r + k)
    oc = oracle_of(f)
    g = complex_gaussian(np.random.default_rng(k), (p.n, k))
    gd = torch.from_numpy(g).cuda()
    pl = f.plan()
    y = pl.apply(gd)
    assert rel(y, ochain.apply(oc, g)) <= TOL128
    assert rel(pl.apply(gd, adjoint=True), ochain.apply(oc, g, adjoint=True)) <= TOL128
    assert torch.equal(pl.apply(gd), y)


@pytest.mark.parametrize("n,leaf,r,k", [(1 << 18, 16, 16, 1), (1 << 16, 16, 8, 64)])
def test_pinned_host_pipeline_bitwise(n, leaf, r, k):
    """bf_apply_host with page-locked buffers pipelines H2D/D2H chunks against the chain
    (part views + separate middle kernel): bitwise equal to the device path, both directions."""
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=7, device="cuda")
    g = torch.from_numpy(complex_gaussian(np.random.default_rng(2), (n, k)))
    g_pin = g.pin_memory()
    o_pin = torch.empty_like(g_pin).pin_memory()
    pl = f.plan()
    for adjoint in (False, True):
        dev = pl.apply(g.cuda(), adjoint=adjoint).cpu().numpy()
        for _ in range(2):      # first call captures the pipeline graph, second replays it
            host = pl.apply(g_pin.numpy(), adjoint=adjoint, out=o_pin.numpy())
            assert np.array_equal(host, dev)


def test_pinned_host_pipeline_regrow():
    """k=1 -> k=4 -> k=1 on the same pinned buffers: the k=4 call grows the plan's device
    buffers, so the k=1 graph cached before it must not be replayed against the freed ones."""
    p = bf.make_partition(1 << 18, 16)
    f = synthetic_chain(p, 16, seed=3, device="cuda")
    pl = f.plan()
    g4 = torch.from_numpy(complex_gaussian(np.random.default_rng(5), (p.n, 4))).pin_memory()
    o4 = torch.empty_like(g4).pin_memory()
    g1 = g4[:, :1].contiguous().pin_memory()
    o1 = torch.empty_like(g1).pin_memory()
    want1 = pl.apply(g1.cuda()).cpu().numpy()
    want4 = pl.apply(g4.cuda()).cpu().numpy()
    for _ in range(2):
        assert np.array_equal(pl.apply(g1.numpy(), out=o1.numpy()), want1)
        assert np.array_equal(pl.apply(g4.numpy(), out=o4.numpy()), want4)
        assert np.array_equal(pl.apply(g1.numpy(), out=o1.numpy()), want1)


@pytest.mark.parametrize("n,levels,r,k", [
    (4, 2, 1, 1),       # smallest partition: m = 2, side = 2
    (4, 2, 2, 3),
    (16, 8, 3, 2),      # leaf 1/16: the middle level itself is merge-only (side = 1)
    (64, 12, 2, 5),     # leaf 1/64, every level merge-only
    (32, 10, 4, 9),     # many-RHS kernels on merge-only levels
])
def test_edge_geometries(n, levels, r, k):
    p = bf.DyadicPartition(n, levels)
    f = synthetic_chain(p, r, seed=n * levels + r)
    oc = oracle_of(f)
    g = complex_gaussian(np.random.default_rng(k), (n, k))
    gd = torch.from_numpy(g).cuda()
    assert rel(f.plan().apply(gd), ochain.apply(oc, g)) <= TOL128
    assert rel(f.plan().apply(gd, adjoint=True), ochain.apply(oc, g, adjoint=True)) <= TOL128
    assert rel(f.plan("c64").apply(gd).to(torch.complex128), ochain.apply(oc, g)) <= TOL64
    # shapes: (n,) -> (n,), (n, 1) -> (n, 1)
    assert f.apply(g[:, 0]).shape == (n,) and f.apply(g[:, :1]).shape == (n, 1)


def test_plan_rejects_mismatched_factors():
    p = bf.make_partition(256, 16)
    f = synthetic_chain(p, 4, seed=1)
    bad = bf.ButterflyFactors(p, 4, f.u_outer, f.g_chain[:-1], f.middle, f.h_chain, f.v_outer)
    with pytest.raises(ValueError):
        bad.apply(np.zeros(256))
    wrong = bf.ButterflyFactors(p, 4, bf.BlockDiagonalFactor(f.u_outer.blocks[:, :, :3]), f.g_chain, f.middle,
                                f.h_chain, f.v_outer)
    with pytest.raises(ValueError):
        wrong.apply(np.zeros(256))


@pytest.mark.parametrize("leaf", [16, 1, 0.25])
def test_many_rhs_shape_sweep(leaf):
    """Many-RHS consumers across warp-tile choices (DMMA 2x4 / 2x2 / 1x2, in-place outputs,
    k-tiles with partial last tiles, merge-only levels) and the complex64 FFMA tiles."""
    n = 1 << 12
    for r in (5, 12, 16):
        f = synthetic_chain(bf.make_partition(n, leaf), r, seed=7 * r + int(4 * leaf))
        oc = oracle_of(f)
        for k in (8, 24, 40, 130):
            g = complex_gaussian(np.random.default_rng(k + r), (n, k))
            gd = torch.from_numpy(g).cuda()
            for adj in (False, True):
                want = ochain.apply(oc, g, adjoint=adj)
                assert rel(f.plan().apply(gd, adjoint=adj), want) <= TOL128, (r, k, adj)
                assert rel(f.plan("c64").apply(gd, adjoint=adj).to(torch.complex128), want) <= TOL64, (r, k, adj)


def test_c64_tensor_core_levels():
    """complex64 levels on tcgen05 (kind::tf32, 3xTF32 split, accumulators in TMEM;
    csrc/tc_kernel.cuh), opt-in BF_TC=1, run in a subprocess with the switch set: forward
    and adjoint within the c64 tolerance of the oracle, partial 128-RHS tiles, leaf and
    transfer levels, the fused middle factor."""
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_1502_01379_b200 as bf
from oracle import chain as ochain
from paper_1502_01379_b200.synthetic import synthetic_chain
for n, leaf, r, k in [(1 << 12, 16, 16, 128), (1 << 14, 16, 8, 256), (1 << 12, 16, 16, 300), (1 << 12, 1, 4, 130),
                      (1 << 12, 16, 16, 129)]:
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=n + r + k)
    oc = ochain.Chain.from_reference(f)
    rng = np.random.default_rng(k)
    g = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    plan = f.plan("c64")
    for adj in (False, True):
        got = plan.apply(torch.from_numpy(g).cuda(), adjoint=adj).to(torch.complex128).cpu().numpy()
        want = ochain.apply(oc, g, adjoint=adj)
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err <= 1e-5, (n, k, adj, err)
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                         env={**os.environ, "BF_TC": "1"})
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
