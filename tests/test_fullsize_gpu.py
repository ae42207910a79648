"""Apply parity at the benchmarked sizes (the index math at L = 16-20 with many right-hand
sides, not only the kernel shapes), against the oracle's restatement of
ButterflyFactors._chain (factors.py:217-237) on a few output columns:

  cfg2   FIO geometry N=2^20, r=16, L=16, 256 RHS (two-CTA in-place DMMA levels)
  cfg4b  2-D quadtree n=1024^2, r=25, depth 8, 16 RHS (whole-unit 200 KB stages)
  cfg4a  N=2^24, r=16, L=20, 64 RHS, sharded over P=8 parts: parts 0
         and 5 built from their own 22.6 GB slices; their down and up halves against the
         oracle on the same slices (the V/H side is block-diagonal per column node, the
         G/U side per row node, so a part's half is the oracle's chain on its slices),
         and the pack -> unpack index maps on the part's own (diagonal) exchange chunk.

RHS columns are independent (reference test_factors.py:46-51), so the oracle runs on 1-4
columns of the same inputs. Tolerance: rel. 2-norm <= 1e-11 (complex128, north_star).
"""

import numpy as np
import pytest

import paper_1502_01379_b200 as bf
from oracle import chain as ochain
from paper_1502_01379_b200.synthetic import bench_chain, bench_slices

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def gauss(seed, shape):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def oracle_of(f):
    return ochain.Chain.from_reference(f)


@pytest.mark.parametrize("kind,k,cols", [("cfg2", 256, (0, 97, 255)), ("cfg4b", 16, (0, 15))])
def test_benchmark_sizes_vs_oracle(kind, k, cols):
    if kind == "cfg2":
        p, r = bf.make_partition(1 << 20, 16), 16
    else:
        p, r = bf.make_quadtree_partition(1024, 4), 25
    f = bench_chain(p, r, seed=11)
    plan = f.plan()
    oc = oracle_of(f)
    g = gauss(3, (p.n, k))
    gd = torch.from_numpy(g).cuda()
    sel = list(cols)
    for adjoint in (False, True):
        got = plan.apply(gd, adjoint=adjoint)[:, sel].cpu().numpy()
        want = ochain.apply(oc, np.ascontiguousarray(g[:, sel]), adjoint=adjoint)
        err = rel(got, want)
        print(f"\n{kind} k={k} {'adjoint' if adjoint else 'forward'}: columns {sel} rel {err:.2e}")
        assert err <= TOL


def _down_oracle(sl, x, adjoint):
    """A part's down half on its slices: V^L*, H^{L-1}*..H^h* (forward) or U^L*, G^{L-1}*..G^h*."""
    leaf, lv = (sl["u_leaf"], sl["g"]) if adjoint else (sl["v_leaf"], sl["h"])
    w = ochain.leaf_adjoint(leaf, x)
    for _, b in reversed(lv):
        w = ochain.transfer_adjoint(b, w)
    return w


def _up_oracle(sl, w, adjoint):
    """A part's up half: G^h..G^{L-1}, U^L (forward) or H^h..H^{L-1}, V^L (adjoint)."""
    leaf, lv = (sl["v_leaf"], sl["h"]) if adjoint else (sl["u_leaf"], sl["g"])
    for _, b in lv:
        w = ochain.transfer_forward(b, w)
    return ochain.leaf_forward(leaf, w)


@pytest.mark.parametrize("part", [0, 5])
def test_cfg4a_sharded_part_vs_oracle(part):
    """BASELINE config 4a (N=2^24, r=16, leaf 16 -> L=20, m=1024, 64 RHS) at P=8: one part's
    local halves and its diagonal exchange chunk at full size."""
    from paper_1502_01379_b200.sharded import ShardedPlan
    P, k, r = 8, 64, 16
    p = bf.make_partition(1 << 24, 16)
    sl = bench_slices(p, r, part, P, seed=7)
    sp = ShardedPlan(p, r, part, P, sl)
    nl, m = sp.n_local, p.mid_nodes
    sel = [0, 63]
    x = gauss(part, (nl, k))
    xd = torch.from_numpy(x).cuda()
    for adjoint in (False, True):
        mid = sp.down(xd, adjoint)
        want = _down_oracle(sl, np.ascontiguousarray(x[:, sel]), adjoint)
        err = rel(mid[:, sel].cpu().numpy(), want)
        print(f"\ncfg4a part {part}/{P} down {'adjoint' if adjoint else 'forward'}: rel {err:.2e}")
        assert err <= TOL
        # exchange index maps: only this part's own chunk (rows i in I_d, columns j in J_d) is
        # filled, as if every other part sent zeros; unpack must hold W-scaled mid_in[j, i]
        send = sp.pack(mid, adjoint)
        recv = torch.zeros_like(send)
        c = sp.chunk_rows
        recv[part * c:(part + 1) * c] = send[part * c:(part + 1) * c]
        got = sp.unpack(recv, adjoint).cpu().numpy().reshape(sp.mp, m, r, k)
        mp, d0 = sp.mp, part * sp.mp
        mid_h = mid.cpu().numpy().reshape(sp.mp, m, r, k)          # [j_local, i, rho]
        w = sl["weights"]
        # forward: out[i, j] = W[i, j] in[j, i]; adjoint: out[j, i] = W[i, j] in[i, j] (factors.py:180-190)
        blk = mid_h[:, d0:d0 + mp]                                     # [j_local, i_local]
        wt = w[d0:d0 + mp, d0:d0 + mp]                                 # [i_local, j_local]
        exp = (wt[:, :, :, None] * blk.swapaxes(0, 1)) if not adjoint else \
            (wt.swapaxes(0, 1)[:, :, :, None] * blk.swapaxes(0, 1))
        assert rel(got[:, d0:d0 + mp], exp) <= 1e-15
        assert not np.any(got[:, :d0]) and not np.any(got[:, d0 + mp:])
        # up half on an arbitrary middle slice
        y = gauss(10 + part, (sp.mid_rows, k))
        out = sp.up(torch.from_numpy(y).cuda(), adjoint)
        want = _up_oracle(sl, np.ascontiguousarray(y[:, sel]), adjoint)
        err = rel(out[:, sel].cpu().numpy(), want)
        print(f"cfg4a part {part}/{P} up {'adjoint' if adjoint else 'forward'}: rel {err:.2e}")
        assert err <= TOL
    del sp
    torch.cuda.empty_cache()
