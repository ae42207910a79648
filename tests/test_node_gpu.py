"""Node kernels (csrc/node_kernel.cuh): each half of the chain as one launch, one CTA per
(middle node, right-hand-side chunk), used for chains whose factors sit in L2 (BASELINE
configs 0 and 1). Parity against the oracle's restatement of ButterflyFactors._chain
(factors.py:217-237), forward and adjoint, on the FMA (k < 8) and DMMA (k >= 8) paths,
full and partial RHS chunks, and against the reference's own golden apply outputs."""

import numpy as np
import pytest

import paper_1502_01379_b200 as bf
from conftest import chain_from_golden, complex_gaussian, golden
from oracle import chain as ochain
from paper_1502_01379_b200.synthetic import synthetic_chain

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-13


def rel(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else a
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,leaf,r,k", [
    (1 << 10, 8, 12, 1),      # BASELINE config 0 geometry (FMA path)
    (1 << 10, 8, 12, 3),
    (1 << 12, 16, 8, 5),
    (1 << 12, 1, 4, 2),       # leaf 1: one-row leaf blocks
    (1 << 16, 16, 8, 64),     # BASELINE config 1 geometry (DMMA, 16-RHS chunks)
    (1 << 16, 16, 8, 20),     # partial last chunk
    (1 << 14, 16, 16, 8),     # r = 16: 8-RHS chunks
    (1 << 12, 16, 12, 11),    # r = 12: partial 8-row tiles
])
def test_node_path_vs_oracle(n, leaf, r, k):
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=n + r + k)
    oc = ochain.Chain.from_reference(f)
    g = complex_gaussian(np.random.default_rng(k), (n, k))
    plan = f.plan()
    gd = torch.from_numpy(g).cuda()
    for adjoint in (False, True):
        got = plan.apply(gd, adjoint=adjoint)
        err = rel(got, ochain.apply(oc, g, adjoint=adjoint))
        assert err <= TOL, (adjoint, err)
    # zero in -> exactly zero out; run-to-run deterministic
    assert not plan.apply(torch.zeros_like(gd)).abs().max().item()
    assert torch.equal(plan.apply(gd), plan.apply(gd))


def test_node_path_cfg0_golden():
    """The reference's own cfg0 factors and apply output (oracle/gen_golden.py)."""
    d = golden("apply_cfg0_fio_n1024_r12_leaf8.npz")
    oc = chain_from_golden(d)
    f = bf.from_arrays(oc.n, oc.levels, oc.rank, oc.u_leaf, oc.g_levels, oc.weights, oc.h_levels, oc.v_leaf)
    gd = torch.from_numpy(d["g"]).cuda()
    assert rel(f.plan().apply(gd), d["fwd"]) <= 1e-11
    assert rel(f.plan().apply(gd, adjoint=True), d["adj"]) <= 1e-11


def test_node_mma_opt_in_subprocess():
    """The staged many-RHS node kernel (node_mma.cuh, opt-in BF_NODE_MMA=1: slower than the
    level kernels at cfg1, kept as a measured alternative) stays correct: cfg1 geometry,
    forward and adjoint, against the oracle, in a process with the switch set."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_1502_01379_b200 as bf
from oracle import chain as ochain
from paper_1502_01379_b200.synthetic import synthetic_chain
for n, leaf, r, k in [(1 << 16, 16, 8, 64), (1 << 14, 16, 16, 12)]:
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=3)
    oc = ochain.Chain.from_reference(f)
    g = np.random.default_rng(0).standard_normal((n, k)) + 1j
    for adj in (False, True):
        got = f.plan().apply(torch.from_numpy(g).cuda(), adjoint=adj).cpu().numpy()
        want = ochain.apply(oc, g, adjoint=adj)
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err <= 1e-13, (n, k, adj, err)
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                         env={**os.environ, "BF_NODE_MMA": "1"})
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
