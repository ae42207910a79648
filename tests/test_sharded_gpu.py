"""libbfly's sharded steps (bf_apply_down / bf_middle_pack / bf_middle_unpack /
bf_apply_up) for P parts, emulated in one process on one GPU: each part's
steps run in turn and the all-to-all is done by slicing the send buffers (no
part waits on another). The concatenated outputs must equal the full apply."""

import numpy as np
import pytest

import paper_1502_01379_b200 as bf
from conftest import complex_gaussian
from paper_1502_01379_b200.sharded import ShardedPlan
from paper_1502_01379_b200.synthetic import synthetic_chain

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def emulate(plans, g, adjoint):
    P = len(plans)
    n_local = plans[0].n_local
    sends = [pl.pack(pl.down(g[d * n_local:(d + 1) * n_local], adjoint), adjoint) for d, pl in enumerate(plans)]
    chunk = plans[0].chunk_rows
    outs = []
    for e, pl in enumerate(plans):
        recv = torch.cat([sends[d][e * chunk:(e + 1) * chunk] for d in range(P)])
        outs.append(pl.up(pl.unpack(recv, adjoint), adjoint))
    return torch.cat(outs)


@pytest.mark.parametrize("n,leaf,r,k,P,dtype", [
    (1 << 12, 16, 8, 1, 2, "c128"),
    (1 << 14, 16, 16, 3, 4, "c128"),
    (1 << 12, 0.25, 4, 2, 8, "c128"),
    (1 << 16, 16, 8, 64, 8, "c128"),   # config-1 geometry, many-RHS kernel
    (1 << 14, 16, 16, 1, 4, "c64"),
    (1 << 14, 16, 16, 16, 4, "c128"),  # rank 16, many RHS: every part runs on its branching-4 twin
    (1 << 14, 16, 16, 64, 2, "c64"),
])
def test_sharded_steps_match_full_apply(n, leaf, r, k, P, dtype):
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=n + P)
    plans = [ShardedPlan.from_factors(f, d, P, dtype=dtype) for d in range(P)]
    g = torch.from_numpy(complex_gaussian(np.random.default_rng(1), (n, k))).cuda()
    full = f.plan(dtype)
    tol = 1e-13 if dtype == "c128" else 1e-6
    for adjoint in (False, True):
        want = full.apply(g, adjoint=adjoint)
        got = emulate(plans, g, adjoint)
        err = (torch.linalg.norm(got - want) / torch.linalg.norm(want)).item()
        assert err <= tol, (adjoint, err)


def test_sharded_plan_rejects_full_apply_and_bad_parts():
    p = bf.make_partition(1 << 12, 16)
    f = synthetic_chain(p, 4, seed=3)
    pl = ShardedPlan.from_factors(f, 0, 2)
    from paper_1502_01379_b200 import _lib
    import ctypes
    x = torch.zeros((p.n, 1), dtype=torch.complex128, device="cuda")
    ws = torch.empty(pl.lib.bf_apply_workspace_bytes(pl._h, 1), dtype=torch.uint8, device="cuda")
    rc = pl.lib.bf_apply(pl._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(x.data_ptr()), 1, 0,
                         ctypes.c_void_p(ws.data_ptr()), ws.numel(), None)
    assert rc == _lib.BF_EINVAL
    with pytest.raises(ValueError):
        ShardedPlan.from_factors(f, 0, 3)


def test_sharded_quadtree_steps():
    p = bf.make_quadtree_partition(64, 4)
    f = synthetic_chain(p, 8, seed=4)
    plans = [ShardedPlan.from_factors(f, d, 4) for d in range(4)]
    g = torch.from_numpy(complex_gaussian(np.random.default_rng(2), (p.n, 2))).cuda()
    for adjoint in (False, True):
        want = f.plan().apply(g, adjoint=adjoint)
        got = emulate(plans, g, adjoint)
        assert (torch.linalg.norm(got - want) / torch.linalg.norm(want)).item() <= 1e-13


@pytest.mark.parametrize("n,leaf,r,k,P", [(1 << 12, 16, 8, 1, 2), (1 << 14, 16, 16, 3, 4), (1 << 16, 16, 8, 64, 8),
                                         (1 << 14, 16, 16, 32, 4)])
def test_fused_push_exchange_emulated(n, leaf, r, k, P):
    """bf_apply_down_push: the last down level stores (weights applied) straight into every
    part's receive buffer — emulated with P local buffers on one GPU (each part's push runs
    in turn; nothing waits on another part). Unpack + up of each part must reproduce the
    full apply, bitwise equal to the pack + all-to-all path."""
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=n + 3 * P)
    plans = [ShardedPlan.from_factors(f, d, P) for d in range(P)]
    g = torch.from_numpy(complex_gaussian(np.random.default_rng(1), (n, k))).cuda()
    nl, chunk = plans[0].n_local, plans[0].chunk_rows
    for adjoint in (False, True):
        recv = [torch.zeros((P * chunk, k), dtype=torch.complex128, device="cuda") for _ in range(P)]
        for d, pl in enumerate(plans):
            pl.down_push(g[d * nl:(d + 1) * nl], adjoint, [b.data_ptr() for b in recv])
        got = torch.cat([pl.up(pl.unpack(recv[e], adjoint), adjoint) for e, pl in enumerate(plans)])
        want = f.plan().apply(g, adjoint=adjoint)
        assert (torch.linalg.norm(got - want) / torch.linalg.norm(want)).item() <= 1e-13
        assert torch.equal(got, emulate(plans, g, adjoint))


class _Loopback:
    """In-process stand-in for the all-to-all / all-gather of factorize_part: parts run in
    Python threads on one GPU and meet at host barriers (no kernel waits on another)."""

    def __init__(self, n):
        import threading
        self.n, self.bar, self.slots = n, threading.Barrier(n), [None] * n

    def exchange(self, part):
        def run(send):
            torch.cuda.synchronize()
            self.slots[part] = send
            self.bar.wait()
            recv = torch.stack([self.slots[e][part].clone() for e in range(self.n)])
            torch.cuda.synchronize()
            self.bar.wait()
            return recv
        return run

    def gather(self, part):
        def run(rows):
            torch.cuda.synchronize()
            self.slots[part] = rows
            self.bar.wait()
            out = torch.cat([self.slots[e].clone() for e in range(self.n)])
            torch.cuda.synchronize()
            self.bar.wait()
            return out
        return run


@pytest.mark.parametrize("n,leaf,r,nparts", [(1024, 8, 12, 2), (4096, 16, 8, 4)])
def test_sharded_construction_bitwise_equal_to_factorize(n, leaf, r, nparts):
    """factorize_part's slices == shard_slices(factorize(...)) bit for bit (every block has
    its own SeedSequence, so the split over parts cannot change a number)."""
    import threading

    from paper_1502_01379_b200 import construct as bc
    from paper_1502_01379_b200.sharded import shard_slices
    p = bf.make_partition(n, leaf)
    ker = bf.FioKernel(n)
    full = bf.factorize(ker, p, r, seed=3)
    lb = _Loopback(nparts)
    out = [None] * nparts
    errs = []

    def work(d):
        try:
            out[d] = bc.factorize_part(ker, p, r, d, nparts, seed=3, exchange=lb.exchange(d), gather=lb.gather(d))
        except Exception as exc:  # surfaced below
            errs.append(exc)
            lb.bar.abort()

    ths = [threading.Thread(target=work, args=(d,)) for d in range(nparts)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    assert not errs, errs
    for d in range(nparts):
        want = shard_slices(full, d, nparts)
        got = out[d]
        assert torch.equal(got["weights"], want["weights"])
        assert torch.equal(got["u_leaf"], want["u_leaf"]) and torch.equal(got["v_leaf"], want["v_leaf"])
        for key in ("g", "h"):
            for (l1, b1), (l2, b2) in zip(got[key], want[key]):
                assert l1 == l2 and torch.equal(b1, b2), (key, l1)
