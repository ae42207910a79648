"""Multi-process (gloo, world size 2 and 4) check of the sharded apply's host
logic: factor slicing, the middle pack/exchange/unpack and the down/up split
reproduce the full chain. Local steps here are the oracle's
per-factor maps (test-only subclass); on the GPU they are libbfly.so."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1502_01379_b200 as bf
from oracle import chain as ochain
from paper_1502_01379_b200.sharded import ShardedApply, shard_slices
from paper_1502_01379_b200.synthetic import synthetic_chain


class OracleShard(ShardedApply):
    def __init__(self, f, part, nparts):
        super().__init__(f.partition, f.rank, part, nparts)
        self.s = shard_slices(f, part, nparts)

    def down(self, x, adjoint):
        w = x.numpy().reshape(self.n_local, -1)
        lead, levels = (self.s["u_leaf"], self.s["g"]) if adjoint else (self.s["v_leaf"], self.s["h"])
        w = ochain.leaf_adjoint(lead, w)
        for _, b in reversed(levels):
            w = ochain.transfer_adjoint(b, w)
        return torch.from_numpy(np.ascontiguousarray(w))

    def pack(self, mid, adjoint):
        m, mp_, r, P = self.p.mid_nodes, self.mp, self.r, self.nparts
        W = self.s["weights"]
        x = mid.numpy().reshape(mp_, m, r, -1)
        out = np.empty((P, mp_, mp_, r, x.shape[-1]), dtype=complex)
        for e in range(P):
            for a in range(mp_):
                own = self.part * mp_ + a
                for bl in range(mp_):
                    other = e * mp_ + bl
                    wv = W[own, other] if adjoint else W[other, own]
                    out[e, a, bl] = wv[:, None] * x[a, other]
        return torch.from_numpy(out.reshape(P * mp_ * mp_ * r, -1))

    def unpack(self, recv, adjoint):
        m, mp_, r, P = self.p.mid_nodes, self.mp, self.r, self.nparts
        x = recv.numpy().reshape(P, mp_, mp_, r, -1)
        out = np.empty((mp_, m, r, x.shape[-1]), dtype=complex)
        for d in range(P):
            for a in range(mp_):
                out[:, d * mp_ + a] = x[d, a]
        return torch.from_numpy(out.reshape(mp_ * m * r, -1))

    def up(self, mid, adjoint):
        w = mid.numpy()
        levels, trail = (self.s["h"], self.s["v_leaf"]) if adjoint else (self.s["g"], self.s["u_leaf"])
        for _, b in levels:
            w = ochain.transfer_forward(b, w)
        return torch.from_numpy(ochain.leaf_forward(trail, w))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, leaf, r, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = bf.make_partition(n, leaf)
        f = synthetic_chain(p, r, seed=77)
        g = np.random.default_rng(5).standard_normal((n, k)) + 1j * np.random.default_rng(6).standard_normal((n, k))
        sh = OracleShard(f, rank, world)
        rows = slice(rank * n // world, (rank + 1) * n // world)
        res = []
        for adjoint in (False, True):
            out = sh.apply(torch.from_numpy(g[rows]), adjoint=adjoint)
            parts = [torch.empty_like(out) for _ in range(world)]
            dist.all_gather(parts, out)
            res.append(torch.cat(parts).numpy())
        if rank == 0:
            c = ochain.Chain(n, p.levels, r, f.u_outer.blocks, [(t.level, t.blocks) for t in f.g_chain],
                             f.middle.weights, [(t.level, t.blocks) for t in f.h_chain], f.v_outer.blocks)
            errs = [np.linalg.norm(res[i] - ochain.apply(c, g, adjoint=bool(i))) / np.linalg.norm(res[i])
                    for i in range(2)]
            q.put(errs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,leaf,r,k", [(2, 1024, 8, 4, 3), (4, 4096, 16, 5, 2), (2, 256, 0.25, 3, 1)])
def test_sharded_chain_matches_full_apply(world, n, leaf, r, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, world, port, n, leaf, r, k, q)) for i in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    assert all(pr.exitcode == 0 for pr in procs)
    errs = q.get(timeout=5)
    assert max(errs) <= 1e-13, errs


def test_shard_slices_geometry():
    p = bf.make_partition(1024, 8)
    f = synthetic_chain(p, 4, seed=1)
    s = shard_slices(f, 1, 4)
    assert s["u_leaf"].shape[0] == f.u_outer.blocks.shape[0] // 4
    for (lvl, b), t in zip(s["g"], f.g_chain):
        assert lvl == t.level and b.shape[0] == t.blocks.shape[0] // 4
    with pytest.raises(ValueError):
        shard_slices(f, 0, 3)
