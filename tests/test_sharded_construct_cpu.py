"""Multi-process (gloo, world size 2 and 4) check of the sharded construction's
orchestration (construct.factorize_part): each part computes
only its block rows, the v0 sigma0 pieces reach the owners of their columns by
one all-to-all per row step, the weight rows are all-gathered, and every part
ends with exactly the slices shard_slices cuts from the single-part result.
The middle blocks and the recursion are host fakes here (deterministic
functions of the block / slab); on the GPU they are libbfly.so and the full
equality is tested in tests/test_sharded_gpu.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1502_01379_b200 as bf
from oracle import construct as ocons
from paper_1502_01379_b200 import construct as bc


def fake_blocks(p, r):
    side, m = p.mid_side, p.mid_nodes

    def blocks(ij):
        uu, vv, ww = [], [], []
        for i, j in ij:
            g = np.random.default_rng(1000 * i + j)
            uu.append(g.standard_normal((side, r)) + 1j * g.standard_normal((side, r)))
            vv.append(g.standard_normal((side, r)) + 1j * g.standard_normal((side, r)))
            ww.append(g.uniform(0.5, 1.5, r))
        return (torch.from_numpy(np.array(uu)), torch.from_numpy(np.array(vv)), torch.from_numpy(np.array(ww)))
    return blocks


def host_recurse(slabs, p, r):
    leaf, pieces = ocons.recurse(slabs.numpy(), p.n, p.levels, r)
    return torch.from_numpy(leaf), [(lvl, torch.from_numpy(b)) for lvl, b in pieces]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cut(a, part, nparts):
    n0 = a.shape[0]
    return a[part * n0 // nparts:(part + 1) * n0 // nparts]


def _worker(rank, world, port, n, leaf, r, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = bf.make_partition(n, leaf)
        got = bc.factorize_part(None, p, r, rank, world, device="cpu", blocks_fn=fake_blocks(p, r),
                                recurse_fn=host_recurse)
        full = bc.factorize_part(None, p, r, 0, 1, device="cpu", blocks_fn=fake_blocks(p, r),
                                 recurse_fn=host_recurse)
        ok = torch.equal(got["weights"], full["weights"])
        ok &= torch.equal(got["u_leaf"], _cut(full["u_leaf"], rank, world))
        ok &= torch.equal(got["v_leaf"], _cut(full["v_leaf"], rank, world))
        for key in ("g", "h"):
            for (l1, b1), (l2, b2) in zip(got[key], full[key]):
                ok &= l1 == l2 and torch.equal(b1, _cut(b2, rank, world))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,leaf,r", [(2, 256, 4, 3), (4, 1024, 16, 4)])
def test_sharded_construction_matches_single_part(world, n, leaf, r):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, world, port, n, leaf, r, q)) for i in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    assert all(pr.exitcode == 0 for pr in procs)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(res.values()), res


def test_factorize_part_rejects_bad_split():
    p = bf.make_partition(256, 4)
    with pytest.raises(ValueError):
        bc.factorize_part(None, p, 3, 0, 3, device="cpu", blocks_fn=fake_blocks(p, 3), recurse_fn=host_recurse)
