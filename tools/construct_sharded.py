"""Node-sharded construction + apply on P GPUs, never materialising the whole chain:
each rank builds its slices with factorize_part (NCCL all-to-all of the v0 sigma0
pieces, all-gather of the weights), wraps them in a ShardedPlan and applies.

  torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/construct_sharded.py [cfg0|cfg1|cfg2]

Rank 0 prints construction time (max over ranks) and the sampled-row accuracy
eps_a of the sharded chain against direct row sums (bench.py:84-97's metric).
"""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200.construct import factorize_part  # noqa: E402
from paper_1502_01379_b200.sharded import ShardedPlan  # noqa: E402

CFG = {"cfg0": ("fio", 1 << 10, 12, 8), "cfg1": ("dftp", 1 << 16, 8, 16), "cfg2": ("fio", 1 << 20, 16, 16)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    kind, n, r, leaf = CFG[name]
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl" if world > 1 else "gloo", init_method="env://") if world > 1 else None
    p = bf.make_partition(n, leaf)
    ker = bf.FioKernel(n) if kind == "fio" else bf.DftPlusKernel(n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    slices = factorize_part(ker, p, r, rank, world, seed=0)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    sp = ShardedPlan(p, r, rank, world, slices)
    rng = np.random.default_rng(np.random.SeedSequence(0, spawn_key=(4, 0)))
    sample = np.sort(rng.choice(n, size=min(256, n), replace=False))
    g = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    nl = n // world
    out = sp.apply(torch.from_numpy(g[rank * nl:(rank + 1) * nl].reshape(nl, 1)).cuda())
    if world > 1:
        parts = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(parts, out)
        out = torch.cat(parts)
        tt = torch.tensor([t], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    if rank == 0:
        exact = bf.RowSampledReference(ker).rows(g, sample)
        err = np.linalg.norm(out.cpu().numpy()[sample, 0] - exact) / np.linalg.norm(exact)
        print(json.dumps({"config": name, "parts": world, "construction_s": t, "eps_a": float(err)}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
