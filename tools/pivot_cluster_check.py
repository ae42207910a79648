"""Middle-block factors of one block-row (cfg1 / cfg2 geometry) with the current
pivot-kernel selection, saved for a bitwise comparison between runs with and
without BF_NO_PIVOT_CLUSTER=1. Usage: python tools/pivot_cluster_check.py OUT.pt"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200 import construct as bc  # noqa: E402

res = {}
for name, (kern, n, r, leaf, rows) in {"cfg1": (bf.DftPlusKernel, 1 << 16, 8, 16, [0, 17]),
                                       "cfg2": (bf.FioKernel, 1 << 20, 16, 16, [5])}.items():
    p = bf.make_partition(n, leaf)
    ms = bc.MiddleSampler(kern(n), p, r, seed=0)
    ij = [(i, j) for i in rows for j in range(p.mid_nodes)]
    u, v, w = ms.blocks(ij)
    res[name] = (u.cpu(), v.cpu(), w.cpu())
torch.save(res, sys.argv[1])
print("saved", sys.argv[1])
