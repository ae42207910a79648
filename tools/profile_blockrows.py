"""ncu driver: one middle launch of cfg2 block-rows (4 rows = 1,024 blocks, factorize's batch)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200 import construct as bc  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n, r, leaf = 1 << 20, 16, 16
p = bf.make_partition(n, leaf)
ms = bc.MiddleSampler(bf.FioKernel(n), p, r, seed=0)
for rep in range(2):
    u, v, w = ms.blocks([(i, j) for i in range(rows) for j in range(p.mid_nodes)])
torch.cuda.synchronize()
print("ok")
