"""ncu driver: one block-row of cfg2 middle blocks + one slab recursion."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200 import construct as bc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n, r, leaf = {"cfg1": (1 << 16, 8, 16), "cfg2": (1 << 20, 16, 16)}[name]
p = bf.make_partition(n, leaf)
ker = bf.FioKernel(n) if name == "cfg2" else bf.DftPlusKernel(n)
ms = bc.MiddleSampler(ker, p, r, seed=0)
u, v, w = ms.blocks([(0, j) for j in range(p.mid_nodes)])
slab = u.permute(1, 0, 2).reshape(1, p.mid_side, p.mid_nodes, r)
bc.recurse(slab, p, r)
torch.cuda.synchronize()
print("ok")
