"""Minimal driver for ncu: build the config-2 plan (synthetic factors) and run
a few forward applies. Usage: python tools/profile_apply.py [cfg2|cfg1|cfg0] [c128|c64] [k] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200.synthetic import synthetic_chain  # noqa: E402

CFG = {"cfg0": (1 << 10, 12, 8), "cfg1": (1 << 16, 8, 16), "cfg2": (1 << 20, 16, 16), "cfg3": (256, 25, 4),
       "cfg4b": (1024, 25, 4)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dtype = sys.argv[2] if len(sys.argv) > 2 else "c128"
k = int(sys.argv[3]) if len(sys.argv) > 3 else 1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
n, r, leaf = CFG[name]
p = bf.make_quadtree_partition(n, leaf) if name in ("cfg3", "cfg4b") else bf.make_partition(n, leaf)
n = p.n
f = synthetic_chain(p, r, device="cuda")
pl = f.plan(dtype)
g = torch.randn((n, k), dtype=torch.complex128, device="cuda").to(pl.torch_dtype)
for _ in range(reps):
    out = pl.apply(g)
torch.cuda.synchronize()
print("ok", name, dtype, k, float(out.abs().sum()))
