"""Device time of the forward apply on a device-drawn synthetic chain (CUDA events around
`reps` applies after a warm-up). Usage: python tools/time_apply.py [cfg] [c128|c64] [k] [reps]
Prints one line: cfg dtype k ms_per_apply plus the BF_* switches set in the environment."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200.synthetic import synthetic_chain  # noqa: E402

CFG = {"cfg0": (1 << 10, 12, 8), "cfg1": (1 << 16, 8, 16), "cfg2": (1 << 20, 16, 16), "cfg3": (256, 25, 4),
       "cfg4b": (1024, 25, 4), "cfg2r4": (1024, 16, 4), "cfg1r4": (256, 8, 4)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dtype = sys.argv[2] if len(sys.argv) > 2 else "c128"
k = int(sys.argv[3]) if len(sys.argv) > 3 else 1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
n, r, leaf = CFG[name]
p = bf.make_quadtree_partition(n, leaf) if name in ("cfg3", "cfg4b", "cfg2r4", "cfg1r4") else bf.make_partition(n, leaf)
n = p.n
f = synthetic_chain(p, r, device="cuda")
pl = f.plan(dtype)
g = torch.randn((n, k), dtype=torch.complex128, device="cuda").to(pl.torch_dtype)
ref = None
for _ in range(3):
    out = pl.apply(g)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    out = pl.apply(g)
e1.record()
torch.cuda.synchronize()
sw = " ".join(f"{a}={b}" for a, b in sorted(os.environ.items()) if a.startswith("BF_"))
print(f"{name} {dtype} k={k} {e0.elapsed_time(e1) / reps:.4f} ms/apply  checksum {float(out.abs().sum()):.10e}  [{sw}]", flush=True)
