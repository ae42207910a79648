"""Device time of one apply (bf_apply graph replay, CUDA events over many steps) for a
list of chain geometries: `python tools/time_chain.py n:leaf:r:k [...]` (binary trees,
synthetic factors). Used to compare launch paths (BF_NO_NODE, BF_NO_PDL, ...)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200.synthetic import synthetic_chain  # noqa: E402


def time_one(n, leaf, r, k, steps=200):
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=1, device="cuda")
    plan = f.plan()
    g = torch.randn((n, k), dtype=torch.complex128, device="cuda")
    out = torch.empty_like(g)
    ws = torch.empty(plan.workspace_bytes(k), dtype=torch.uint8, device="cuda")
    for _ in range(10):
        plan.apply(g, out=out, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        plan.apply(g, out=out, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    host = e0.elapsed_time(e1) / steps * 1e3
    # device time: `reps` applies captured into one CUDA graph (no host launch cost per apply)
    reps = 50
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg, capture_error_mode="thread_local"):
        for _ in range(reps):
            plan.apply(g, out=out, workspace=ws)
    cg.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        cg.replay()
    e1.record()
    torch.cuda.synchronize()
    return host, e0.elapsed_time(e1) / (4 * reps) * 1e3


if __name__ == "__main__":
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("BF_"))
    for spec in sys.argv[1:]:
        n, leaf, r, k = spec.split(":")
        leaf = float(leaf) if "." in leaf else int(leaf)
        host, dev = time_one(int(n), leaf, int(r), int(k))
        print(f"{spec:>20} host-loop {host:9.2f} us  device (graph of applies) {dev:9.2f} us  {tag}")
