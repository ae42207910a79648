"""Break down the host-buffer (e2e) apply of cfg2: device chain alone, H2D/D2H
alone (pinned), and the pipelined bf_apply_host. Usage: python tools/e2e_probe.py [reps]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200.synthetic import synthetic_chain  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
p = bf.make_partition(1 << 20, 16)
f = synthetic_chain(p, 16, device="cuda")
pl = f.plan()
n = p.n
g = torch.randn((n, 1), dtype=torch.complex128, device="cuda")
gh = g.cpu().pin_memory()
oh = torch.empty_like(gh).pin_memory()


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2] * 1e3


out = torch.empty_like(g)
print("device chain ms", timeit(lambda: pl.apply(g, out=out)))
print("h2d 16.8MB ms", timeit(lambda: g.copy_(gh, non_blocking=True)))
print("d2h 16.8MB ms", timeit(lambda: oh.copy_(g, non_blocking=True)))
print("host apply ms (chunks=%s)" % os.environ.get("BF_PIPE_CHUNKS", "default 4"), timeit(lambda: pl.apply(gh.numpy(), out=oh.numpy())))
