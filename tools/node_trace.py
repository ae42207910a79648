"""Per-CTA %globaltimer stamps of the node kernels (bf_debug_node_trace) for one apply:
where a half's time goes (prefetch issue, wait on the previous kernel, input staging,
each step). `python tools/node_trace.py n:leaf:r:k`."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200 import _lib  # noqa: E402
from paper_1502_01379_b200.synthetic import synthetic_chain  # noqa: E402

for spec in sys.argv[1:]:
    n, leaf, r, k = (int(x) for x in spec.split(":"))
    p = bf.make_partition(n, leaf)
    f = synthetic_chain(p, r, seed=1, device="cuda")
    plan = f.plan()
    buf = torch.zeros(2 * 4096 * 32, dtype=torch.int64, device="cuda")
    _lib.load().bf_debug_node_trace(ctypes.c_void_p(buf.data_ptr()))
    g = torch.randn((n, k), dtype=torch.complex128, device="cuda")
    out = torch.empty_like(g)
    ws = torch.empty(plan.workspace_bytes(k), dtype=torch.uint8, device="cuda")
    for _ in range(5):
        plan.apply(g, out=out, workspace=ws)
    torch.cuda.synchronize()
    flat = buf.cpu().numpy()
    _lib.load().bf_debug_node_trace(None)
    ctas = int((flat.reshape(-1, 32)[:, 0] > 0).sum()) // 2
    t = flat[:2 * ctas * 32].reshape(2, ctas, 32)
    t0 = t[0, :ctas, 0].min()
    for half, name in ((0, "down"), (1, "up")):
        x = t[half, :ctas].astype(np.float64)
        x[x == 0] = np.nan
        rel = (x - t0) / 1e3
        print(f"{spec} {name}: stamps (us from down start), CTA median / max")
        print("   ", " ".join(f"{i}:{np.nanmedian(rel[:, i]):.2f}/{np.nanmax(rel[:, i]):.2f}"
                               for i in range(23) if not np.all(np.isnan(rel[:, i]))))
        cyc = t[half, :ctas, 23:29].astype(np.int64)
        if cyc[:, 0].any():
            med = lambda j, i: int(np.median(cyc[:, j] - cyc[:, i]))  # noqa: E731
            print("    last deferred step, SM cycles (CTA median): setup", med(3, 0), "dot loop", med(4, 3),
                  "shuffles", med(5, 4), "to barrier", med(1, 5), "barrier", med(2, 1))
