"""clock64 phases of CTA 0 of the tcgen05 complex64 level kernel (bf_debug_node_trace):
wait for the raw tile, split, MMA issue, MMA completion, epilogue. `python tools/tc_trace.py n leaf r k`"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200 import _lib  # noqa: E402
from paper_1502_01379_b200.synthetic import synthetic_chain  # noqa: E402

n, leaf, r, k = (int(x) for x in sys.argv[1:5])
f = synthetic_chain(bf.make_partition(n, leaf), r, seed=1, device="cuda")
plan = f.plan("c64")
x = torch.randn((n, k), dtype=torch.complex64, device="cuda")
tr = torch.zeros(4096, dtype=torch.int64, device="cuda")
lib = _lib.load()
ws = torch.empty(plan.workspace_bytes(k), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
plan.apply(x, out=out, workspace=ws)
torch.cuda.synchronize()
lib.bf_debug_node_trace(ctypes.c_void_p(tr.data_ptr()))
out = torch.empty_like(x)   # new buffers: a fresh graph captures the trace pointer
lib.bf_apply(plan._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), k, 0,
             ctypes.c_void_p(ws.data_ptr()), ws.numel(), None)
torch.cuda.synchronize()
lib.bf_debug_node_trace(None)
t = tr.cpu().numpy()[:128].reshape(16, 8).astype(np.int64)
# split warp 0: 0 planes free, 1 raw landed, 2 planes written; epilogue warp 4: 3 tile stored
for it in range(16):
    if not t[it, 0]:
        continue
    print(it, "wait raw", t[it, 1] - t[it, 0], "split", t[it, 2] - t[it, 1], "| epilogue done at +",
          t[it, 3] - t[0, 0], "split done at +", t[it, 2] - t[0, 0])
