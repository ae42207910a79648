"""Per-level timing of bf_recurse_level on a cfg2-shaped slab (1, 4096, 256, 16)."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200 import _lib  # noqa: E402

p = bf.make_partition(1 << 20, 16)
r = 16
lib = _lib.load()
nslab = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cur = torch.randn((nslab, p.mid_side, p.mid_nodes, r, 2), dtype=torch.float64, device="cuda")
cur = torch.view_as_complex(cur).contiguous()
for lvl in range(p.half, p.levels):
    nb, rows, groups, _ = cur.shape
    pairs = groups // 2
    blocks = torch.empty((nb, 2, pairs, r, 2 * r), dtype=torch.complex128, device="cuda")
    nxt = torch.empty((2 * nb, rows // 2, pairs, r), dtype=torch.complex128, device="cuda")
    need = ctypes.c_uint64(0)
    lib.bf_recurse_level(r, 2, nb, rows, groups, None, None, None, None, ctypes.byref(need), None)
    ws = torch.empty(max(int(need.value), 16), dtype=torch.uint8, device="cuda")
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(lib.bf_recurse_level(r, 2, nb, rows, groups, ctypes.c_void_p(cur.data_ptr()),
                                        ctypes.c_void_p(blocks.data_ptr()), ctypes.c_void_p(nxt.data_ptr()),
                                        ctypes.c_void_p(ws.data_ptr()), ctypes.byref(need), None))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"level {lvl}: problems {nb * 2 * pairs} of ({rows // 2} x {2 * r}): {dt * 1e3:.2f} ms")
    cur = nxt
