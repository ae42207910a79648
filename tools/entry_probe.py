"""Device entries vs the reference's golden entries (tests/golden/entries.npz): size of
the differences, and which part of the phase they come from."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1502_01379_b200 as bf

d = dict(np.load(os.path.join(ROOT, "tests", "golden", "entries.npz")))
for n in (1024, 1 << 16, 1 << 20, 1 << 24):
    rows, cols, want = d[f"fio_{n}_rows"], d[f"fio_{n}_cols"], d[f"fio_{n}"]
    got = bf.FioKernel(n).block(rows, cols)
    diff = np.abs(got - want)
    print(n, "max |diff| %.3e  nonzero %d/%d" % (diff.max(), (diff > 0).sum(), diff.size))
