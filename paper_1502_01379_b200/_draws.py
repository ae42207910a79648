"""Per-block rng.choice draw tables of the sampling construction (host side).

Kept free of torch / CUDA imports so a process pool can start its workers
with the "spawn" method (forking a CUDA-initialised, multi-threaded process is
unsafe): each worker imports only NumPy and this module.
"""

from __future__ import annotations

import numpy as np

SAMPLING_DOMAIN = 0  # construct.py:26


def block_rng(seed, *key) -> np.random.Generator:
    """Independent generator for one construction sub-task (construct.py:31-33)."""
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=key))


def draws_for(args):
    """Draw tables of a list of blocks: 2*(iters+1) rng.choice(side, rqs) per block, in the
    reference's consumption order row, col, row, col, ... (lowrank.py:237-251)."""
    seed, side, rqs, iters, blocks = args
    out = np.empty((len(blocks), 2 * (iters + 1), rqs), dtype=np.int32)
    for b, (i, j) in enumerate(blocks):
        rng = block_rng(seed, SAMPLING_DOMAIN, int(i), int(j))
        for s in range(2 * (iters + 1)):
            out[b, s] = rng.choice(side, size=rqs, replace=False)
    return out
