"""Per-block rng.choice draw tables of the sampling construction (host side).

Kept free of torch / CUDA imports: large tables are made by running this module
as a fresh helper process (``python -m paper_1502_01379_b200._draws``) that forks
its own NumPy-only workers, so the CUDA-initialised, multi-threaded caller is
never forked and no start method has to re-run the caller's ``__main__``.
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


def draw_tables_parallel(seed, side, rqs, iters, blocks, workers):
    """All blocks' tables with a fork pool — only ever called inside the helper process."""
    import multiprocessing
    from concurrent.futures import ProcessPoolExecutor
    chunks = [blocks[k::workers] for k in range(workers)]
    with ProcessPoolExecutor(workers, mp_context=multiprocessing.get_context("fork")) as ex:
        parts = list(ex.map(draws_for, [(seed, side, rqs, iters, c) for c in chunks]))
    out = np.empty((len(blocks), 2 * (iters + 1), rqs), dtype=np.int32)
    for k, part in enumerate(parts):
        out[k::workers] = part
    return out


if __name__ == "__main__":
    import pickle
    import sys
    seed, side, rqs, iters, blocks, workers = pickle.load(sys.stdin.buffer)
    tab = draw_tables_parallel(seed, side, rqs, iters, [tuple(b) for b in blocks.tolist()], workers)
    sys.stdout.buffer.write(np.ascontiguousarray(tab).tobytes())
    sys.stdout.buffer.flush()
