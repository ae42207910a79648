"""Seeded synthetic factor chains at exact ``_level_geometry`` shapes.

Benchmark inputs for configs whose CPU construction is infeasible (BASELINE
config 2 takes ~10-19 h in the reference, config 4a does not fit host RAM):
blocks are complex Gaussians scaled by 1/sqrt(2*cols) (so every level
roughly preserves the vector norm), middle weights U(0.5, 1.5) as in the
reference's ``conftest.random_exact_chain`` (pkg/tests/conftest.py:20-39),
drawn in the order V^L, H levels ascending, M, G levels ascending, U^L.
``random_exact_chain`` itself is not used: it requires leaf rows <= r and
fails at leaf 16.
"""

from __future__ import annotations

import numpy as np

from .factors import BlockDiagonalFactor, ButterflyFactors, MiddleFactor, TransferFactor
from .partition import DyadicPartition, level_geometry


def synthetic_chain(p: DyadicPartition, r: int, seed: int = 20240801, device=None) -> ButterflyFactors:
    """Host (NumPy, ``device=None``) or device (torch CUDA tensors) synthetic chain."""
    shapes, leaf_shape = level_geometry(p, r)
    if device is None:
        rng = np.random.default_rng(seed)

        def draw(shape):
            scale = 1.0 / np.sqrt(2.0 * shape[-1])
            out = np.empty(shape, dtype=np.complex128)
            out.real = rng.standard_normal(shape) * scale
            out.imag = rng.standard_normal(shape) * scale
            return out

        def weights():
            return rng.uniform(0.5, 1.5, size=(p.mid_nodes, p.mid_nodes, r))
    else:
        import torch
        gen = torch.Generator(device=device)
        gen.manual_seed(seed)

        def draw(shape):
            scale = 1.0 / np.sqrt(2.0 * shape[-1])
            t = torch.randn(tuple(shape) + (2,), dtype=torch.float64, device=device, generator=gen)
            t.mul_(scale)
            return torch.view_as_complex(t)

        def weights():
            w = torch.rand((p.mid_nodes, p.mid_nodes, r), dtype=torch.float64, device=device, generator=gen)
            return w.add_(0.5)

    v = draw(leaf_shape)
    h = tuple(TransferFactor(lvl, draw(shape)) for lvl, _, shape in shapes)
    w = weights()
    g = tuple(TransferFactor(lvl, draw(shape)) for lvl, _, shape in shapes)
    u = draw(leaf_shape)
    return ButterflyFactors(p, r, BlockDiagonalFactor(u), g, MiddleFactor(w), h, BlockDiagonalFactor(v))


BENCH_CHUNK = 1 << 22   # complex values per independently seeded chunk (thread-count invariant)


def _fill(specs, seed, key0=(), threads=None):
    """Allocate and fill [(kind, shape)] ("c": complex Gaussian / sqrt(2 cols), "w": U(0.5, 1.5))
    chunk by chunk, chunk c of array a from SeedSequence(seed, spawn_key=key0 + (a, c)), on a
    thread pool (NumPy's generators release the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    import os

    arrays = [np.empty(s, dtype=np.complex128 if kind == "c" else np.float64) for kind, s in specs]
    jobs = []
    for fi, ((kind, shape), arr) in enumerate(zip(specs, arrays)):
        flat = arr.reshape(-1)
        for ci, lo in enumerate(range(0, flat.size, BENCH_CHUNK)):
            jobs.append((fi, ci, kind, shape, flat[lo:lo + BENCH_CHUNK]))

    def fill(job):
        fi, ci, kind, shape, out = job
        rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=tuple(key0) + (fi, ci)))
        if kind == "w":
            out[:] = rng.uniform(0.5, 1.5, size=out.size)
            return
        v = out.view(np.float64)                      # interleaved (re, im)
        rng.standard_normal(out=v)
        v *= 1.0 / np.sqrt(2.0 * shape[-1])

    with ThreadPoolExecutor(max_workers=threads or min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(fill, jobs))
    return arrays


def bench_chain(p, r: int, seed: int = 20240801, threads: int | None = None) -> ButterflyFactors:
    """Host (NumPy) synthetic chain for the benchmark, identical bytes in both bench arms.

    Same distribution and factor order as ``synthetic_chain`` (V^L, H ascending, M, G
    ascending, U^L), but every factor is split into fixed chunks of ``BENCH_CHUNK`` values,
    each drawn from its own ``SeedSequence(seed, spawn_key=(factor, chunk))`` generator, so
    the chunks can be filled by a thread pool and the result does not depend on the thread
    count. cfg2 (9.1 GB) draws in a few seconds instead of ~25 s sequentially."""
    shapes, leaf_shape = level_geometry(p, r)
    specs = [("c", leaf_shape)] + [("c", s) for _, _, s in shapes] + [("w", (p.mid_nodes, p.mid_nodes, r))] \
        + [("c", s) for _, _, s in shapes] + [("c", leaf_shape)]
    arrays = _fill(specs, seed, threads=threads)
    nl = len(shapes)
    v = arrays[0]
    h = tuple(TransferFactor(lvl, a) for (lvl, _, _), a in zip(shapes, arrays[1:1 + nl]))
    w = arrays[1 + nl]
    g = tuple(TransferFactor(lvl, a) for (lvl, _, _), a in zip(shapes, arrays[2 + nl:2 + 2 * nl]))
    u = arrays[-1]
    return ButterflyFactors(p, r, BlockDiagonalFactor(u), g, MiddleFactor(w), h, BlockDiagonalFactor(v))


def bench_slices(p, r: int, part: int, nparts: int, seed: int = 20240801, threads: int | None = None) -> dict:
    """One part's factor slices (the ``shard_slices`` layout: leading index range
    [part/nparts, (part+1)/nparts) of every factor, full weights) drawn on the host, seeded
    per part (spawn keys (1000 + part, factor, chunk)); weights as in ``bench_chain``. For
    chains no host or GPU holds whole (BASELINE config 4a: 180 GB in complex128)."""
    shapes, leaf_shape = level_geometry(p, r)
    loc = lambda s: (s[0] // nparts,) + tuple(s[1:])  # noqa: E731
    specs = [("c", loc(leaf_shape))] + [("c", loc(s)) for _, _, s in shapes] \
        + [("c", loc(s)) for _, _, s in shapes] + [("c", loc(leaf_shape))]
    arrays = _fill(specs, seed, key0=(1000 + part,), threads=threads)
    w = _fill([("w", (p.mid_nodes, p.mid_nodes, r))], seed, key0=(2000,), threads=threads)[0]
    nl = len(shapes)
    return {"v_leaf": arrays[0], "h": [(lvl, a) for (lvl, _, _), a in zip(shapes, arrays[1:1 + nl])],
            "weights": w, "g": [(lvl, a) for (lvl, _, _), a in zip(shapes, arrays[1 + nl:1 + 2 * nl])],
            "u_leaf": arrays[-1]}


def to_host(f: ButterflyFactors) -> ButterflyFactors:
    """NumPy copy of a (possibly device-resident) chain."""
    def h(a):
        return a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)

    return ButterflyFactors(f.partition, f.rank, BlockDiagonalFactor(h(f.u_outer.blocks)),
                            tuple(TransferFactor(t.level, h(t.blocks)) for t in f.g_chain),
                            MiddleFactor(h(f.middle.weights)),
                            tuple(TransferFactor(t.level, h(t.blocks)) for t in f.h_chain),
                            BlockDiagonalFactor(h(f.v_outer.blocks)))


def synthetic_slices(p, r: int, part: int, nparts: int, seed: int = 20240801, device=None) -> dict:
    """One part's factor slices (the ``shard_slices`` layout) drawn directly, seeded per part,
    for chains too large to materialise whole (BASELINE config 4a: 180 GB in complex128).
    Equivalent in distribution to slicing a synthetic chain; weights are shared by all parts."""
    import torch
    shapes, leaf_shape = level_geometry(p, r)
    gen = torch.Generator(device=device or "cpu")
    gen.manual_seed(seed * 1009 + part)
    dev = device or "cpu"

    def draw(shape):
        shape = (shape[0] // nparts,) + tuple(shape[1:])
        t = torch.randn(shape + (2,), dtype=torch.float64, device=dev, generator=gen)
        t.mul_(1.0 / np.sqrt(2.0 * shape[-1]))
        return torch.view_as_complex(t)

    wgen = torch.Generator(device=dev)
    wgen.manual_seed(seed)
    weights = torch.rand((p.mid_nodes, p.mid_nodes, r), dtype=torch.float64, device=dev, generator=wgen).add_(0.5)
    return {"v_leaf": draw(leaf_shape), "h": [(lvl, draw(s)) for lvl, _, s in shapes], "weights": weights,
            "g": [(lvl, draw(s)) for lvl, _, s in shapes], "u_leaf": draw(leaf_shape)}
