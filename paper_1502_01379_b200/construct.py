"""Sampling construction of the factor chain on the B200 — the reference's
``construct.py`` entry point ``factorize`` (same signature, modes, errors),
with every numeric stage in libbfly.so:

* middle level: ``bf_middle_blocks`` — one CTA per block runs the randomized
  sampling SVD (lowrank.py:219-258) on entries evaluated on the device;
* recursion: ``bf_recurse_level`` — batched SVD of the (rows/2 x 2r) stacks
  (construct.py:127-163);
* matvec mode: probe products through the operator oracle (device-resident for
  this package's own chains and ComposedOperator), then ``bf_middle_probes`` —
  one CTA per block finishes svd_from_probes (lowrank.py:204-216).

The host keeps only geometry and the random draws: each block's
``rng.choice`` draws come from the reference's own generator
``SeedSequence(seed, spawn_key=(0, i, j))`` (construct.py:31-33), which makes
them identical to the reference's and independent of the schedule — so
"sampling" and "streaming" produce bitwise-identical factors, as in the
reference (pkg/tests/test_construct.py:197-202).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._draws import block_rng, draws_for
from .factors import BlockDiagonalFactor, ButterflyFactors, MiddleFactor, TransferFactor
from .kernels import is_entry_oracle, is_operator_oracle
from .partition import DyadicPartition, level_geometry

SAMPLING_DOMAIN = 0   # construct.py:26
COL_PROBE_DOMAIN = 1  # construct.py:27
ROW_PROBE_DOMAIN = 2  # construct.py:28


@dataclass(frozen=True)
class OversamplingParams:
    """p extra probe columns, q sample multiplier, iters skeleton sweeps (lowrank.py:33-48)."""

    p: int = 5
    q: int = 3
    iters: int = 3

    def __post_init__(self):
        if self.p < 0 or self.q < 1 or self.iters < 1:
            raise ValueError(f"invalid oversampling parameters {self}")


DEFAULT_PARAMS = OversamplingParams()


_draws_for = draws_for


def draw_tables(seed, side: int, r: int, params: OversamplingParams, blocks) -> np.ndarray:
    """The reference's per-block rng.choice draws, in consumption order."""
    rqs = min(r * params.q, side)
    blocks = list(blocks)
    if len(blocks) < 2048:
        return _draws_for((seed, side, rqs, params.iters, blocks))
    # large tables: a fresh helper interpreter (NumPy only) forks its own workers, so this
    # CUDA-initialised, multi-threaded process is never forked (see _draws.py)
    import pickle
    import subprocess
    import sys
    workers = min(16, os.cpu_count() or 1)
    arr = np.asarray(blocks, dtype=np.int64).reshape(-1, 2)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {**os.environ, "PYTHONPATH": root + os.pathsep + os.environ.get("PYTHONPATH", "")}
    res = subprocess.run([sys.executable, "-m", "paper_1502_01379_b200._draws"],
                         input=pickle.dumps((seed, side, rqs, params.iters, arr, workers)),
                         capture_output=True, env=env, check=False)
    if res.returncode != 0:
        raise RuntimeError("draw-table helper failed: " + res.stderr.decode(errors="replace")[-2000:])
    return np.frombuffer(res.stdout, dtype=np.int32).reshape(len(blocks), 2 * (params.iters + 1), rqs).copy()


class _DeviceOracle:
    """How the device reads an entry oracle (SURVEY.md §8(b) "entry-oracle plugin protocol").

    * analytic kernels by id (FIO, the config-1 DFT(+), the reference's centered DftKernel,
      the 2-D Radon kernel), recognised by ``kernel_id`` or, for the reference's own
      classes, by type name and ``n``;
    * an explicit matrix (``DenseOracle``) or a cached Hankel table: a dense device source;
    * anything else with ``.block(rows, cols)`` — including an uncached or too-large
      Hankel kernel — through per-middle-block windows (``tiles``): each block's
      side x side window is evaluated (host ``oracle.block`` through the BlockView
      offsets, oracles.py:57-68, or a device producer) and uploaded batch by batch, so
      memory stays bounded by the batch instead of the dense n x n matrix."""

    def __init__(self, oracle, n):
        torch = _lib.require_cuda()
        self.oracle, self.n = oracle, n
        self.dense = None
        self.tiles = None           # callable(list of (i, j), side) -> device (nb, side, side)
        kid = getattr(oracle, "kernel_id", None)
        name = type(oracle).__name__
        if kid in (_lib.BF_KERNEL_FIO, _lib.BF_KERNEL_DFTP, _lib.BF_KERNEL_RADON2D, _lib.BF_KERNEL_DFT):
            self.kernel_id = kid
        elif name == "FioKernel" and getattr(oracle, "n", None) == n:   # the reference's own class
            self.kernel_id = _lib.BF_KERNEL_FIO
        elif name == "DftKernel" and getattr(oracle, "n", None) == n:   # the reference's own class
            self.kernel_id = _lib.BF_KERNEL_DFT
        elif name == "HankelKernel" and getattr(oracle, "n", None) == n:
            from .kernels import HankelKernel
            mine = oracle if hasattr(oracle, "device_table") else \
                HankelKernel(n, cache=bool(getattr(oracle, "_cache_rows", n <= HankelKernel.TABLE_CAP)))
            if mine._cache and n <= HankelKernel.TABLE_CAP:
                self.dense = mine.device_table()       # the reference's row cache, filled from empty
                self.kernel_id = _lib.BF_KERNEL_DENSE
            else:                                      # uncached rows: one order sweep per window
                self.tiles = mine.device_windows
                self.kernel_id = _lib.BF_KERNEL_TILES
        elif getattr(oracle, "matrix", None) is not None:
            self.dense = torch.as_tensor(np.ascontiguousarray(oracle.matrix, dtype=np.complex128)).cuda()
            self.kernel_id = _lib.BF_KERNEL_DENSE
        else:
            self.tiles = self._host_windows
            self.kernel_id = _lib.BF_KERNEL_TILES

    def _host_windows(self, blocks, side):
        torch = _lib.require_cuda()
        out = np.empty((len(blocks), side, side), dtype=np.complex128)
        ar = np.arange(side, dtype=np.intp)
        for b, (i, j) in enumerate(blocks):
            try:
                out[b] = self.oracle.block(ar + i * side, ar + j * side)
            except Exception as exc:
                raise _lib.OracleError(f"entry oracle failed on middle block ({i}, {j})") from exc
        return torch.from_numpy(out).cuda()


TILE_BUDGET = 2 << 30   # bytes of per-block entry windows uploaded per launch (BF_KERNEL_TILES)


class MiddleSampler:
    """Batched middle-level blocks on the device (construct.py:43-68)."""

    def __init__(self, oracle, p: DyadicPartition, r: int, params=DEFAULT_PARAMS, seed=0):
        self.torch = _lib.require_cuda()
        self.lib = _lib.load()
        self.p, self.r, self.params, self.seed = p, r, params, seed
        self.m, self.side = p.mid_nodes, p.mid_side
        if self.side < r:
            raise ValueError(f"middle blocks are {self.side} wide, below rank {r}")
        self.dev = _DeviceOracle(oracle, p.n)
        self.branching = getattr(p, "branching", 2)
        self.dense_branch = r * params.q >= self.side
        self._all_draws = None
        self._row0 = 0

    def prepare_draws(self, rows=None):
        """Draw tables of the middle blocks of block rows `rows` (default: all) up front
        (process pool), consumed per batch."""
        if not self.dense_branch and self._all_draws is None:
            m = self.m
            rows = range(m) if rows is None else rows
            self._row0 = rows.start
            self._all_draws = draw_tables(self.seed, self.side, self.r, self.params,
                                          [(i, j) for i in rows for j in range(m)])

    # BlockState of construct.cu (int64 r0, c0; 8 int32 counters; six int32[128] index sets)
    _STATE = np.dtype([("r0", "<i8"), ("c0", "<i8"), ("nrows", "<i4"), ("ncols", "<i4"), ("nskr", "<i4"),
                       ("nskc", "<i4"), ("tc", "<i4"), ("tr", "<i4"), ("t", "<i4"), ("pad", "<i4"),
                       ("rows", "<i4", 128), ("cols", "<i4", 128), ("skr", "<i4", 128), ("skc", "<i4", 128),
                       ("pivc", "<i4", 128), ("pivr", "<i4", 128)])

    def blocks(self, ij, trace=False):
        """(u0*sigma0, v0*sigma0, floored_inverse(sigma0)) for blocks ij, on the device.

        trace=True also returns, per block, the index sets the sampling SVD ended with
        (lowrank.py:238-256): the last sweep's sorted skeletons Pi_col / Pi_row, the
        least-squares row/column sets and the two basis pivot lists in pick order."""
        torch = self.torch
        ij = np.asarray(ij, dtype=np.int32).reshape(-1, 2)
        nb = ij.shape[0]
        side, r = self.side, self.r
        u = torch.empty((nb, side, r), dtype=torch.complex128, device="cuda")
        v = torch.empty_like(u)
        w = torch.empty((nb, r), dtype=torch.float64, device="cuda")
        def upload(arr):   # pinned + non-blocking: the host never waits for queued kernels
            return torch.from_numpy(np.ascontiguousarray(arr)).pin_memory().cuda(non_blocking=True)

        ij_d = upload(ij)
        if self.dense_branch:
            draws_d = None
        elif self._all_draws is not None:
            idx = (ij[:, 0] - self._row0) * self.m + ij[:, 1]
            draws_d = upload(self._all_draws[idx])
        else:
            # this batch's draws on the host while the device still runs the previous batch
            draws_d = upload(draw_tables(self.seed, side, r, self.params, ij.tolist()))
        wsb = int(self.lib.bf_middle_workspace_bytes(self.p.n, self.p.levels, self.branching, r, self.params.q, nb))
        if wsb == 0:
            raise ValueError("geometry/rank not supported by the batched sampling kernels (need r*(q+1) <= 128)")
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        P = ctypes.c_void_p
        if self.dev.tiles is None:
            dense = P(self.dev.dense.data_ptr()) if self.dev.dense is not None else None
            rc = self.lib.bf_middle_blocks(self.dev.kernel_id, self.p.n, self.p.levels, self.branching, r,
                                           self.params.q, self.params.iters, dense, nb, P(ij_d.data_ptr()),
                                           P(draws_d.data_ptr()) if draws_d is not None else None,
                                           P(u.data_ptr()), P(v.data_ptr()), P(w.data_ptr()), P(ws.data_ptr()), wsb,
                                           stream)
            self._raise(rc, ij)
            states = ws[:nb * self._STATE.itemsize].cpu().numpy().view(self._STATE) if trace else None
        else:
            # per-block entry windows, uploaded in batches bounded by TILE_BUDGET
            per = max(1, TILE_BUDGET // (16 * side * side))
            slot = torch.full((self.m * self.m,), -1, dtype=torch.int32, device="cuda")
            states = []
            for lo in range(0, nb, per):
                hi = min(nb, lo + per)
                sub = [tuple(int(t) for t in x) for x in ij[lo:hi]]
                tiles = self.dev.tiles(sub, side)
                slot.fill_(-1)
                slot[torch.as_tensor([i * self.m + j for i, j in sub], device="cuda")] = \
                    torch.arange(hi - lo, dtype=torch.int32, device="cuda")
                rc = self.lib.bf_middle_blocks_tiled(
                    self.p.n, self.p.levels, self.branching, r, self.params.q, self.params.iters,
                    P(tiles.data_ptr()), P(slot.data_ptr()), hi - lo, P(ij_d[lo:hi].data_ptr()),
                    P(draws_d[lo:hi].data_ptr()) if draws_d is not None else None,
                    P(u[lo:hi].data_ptr()), P(v[lo:hi].data_ptr()), P(w[lo:hi].data_ptr()), P(ws.data_ptr()), wsb,
                    stream)
                self._raise(rc, ij[lo:hi])
                if trace:
                    states.append(ws[:(hi - lo) * self._STATE.itemsize].cpu().numpy().view(self._STATE).copy())
                del tiles
            states = np.concatenate(states) if trace else None
        if not trace:
            return u, v, w
        raw = states
        tr = []
        for st in raw:
            if st["tc"] < 0:        # dense branch: no pivots
                tr.append({})
                continue
            tr.append({"skc": st["skc"][:st["nskc"]].tolist(), "skr": st["skr"][:st["nskr"]].tolist(),
                       "rows": st["rows"][:st["nrows"]].tolist(), "cols": st["cols"][:st["ncols"]].tolist(),
                       "pivc": st["pivc"][:st["tc"]].tolist(), "pivr": st["pivr"][:st["tr"]].tolist()})
        return u, v, w, tr

    @staticmethod
    def _raise(rc, ij):
        if rc != _lib.BF_OK:
            msg = _lib.last_error()
            if rc == _lib.BF_EINVAL:
                raise ValueError(msg)
            raise _lib.OracleError(f"entry oracle failed on middle blocks {ij[:1].tolist()}...: {msg}")

    def batch_rows(self) -> int:
        """Block-rows per launch: enough CTAs to fill the GPU, bounded workspace."""
        per_block = max(1, int(self.lib.bf_middle_workspace_bytes(self.p.n, self.p.levels, self.branching, self.r,
                                                                  self.params.q, 1)))
        # up to 1024 blocks per launch (cfg2: 4 rows, 17.8 GB of workspace): 62.0 ms per row
        # against 66.7 ms with one 256-block row (1.7 waves of one CTA per SM)
        by_mem = max(1, (20 << 30) // (per_block * self.m))
        return max(1, min(self.m, max(1, 1024 // self.m), by_mem))


def complex_normal(rng: np.random.Generator, shape) -> np.ndarray:
    """Independent N(0,1) real and imaginary parts, real block drawn first (lowrank.py:97-99)."""
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def probe_blocks(p: DyadicPartition, width: int, seed, domain) -> np.ndarray:
    """Diagonal blocks (m, side, width) of block_diagonal_probe (construct.py:78-86), drawn
    on the host with the reference's generator block_rng(seed, domain, j) so the probes
    are the reference's bit for bit."""
    m, side = p.mid_nodes, p.mid_side
    return np.stack([complex_normal(block_rng(seed, domain, j), (side, width)) for j in range(m)])


def block_diagonal_probe(p: DyadicPartition, width: int, seed, domain) -> np.ndarray:
    """(n, m*width) Gaussian probe with one (side x width) block per middle node (construct.py:78-86)."""
    blocks = probe_blocks(p, width, seed, domain)
    m, side, _ = blocks.shape
    probe = np.zeros((p.n, m * width), dtype=np.complex128)
    for j in range(m):
        probe[j * side:(j + 1) * side, j * width:(j + 1) * width] = blocks[j]
    return probe


def _probe_products(op, blocks_d, p: DyadicPartition, width: int, adjoint: bool, chunk: int = 128):
    """K @ probe (or K* @ probe) as a device (n, m*width) array, 128 probe columns per
    application (_apply_chunked, construct.py:71-75). Device operators (ButterflyFactors,
    ComposedOperator: ``accepts_device``) get device probes; any other operator oracle is
    called on host chunks, the products uploaded."""
    torch = _lib.require_cuda()
    m, side = p.mid_nodes, p.mid_side
    ncol = m * width
    out = torch.empty((p.n, ncol), dtype=torch.complex128, device="cuda")
    fn = op.apply_adjoint if adjoint else op.apply
    on_device = bool(getattr(op, "accepts_device", False))
    for c0 in range(0, ncol, chunk):
        c1 = min(ncol, c0 + chunk)
        probe = torch.zeros((p.n, c1 - c0), dtype=torch.complex128, device="cuda")
        for j in range(c0 // width, (c1 - 1) // width + 1):
            lo, hi = max(c0, j * width), min(c1, (j + 1) * width)
            probe[j * side:(j + 1) * side, lo - c0:hi - c0] = blocks_d[j, :, lo - j * width:hi - j * width]
        try:
            if on_device:
                y = fn(probe)
            else:
                y = torch.as_tensor(np.ascontiguousarray(fn(probe.cpu().numpy()), dtype=np.complex128)).cuda()
        except Exception as exc:
            raise _lib.OracleError("operator oracle failed on the probe block") from exc
        out[:, c0:c1] = y
    return out


def middle_factorization_matvec(op, p: DyadicPartition, r: int, params=DEFAULT_PARAMS, seed=0):
    """U^h, M, V^h from black-box applications of K and K* (construct.py:89-124), device tensors.

    One block-diagonal probe per side covers every middle block; each block's rank-r SVD is
    then finished from the stored products on the device (``bf_middle_probes``: pivots,
    bases, floored least squares and the middle SVD of svd_from_probes, lowrank.py:204-216)."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    m, side = p.mid_nodes, p.mid_side
    if side < r:
        raise ValueError(f"middle blocks are {side} wide, below rank {r}")
    width = min(r + params.p, side)
    branching = getattr(p, "branching", 2)
    col_d = torch.as_tensor(probe_blocks(p, width, seed, COL_PROBE_DOMAIN)).cuda()
    row_d = torch.as_tensor(probe_blocks(p, width, seed, ROW_PROBE_DOMAIN)).cuda().contiguous()
    k_cols = _probe_products(op, col_d, p, width, adjoint=False)
    k_rows = _probe_products(op, row_d, p, width, adjoint=True)
    del col_d
    u = torch.zeros((m, side, m, r), dtype=torch.complex128, device="cuda")
    v = torch.zeros_like(u)
    w = torch.zeros((m, m, r), dtype=torch.float64, device="cuda")
    per_block = max(1, int(lib.bf_probe_workspace_bytes(p.n, p.levels, branching, r, width, 1)))
    if int(lib.bf_probe_workspace_bytes(p.n, p.levels, branching, r, width, 1)) == 0:
        raise ValueError(f"probe width {width} not supported by the batched probe kernels (<= 128)")
    step_rows = max(1, min(m, (2 << 30) // (per_block * m)))
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for i0 in range(0, m, step_rows):
        rows = range(i0, min(m, i0 + step_rows))
        ij = np.array([(i, j) for i in rows for j in range(m)], dtype=np.int32)
        nb = ij.shape[0]
        ub = torch.empty((nb, side, r), dtype=torch.complex128, device="cuda")
        vb = torch.empty_like(ub)
        wb = torch.empty((nb, r), dtype=torch.float64, device="cuda")
        ij_d = torch.from_numpy(ij).cuda()
        wsb = int(lib.bf_probe_workspace_bytes(p.n, p.levels, branching, r, width, nb))
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        _lib.check(lib.bf_middle_probes(p.n, p.levels, branching, r, width, nb, ctypes.c_void_p(ij_d.data_ptr()),
                                        ctypes.c_void_p(k_cols.data_ptr()), m * width,
                                        ctypes.c_void_p(k_rows.data_ptr()), m * width,
                                        ctypes.c_void_p(row_d.data_ptr()), ctypes.c_void_p(ub.data_ptr()),
                                        ctypes.c_void_p(vb.data_ptr()), ctypes.c_void_p(wb.data_ptr()),
                                        ctypes.c_void_p(ws.data_ptr()), wsb, stream), "bf_middle_probes")
        k = len(rows)
        u[i0:i0 + k] = ub.reshape(k, m, side, r).permute(0, 2, 1, 3)          # u[i, :, j, :]
        v[:, :, i0:i0 + k, :] = vb.reshape(k, m, side, r).permute(1, 2, 0, 3)  # v[j, :, i, :]
        w[i0:i0 + k] = wb.reshape(k, m, r)
    return (BlockDiagonalFactor(u.reshape(m, side, m * r)), MiddleFactor(w),
            BlockDiagonalFactor(v.reshape(m, side, m * r)))


def recurse(cur, p: DyadicPartition, r: int):
    """_recurse (construct.py:127-163) on a device stack (nodes, rows, groups, r)."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    b = getattr(p, "branching", 2)
    pieces = []
    cur = cur.contiguous()
    for lvl in range(p.half, p.levels):
        nb, rows, groups, _ = cur.shape
        pairs = groups // b
        if rows >= b:
            blocks = torch.empty((nb, b, pairs, r, b * r), dtype=torch.complex128, device="cuda")
            nxt = torch.empty((b * nb, rows // b, pairs, r), dtype=torch.complex128, device="cuda")
        else:
            blocks = torch.empty((nb, pairs, r, b * r), dtype=torch.complex128, device="cuda")
            nxt = torch.empty((nb, 1, pairs, r), dtype=torch.complex128, device="cuda")
        need = ctypes.c_uint64(0)
        _lib.check(lib.bf_recurse_level(r, b, nb, rows, groups, None, None, None, None, ctypes.byref(need), stream))
        ws = torch.empty(max(int(need.value), 16), dtype=torch.uint8, device="cuda")
        _lib.check(lib.bf_recurse_level(r, b, nb, rows, groups, ctypes.c_void_p(cur.data_ptr()),
                                        ctypes.c_void_p(blocks.data_ptr()), ctypes.c_void_p(nxt.data_ptr()),
                                        ctypes.c_void_p(ws.data_ptr()), ctypes.byref(need), stream),
                   "bf_recurse_level")
        pieces.append((lvl, blocks))
        cur = nxt
    return cur[:, :, 0, :].contiguous(), pieces


def recursive_factor_u(u_h: BlockDiagonalFactor, p: DyadicPartition, r: int):
    """Expand the middle left factor into leaf factor + transfer chain (construct.py:171-176)."""
    torch = _lib.require_cuda()
    blocks = u_h.blocks if hasattr(u_h.blocks, "data_ptr") else torch.as_tensor(np.asarray(u_h.blocks)).cuda()
    cur = blocks.to(torch.complex128).reshape(p.mid_nodes, p.mid_side, p.mid_nodes, r)
    leaf, pieces = recurse(cur, p, r)
    return BlockDiagonalFactor(leaf), tuple(TransferFactor(lvl, b) for lvl, b in pieces)


def _recurse_full(h: BlockDiagonalFactor, p: DyadicPartition, r: int):
    """recursive_factor_u over the whole (m, side, m r) middle factor, slabs batched per
    launch as in factorize (the reference recurses all m slabs at once, construct.py:171-176)."""
    torch = _lib.require_cuda()
    m, side = p.mid_nodes, p.mid_side
    cur = h.blocks.reshape(m, side, m, r)
    shapes, leaf_shape = level_geometry(p, r)
    chain = {lvl: torch.zeros(shape, dtype=torch.complex128, device="cuda") for lvl, _, shape in shapes}
    leaf = torch.zeros(leaf_shape, dtype=torch.complex128, device="cuda")
    kb = recursion_batch(m, side, r)
    for k0 in range(0, m, kb):
        cnt = min(kb, m - k0)
        leaf_k, pieces = recurse(cur[k0:k0 + cnt], p, r)
        _place(chain, leaf, k0, cnt, leaf_k, pieces)
    return BlockDiagonalFactor(leaf), tuple(TransferFactor(lvl, chain[lvl]) for lvl, _, _ in shapes)


def recursive_factor_v(v_h: BlockDiagonalFactor, p: DyadicPartition, r: int):
    """Same expansion for the right factor (construct.py:179-181)."""
    return recursive_factor_u(v_h, p, r)


def middle_factorization_sampling(entry, p: DyadicPartition, r: int, params=DEFAULT_PARAMS, seed=0):
    """U^h, M, V^h of the sampling construction (construct.py:53-68), device tensors."""
    torch = _lib.require_cuda()
    ms = MiddleSampler(entry, p, r, params, seed)
    m, side = ms.m, ms.side
    u = torch.zeros((m, side, m, r), dtype=torch.complex128, device="cuda")
    v = torch.zeros_like(u)
    w = torch.zeros((m, m, r), dtype=torch.float64, device="cuda")
    step = ms.batch_rows()
    for i0 in range(0, m, step):
        rows = range(i0, min(m, i0 + step))
        uu, vv, ww = ms.blocks([(i, j) for i in rows for j in range(m)])
        k = len(rows)
        u[i0:i0 + k] = uu.reshape(k, m, side, r).permute(0, 2, 1, 3)      # u[i, :, j, :]
        v[:, :, i0:i0 + k, :] = vv.reshape(k, m, side, r).permute(1, 2, 0, 3)  # v[j, :, i, :]
        w[i0:i0 + k] = ww.reshape(k, m, r)
    return (BlockDiagonalFactor(u.reshape(m, side, m * r)), MiddleFactor(w),
            BlockDiagonalFactor(v.reshape(m, side, m * r)))


def _place(chain, leaf, k0, cnt, leaf_k, pieces):
    """Scatter the recursion of slabs k0 .. k0+cnt-1 (node-major) into the full chain."""
    for lvl, blocks in pieces:
        nb = blocks.shape[0] // cnt
        chain[lvl][k0 * nb:(k0 + cnt) * nb] = blocks
    nb = leaf_k.shape[0] // cnt
    leaf[k0 * nb:(k0 + cnt) * nb] = leaf_k


def recursion_batch(m: int, side: int, r: int) -> int:
    """Slabs per recursion launch: >= BF_RECURSION_PROBLEMS (default 2048) first-level
    problems (the level kernels are latency-bound per problem, so the GPU needs many in
    flight — and several machine-fills of them, so that the last partial fill is a small
    share), <= 4 GiB of slabs."""
    target = max(1, int(os.environ.get("BF_RECURSION_PROBLEMS", "2048")))
    slab_bytes = 16 * side * m * r
    return max(1, min(m, -(-target // m), (4 << 30) // max(1, slab_bytes)))


def factorize(oracle, p: DyadicPartition, r: int, params=DEFAULT_PARAMS, seed=0,
              mode="sampling") -> ButterflyFactors:
    """Build the full sparse chain for the operator behind ``oracle`` (construct.py:184-213).

    mode="sampling"   entry oracle; every middle block sampled once (V^h held on the device);
    mode="streaming"  entry oracle; one middle block row/column at a time, O(n log n) memory,
                      each block sampled twice — bitwise identical to "sampling";
    mode="matvec"     operator oracle (.apply / .apply_adjoint); block-diagonal probes, every
                      block finished from the probe products on the device (construct.py:89-124).
    """
    if params is None:
        params = DEFAULT_PARAMS
    if r < 1:
        raise ValueError(f"rank must be positive, got {r}")
    if mode in ("sampling", "streaming") and not is_entry_oracle(oracle):
        raise ValueError(f"mode={mode!r} needs an entry oracle")
    if mode == "matvec" and not is_operator_oracle(oracle):
        raise ValueError("mode='matvec' needs an operator oracle")
    if mode not in ("sampling", "streaming", "matvec"):
        raise ValueError(f"unknown mode {mode!r}")
    torch = _lib.require_cuda()
    if mode == "matvec":
        u_h, middle, v_h = middle_factorization_matvec(oracle, p, r, params, seed)
        (u_outer, g_chain), (v_outer, h_chain) = (_recurse_full(u_h, p, r), _recurse_full(v_h, p, r))
        return ButterflyFactors(p, r, u_outer, g_chain, middle, h_chain, v_outer)
    # each batch draws its own tables on the host (draw_tables) while the device works on
    # the previous batch: the ~4 s of NumPy draws at cfg2 stay off the critical path
    ms = MiddleSampler(oracle, p, r, params, seed)
    m, side = ms.m, ms.side
    shapes, leaf_shape = level_geometry(p, r)
    weights = torch.zeros((m, m, r), dtype=torch.float64, device="cuda")
    sides = []
    v_full = None
    if mode == "sampling":
        v_full = torch.zeros((m, side, m, r), dtype=torch.complex128, device="cuda")
    for axis in ("u", "v"):
        chain = {lvl: torch.zeros(shape, dtype=torch.complex128, device="cuda") for lvl, _, shape in shapes}
        leaf = torch.zeros(leaf_shape, dtype=torch.complex128, device="cuda")
        kb = recursion_batch(m, side, r)
        if axis == "v" and mode == "sampling":
            for k0 in range(0, m, kb):
                cnt = min(kb, m - k0)
                leaf_k, pieces = recurse(v_full[k0:k0 + cnt], p, r)
                _place(chain, leaf, k0, cnt, leaf_k, pieces)
        else:
            # slab recursions run on a side stream, overlapping the next block-rows' middle
            # kernels (both are latency-bound at low occupancy); two slab buffers alternate
            main = torch.cuda.current_stream()
            side_stream = torch.cuda.Stream()
            bufs = [torch.empty((kb, side, m, r), dtype=torch.complex128, device="cuda") for _ in range(2)]
            done = [None, None]
            cb = 0
            buf = bufs[cb]
            filled, k_first = 0, 0
            step = ms.batch_rows()
            for k0 in range(0, m, step):
                ks = range(k0, min(m, k0 + step))
                ij = [((k, o) if axis == "u" else (o, k)) for k in ks for o in range(m)]
                uu, vv, ww = ms.blocks(ij)
                for idx, k in enumerate(ks):
                    sl = slice(idx * m, (idx + 1) * m)
                    if filled == 0 and done[cb] is not None:
                        main.wait_event(done[cb])                                  # buffer free again
                    if axis == "u":
                        buf[filled] = uu[sl].permute(1, 0, 2)                      # slab[:, j, :]
                        weights[k] = ww[sl]
                        if v_full is not None:
                            v_full[:, :, k, :] = vv[sl]                            # v[j, :, i=k, :]
                    else:
                        buf[filled] = vv[sl].permute(1, 0, 2)                      # slab[:, i, :]
                    if filled == 0:
                        k_first = k
                    filled += 1
                    if filled == kb or k == m - 1:
                        side_stream.wait_stream(main)
                        with torch.cuda.stream(side_stream):
                            leaf_k, pieces = recurse(buf[:filled], p, r)
                            _place(chain, leaf, k_first, filled, leaf_k, pieces)
                            done[cb] = torch.cuda.Event()
                            done[cb].record(side_stream)
                        buf.record_stream(side_stream)
                        cb ^= 1
                        buf = bufs[cb]
                        filled = 0
            main.wait_stream(side_stream)
            del buf, bufs
        sides.append((BlockDiagonalFactor(leaf), tuple(TransferFactor(lvl, chain[lvl]) for lvl, _, _ in shapes)))
    del v_full
    (u_outer, g_chain), (v_outer, h_chain) = sides
    return ButterflyFactors(p, r, u_outer, g_chain, MiddleFactor(weights), h_chain, v_outer)


def _dist_exchange(group=None):
    """All-to-all of equal per-part chunks (leading dim = parts) over torch.distributed."""
    def run(send):
        import torch
        import torch.distributed as dist
        recv = torch.empty_like(send)
        sr = torch.view_as_real(send) if send.is_complex() else send
        rr = torch.view_as_real(recv) if recv.is_complex() else recv
        dist.all_to_all_single(rr.reshape(-1), sr.reshape(-1), group=group)
        return recv

    def gather(rows):
        import torch
        import torch.distributed as dist
        out = [torch.empty_like(rows) for _ in range(dist.get_world_size(group))]
        dist.all_gather(out, rows.contiguous(), group=group)
        return torch.cat(out)

    return run, gather


def factorize_part(oracle, p: DyadicPartition, r: int, part: int, nparts: int, params=DEFAULT_PARAMS, seed=0,
                   exchange=None, gather=None, device="cuda", blocks_fn=None, recurse_fn=None) -> dict:
    """Part `part` of `nparts` of a node-sharded sampling construction (SURVEY.md §8(e):
    "construction shards trivially over (i, j) middle blocks"): returns the slices
    ``sharded.shard_slices(factorize(...), part, nparts)`` would cut — bit for bit, since
    every block draws from its own SeedSequence(seed, spawn_key=(0, i, j)).

    Part d computes the middle blocks of its rows i in I_d (all columns j) and recurses
    its U slabs into its G / U^L slices. Each block's v0 sigma0 belongs to the owner of
    column j: one all-to-all per row step moves (m/P) x side x r complex values to every
    part; the V slabs a part then holds are recursed into its H / V^L slices. The weight
    rows are all-gathered (the sharded apply scales by W[:, J_d] in its pack / push).

    exchange(send (P, ...)) -> recv (P, ...) and gather(rows) -> all rows default to
    torch.distributed (NCCL on GPUs); blocks_fn / recurse_fn default to the device
    kernels (tests substitute host fakes to check the orchestration)."""
    import torch
    m, side = p.mid_nodes, p.mid_side
    if m % nparts:
        raise ValueError(f"{nparts} parts do not divide the {m} middle nodes")
    if r < 1:
        raise ValueError(f"rank must be positive, got {r}")
    mp = m // nparts
    own = range(part * mp, (part + 1) * mp)
    if exchange is None or gather is None:
        if nparts == 1:
            exchange, gather = (lambda x: x.clone()), (lambda x: x)
        else:
            exchange, gather = _dist_exchange()
    if blocks_fn is None:
        if not is_entry_oracle(oracle):
            raise ValueError("the sharded construction needs an entry oracle")
        ms = MiddleSampler(oracle, p, r, params, seed)
        if mp * m >= 1024:
            ms.prepare_draws(own)
        blocks_fn, step = ms.blocks, ms.batch_rows()
    else:
        step = max(1, min(mp, 2))
    recurse_fn = recurse if recurse_fn is None else recurse_fn
    shapes, leaf_shape = level_geometry(p, r)
    cplx = torch.complex128

    def part_chain():
        chain = {lvl: torch.zeros((shape[0] // nparts,) + tuple(shape[1:]), dtype=cplx, device=device)
                 for lvl, _, shape in shapes}
        leaf = torch.zeros((leaf_shape[0] // nparts,) + tuple(leaf_shape[1:]), dtype=cplx, device=device)
        return chain, leaf

    w_rows = torch.zeros((mp, m, r), dtype=torch.float64, device=device)
    v_slabs = torch.zeros((mp, side, m, r), dtype=cplx, device=device)   # [j local, row, i, rho]
    u_chain, u_leaf = part_chain()
    kb = recursion_batch(m, side, r)
    buf = torch.empty((min(kb, mp), side, m, r), dtype=cplx, device=device)
    filled, first = 0, 0
    for s0 in range(0, mp, step):
        rows = list(own[s0:s0 + step])
        uu, vv, ww = blocks_fn([(i, j) for i in rows for j in range(m)])
        nr = len(rows)
        vv = vv.reshape(nr, nparts, mp, side, r)                  # [row i, owner e of j, j local, ., .]
        recv = exchange(vv.permute(1, 0, 2, 3, 4).contiguous())   # [source e, row step, j local (mine), ., .]
        for e in range(nparts):
            for idx in range(nr):
                v_slabs[:, :, e * mp + s0 + idx, :] = recv[e, idx]
        for idx, i in enumerate(rows):
            sl = slice(idx * m, (idx + 1) * m)
            w_rows[i - own.start] = ww[sl]
            buf[filled] = uu[sl].permute(1, 0, 2)                  # slab[:, j, :]
            if filled == 0:
                first = i - own.start
            filled += 1
            if filled == buf.shape[0] or i == own[-1]:
                leaf_k, pieces = recurse_fn(buf[:filled], p, r)
                _place(u_chain, u_leaf, first, filled, leaf_k, pieces)
                filled = 0
    del buf
    weights = gather(w_rows)
    v_chain, v_leaf = part_chain()
    for k0 in range(0, mp, kb):
        cnt = min(kb, mp - k0)
        leaf_k, pieces = recurse_fn(v_slabs[k0:k0 + cnt], p, r)
        _place(v_chain, v_leaf, k0, cnt, leaf_k, pieces)
    return {"u_leaf": u_leaf, "v_leaf": v_leaf, "weights": weights,
            "g": [(lvl, u_chain[lvl]) for lvl, _, _ in shapes], "h": [(lvl, v_chain[lvl]) for lvl, _, _ in shapes]}
