"""Factor chain storage and its application — the reference's ``factors.py``
API (same classes, fields, layouts and errors), applied on the B200 through
libbfly.so (include/bfly.h).

The dataclasses hold the factor arrays in the reference layout
(factors.py:23-203) as NumPy arrays (or, for device-generated factor sets,
contiguous torch CUDA tensors). ``ButterflyFactors.apply`` uploads them once
into an immutable device plan (``DevicePlan``) and runs the CUDA chain; there
is no NumPy compute path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .partition import DyadicPartition, level_geometry


def _np(a):
    """Host view of a factor array (NumPy or torch)."""
    if hasattr(a, "detach"):
        return a.detach().cpu().numpy()
    return np.asarray(a)


@dataclass(frozen=True)
class BlockDiagonalFactor:
    """Uniform block diagonal: blocks[b] sits at (b*rows, b*cols) (factors.py:23-56)."""

    blocks: object  # (nb, rows, cols) complex

    @property
    def nnz(self) -> int:
        return int(np.prod(self.blocks.shape))

    @property
    def shape(self):
        nb, rows, cols = self.blocks.shape
        return (nb * rows, nb * cols)

    def iter_blocks(self):
        b = _np(self.blocks)
        nb, rows, cols = b.shape
        for i in range(nb):
            yield i * rows, i * cols, b[i]

    def dense(self) -> np.ndarray:
        out = np.zeros(self.shape, dtype=np.complex128)
        for r0, c0, blk in self.iter_blocks():
            out[r0:r0 + blk.shape[0], c0:c0 + blk.shape[1]] = blk
        return out


@dataclass(frozen=True)
class TransferFactor:
    """One level: (groups, 2, pairs, r, 2r) splitting or (nodes, pairs, r, 2r) merge-only (factors.py:59-142)."""

    level: int
    blocks: object

    @property
    def splits(self) -> bool:
        return len(self.blocks.shape) == 5

    @property
    def rank(self) -> int:
        return self.blocks.shape[-2]

    @property
    def pairs(self) -> int:
        return self.blocks.shape[-3]

    @property
    def nnz(self) -> int:
        return int(np.prod(self.blocks.shape))

    @property
    def shape(self):
        r, p, c = self.rank, self.pairs, self.blocks.shape[-1]
        if self.splits:
            g, nt = self.blocks.shape[0], self.blocks.shape[1]
            return (nt * g * p * r, g * p * c)
        nodes = self.blocks.shape[0]
        return (nodes * p * r, nodes * p * c)

    def iter_blocks(self):
        """Block offsets exactly as factors.py:97-112 (the .bfac header order); nt row
        parts and c = nt*r columns per block (nt = 2 in the reference, 4 on quadtrees)."""
        b = _np(self.blocks)
        r, p, c = self.rank, self.pairs, b.shape[-1]
        if self.splits:
            nt = b.shape[1]
            for g in range(b.shape[0]):
                for t in range(nt):
                    for j in range(p):
                        yield (nt * g + t) * p * r + j * r, g * p * c + j * c, b[g, t, j]
        else:
            for node in range(b.shape[0]):
                for j in range(p):
                    yield node * p * r + j * r, node * p * c + j * c, b[node, j]

    def dense(self) -> np.ndarray:
        out = np.zeros(self.shape, dtype=np.complex128)
        for r0, c0, blk in self.iter_blocks():
            out[r0:r0 + blk.shape[0], c0:c0 + blk.shape[1]] = blk
        return out


@dataclass(frozen=True)
class MiddleFactor:
    """Weighted block permutation: weights[i, j] on the (j, i) slot (factors.py:145-190)."""

    weights: object  # (m, m, r) real

    @property
    def m(self) -> int:
        return self.weights.shape[0]

    @property
    def rank(self) -> int:
        return self.weights.shape[2]

    @property
    def nnz(self) -> int:
        return int(np.prod(self.weights.shape))

    @property
    def shape(self):
        n = self.m * self.m * self.rank
        return (n, n)

    def iter_blocks(self):
        w = _np(self.weights)
        m, r = self.m, self.rank
        for i in range(m):
            for j in range(m):
                yield i * m * r + j * r, j * m * r + i * r, w[i, j]

    def dense(self) -> np.ndarray:
        out = np.zeros(self.shape, dtype=np.complex128)
        for r0, c0, w in self.iter_blocks():
            out[r0:r0 + self.rank, c0:c0 + self.rank] = np.diag(w)
        return out


_DTYPES = {"c128": _lib.BF_C128, "c64": _lib.BF_C64}


class DevicePlan:
    """Immutable device copy of one factor chain (a ``bf_plan``).

    ``dtype`` is "c128" (the reference's arithmetic, factors.py:222) or the
    opt-in "c64" mode. Applies accept torch CUDA tensors (zero-copy, result on
    the device) or host arrays (H2D + apply + D2H in one C call).
    """

    def __init__(self, f: "ButterflyFactors", dtype: str = "c128", device=None):
        torch = _lib.require_cuda()
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be one of {sorted(_DTYPES)}")
        lib = _lib.load()
        self.n, self.dtype = f.n, dtype
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.torch_dtype = torch.complex128 if dtype == "c128" else torch.complex64
        self.np_dtype = np.complex128 if dtype == "c128" else np.complex64
        h = ctypes.c_void_p()
        _lib.check(lib.bf_plan_create_tree(ctypes.byref(h), f.n, f.partition.levels, f.rank,
                                           getattr(f.partition, "branching", 2), _DTYPES[dtype], self.device, 0, 1),
                   "bf_plan_create_tree")
        self._h = h
        self._lib = lib
        self._check_geometry(f)
        keep = []

        def ptr(a, real=False):
            if hasattr(a, "data_ptr"):
                want = torch.float64 if real else torch.complex128
                t = a.detach().to(dtype=want).contiguous()
                keep.append(t)
                return t.data_ptr()
            arr = np.ascontiguousarray(a, dtype=np.float64 if real else np.complex128)
            keep.append(arr)
            return arr.ctypes.data

        nl = len(f.g_chain)
        g_ptrs = (ctypes.c_void_p * nl)(*[ptr(tf.blocks) for tf in f.g_chain])
        h_ptrs = (ctypes.c_void_p * nl)(*[ptr(tf.blocks) for tf in f.h_chain])
        _lib.check(lib.bf_plan_upload(h, ptr(f.u_outer.blocks), g_ptrs, ptr(f.middle.weights, real=True),
                                      h_ptrs, ptr(f.v_outer.blocks)), "bf_plan_upload")
        del keep

    @classmethod
    def adopt(cls, f: "ButterflyFactors", handle, dtype: str, device: int) -> "DevicePlan":
        """Wrap an already uploaded bf_plan (e.g. one built by bf_plan_load_bfac)."""
        import torch
        pl = cls.__new__(cls)
        pl._lib = _lib.load()
        pl._h = handle
        pl.n, pl.dtype, pl.device = f.n, dtype, device
        pl.torch_dtype = torch.complex128 if dtype == "c128" else torch.complex64
        pl.np_dtype = np.complex128 if dtype == "c128" else np.complex64
        pl._check_geometry(f)
        return pl

    def _check_geometry(self, f):
        nl = ctypes.c_uint32()
        self._lib.bf_plan_geometry(self._h, ctypes.byref(nl), None, None, None)
        splits = (ctypes.c_int8 * nl.value)()
        dims = (ctypes.c_uint64 * (5 * nl.value))()
        leaf = (ctypes.c_uint64 * 3)()
        _lib.check(self._lib.bf_plan_geometry(self._h, None, splits, dims, leaf))
        shapes, leaf_shape = level_geometry(f.partition, f.rank)
        if nl.value != len(shapes) or len(f.g_chain) != nl.value or len(f.h_chain) != nl.value:
            raise ValueError("factor chain length does not match the partition geometry")
        for i, (lvl, sp, shp) in enumerate(shapes):
            got = tuple(int(x) for x in dims[5 * i:5 * i + len(shp)])
            if bool(splits[i]) != sp or got != shp:
                raise RuntimeError(f"plan geometry {got} != host geometry {shp} at level {lvl}")
            for tf in (f.g_chain[i], f.h_chain[i]):
                if tuple(tf.blocks.shape) != shp or tf.level != lvl:
                    raise ValueError(f"transfer level {tf.level} has shape {tuple(tf.blocks.shape)}, "
                                     f"geometry needs level {lvl} {shp}")
        if tuple(int(x) for x in leaf) != tuple(leaf_shape):
            raise RuntimeError("plan leaf geometry mismatch")
        self._shapes = [shp for _, _, shp in shapes]
        self._leaf = tuple(int(x) for x in leaf)
        self._half = f.partition.half
        for fac in (f.u_outer, f.v_outer):
            if tuple(fac.blocks.shape) != tuple(leaf_shape):
                raise ValueError(f"leaf factor shape {tuple(fac.blocks.shape)} != {tuple(leaf_shape)}")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.bf_plan_destroy(h)
            self._h = None

    def workspace_bytes(self, k: int) -> int:
        return int(self._lib.bf_apply_workspace_bytes(self._h, k))

    def _stream(self, stream):
        import torch
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        return ctypes.c_void_p(s.cuda_stream)

    def apply(self, g, adjoint: bool = False, out=None, workspace=None, stream=None):
        """K @ g (K* @ g when adjoint) — ButterflyFactors._chain (factors.py:217-237)."""
        if hasattr(g, "is_cuda") and g.is_cuda:
            return self._apply_device(g, adjoint, out, workspace, stream)
        return self._apply_host(g, adjoint, out, stream)

    def _apply_device(self, g, adjoint, out, workspace, stream):
        import torch
        if g.shape[0] != self.n:
            raise ValueError(f"input length {g.shape[0]} != {self.n}")
        vec = g.dim() == 1
        w = g.reshape(self.n, -1)
        if w.dtype != self.torch_dtype:
            w = w.to(self.torch_dtype)
        w = w.contiguous()
        k = w.shape[1]
        if out is None:
            out = torch.empty_like(w)
        elif out.shape[0] != self.n or out.numel() != w.numel() or out.dtype != self.torch_dtype or not out.is_contiguous():
            raise ValueError("out must be a contiguous tensor of the input shape and plan dtype")
        wsb = self.workspace_bytes(k)
        if workspace is None or workspace.numel() < wsb:
            workspace = torch.empty(wsb, dtype=torch.uint8, device=w.device)
        _lib.check(self._lib.bf_apply(self._h, ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(out.data_ptr()), k,
                                      int(bool(adjoint)), ctypes.c_void_p(workspace.data_ptr()), wsb,
                                      self._stream(stream)), "bf_apply")
        return out.reshape(-1) if vec else out.reshape(self.n, k)

    def _apply_host(self, g, adjoint, out, stream):
        g = np.asarray(g)
        if g.shape[0] != self.n:
            raise ValueError(f"input length {g.shape[0]} != {self.n}")
        vec = g.ndim == 1
        w = np.ascontiguousarray(g.reshape(self.n, -1), dtype=self.np_dtype)
        k = w.shape[1]
        if out is None:
            res = np.empty_like(w)
        else:
            res = out.reshape(self.n, -1) if out.ndim == 1 else out
            if res.shape != w.shape or res.dtype != self.np_dtype or not res.flags.c_contiguous:
                raise ValueError("out must be a C-contiguous array of the input shape and plan dtype")
        _lib.check(self._lib.bf_apply_host(self._h, ctypes.c_void_p(w.ctypes.data), ctypes.c_void_p(res.ctypes.data),
                                           k, int(bool(adjoint)), self._stream(stream)), "bf_apply_host")
        return res[:, 0] if vec else res

    def apply_factor(self, which: str, level: int, adjoint: bool, x, stream=None):
        """One factor's forward/adjoint on a device (dim, k) tensor (per-level parity)."""
        import torch
        code = {"V": _lib.BF_FACTOR_V, "H": _lib.BF_FACTOR_H, "M": _lib.BF_FACTOR_M,
                "G": _lib.BF_FACTOR_G, "U": _lib.BF_FACTOR_U}[which]
        x = x.to(self.torch_dtype).contiguous()
        x2 = x.reshape(x.shape[0], -1)
        k = x2.shape[1]
        out_rows = self._factor_out_rows(which, level, adjoint, x2.shape[0])
        out = torch.empty((out_rows, k), dtype=self.torch_dtype, device=x.device)
        _lib.check(self._lib.bf_apply_factor(self._h, code, int(level), int(bool(adjoint)),
                                             ctypes.c_void_p(x2.data_ptr()), ctypes.c_void_p(out.data_ptr()), k,
                                             self._stream(stream)), "bf_apply_factor")
        return out

    def _factor_out_rows(self, which, level, adjoint, rows_in):
        """Output length of one factor op: its (rows, cols) shape read R-side / C-side."""
        nb, n0, r = self._leaf
        if which in ("V", "U"):
            return nb * r if adjoint else nb * n0
        if which == "M":
            return rows_in
        shp = self._shapes[level - self._half]
        if len(shp) == 5:
            rows, cols = shp[0] * shp[1] * shp[2] * shp[3], shp[0] * shp[2] * shp[4]
        else:
            rows, cols = shp[0] * shp[1] * shp[2], shp[0] * shp[1] * shp[3]
        return cols if adjoint else rows


@dataclass(frozen=True)
class ButterflyFactors:
    """Complete factor chain plus its partition (factors.py:193-255)."""

    partition: DyadicPartition
    rank: int
    u_outer: BlockDiagonalFactor
    g_chain: tuple
    middle: MiddleFactor
    h_chain: tuple
    v_outer: BlockDiagonalFactor
    _plans: dict = field(default_factory=dict, compare=False, repr=False)
    accepts_device = True   # operator-oracle protocol: apply() takes torch CUDA tensors too

    @property
    def n(self) -> int:
        return self.partition.n

    def plan(self, dtype: str = "c128", device=None) -> DevicePlan:
        """The (cached) device plan of this chain."""
        key = (dtype, device)
        pl = self._plans.get(key)
        if pl is None:
            pl = DevicePlan(self, dtype=dtype, device=device)
            self._plans[key] = pl
        return pl

    def apply(self, g, out=None):
        """Evaluate K @ g through the sparse chain in O(n log n) (factors.py:209-211)."""
        return self.plan().apply(g, adjoint=False, out=out)

    def apply_adjoint(self, g, out=None):
        """Evaluate K* @ g (factors.py:213-215)."""
        return self.plan().apply(g, adjoint=True, out=out)

    def dense(self, chunk: int = 512) -> np.ndarray:
        """Materialise the factored operator column block by column block (factors.py:239-246)."""
        n = self.n
        out = np.empty((n, n), dtype=np.complex128)
        for c0 in range(0, n, chunk):
            eye = np.zeros((n, min(chunk, n - c0)), dtype=np.complex128)
            eye[np.arange(c0, c0 + eye.shape[1]), np.arange(eye.shape[1])] = 1.0
            out[:, c0:c0 + eye.shape[1]] = self.apply(eye)
        return out

    def nnz_report(self) -> "NnzReport":
        return NnzReport(u_outer=self.u_outer.nnz, g={tf.level: tf.nnz for tf in self.g_chain},
                         middle=self.middle.nnz, h={tf.level: tf.nnz for tf in self.h_chain},
                         v_outer=self.v_outer.nnz)


@dataclass(frozen=True)
class NnzReport:
    """Stored-entry counts per factor (factors.py:258-271)."""

    u_outer: int
    g: dict = field(default_factory=dict)
    middle: int = 0
    h: dict = field(default_factory=dict)
    v_outer: int = 0

    @property
    def total(self) -> int:
        return self.u_outer + self.v_outer + self.middle + sum(self.g.values()) + sum(self.h.values())


def factors_equal(a: ButterflyFactors, b: ButterflyFactors) -> bool:
    """Bit-exact equality of two chains (factors.py:274-285)."""
    if a.partition != b.partition or a.rank != b.rank:
        return False
    if len(a.g_chain) != len(b.g_chain) or len(a.h_chain) != len(b.h_chain):
        return False
    pairs = [(a.u_outer.blocks, b.u_outer.blocks), (a.v_outer.blocks, b.v_outer.blocks),
             (a.middle.weights, b.middle.weights)]
    pairs += [(x.blocks, y.blocks) for x, y in zip(a.g_chain, b.g_chain)]
    pairs += [(x.blocks, y.blocks) for x, y in zip(a.h_chain, b.h_chain)]
    return all(tuple(x.shape) == tuple(y.shape) and np.array_equal(_np(x), _np(y)) for x, y in pairs)


def from_arrays(n, levels, rank, u_leaf, g_levels, weights, h_levels, v_leaf, partition=None) -> ButterflyFactors:
    """Assemble a chain from raw arrays; g_levels/h_levels are [(level, blocks)] ascending."""
    p = partition if partition is not None else DyadicPartition(int(n), int(levels))
    return ButterflyFactors(p, int(rank), BlockDiagonalFactor(u_leaf),
                            tuple(TransferFactor(int(l), b) for l, b in g_levels), MiddleFactor(weights),
                            tuple(TransferFactor(int(l), b) for l, b in h_levels), BlockDiagonalFactor(v_leaf))
