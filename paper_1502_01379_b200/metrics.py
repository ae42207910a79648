"""The reference's accuracy metric eps_a on the GPU (reference bench.py:38-97).

eps_a compares the factored operator with the direct row sums of the entry
oracle at |S| sampled rows on one shared Gaussian input. The ground truth
``K[S, :] g`` costs |S| N entry evaluations (4.3e9 at N = 2^24), so it runs on
the device (``bf_sampled_rows``) with the entries computed on the fly.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .construct import _DeviceOracle


class RowSampledReference:
    """Direct row sums of an entry oracle at sampled rows only (bench.py:38-46)."""

    def __init__(self, entry):
        self.entry = entry
        self._dev = None

    def rows(self, g, sample):
        torch = _lib.require_cuda()
        n = self.entry.shape[1]
        if self._dev is None:
            self._dev = _DeviceOracle(self.entry, n)
        g = np.asarray(g)
        vec = g.ndim == 1
        gd = torch.as_tensor(np.ascontiguousarray(g.reshape(n, -1), dtype=np.complex128)).cuda()
        k = gd.shape[1]
        if self._dev.kernel_id == _lib.BF_KERNEL_TILES:
            # an entry oracle the device cannot evaluate per entry: its rows K[S, :] through
            # .block (the reference's own ground truth, bench.py:38-46), chunked to bound
            # memory, the row sums on the device
            sample = np.asarray(sample, dtype=np.intp)
            res = torch.empty((sample.size, k), dtype=torch.complex128, device="cuda")
            step = max(1, (1 << 27) // n)
            for lo in range(0, sample.size, step):
                blk = self.entry.block(sample[lo:lo + step], np.arange(n))
                res[lo:lo + step] = torch.as_tensor(np.ascontiguousarray(blk, dtype=np.complex128)).cuda() @ gd
            res = res.cpu().numpy()
            return res[:, 0] if vec else res
        rows = torch.as_tensor(np.ascontiguousarray(sample, dtype=np.int64)).cuda()
        out = torch.empty((rows.numel(), k), dtype=torch.complex128, device="cuda")
        lib = _lib.load()
        wsb = int(lib.bf_sampled_rows_workspace(n, rows.numel(), k))
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
        dense = ctypes.c_void_p(self._dev.dense.data_ptr()) if self._dev.dense is not None else None
        _lib.check(lib.bf_sampled_rows(self._dev.kernel_id, n, dense, ctypes.c_void_p(rows.data_ptr()), rows.numel(),
                                       ctypes.c_void_p(gd.data_ptr()), k, ctypes.c_void_p(out.data_ptr()),
                                       ctypes.c_void_p(ws.data_ptr()), wsb,
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "bf_sampled_rows")
        res = out.cpu().numpy()
        return res[:, 0] if vec else res


class OperatorReference:
    """Ground truth from a fast black-box operator, e.g. a ComposedOperator (bench.py:60-72)."""

    def __init__(self, op):
        self.op = op

    def rows(self, g, sample):
        out = self.op.apply(g)
        if hasattr(out, "is_cuda"):
            out = out.cpu().numpy()
        return np.asarray(out)[sample]


def sampled_relative_error(u_approx, u_exact):
    """(error, used_absolute_fallback) of the sampled l2 ratio metric (bench.py:75-81)."""
    diff = float(np.linalg.norm(u_approx - u_exact))
    denom = float(np.linalg.norm(u_exact))
    if denom == 0.0:
        return diff, True
    return diff / denom, False


def estimate_eps_a_info(f, reference, sample_count: int, rng):
    """bench.py:90-97: |S| rows without replacement, g = complex_normal, relative l2 error."""
    rng = np.random.default_rng(rng)
    n = f.n
    sample = np.sort(rng.choice(n, size=min(sample_count, n), replace=False))
    g = rng.standard_normal((n,)) + 1j * rng.standard_normal((n,))
    return sampled_relative_error(f.apply(g)[sample], reference.rows(g, sample))


def estimate_eps_a(f, reference, sample_count: int, rng) -> float:
    value, _ = estimate_eps_a_info(f, reference, sample_count, rng)
    return value
