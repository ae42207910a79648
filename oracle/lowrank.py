"""Low-rank engines of the sampling construction — NumPy restatement of
reference ``lowrank.py`` (test infrastructure; see oracle/__init__.py)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PINV_FLOOR = 1e-13   # lowrank.py:22
PIVOT_TIE = 1e-14    # lowrank.py:25
BASIS_TRIM = 1e-11   # lowrank.py:30


@dataclass(frozen=True)
class Params:
    """OversamplingParams defaults (lowrank.py:33-51)."""

    p: int = 5
    q: int = 3
    iters: int = 3


@dataclass(frozen=True)
class Triple:
    """LowRankApprox (lowrank.py:54-67): u0 diag(sigma) v0*."""

    u0: np.ndarray
    sigma0: np.ndarray
    v0: np.ndarray

    def matrix(self):
        return (self.u0 * self.sigma0) @ self.v0.conj().T


def floored_inverse(sigma) -> np.ndarray:
    """1/sigma where sigma > PINV_FLOOR * max(sigma), else 0 (lowrank.py:79-87)."""
    sigma = np.asarray(sigma, dtype=float)
    out = np.zeros_like(sigma)
    if sigma.size:
        mask = sigma > PINV_FLOOR * sigma.max(initial=0.0)
        out[mask] = 1.0 / sigma[mask]
    return out


def pinv_floored(a: np.ndarray) -> np.ndarray:
    """SVD pseudo-inverse with the shared floor (lowrank.py:90-94)."""
    u, s, vh = np.linalg.svd(a, full_matrices=False)
    return (vh.conj().T * floored_inverse(s)) @ u.conj().T


def greedy_pivots(a: np.ndarray, k: int, rel_tol: float = 0.0) -> list:
    """Greedy Gram-Schmidt column pivoting (lowrank.py:102-129).

    Residual norms are downdated, never recomputed; a column within
    2*PIVOT_TIE (relative) of the maximum ties and the lowest index wins.
    """
    work = np.array(a, dtype=np.complex128, copy=True)
    k = min(k, *work.shape)
    resid = (work.real * work.real + work.imag * work.imag).sum(axis=0)
    stop = rel_tol * rel_tol * float(resid.max(initial=0.0))
    picks = []
    while len(picks) < k:
        top = float(resid.max(initial=0.0))
        if top <= stop or top <= 0.0:
            break
        j = int(np.flatnonzero(resid >= top * (1.0 - 2.0 * PIVOT_TIE))[0])
        picks.append(j)
        q = work[:, j] / np.sqrt(resid[j])
        proj = q.conj() @ work
        work -= q[:, None] * proj
        resid -= proj.real * proj.real + proj.imag * proj.imag
        np.maximum(resid, 0.0, out=resid)
        resid[j] = 0.0
    return picks


def pivoted_basis(a: np.ndarray, k: int, pad: bool = True, rel_tol: float = 0.0) -> np.ndarray:
    """Orthonormal basis of the first k pivot columns (lowrank.py:132-154)."""
    rows = a.shape[0]
    if k > rows:
        raise ValueError(f"cannot build {k} orthonormal columns in dimension {rows}")
    piv = greedy_pivots(a, k, rel_tol)
    cols = a[:, piv]
    if len(piv) < k:
        if not pad:
            if not piv:
                return np.zeros((rows, 0), dtype=np.complex128)
            return np.linalg.qr(cols)[0]
        cols = np.concatenate([cols, np.eye(rows, dtype=np.complex128)[:, :k - len(piv)]], axis=1)
    return np.linalg.qr(cols)[0][:, :k]


def complete_basis(part: np.ndarray, k: int) -> np.ndarray:
    """Pad (rows x t) orthonormal columns to k with QR of canonical fillers (lowrank.py:157-165)."""
    rows, t = part.shape
    if t == k:
        return part
    q = np.linalg.qr(np.concatenate([part, np.eye(rows, dtype=np.complex128)[:, :k - t]], axis=1))[0]
    return np.concatenate([part, q[:, t:k]], axis=1)


def truncated_svd(z: np.ndarray, r: int) -> Triple:
    """Dense SVD truncated to rank r (lowrank.py:168-179)."""
    z = np.asarray(z)
    if not 1 <= r <= min(z.shape):
        raise ValueError(f"rank {r} outside [1, {min(z.shape)}]")
    u, s, vh = np.linalg.svd(z, full_matrices=False)
    return Triple(np.ascontiguousarray(u[:, :r], dtype=np.complex128),
                  np.ascontiguousarray(s[:r]),
                  np.ascontiguousarray(vh[:r].conj().T))


def union_sorted(drawn, kept) -> np.ndarray:
    """np.union1d of drawn indices and a skeleton (lowrank.py:280-281)."""
    return np.union1d(np.asarray(drawn, dtype=np.intp), kept)


def assemble(mid, q_col, q_row, r) -> Triple:
    """SVD of the middle matrix, truncate/zero-pad to r (lowrank.py:284-293)."""
    um, sm, vhm = np.linalg.svd(mid, full_matrices=False)
    t = min(r, sm.shape[0])
    sigma = np.zeros(r)
    sigma[:t] = sm[:t]
    return Triple(complete_basis(q_col @ um[:, :t], r), sigma,
                  complete_basis(q_row @ vhm[:t].conj().T, r))


def complex_normal(rng: np.random.Generator, shape) -> np.ndarray:
    """Independent N(0,1) real and imaginary parts, real block drawn first (lowrank.py:97-99)."""
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def probe_svd(y_col, y_row, r_row, r) -> Triple:
    """Rank-r SVD of a block from stored probe products only (svd_from_probes,
    lowrank.py:204-216): y_col = Z C, y_row = Z* R and the row probe R; the
    middle matrix solves R* Q_col M ~ y_row* Q_row in the floored least squares."""
    width = min(y_col.shape[1], y_col.shape[0], y_row.shape[0])
    q_col = pivoted_basis(y_col, width)
    q_row = pivoted_basis(y_row, width)
    mid = pinv_floored(r_row.conj().T @ q_col) @ (y_row.conj().T @ q_row)
    return assemble(mid, q_col, q_row, r)


def draw_tables(rng, m: int, n: int, r: int, params: Params = Params()):
    """The 8 RNG draws of one sampling SVD, in consumption order (lowrank.py:237-251).

    Draws never depend on pivot results, so the whole table can be made up
    front; returns ``(row_draws[iters+1], col_draws[iters+1])``.
    """
    rq = r * params.q
    rows, cols = [], []
    for _ in range(params.iters + 1):
        rows.append(np.asarray(rng.choice(m, size=min(rq, m), replace=False), dtype=np.intp))
        cols.append(np.asarray(rng.choice(n, size=min(rq, n), replace=False), dtype=np.intp))
    return rows, cols


def sampling_svd(entry, m: int, n: int, r: int, params: Params = Params(), rng=None,
                 trace: dict | None = None) -> Triple:
    """Randomized sampling SVD (lowrank.py:219-258; paper section 2.2).

    ``trace`` (optional) receives the stage intermediates used by staged
    parity tests: skeleton lists per sweep, final sets, bases and mid matrix.
    """
    rng = np.random.default_rng(rng)
    if not 1 <= r <= min(m, n):
        raise ValueError(f"rank {r} outside [1, {min(m, n)}]")
    if r * params.q >= max(m, n):
        return truncated_svd(entry(np.arange(m), np.arange(n)), r)
    all_rows, all_cols = np.arange(m), np.arange(n)
    row_draws, col_draws = draw_tables(rng, m, n, r, params)
    sk_row = np.empty(0, dtype=np.intp)
    sk_col = np.empty(0, dtype=np.intp)
    for s in range(params.iters):
        rows = union_sorted(row_draws[s], sk_row)
        sk_col = np.asarray(sorted(greedy_pivots(entry(rows, all_cols), r)), dtype=np.intp)
        cols = union_sorted(col_draws[s], sk_col)
        sk_row = np.asarray(sorted(greedy_pivots(entry(all_rows, cols).conj().T, r)), dtype=np.intp)
        if trace is not None:
            trace.setdefault("sk_col", []).append(sk_col)
            trace.setdefault("sk_row", []).append(sk_row)
    rows = union_sorted(row_draws[-1], sk_row)
    cols = union_sorted(col_draws[-1], sk_col)
    width = max(r, min(rows.size, cols.size) - r)
    q_col = pivoted_basis(entry(all_rows, cols), min(width, m), pad=False, rel_tol=BASIS_TRIM)
    q_row = pivoted_basis(entry(rows, all_cols).conj().T, min(width, n), pad=False, rel_tol=BASIS_TRIM)
    mid = pinv_floored(q_col[rows, :]) @ entry(rows, cols) @ pinv_floored(q_row[cols, :].conj().T)
    if trace is not None:
        trace.update(rows=rows, cols=cols, q_col=q_col, q_row=q_row, mid=mid)
    return assemble(mid, q_col, q_row, r)
