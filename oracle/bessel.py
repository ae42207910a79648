"""Bessel J_m, Y_m and Hankel H1_m order sweeps — NumPy restatement of the
reference ``bessel.py`` (test infrastructure; see oracle/__init__.py).

Algorithm (published, Cephes j0/j1/y0/y1 + Miller's method): orders 0 and 1
from rational approximations (|x| <= 5) or the Hankel asymptotic form
(x > 5); Y upward by the three-term recurrence; J by the normalised backward
recurrence from start = int(max(x + 10 cbrt(x) + 40)) (at least max_order+15)
with the sum rule J0 + 2 (J2 + J4 + ...) = 1 and a 1e-200 rescale checked every
16 steps (reference bessel.py:178-230). The coefficients are Cephes' published
constants, written here as exact hexadecimal doubles.
"""

from __future__ import annotations

import numpy as np

H = float.fromhex
# Cephes tables, grouped per function: (numerator, denominator) coefficient lists
CEPHES = {
    "j0_small": ([H(v) for v in ("-0x1.1dc53ad1c8325p+32", "0x1.c7751c772990dp+40", "-0x1.c5614e0d900f7p+47",
                                 "0x1.13ef869ff5fb4p+53")],
                 [H(v) for v in ("0x1.f3902a696b78cp+8", "0x1.536cb36a21a67p+17", "0x1.719342eac0634p+25",
                                 "0x1.4d5b009444914p+33", "0x1.ebeb372182e46p+40", "0x1.1a6a28c9748e9p+48",
                                 "0x1.c41417e7b2e9cp+54", "0x1.7be34c7b662ccp+60")]),
    "y0_small": ([H(v) for v in ("0x1.e7437e896898fp+13", "-0x1.bf81f32e48896p+23", "0x1.43f78f0284cddp+32",
                                 "-0x1.c957be1d6bd2bp+39", "0x1.3ea723cc3ac2dp+46", "-0x1.8a121d1d8cc02p+51",
                                 "0x1.3a94b660b4003p+55", "-0x1.06d4b5906367bp+54")],
                 [H(v) for v in ("0x1.04522576dfcb6p+10", "0x1.31b76a907bc0cp+19", "0x1.007635164d101p+28",
                                 "0x1.41ddb2b8664bcp+36", "0x1.275fcc57e828ep+44", "0x1.68910dfeb596dp+51",
                                 "0x1.bd25fbcf9b5d0p+57")]),
    "p0": ([H(v) for v in ("0x1.a1d30983b6b27p-11", "0x1.534b0b35dd1cfp-4", "0x1.3d5214e680b98p+0",
                           "0x1.5c9fbe97a0956p+2", "0x1.17e8c69409888p+3", "0x1.53684a59425a1p+2", "0x1p+0")],
           [H(v) for v in ("0x1.e4a80ce039737p-11", "0x1.5ebc5ab5454e3p-4", "0x1.40e72c9b3069fp+0",
                           "0x1.5e247e68162bbp+2", "0x1.18618ea1b21a1p+3", "0x1.53965ed423a19p+2", "0x1p+0")]),
    "q0": ([H(v) for v in ("-0x1.7474238a5384ap-7", "-0x1.4853b3a321174p+0", "-0x1.38dcff50e2c0cp+4",
                           "-0x1.74d2f5a6de8c4p+6", "-0x1.635cc20cae8eap+7", "-0x1.2627aec17392dp+7",
                           "-0x1.9b48c55b218cdp+5", "-0x1.83358d1b9a1ddp+2")],
           [H(v) for v in ("0x1.01457413c25acp+6", "0x1.ac370b1759c7fp+9", "0x1.e54cdbd748cb5p+11",
                           "0x1.c4877bdefd63ep+12", "0x1.72aba1d733b11p+12", "0x1.01c2fc7319e82p+11",
                           "0x1.e402f06280a54p+7")]),
    "j1_small": ([H(v) for v in ("-0x1.ad23c4cda4fc5p+29", "0x1.a52ba0d438c6bp+38", "-0x1.08a92e6ccf175p+46",
                                 "0x1.a2b42a697c482p+51")],
                 [H(v) for v in ("0x1.366b11b7086e7p+9", "0x1.f5eda0dd701b2p+17", "0x1.3e954dc92a1b1p+26",
                                 "0x1.4a13f7befeac1p+34", "0x1.146fb8076ffa8p+42", "0x1.64b0a3eccf45fp+49",
                                 "0x1.3e0bff4653f81p+56", "0x1.2779576702939p+62")]),
    "y1_small": ([H(v) for v in ("0x1.2d2be62f9b6c5p+30", "-0x1.2d72d58836521p+39", "0x1.a0954b0910fefp+46",
                                 "-0x1.ce01a37a1b083p+52", "0x1.679ad0b7366b1p+57", "-0x1.59e415dde2b17p+59")],
                 [H(v) for v in ("0x1.29269a93f7ac2p+9", "0x1.cc160be58ef7fp+17", "0x1.184efa9c8aceep+26",
                                 "0x1.178c3906b7b83p+34", "0x1.c3f5efda99316p+41", "0x1.1a326d71d1e4ep+49",
                                 "0x1.e83e3c547a488p+55", "0x1.b90f190f6747fp+61")]),
    "p1": ([H(v) for v in ("0x1.8f92c4c6c651bp-11", "0x1.2b948a3fec4b6p-4", "0x1.208fec21596d6p+0",
                           "0x1.472c4f8b13a6ap+2", "0x1.0d91c8b5d2f16p+3", "0x1.4dbaa142f81a2p+2", "0x1p+0")],
           [H(v) for v in ("0x1.2b89b13443d69p-11", "0x1.19fdd5948aa83p-4", "0x1.1aea9b850eed6p+0",
                           "0x1.44ba2f7d251a1p+2", "0x1.0ccb9dda2fd65p+3", "0x1.4d6dd4762b4d9p+2", "0x1p+0")]),
    "q1": ([H(v) for v in ("0x1.a27fa6b70ba40p-5", "0x1.3edb5c66d8fd6p+2", "0x1.2f4b99acf1c67p+6",
                           "0x1.6ec7947aa180dp+8", "0x1.636d9b66f6e50p+9", "0x1.2abeab9e802d0p+9",
                           "0x1.a760a4c54bb0bp+7", "0x1.934ff4d159eb5p+4")],
           [H(v) for v in ("0x1.28f3060895077p+6", "0x1.081cba20e5f6fp+10", "0x1.37a691bfdfe81p+12",
                           "0x1.2ad28d280d118p+13", "0x1.f3d0aa6973d14p+12", "0x1.61462b4bd1781p+11",
                           "0x1.5017f6ae75997p+8")]),
}
J0_ROOTS2 = (H("0x1.721fb80462bbbp+2"), H("0x1.e78a4a621dd6fp+4"))   # squares of the first J0 zeros
J1_ROOTS2 = (H("0x1.d5d2b4189822cp+3"), H("0x1.89bf66072a432p+5"))   # squares of the first J1 zeros
TWO_OVER_PI = H("0x1.45f306dc9c883p-1")
QUARTER_PI = H("0x1.921fb54442d18p-1")
THREE_QUARTER_PI = H("0x1.2d97c7f3321d2p+1")
SQRT_TWO_OVER_PI = H("0x1.9884533d43651p-1")
RESCALE = 1e-200


def horner(z, coef, monic=False):
    """sum c_k z^(n-k) by Horner's rule, separate multiply and add (no FMA);
    monic: an implicit leading 1 (Cephes p1evl)."""
    acc = (z + coef[0]) if monic else np.full_like(z, coef[0])
    for c in coef[1:]:
        acc = acc * z + c
    return acc


def _far(x, order):
    """Hankel asymptotic pieces for x > 5: (p, q, x - phase, sqrt(2/pi)/sqrt(x))."""
    pk, qk, phase = ("p0", "q0", QUARTER_PI) if order == 0 else ("p1", "q1", THREE_QUARTER_PI)
    w = 5.0 / x
    z = w * w
    p = horner(z, CEPHES[pk][0]) / horner(z, CEPHES[pk][1])
    q = horner(z, CEPHES[qk][0]) / horner(z, CEPHES[qk][1], monic=True)
    return p, q, x - phase, SQRT_TWO_OVER_PI / np.sqrt(x)


def j0(x):
    x = np.abs(np.asarray(x, dtype=float))
    out = np.empty_like(x)
    near = x <= 5.0
    z = x[near] * x[near]
    val = (z - J0_ROOTS2[0]) * (z - J0_ROOTS2[1]) * horner(z, CEPHES["j0_small"][0]) \
        / horner(z, CEPHES["j0_small"][1], monic=True)
    out[near] = np.where(x[near] < 1e-5, 1.0 - z / 4.0, val)
    xf = x[~near]
    p, q, xn, amp = _far(xf, 0)
    out[~near] = amp * (p * np.cos(xn) - (5.0 / xf) * q * np.sin(xn))
    return out


def y0(x):
    x = np.asarray(x, dtype=float)
    if (x <= 0).any():
        raise ValueError("y0 requires x > 0")
    out = np.empty_like(x)
    near = x <= 5.0
    xs = x[near]
    z = xs * xs
    out[near] = horner(z, CEPHES["y0_small"][0]) / horner(z, CEPHES["y0_small"][1], monic=True) \
        + TWO_OVER_PI * np.log(xs) * j0(xs)
    xf = x[~near]
    p, q, xn, amp = _far(xf, 0)
    out[~near] = amp * (p * np.sin(xn) + (5.0 / xf) * q * np.cos(xn))
    return out


def j1(x):
    x = np.asarray(x, dtype=float)
    sgn = np.sign(x)
    x = np.abs(x)
    out = np.empty_like(x)
    near = x <= 5.0
    z = x[near] * x[near]
    out[near] = x[near] * (z - J1_ROOTS2[0]) * (z - J1_ROOTS2[1]) * horner(z, CEPHES["j1_small"][0]) \
        / horner(z, CEPHES["j1_small"][1], monic=True)
    xf = x[~near]
    p, q, xn, amp = _far(xf, 1)
    out[~near] = amp * (p * np.cos(xn) - (5.0 / xf) * q * np.sin(xn))
    return sgn * out


def y1(x):
    x = np.asarray(x, dtype=float)
    if (x <= 0).any():
        raise ValueError("y1 requires x > 0")
    out = np.empty_like(x)
    near = x <= 5.0
    xs = x[near]
    z = xs * xs
    out[near] = xs * horner(z, CEPHES["y1_small"][0]) / horner(z, CEPHES["y1_small"][1], monic=True) \
        + TWO_OVER_PI * (j1(xs) * np.log(xs) - 1.0 / xs)
    xf = x[~near]
    p, q, xn, amp = _far(xf, 1)
    out[~near] = amp * (p * np.sin(xn) + (5.0 / xf) * q * np.cos(xn))
    return out


def sweep_start(x, max_order: int) -> int:
    """Backward-recurrence start index of a batch (reference bessel.py:196-197)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    return max(int(np.max(x + 10.0 * np.cbrt(x) + 40.0)), max_order + 15)


def jy_orders(x, max_order: int, start: int | None = None):
    """J_m(x), Y_m(x) for m = 0..max_order over a batch of x > 0 (bessel.py:178-222).
    ``start`` defaults to the batch's own sweep_start (what the reference uses)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    if (x <= 0).any():
        raise ValueError("order sweep requires x > 0")
    nx, width = x.shape[0], max_order + 1
    ys = np.empty((nx, width))
    ys[:, 0] = y0(x)
    if max_order >= 1:
        ys[:, 1] = y1(x)
    for m in range(1, max_order):
        ys[:, m + 1] = (2.0 * m / x) * ys[:, m] - ys[:, m - 1]
    if start is None:
        start = sweep_start(x, max_order)
    js = np.empty((nx, width))
    prev, cur = np.zeros(nx), np.full(nx, 1e-150)
    norm = 2.0 * cur if start % 2 == 0 else np.zeros(nx)
    for m in range(start, 0, -1):
        prev, cur = cur, (2.0 * m / x) * cur - prev
        order = m - 1
        if order <= max_order:
            js[:, order] = cur
        if order > 0 and order % 2 == 0:
            norm = norm + 2.0 * cur
        if m % 16 == 0:
            big = np.abs(cur) > 1e200
            if big.any():
                prev[big] *= RESCALE
                cur[big] *= RESCALE
                norm[big] *= RESCALE
                if order <= max_order:
                    js[big, order:] *= RESCALE
    norm = norm + cur
    return js / norm[:, None], ys


def hankel1_orders(x, max_order: int, start: int | None = None) -> np.ndarray:
    """H1_m(x) = J_m(x) + i Y_m(x), m = 0..max_order (bessel.py:225-230)."""
    js, ys = jy_orders(x, max_order, start)
    return js + 1j * ys


def hankel_points(n: int, rows) -> np.ndarray:
    """x_i = n + (2 pi / 3) i (HankelKernel.point, kernels.py:60-61)."""
    return n + (2.0 * np.pi / 3.0) * np.asarray(rows, dtype=np.intp).astype(float)


def hankel_table(n: int, batch: int = 256) -> np.ndarray:
    """The full (n x n) Hankel matrix filled the way the reference's cached
    HankelKernel fills it from empty on block(arange(n), arange(n)): sorted rows in
    batches of `batch`, each batch one sweep to order n-1 (kernels.py:63-82)."""
    out = np.empty((n, n), dtype=np.complex128)
    for lo in range(0, n, batch):
        rows = np.arange(lo, min(n, lo + batch))
        out[rows] = hankel1_orders(hankel_points(n, rows), n - 1)
    return out
