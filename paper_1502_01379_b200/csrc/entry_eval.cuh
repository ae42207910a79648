// entry_eval.cuh — device evaluation of the kernel entries K(x_i, xi_j).
// See entries.cu for the reference expressions and rounding rules.
#pragma once

#include "common.cuh"
#include "../../include/bfly.h"
#include "crmath.cuh"

namespace bfly {

constexpr double kTwoPi = 6.283185307179586;  // fl(2 * pi), the reference's 2.0 * np.pi

// tab[i] = c(x_i) = (2 + sin(2 pi x_i))/8 with a correctly rounded sine (row_table)
__device__ __forceinline__ double2 fio_entry(uint64_t n, const double* __restrict__ tab, int64_t i, int64_t j) {
  const double nd = static_cast<double>(n);
  const double x = __ddiv_rn(static_cast<double>(i), nd);
  const double xi = __dsub_rn(static_cast<double>(j), __ddiv_rn(nd, 2.0));
  const double phase = __dadd_rn(__dmul_rn(x, xi), __dmul_rn(tab[i], fabs(xi)));
  double s, c;
  sincos(__dmul_rn(kTwoPi, phase), &s, &c);
  return make_double2(c, s);
}

// the table entry itself: the reference's float64 ops on a correctly rounded sine
__device__ __forceinline__ double fio_speed(uint64_t n, uint64_t i) {
  const double x = __ddiv_rn(static_cast<double>(i), static_cast<double>(n));
  double s, c;
  cr::sincos_cr(__dmul_rn(kTwoPi, x), &s, &c);
  return __ddiv_rn(__dadd_rn(2.0, s), 8.0);
}

__device__ __forceinline__ double2 dftp_entry(uint64_t n, int64_t i, int64_t j) {
  const uint64_t t = (static_cast<uint64_t>(i) * static_cast<uint64_t>(j)) % n;
  const double frac = __ddiv_rn(static_cast<double>(t), static_cast<double>(n));
  double s, c;
  sincos(__dmul_rn(kTwoPi, frac), &s, &c);
  return make_double2(c, s);
}


// BASELINE configs 3/4b: the 2-D generalized Radon kernel on an n_side^2 grid
// with Morton (Z-order) indices (oracle/entries.py:radon2d_block defines the
// convention and the rounding order, followed here with _rn intrinsics).
__device__ __forceinline__ void morton_decode(uint64_t z, uint32_t bits, uint32_t* a1, uint32_t* a2) {
  uint32_t x = 0, y = 0;
  for (uint32_t k = 0; k < bits; ++k) {
    y |= static_cast<uint32_t>((z >> (2 * k)) & 1u) << k;
    x |= static_cast<uint32_t>((z >> (2 * k + 1)) & 1u) << k;
  }
  *a1 = x;
  *a2 = y;
}

// tab[a] = sin(t), tab[ns + a] = cos(t), t = fl(2 pi a/ns), correctly rounded (row_table)
__device__ __forceinline__ double2 radon2d_entry(uint64_t n, const double* __restrict__ tab, int64_t i, int64_t j) {
  const uint32_t bits = (63 - __clzll(static_cast<long long>(n))) / 2;
  const uint32_t nsi = 1u << bits;
  const double ns = static_cast<double>(nsi);
  uint32_t a1, a2, b1, b2;
  morton_decode(static_cast<uint64_t>(i), bits, &a1, &a2);
  morton_decode(static_cast<uint64_t>(j), bits, &b1, &b2);
  const double x1 = __ddiv_rn(static_cast<double>(a1), ns), x2 = __ddiv_rn(static_cast<double>(a2), ns);
  const double half = __ddiv_rn(ns, 2.0);
  const double xi1 = __dsub_rn(static_cast<double>(b1), half), xi2 = __dsub_rn(static_cast<double>(b2), half);
  const double c1 = __ddiv_rn(__dadd_rn(2.0, __dmul_rn(tab[a1], tab[a2])), 16.0);
  const double c2 = __ddiv_rn(__dadd_rn(2.0, __dmul_rn(tab[nsi + a1], tab[nsi + a2])), 16.0);
  const double q = __dadd_rn(__dmul_rn(__dmul_rn(c1, c1), __dmul_rn(xi1, xi1)),
                             __dmul_rn(__dmul_rn(c2, c2), __dmul_rn(xi2, xi2)));
  const double phase = __dadd_rn(__dadd_rn(__dmul_rn(x1, xi1), __dmul_rn(x2, xi2)), __dsqrt_rn(q));
  double s, c;
  sincos(__dmul_rn(kTwoPi, phase), &s, &c);
  return make_double2(c, s);
}

// The reference's centered transform DftKernel.block (kernels.py:87-97):
// xi = row - n/2, x = col/n, exp(-2j*pi*xi*x) evaluated by NumPy as
// ((-2j*pi)*xi)*x with complex-by-real products, i.e. angle fl(fl(-fl(2 pi) xi) x)
// and a real part of +-0 (exp(+-0) = 1 exactly): (cos a, sin a), no FMA.
__device__ __forceinline__ double2 dft_entry(uint64_t n, int64_t i, int64_t j) {
  const double xi = __dsub_rn(static_cast<double>(i), 0.5 * static_cast<double>(n));
  const double x = __ddiv_rn(static_cast<double>(j), static_cast<double>(n));
  double s, c;
  sincos(__dmul_rn(__dmul_rn(-kTwoPi, xi), x), &s, &c);
  return make_double2(c, s);
}

// A device-evaluable entry oracle: analytic kernels by id, an explicit row-major
// matrix (the reference's DenseOracle, oracles.py:39-54), or per-middle-block
// windows of any entry oracle evaluated elsewhere (BF_KERNEL_TILES: the window of
// block (bi, bj) is tile slot[bi m + bj], side x side row-major).
struct EntrySrc {
  int kind;             // BF_KERNEL_FIO | DFTP | DENSE | RADON2D | DFT | TILES
  uint64_t n;
  const double2* dense; // BF_KERNEL_DENSE: n x n row-major; BF_KERNEL_TILES: the tiles
  const double* tab;    // BF_KERNEL_FIO / BF_KERNEL_RADON2D: row_table(kind, n)
  const int32_t* slot;  // BF_KERNEL_TILES: (m, m) tile index per middle block, -1 = absent
  uint64_t side, m;     // BF_KERNEL_TILES: middle block side and count per dimension
};

__device__ __forceinline__ double2 entry_eval(const EntrySrc& s, int64_t i, int64_t j) {
  if (s.kind == BF_KERNEL_FIO) return fio_entry(s.n, s.tab, i, j);
  if (s.kind == BF_KERNEL_DFTP) return dftp_entry(s.n, i, j);
  if (s.kind == BF_KERNEL_RADON2D) return radon2d_entry(s.n, s.tab, i, j);
  if (s.kind == BF_KERNEL_DFT) return dft_entry(s.n, i, j);
  if (s.kind == BF_KERNEL_TILES) {
    const uint64_t bi = static_cast<uint64_t>(i) / s.side, bj = static_cast<uint64_t>(j) / s.side;
    const uint64_t t = static_cast<uint64_t>(s.slot[bi * s.m + bj]);
    return s.dense[(t * s.side + (static_cast<uint64_t>(i) - bi * s.side)) * s.side +
                   (static_cast<uint64_t>(j) - bj * s.side)];
  }
  return s.dense[static_cast<uint64_t>(i) * s.n + j];
}

// Host side (entries.cu): the per-N table of the row-only transcendental terms, built on
// the device once per (device, kind, n) and kept for the process (n doubles for FIO,
// 2 n_side for the 2-D kernel; NULL with the error set on failure).
const double* row_table(int kind, uint64_t n, cudaStream_t st);

}  // namespace bfly
