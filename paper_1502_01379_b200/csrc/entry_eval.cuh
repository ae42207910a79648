// entry_eval.cuh — device evaluation of the kernel entries K(x_i, xi_j).
// See entries.cu for the reference expressions and rounding rules.
#pragma once

#include "common.cuh"
#include "../../include/bfly.h"

namespace bfly {

constexpr double kTwoPi = 6.283185307179586;  // fl(2 * pi), the reference's 2.0 * np.pi

__device__ __forceinline__ double2 fio_entry(uint64_t n, int64_t i, int64_t j) {
  const double nd = static_cast<double>(n);
  const double x = __ddiv_rn(static_cast<double>(i), nd);
  const double xi = __dsub_rn(static_cast<double>(j), __ddiv_rn(nd, 2.0));
  const double speed = __ddiv_rn(__dadd_rn(2.0, sin(__dmul_rn(kTwoPi, x))), 8.0);
  const double phase = __dadd_rn(__dmul_rn(x, xi), __dmul_rn(speed, fabs(xi)));
  double s, c;
  sincos(__dmul_rn(kTwoPi, phase), &s, &c);
  return make_double2(c, s);
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

__device__ __forceinline__ double2 radon2d_entry(uint64_t n, int64_t i, int64_t j) {
  const uint32_t bits = (63 - __clzll(static_cast<long long>(n))) / 2;
  const double ns = static_cast<double>(1u << bits);
  uint32_t a1, a2, b1, b2;
  morton_decode(static_cast<uint64_t>(i), bits, &a1, &a2);
  morton_decode(static_cast<uint64_t>(j), bits, &b1, &b2);
  const double x1 = __ddiv_rn(static_cast<double>(a1), ns), x2 = __ddiv_rn(static_cast<double>(a2), ns);
  const double half = __ddiv_rn(ns, 2.0);
  const double xi1 = __dsub_rn(static_cast<double>(b1), half), xi2 = __dsub_rn(static_cast<double>(b2), half);
  const double t1 = __dmul_rn(kTwoPi, x1), t2 = __dmul_rn(kTwoPi, x2);
  const double c1 = __ddiv_rn(__dadd_rn(2.0, __dmul_rn(sin(t1), sin(t2))), 16.0);
  const double c2 = __ddiv_rn(__dadd_rn(2.0, __dmul_rn(cos(t1), cos(t2))), 16.0);
  const double q = __dadd_rn(__dmul_rn(__dmul_rn(c1, c1), __dmul_rn(xi1, xi1)),
                             __dmul_rn(__dmul_rn(c2, c2), __dmul_rn(xi2, xi2)));
  const double phase = __dadd_rn(__dadd_rn(__dmul_rn(x1, xi1), __dmul_rn(x2, xi2)), __dsqrt_rn(q));
  double s, c;
  sincos(__dmul_rn(kTwoPi, phase), &s, &c);
  return make_double2(c, s);
}

// A device-evaluable entry oracle: analytic kernels by id, or an explicit
// row-major matrix (the reference's DenseOracle, oracles.py:39-54).
struct EntrySrc {
  int kind;             // BF_KERNEL_FIO | BF_KERNEL_DFTP | BF_KERNEL_DENSE | BF_KERNEL_RADON2D
  uint64_t n;
  const double2* dense; // BF_KERNEL_DENSE: n x n row-major
};

__device__ __forceinline__ double2 entry_eval(const EntrySrc& s, int64_t i, int64_t j) {
  if (s.kind == BF_KERNEL_FIO) return fio_entry(s.n, i, j);
  if (s.kind == BF_KERNEL_DFTP) return dftp_entry(s.n, i, j);
  if (s.kind == BF_KERNEL_RADON2D) return radon2d_entry(s.n, i, j);
  return s.dense[static_cast<uint64_t>(i) * s.n + j];
}

}  // namespace bfly
