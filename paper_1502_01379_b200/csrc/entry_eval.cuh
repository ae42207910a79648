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


// A device-evaluable entry oracle: analytic kernels by id, or an explicit
// row-major matrix (the reference's DenseOracle, oracles.py:39-54).
struct EntrySrc {
  int kind;             // BF_KERNEL_FIO | BF_KERNEL_DFTP | BF_KERNEL_DENSE
  uint64_t n;
  const double2* dense; // BF_KERNEL_DENSE: n x n row-major
};

__device__ __forceinline__ double2 entry_eval(const EntrySrc& s, int64_t i, int64_t j) {
  if (s.kind == BF_KERNEL_FIO) return fio_entry(s.n, i, j);
  if (s.kind == BF_KERNEL_DFTP) return dftp_entry(s.n, i, j);
  return s.dense[static_cast<uint64_t>(i) * s.n + j];
}

}  // namespace bfly
