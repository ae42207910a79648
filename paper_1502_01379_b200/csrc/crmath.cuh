// crmath.cuh — correctly rounded sin/cos of moderate float64 arguments, in double-double.
//
// The FIO phase speed c(x) = (2 + sin 2 pi x)/8 and the 2-D Radon speeds c1, c2 are
// multiplied by |xi| <= N/2 inside the phase, so a one-ulp difference between the device
// sin and glibc's (the reference's np.sin) grows into a phase error of up to ulp(c) N/2:
// 4.7e-10 at N = 2^20, 7.5e-9 at 2^24, a million times the rounding noise the staged
// parity envelope is calibrated to (SURVEY.md §8(c) stage 4). Evaluating these sines in
// double-double and rounding once gives the correctly rounded value, which is what glibc
// returns for every x = i/N (checked exhaustively for N = 2^24 against NumPy,
// tests/test_entries_gpu.py). They depend on the row point only, so each plan-free entry
// source tabulates them once per N (entries.cu: row_table).
#pragma once

#include <cstdint>

namespace bfly {
namespace cr {

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}

__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}

__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}

__device__ __forceinline__ dd add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = quick_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return quick_two_sum(s.hi, s.lo);
}

__device__ __forceinline__ dd mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
  return quick_two_sum(p.hi, p.lo);
}

__device__ __forceinline__ dd div_d(dd a, double b) {
  const double q1 = __ddiv_rn(a.hi, b);
  const dd p = two_prod(q1, b);
  dd r = two_sum(a.hi, -p.hi);
  r.lo = __dadd_rn(r.lo, __dsub_rn(a.lo, p.lo));
  const double q2 = __ddiv_rn(__dadd_rn(r.hi, r.lo), b);
  return quick_two_sum(q1, q2);
}

// pi/2 = P1 + P2 + P3 to ~1e-49
constexpr double kP1 = 1.5707963267948966e+00;
constexpr double kP2 = 6.123233995736766e-17;
constexpr double kP3 = -1.4973849048591698e-33;

// sin and cos of x (|x| <= 1e3), each correctly rounded to float64 except in cases
// closer to a rounding boundary than ~2^-100 relative.
__device__ inline void sincos_cr(double x, double* sn, double* cs) {
  const double k = rint(__dmul_rn(x, 0.6366197723675814));  // x * 2/pi
  const dd p1 = two_prod(k, kP1);
  dd r = two_sum(x, -p1.hi);      // exact (Sterbenz) for the quadrant's k
  r = add(r, dd{-p1.lo, 0.0});
  const dd p2 = two_prod(k, kP2);
  r = add(r, dd{-p2.hi, -p2.lo});
  r = add(r, dd{__dmul_rn(-k, kP3), 0.0});
  const dd t = mul(r, r);
  // Taylor series in double-double: |r| <= pi/4, terms to r^27/27! (< 2e-31 relative)
  dd ps{0.0, 0.0}, pc{0.0, 0.0};
  dd fs{1.0, 0.0}, fc{1.0, 0.0};  // 1/(2j+1)! and 1/(2j)!
  dd cs_coef[14], sn_coef[14];
  for (int j = 0; j < 14; ++j) {
    sn_coef[j] = (j & 1) ? dd{-fs.hi, -fs.lo} : fs;
    cs_coef[j] = (j & 1) ? dd{-fc.hi, -fc.lo} : fc;
    fs = div_d(fs, static_cast<double>((2 * j + 2) * (2 * j + 3)));
    fc = div_d(fc, static_cast<double>((2 * j + 1) * (2 * j + 2)));
  }
  for (int j = 13; j >= 0; --j) {
    ps = add(sn_coef[j], mul(t, ps));
    pc = add(cs_coef[j], mul(t, pc));
  }
  const dd s = mul(r, ps);
  const dd c = pc;
  const int q = static_cast<int>(static_cast<int64_t>(k) & 3);
  const double sv = q == 0 ? s.hi : q == 1 ? c.hi : q == 2 ? -s.hi : -c.hi;
  const double cv = q == 0 ? c.hi : q == 1 ? -s.hi : q == 2 ? -c.hi : s.hi;
  *sn = sv;
  *cs = cv;
}

}  // namespace cr
}  // namespace bfly
