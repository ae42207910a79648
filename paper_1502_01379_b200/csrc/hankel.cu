// hankel.cu — Hankel-kernel entries K[i, j] = H1_j(x_i) on the device
// (reference kernels.py:45-84, bessel.py:178-230; §8(f) rank 4).
//
// One thread per point x: orders 0/1 from the Cephes rational / asymptotic
// forms, Y_m upward by the three-term recurrence, J_m by Miller's normalised
// backward recurrence from the caller's `start` (the reference takes
// int(max(x + 10 cbrt(x) + 40)) over its batch, at least max_order + 15; the
// host computes it with NumPy so the J sweep is the reference's bit for bit).
// Every operation is an explicitly rounded IEEE op (no FMA contraction), in
// NumPy's evaluation order; only sin/cos/log of the order-0/1 seeds can differ
// from the host libm by an ulp. The reference's retroactive 1e-200 rescale of
// already stored J's (`js[big, order:] *= 1e-200`) is replayed at the end from
// a per-thread list of rescale orders, multiplication by multiplication.
#include "common.cuh"
#include "plan.h"

namespace bfly {
namespace {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// Cephes j0/j1/y0/y1 coefficient tables (published constants, exact hex doubles)
__constant__ double kJ0N[4] = {-0x1.1dc53ad1c8325p+32, 0x1.c7751c772990dp+40, -0x1.c5614e0d900f7p+47,
                               0x1.13ef869ff5fb4p+53};
__constant__ double kJ0D[8] = {0x1.f3902a696b78cp+8,  0x1.536cb36a21a67p+17, 0x1.719342eac0634p+25,
                               0x1.4d5b009444914p+33, 0x1.ebeb372182e46p+40, 0x1.1a6a28c9748e9p+48,
                               0x1.c41417e7b2e9cp+54, 0x1.7be34c7b662ccp+60};
__constant__ double kY0N[8] = {0x1.e7437e896898fp+13, -0x1.bf81f32e48896p+23, 0x1.43f78f0284cddp+32,
                               -0x1.c957be1d6bd2bp+39, 0x1.3ea723cc3ac2dp+46, -0x1.8a121d1d8cc02p+51,
                               0x1.3a94b660b4003p+55, -0x1.06d4b5906367bp+54};
__constant__ double kY0D[7] = {0x1.04522576dfcb6p+10, 0x1.31b76a907bc0cp+19, 0x1.007635164d101p+28,
                               0x1.41ddb2b8664bcp+36, 0x1.275fcc57e828ep+44, 0x1.68910dfeb596dp+51,
                               0x1.bd25fbcf9b5d0p+57};
__constant__ double kP0N[7] = {0x1.a1d30983b6b27p-11, 0x1.534b0b35dd1cfp-4, 0x1.3d5214e680b98p+0,
                               0x1.5c9fbe97a0956p+2,  0x1.17e8c69409888p+3, 0x1.53684a59425a1p+2, 0x1p+0};
__constant__ double kP0D[7] = {0x1.e4a80ce039737p-11, 0x1.5ebc5ab5454e3p-4, 0x1.40e72c9b3069fp+0,
                               0x1.5e247e68162bbp+2,  0x1.18618ea1b21a1p+3, 0x1.53965ed423a19p+2, 0x1p+0};
__constant__ double kQ0N[8] = {-0x1.7474238a5384ap-7, -0x1.4853b3a321174p+0, -0x1.38dcff50e2c0cp+4,
                               -0x1.74d2f5a6de8c4p+6, -0x1.635cc20cae8eap+7, -0x1.2627aec17392dp+7,
                               -0x1.9b48c55b218cdp+5, -0x1.83358d1b9a1ddp+2};
__constant__ double kQ0D[7] = {0x1.01457413c25acp+6,  0x1.ac370b1759c7fp+9,  0x1.e54cdbd748cb5p+11,
                               0x1.c4877bdefd63ep+12, 0x1.72aba1d733b11p+12, 0x1.01c2fc7319e82p+11,
                               0x1.e402f06280a54p+7};
__constant__ double kJ1N[4] = {-0x1.ad23c4cda4fc5p+29, 0x1.a52ba0d438c6bp+38, -0x1.08a92e6ccf175p+46,
                               0x1.a2b42a697c482p+51};
__constant__ double kJ1D[8] = {0x1.366b11b7086e7p+9,  0x1.f5eda0dd701b2p+17, 0x1.3e954dc92a1b1p+26,
                               0x1.4a13f7befeac1p+34, 0x1.146fb8076ffa8p+42, 0x1.64b0a3eccf45fp+49,
                               0x1.3e0bff4653f81p+56, 0x1.2779576702939p+62};
__constant__ double kY1N[6] = {0x1.2d2be62f9b6c5p+30, -0x1.2d72d58836521p+39, 0x1.a0954b0910fefp+46,
                               -0x1.ce01a37a1b083p+52, 0x1.679ad0b7366b1p+57, -0x1.59e415dde2b17p+59};
__constant__ double kY1D[8] = {0x1.29269a93f7ac2p+9,  0x1.cc160be58ef7fp+17, 0x1.184efa9c8aceep+26,
                               0x1.178c3906b7b83p+34, 0x1.c3f5efda99316p+41, 0x1.1a326d71d1e4ep+49,
                               0x1.e83e3c547a488p+55, 0x1.b90f190f6747fp+61};
__constant__ double kP1N[7] = {0x1.8f92c4c6c651bp-11, 0x1.2b948a3fec4b6p-4, 0x1.208fec21596d6p+0,
                               0x1.472c4f8b13a6ap+2,  0x1.0d91c8b5d2f16p+3, 0x1.4dbaa142f81a2p+2, 0x1p+0};
__constant__ double kP1D[7] = {0x1.2b89b13443d69p-11, 0x1.19fdd5948aa83p-4, 0x1.1aea9b850eed6p+0,
                               0x1.44ba2f7d251a1p+2,  0x1.0ccb9dda2fd65p+3, 0x1.4d6dd4762b4d9p+2, 0x1p+0};
__constant__ double kQ1N[8] = {0x1.a27fa6b70ba40p-5, 0x1.3edb5c66d8fd6p+2, 0x1.2f4b99acf1c67p+6,
                               0x1.6ec7947aa180dp+8, 0x1.636d9b66f6e50p+9, 0x1.2abeab9e802d0p+9,
                               0x1.a760a4c54bb0bp+7, 0x1.934ff4d159eb5p+4};
__constant__ double kQ1D[7] = {0x1.28f3060895077p+6,  0x1.081cba20e5f6fp+10, 0x1.37a691bfdfe81p+12,
                               0x1.2ad28d280d118p+13, 0x1.f3d0aa6973d14p+12, 0x1.61462b4bd1781p+11,
                               0x1.5017f6ae75997p+8};
constexpr double kJ0Z1 = 0x1.721fb80462bbbp+2, kJ0Z2 = 0x1.e78a4a621dd6fp+4;  // squared J0 zeros
constexpr double kJ1Z1 = 0x1.d5d2b4189822cp+3, kJ1Z2 = 0x1.89bf66072a432p+5;  // squared J1 zeros
constexpr double kTwoOverPi = 0x1.45f306dc9c883p-1, kPiO4 = 0x1.921fb54442d18p-1;
constexpr double k3PiO4 = 0x1.2d97c7f3321d2p+1, kSqrt2OPi = 0x1.9884533d43651p-1;

template <int N>
__device__ __forceinline__ double horner(double z, const double (&c)[N]) {
  double acc = c[0];
#pragma unroll
  for (int k = 1; k < N; ++k) acc = add(mul(acc, z), c[k]);
  return acc;
}
template <int N>
__device__ __forceinline__ double horner_monic(double z, const double (&c)[N]) {
  double acc = add(z, c[0]);
#pragma unroll
  for (int k = 1; k < N; ++k) acc = add(mul(acc, z), c[k]);
  return acc;
}

// order 0 (first = J0, second = Y0) and order 1 seeds at x > 0
__device__ void seeds(double x, double* j0, double* y0, double* j1, double* y1) {
  if (x <= 5.0) {
    const double z = mul(x, x);
    double j0v = dvd(mul(mul(sub(z, kJ0Z1), sub(z, kJ0Z2)), horner(z, kJ0N)), horner_monic(z, kJ0D));
    if (x < 1e-5) j0v = sub(1.0, dvd(z, 4.0));
    const double lg = log(x);
    const double j1v = dvd(mul(mul(mul(x, sub(z, kJ1Z1)), sub(z, kJ1Z2)), horner(z, kJ1N)), horner_monic(z, kJ1D));
    *j0 = j0v;
    *y0 = add(dvd(horner(z, kY0N), horner_monic(z, kY0D)), mul(mul(kTwoOverPi, lg), j0v));
    *j1 = j1v;
    *y1 = add(dvd(mul(x, horner(z, kY1N)), horner_monic(z, kY1D)), mul(kTwoOverPi, sub(mul(j1v, lg), dvd(1.0, x))));
    return;
  }
  const double w = dvd(5.0, x), z = mul(w, w), amp = dvd(kSqrt2OPi, sqrt(x)), f = dvd(5.0, x);
  {
    const double p = dvd(horner(z, kP0N), horner(z, kP0D)), q = dvd(horner(z, kQ0N), horner_monic(z, kQ0D));
    const double xn = sub(x, kPiO4), s = sin(xn), c = cos(xn);
    *j0 = mul(amp, sub(mul(p, c), mul(mul(f, q), s)));
    *y0 = mul(amp, add(mul(p, s), mul(mul(f, q), c)));
  }
  {
    const double p = dvd(horner(z, kP1N), horner(z, kP1D)), q = dvd(horner(z, kQ1N), horner_monic(z, kQ1D));
    const double xn = sub(x, k3PiO4), s = sin(xn), c = cos(xn);
    *j1 = mul(amp, sub(mul(p, c), mul(mul(f, q), s)));
    *y1 = mul(amp, add(mul(p, s), mul(mul(f, q), c)));
  }
}

constexpr int kMaxRescale = 16;

__global__ void k_hankel_orders(const double* __restrict__ xs, int nx, int max_order, int64_t start,
                                double2* __restrict__ out, int64_t ld, int* __restrict__ status) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nx) return;
  const double x = xs[t];
  double2* row = out + static_cast<int64_t>(t) * ld;
  if (!(x > 0.0)) {
    atomicExch(status, 1);
    return;
  }
  double j0, y0, j1, y1;
  seeds(x, &j0, &y0, &j1, &y1);
  // Y upward: ys[m+1] = (2m / x) ys[m] - ys[m-1]
  row[0].y = y0;
  if (max_order >= 1) {
    row[1].y = y1;
    double ym1 = y0, ym = y1;
    for (int m = 1; m < max_order; ++m) {
      const double yn = sub(mul(dvd(2.0 * m, x), ym), ym1);
      row[m + 1].y = yn;
      ym1 = ym;
      ym = yn;
    }
  }
  // J backward (Miller), raw values stored, rescale orders remembered
  int resc[kMaxRescale];
  int nres = 0;
  double prev = 0.0, cur = 1e-150;
  double norm = (start % 2 == 0) ? mul(2.0, cur) : 0.0;
  for (int64_t m = start; m > 0; --m) {
    const double nx_ = sub(mul(dvd(2.0 * static_cast<double>(m), x), cur), prev);
    prev = cur;
    cur = nx_;
    const int64_t order = m - 1;
    if (order <= max_order) row[order].x = cur;
    if (order > 0 && order % 2 == 0) norm = add(norm, mul(2.0, cur));
    if (m % 16 == 0 && fabs(cur) > 1e200) {
      prev = mul(prev, 1e-200);
      cur = mul(cur, 1e-200);
      norm = mul(norm, 1e-200);
      if (order <= max_order) {
        if (nres == kMaxRescale) {
          atomicExch(status, 2);
          return;
        }
        resc[nres++] = static_cast<int>(order);
      }
    }
  }
  norm = add(norm, cur);
  // replay the retroactive rescales (each stored order o saw every event at order <= o,
  // in event order), then js /= norm
  for (int o = 0; o <= max_order; ++o) {
    double v = row[o].x;
    for (int e = 0; e < nres; ++e)
      if (resc[e] <= o) v = mul(v, 1e-200);
    row[o].x = dvd(v, norm);
  }
}

}  // namespace
}  // namespace bfly

using namespace bfly;

extern "C" int bf_hankel_orders(const double* x, uint32_t nx, uint32_t max_order, int64_t start, void* out,
                                uint64_t ld, void* stream) {
  if (!nx) return BF_OK;
  if (!x || !out) return fail(BF_EINVAL, "null pointer");
  if (ld < static_cast<uint64_t>(max_order) + 1) return fail(BF_EINVAL, "row stride below max_order + 1");
  if (start < static_cast<int64_t>(max_order) + 15) return fail(BF_EINVAL, "sweep start below max_order + 15");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* status = nullptr;
  BF_CUDA(cudaMallocAsync(&status, sizeof(int), st));
  BF_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
  k_hankel_orders<<<(nx + 127) / 128, 128, 0, st>>>(x, static_cast<int>(nx), static_cast<int>(max_order), start,
                                                    static_cast<double2*>(out), static_cast<int64_t>(ld), status);
  int h = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(status, st);
  if (e != cudaSuccess) return cuda_fail(e, "bf_hankel_orders");
  if (h == 1) return fail(BF_EINVAL, "order sweep requires x > 0");
  if (h == 2) return fail(BF_EINVAL, "order sweep: too many rescale events");
  return BF_OK;
}
