// linalg.cuh — CTA-level dense kernels for the construction: block
// reductions, a complex one-sided Jacobi SVD on shared-memory matrices, and
// the floored inverse of lowrank.py. One CTA owns one small problem.
#pragma once

#include <cfloat>

#include "common.cuh"

namespace bfly {

constexpr double kPinvFloor = 1e-13;  // lowrank.py:22 PINV_FLOOR
constexpr double kPivotTie = 1e-14;   // lowrank.py:25 PIVOT_TIE
constexpr double kBasisTrim = 1e-11;  // lowrank.py:30 BASIS_TRIM

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double abs2(double2 a) { return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)); }

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  return v;
}

// Block-wide reductions (blockDim.x multiple of 32, <= 1024); scratch >= 32 doubles.
__device__ double block_max(double v, double* scratch) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  v = l < nw ? scratch[l] : -DBL_MAX;
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ int block_min_int(int v, int* scratch) {
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  v = l < nw ? scratch[l] : INT_MAX;
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// Fixed-order (deterministic) block sum.
__device__ double block_sum(double v, double* scratch) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  v = l < nw ? scratch[l] : 0.0;
  return warp_sum(v);
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum; PW_BLOCKSIZE 128): the order np.sum uses along a contiguous
// axis. Used so the initial pivot norms are bit-identical to the reference's
// whenever the reference reduces over a contiguous axis. Single thread.
template <typename F>
__device__ __forceinline__ double pairwise_leaf(const F& get, int lo, int n) {
  if (n < 8) {
    double res = -0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, get(lo + i));
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = get(lo + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], get(lo + i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, get(lo + i));
  return res;
}

// The recursion pairwise(lo, n) = pairwise(lo, n2) + pairwise(lo + n2, n - n2),
// n2 = n/2 - (n/2) % 8, evaluated iteratively (explicit post-order stack) so no
// device call stack is needed.
template <typename F>
__device__ double pairwise_sum(const F& get, int lo0, int n0) {
  int los[24], ns[24], ph[24];
  double left[24];
  int sp = 0;
  los[0] = lo0;
  ns[0] = n0;
  ph[0] = 0;
  double ret = 0.0;
  bool returning = false;
  while (true) {
    if (returning) {
      if (sp < 0) return ret;
      if (ph[sp] == 1) {
        left[sp] = ret;
        ph[sp] = 2;
        const int n2 = ns[sp] / 2 - (ns[sp] / 2) % 8;
        los[sp + 1] = los[sp] + n2;
        ns[sp + 1] = ns[sp] - n2;
        ph[sp + 1] = 0;
        ++sp;
        returning = false;
      } else {
        ret = __dadd_rn(left[sp], ret);
        --sp;
      }
      continue;
    }
    if (ns[sp] <= 128) {
      ret = pairwise_leaf(get, los[sp], ns[sp]);
      --sp;
      returning = true;
      continue;
    }
    ph[sp] = 1;
    const int n2 = ns[sp] / 2 - (ns[sp] / 2) % 8;
    los[sp + 1] = los[sp];
    ns[sp + 1] = n2;
    ph[sp + 1] = 0;
    ++sp;
  }
}

// Sequential sum (np.sum over a non-contiguous axis walks it in order).
template <typename F>
__device__ double sequential_sum(const F& get, int n) {
  double res = 0.0;
  for (int i = 0; i < n; ++i) res = __dadd_rn(res, get(i));
  return res;
}

// ---------------------------------------------------------------- Jacobi SVD
// One-sided (Hestenes) Jacobi on the columns of A (m x n, m >= n) held
// COLUMN-major in shared memory (element (i, c) at A[c * lda + i]) so the 32
// lanes of a warp touch 32 consecutive elements of a column: no bank
// conflicts. On return A holds U*Sigma (unsorted, unnormalised) and V (n x n,
// also column-major, ldv) the accumulated unitary. Pairs run in round-robin
// tournament order, one warp per pair; every reduction has a fixed order, so
// the result is deterministic.
#ifdef BF_JACOBI_STATS
__device__ int g_jacobi_sweeps;
#endif
__device__ void jacobi_cols(double2* A, int m, int n, int lda, double2* V, int ldv, int* flag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int c = i / n, r = i % n;
    V[c * ldv + r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  const int nn = n + (n & 1);  // tournament over an even count (a dummy column if n is odd)
  const double tol = (m > 8 ? m : 8) * 2.220446049250313e-16;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int round = 0; round < nn - 1; ++round) {
      for (int pi = warp; pi < nn / 2; pi += nw) {
        // circle method: position 0 fixed, others rotate
        int a = pi == 0 ? 0 : 1 + (pi - 1 + round) % (nn - 1);
        int b = 1 + (nn - 2 - pi + round) % (nn - 1);
        if (a > b) { const int t = a; a = b; b = t; }
        if (b >= n) continue;
        double2* ca = A + a * lda;
        double2* cb = A + b * lda;
        double al = 0, be = 0;
        double2 ga = make_double2(0, 0);
        for (int i = lane; i < m; i += 32) {
          const double2 x = ca[i], y = cb[i];
          al += x.x * x.x + x.y * x.y;
          be += y.x * y.x + y.y * y.y;
          const double2 g = cmulc(x, y);
          ga.x += g.x;
          ga.y += g.y;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum2(ga);
        // converged pair: |a^H b| <= m eps |a| |b| (the rounding level of the dot product
        // itself; a tighter test can keep rotating noise and never terminate)
        const double g2 = ga.x * ga.x + ga.y * ga.y;
        if (g2 == 0.0 || g2 <= tol * tol * al * be) continue;
        if (lane == 0) *flag = 1;
        // rotation from one rsqrt / sqrt / div / rsqrt chain (the pair's latency
        // is the Jacobi's critical path)
        const double ig = rsqrt(g2);
        const double zeta = (be - al) * 0.5 * ig;
        const double az = fabs(zeta), sgn = zeta >= 0 ? 1.0 : -1.0;
        const double t = az > 1e150 ? sgn * 0.5 / az : sgn / (az + sqrt(1.0 + zeta * zeta));
        const double c = rsqrt(1.0 + t * t), s = c * t;
        const double2 ph = make_double2(ga.x * ig, -ga.y * ig);  // e^{-i phi}
        // [a', b'] = [a, b] [[c, s], [-s e^{-i phi}, c e^{-i phi}]]
        for (int i = lane; i < m; i += 32) {
          const double2 x = ca[i], y = cmul(cb[i], ph);
          ca[i] = make_double2(c * x.x - s * y.x, c * x.y - s * y.y);
          cb[i] = make_double2(s * x.x + c * y.x, s * x.y + c * y.y);
        }
        double2* va = V + a * ldv;
        double2* vb = V + b * ldv;
        for (int i = lane; i < n; i += 32) {
          const double2 x = va[i], y = cmul(vb[i], ph);
          va[i] = make_double2(c * x.x - s * y.x, c * x.y - s * y.y);
          vb[i] = make_double2(s * x.x + c * y.x, s * x.y + c * y.y);
        }
      }
      __syncthreads();
    }
    const int any = *flag;
    __syncthreads();
#ifdef BF_JACOBI_STATS
    if (threadIdx.x == 0) atomicAdd(&g_jacobi_sweeps, 1);
#endif
    if (!any) break;
  }
}

// Thin SVD of a small matrix M (m x n) given in shared memory (row-major, ld).
// Outputs U (m x k), sig (k), Vo (n x k) with k = min(m, n), singular values in
// descending order (ties by column index). W (max*min) and Vt (min*min) are
// shared-memory work buffers (used column-major); flag/perm/ssc are shared scratch.
__device__ void svd_small(const double2* M, int m, int n, int ld, double2* U, int ldu, double2* Vo, int ldv,
                          double* sig, double2* W, double2* Vt, int* flag, int* perm, double* ssc) {
  const bool tall = m >= n;
  const int rr = tall ? m : n, cc = tall ? n : m;  // work on M (tall) or M^H
  // W column-major: W(r, c) = W[c * rr + r]
  for (int i = threadIdx.x; i < rr * cc; i += blockDim.x) {
    const int c = i / rr, r = i % rr;
    W[c * rr + r] = tall ? M[r * ld + c] : cconj(M[c * ld + r]);
  }
  __syncthreads();
  jacobi_cols(W, rr, cc, rr, Vt, cc, flag);
  __syncthreads();
  // column norms (fixed order) and descending order
  for (int c = threadIdx.x >> 5; c < cc; c += blockDim.x >> 5) {
    double acc = 0;
    for (int i = threadIdx.x & 31; i < rr; i += 32) acc += W[c * rr + i].x * W[c * rr + i].x + W[c * rr + i].y * W[c * rr + i].y;
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) ssc[c] = sqrt(acc);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < cc; c += blockDim.x) {
    int rank = 0;
    for (int d = 0; d < cc; ++d) rank += (ssc[d] > ssc[c]) || (ssc[d] == ssc[c] && d < c);
    perm[rank] = c;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < cc; k += blockDim.x) sig[k] = ssc[perm[k]];
  __syncthreads();
  // left vectors of the worked matrix: W[:, c] / sigma ; right vectors: Vt[:, c]
  double2* L = tall ? U : Vo;
  const int ldl = tall ? ldu : ldv;
  double2* R = tall ? Vo : U;
  const int ldr = tall ? ldv : ldu;
  for (int i = threadIdx.x; i < rr * cc; i += blockDim.x) {
    const int k = i / rr, r = i % rr, c = perm[k];
    const double sg = ssc[c];
    const double2 w = W[c * rr + r];
    L[r * ldl + k] = sg > 0 ? make_double2(w.x / sg, w.y / sg) : make_double2(0, 0);
  }
  for (int i = threadIdx.x; i < cc * cc; i += blockDim.x) {
    const int k = i / cc, r = i % cc, c = perm[k];
    R[r * ldr + k] = Vt[c * cc + r];
  }
  __syncthreads();
}

// floored_inverse (lowrank.py:79-87): 1/sigma where sigma > PINV_FLOOR * max, else 0.
__device__ __forceinline__ double floored_inv(double s, double smax) {
  return s > kPinvFloor * smax ? 1.0 / s : 0.0;
}

}  // namespace bfly
