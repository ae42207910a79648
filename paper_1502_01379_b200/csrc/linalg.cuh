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

// ---------------------------------------------------------------- warp Jacobi SVD
// Round-robin partner of column j in round r over nn (even) columns: i + j = r
// (mod nn - 1) pairs i with j; the column with 2 j = r pairs with nn - 1.
__device__ __forceinline__ int rr_partner(int j, int r, int nn) {
  const int q = nn - 1;
  if (j >= nn) return j;
  if (j == q) return (r * (nn >> 1)) % q;
  int p = (r - j) % q;
  if (p < 0) p += q;
  return p == j ? q : p;
}

// One warp: one-sided Jacobi SVD of a small matrix. Lane j holds column j of the
// worked (tall, rr >= cc, rr, cc <= 32) matrix in registers and column j of V in
// the shared scratch Vs (column-major, odd leading dimension 33: conflict-free);
// each round every lane fetches its partner's column by shuffles and both lanes of
// a pair evaluate the same rotation from the same fixed-order sums (deterministic,
// identical in both lanes). The worked matrix is M (tall) or M^H (wide) with
// M(i, c) = src[i * rs + c * cs]. Outputs exactly as svd_small: U (m x k), sig
// (k), Vo (n x k), k = min(m, n), singular values descending (ties by index).
// Vs: 2 * 32 * 33 complex values of shared memory owned by this warp.
constexpr int kWarpSvdLd = 33;

__device__ void warp_svd(const double2* src, int m, int n, int rs, int cs, double2* U, int ldu, double2* Vo,
                         int ldv, double* sig, double2* Vs) {
  const int lane = threadIdx.x & 31;
  const bool tall = m >= n;
  const int rr = tall ? m : n, cc = tall ? n : m;  // worked matrix: rr x cc, columns on lanes
  double2 a[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    double2 x = make_double2(0, 0);
    if (lane < cc && k < rr) x = tall ? src[k * rs + lane * cs] : cconj(src[lane * rs + k * cs]);
    a[k] = x;
  }
  // V double-buffered in shared memory: a rotated lane writes its new column to the
  // other buffer and flips `cur`; a partner reads the slot of the buffer `cur` names
  constexpr int kVbuf = 32 * kWarpSvdLd;
  int cur = 0;
  for (int k = 0; k < cc; ++k) Vs[lane * kWarpSvdLd + k] = make_double2(k == lane ? 1.0 : 0.0, 0.0);
  __syncwarp();
  const int nn = cc + (cc & 1);
  const double tol = (rr > 8 ? rr : 8) * 2.220446049250313e-16;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int round = 0; round < nn - 1; ++round) {
      const int pj = rr_partner(lane, round, nn);
      const bool valid = lane < cc && pj < cc;
      const bool low = lane < pj;
      // own / partner sums; the pair's lower column is "x": both lanes then hold the
      // same (al, be, g) bit for bit (the upper lane's cross sum is the exact conjugate)
      double no = 0, np = 0;
      double2 d = make_double2(0, 0);
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        double2 pk;
        pk.x = __shfl_sync(0xffffffffu, a[k].x, pj);
        pk.y = __shfl_sync(0xffffffffu, a[k].y, pj);
        if (k < rr) {
          // explicitly rounded (no FMA contraction): the upper lane's terms are then the
          // exact conjugates of the lower lane's, and both norms the same sums
          no = __dadd_rn(no, __dadd_rn(__dmul_rn(a[k].x, a[k].x), __dmul_rn(a[k].y, a[k].y)));
          np = __dadd_rn(np, __dadd_rn(__dmul_rn(pk.x, pk.x), __dmul_rn(pk.y, pk.y)));
          d.x = __dadd_rn(d.x, __dadd_rn(__dmul_rn(a[k].x, pk.x), __dmul_rn(a[k].y, pk.y)));
          d.y = __dadd_rn(d.y, __dsub_rn(__dmul_rn(a[k].x, pk.y), __dmul_rn(a[k].y, pk.x)));
        }
      }
      const double al = low ? no : np, be = low ? np : no;
      const double2 g = low ? d : cconj(d);
      const double g2 = g.x * g.x + g.y * g.y;
      const bool rot = valid && !(g2 == 0.0 || g2 <= tol * tol * al * be);
      if (rot) rotated = true;
      // own' = ca own + cb partner: the lower lane (own = x) takes ca = c, cb = -s e^{-i phi};
      // the upper (own = y) ca = c e^{-i phi}, cb = s — [x', y'] = [x, y] [[c, s],
      // [-s e^{-i phi}, c e^{-i phi}]]. Every lane shuffles (uniform control flow).
      double2 ca = make_double2(1, 0), cb = make_double2(0, 0);
      if (rot) {
        const double ig = rsqrt(g2);
        const double zeta = (be - al) * 0.5 * ig;
        const double az = fabs(zeta), sgn = zeta >= 0 ? 1.0 : -1.0;
        const double t = az > 1e150 ? sgn * 0.5 / az : sgn / (az + sqrt(1.0 + zeta * zeta));
        const double c = rsqrt(1.0 + t * t), s_ = c * t;
        const double2 ph = make_double2(g.x * ig, -g.y * ig);  // e^{-i phi}
        ca = low ? make_double2(c, 0) : make_double2(c * ph.x, c * ph.y);
        cb = low ? make_double2(-s_ * ph.x, -s_ * ph.y) : make_double2(s_, 0);
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        double2 pk;
        pk.x = __shfl_sync(0xffffffffu, a[k].x, pj);
        pk.y = __shfl_sync(0xffffffffu, a[k].y, pj);
        if (rot && k < rr) {
          const double2 u = cmul(ca, a[k]), w = cmul(cb, pk);
          a[k] = make_double2(u.x + w.x, u.y + w.y);
        }
      }
      // V columns: read mine and the partner's current ones, write mine to the other buffer
      const int pcur = __shfl_sync(0xffffffffu, cur, pj);
      if (rot) {
        const double2* vm = Vs + cur * kVbuf + lane * kWarpSvdLd;
        const double2* vp = Vs + pcur * kVbuf + pj * kWarpSvdLd;
        double2* vn = Vs + (cur ^ 1) * kVbuf + lane * kWarpSvdLd;
        for (int k = 0; k < cc; ++k) {
          const double2 u = cmul(ca, vm[k]), w = cmul(cb, vp[k]);
          vn[k] = make_double2(u.x + w.x, u.y + w.y);
        }
        cur ^= 1;
      }
      __syncwarp();
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
  }
  // column norms (fixed order), descending rank (ties by index)
  double nrm = 0;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k < rr) nrm += a[k].x * a[k].x + a[k].y * a[k].y;
  nrm = lane < cc ? sqrt(nrm) : -1.0;
  int rank = 0;
  for (int d = 0; d < cc; ++d) {
    const double o = __shfl_sync(0xffffffffu, nrm, d);
    rank += (o > nrm) || (o == nrm && d < lane);
  }
  if (lane < cc) {
    sig[rank] = nrm;
    // left vectors of the worked matrix: a / sigma ; right vectors: V
    double2* L = tall ? U : Vo;
    const int ldl = tall ? ldu : ldv;
    double2* R = tall ? Vo : U;
    const int ldr = tall ? ldv : ldu;
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (k < rr) L[k * ldl + rank] = nrm > 0 ? make_double2(a[k].x / nrm, a[k].y / nrm) : make_double2(0, 0);
    const double2* vm = Vs + cur * kVbuf + lane * kWarpSvdLd;
    for (int k = 0; k < cc; ++k) R[k * ldr + rank] = vm[k];
  }
  __syncwarp();
}

// One warp, columns only: one-sided Jacobi on the columns of a small matrix held one per
// lane in registers (lane j: column j, RR rows, zero padded; cc active columns), with no
// accumulated rotation matrix — the caller wants only the rotated columns W = M J (their
// norms are the singular values, their directions the left singular vectors of M). Used
// on M = R^H in the recursion, whose left singular vectors are the right singular vectors
// of R. The pair's lower lane evaluates the three sums (fused multiply-adds, fixed order)
// and hands them to the upper lane, so both lanes build the same rotation bit for bit.
// `zero` must be 0 at run time without the compiler knowing it (blockIdx.z of a launch
// with gridDim.z = 1): every fourth partner fetch is made to depend on the arithmetic
// before it through `& zero`, which keeps ptxas from hoisting all 2 RR fetches of a pass
// ahead of the arithmetic and spilling the column.
// A shuffle the compiler may not merge with an earlier identical one (the rotation pass
// re-fetches the partner column rather than keeping 2 RR more registers live).
__device__ __forceinline__ double shfl_again(double v, int src) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  asm volatile("shfl.sync.idx.b32 %0, %0, %2, 31, 0xffffffff;\n\tshfl.sync.idx.b32 %1, %1, %2, 31, 0xffffffff;"
               : "+r"(lo), "+r"(hi)
               : "r"(src));
  return __hiloint2double(hi, lo);
}

template <int RR>
__device__ __forceinline__ void warp_jacobi_reg(double2 (&a)[RR], int cc, int zero) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int nn = cc + (cc & 1);
  const double tol = (RR > 8 ? RR : 8) * 2.220446049250313e-16;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int round = 0; round < nn - 1; ++round) {
      const int pj = rr_partner(lane, round, nn);
      const bool valid = lane < cc && pj < cc && pj != lane;
      const bool low = lane < pj;
      int pjv = pj;
      // two accumulators per sum (even / odd rows): the dependent-DFMA chains are the pass's
      // critical path
      double no = 0, np = 0, no1 = 0, np1 = 0;
      double2 d = make_double2(0, 0), d1 = make_double2(0, 0);
#pragma unroll
      for (int k = 0; k < RR; k += 2) {
        // every fourth fetch waits for the sums so far: keeps the partner column from
        // being fetched (and held in registers) whole
        if (k && k % 4 == 0) pjv = pj + ((__double2hiint(d.x) ^ __double2hiint(np1)) & zero);
        double2 pk, pk1;
        pk.x = __shfl_sync(full, a[k].x, pjv);
        pk.y = __shfl_sync(full, a[k].y, pjv);
        pk1.x = __shfl_sync(full, a[k + 1].x, pjv);
        pk1.y = __shfl_sync(full, a[k + 1].y, pjv);
        no = fma(a[k].x, a[k].x, fma(a[k].y, a[k].y, no));
        np = fma(pk.x, pk.x, fma(pk.y, pk.y, np));
        d.x = fma(a[k].x, pk.x, fma(a[k].y, pk.y, d.x));   // conj(own) * partner
        d.y = fma(a[k].x, pk.y, fma(-a[k].y, pk.x, d.y));
        no1 = fma(a[k + 1].x, a[k + 1].x, fma(a[k + 1].y, a[k + 1].y, no1));
        np1 = fma(pk1.x, pk1.x, fma(pk1.y, pk1.y, np1));
        d1.x = fma(a[k + 1].x, pk1.x, fma(a[k + 1].y, pk1.y, d1.x));
        d1.y = fma(a[k + 1].x, pk1.y, fma(-a[k + 1].y, pk1.x, d1.y));
      }
      no += no1;
      np += np1;
      d.x += d1.x;
      d.y += d1.y;
      const int from = low ? lane : pj;  // the pair's lower lane: own = x, partner = y
      const double al = __shfl_sync(full, no, from), be = __shfl_sync(full, np, from);
      double2 g;
      g.x = __shfl_sync(full, d.x, from);
      g.y = __shfl_sync(full, d.y, from);
      const double g2 = g.x * g.x + g.y * g.y;
      const bool rot = valid && !(g2 == 0.0 || g2 <= tol * tol * al * be);
      if (!__any_sync(full, rot)) continue;
      rotated = rotated || rot;
      // [x', y'] = [x, y] [[c, s], [-s e^{-i phi}, c e^{-i phi}]]: own' = ca own + cb partner
      double2 ca = make_double2(1, 0), cb = make_double2(0, 0);
      if (rot) {
        const double ig = rsqrt(g2);
        const double zeta = (be - al) * 0.5 * ig;
        const double az = fabs(zeta), sgn = zeta >= 0 ? 1.0 : -1.0;
        const double t = az > 1e150 ? sgn * 0.5 / az : sgn / (az + sqrt(1.0 + zeta * zeta));
        const double c = rsqrt(1.0 + t * t), s_ = c * t;
        const double2 ph = make_double2(g.x * ig, -g.y * ig);  // e^{-i phi}
        ca = low ? make_double2(c, 0) : make_double2(c * ph.x, c * ph.y);
        cb = low ? make_double2(-s_ * ph.x, -s_ * ph.y) : make_double2(s_, 0);
      }
#pragma unroll
      for (int k = 0; k < RR; ++k) {
        if (k && k % 4 == 0) pjv = pj + ((__double2hiint(a[k - 1].x) ^ __double2hiint(a[k - 1].y)) & zero);
        double2 pk;
        pk.x = shfl_again(a[k].x, pjv);
        pk.y = shfl_again(a[k].y, pjv);
        const double2 u = cmul(ca, a[k]), w = cmul(cb, pk);
        a[k] = make_double2(u.x + w.x, u.y + w.y);
      }
    }
    if (!__any_sync(full, rotated)) break;
  }
}

// floored_inverse (lowrank.py:79-87): 1/sigma where sigma > PINV_FLOOR * max, else 0.
__device__ __forceinline__ double floored_inv(double s, double smax) {
  return s > kPinvFloor * smax ? 1.0 / s : 0.0;
}

}  // namespace bfly
