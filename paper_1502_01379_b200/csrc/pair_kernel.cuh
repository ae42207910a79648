// pair_kernel.cuh — two adjacent transfer levels fused in one kernel for the
// many-RHS complex128 apply ("adjacent levels fused while the working set
// fits in SMEM", BASELINE north star). The intermediate vector of the pair
// never leaves shared memory, so the pair moves its input and output vectors
// once instead of twice.
//
// Geometry (splitting levels, 5-D blocks (G, 2, P, r, 2r)):
// level A = lower index i (G_A, P_A), level B = i + 1 (G_B = 2 G_A, P_B = P_A / 2).
// Forward (G levels, A then B): level-B unit (g', p') reads 2r rows = level-A
// outputs (g'/2, g'%2, 2p') and (g'/2, g'%2, 2p'+1). Work item (g, q), q < P_A/2,
// closes over level-A units (g, 2q), (g, 2q+1) and level-B units (2g, q),
// (2g+1, q): 4 blocks per level. The adjoint (H* levels, B* then A*) is the
// mirror image over the same items.
#pragma once

#include "common.cuh"

namespace bfly {

struct PairArgs {
  const double2* fac_a;  // level A blocks (G_A, 2, P_A, r, 2r)
  const double2* fac_b;  // level B blocks (2 G_A, 2, P_A / 2, r, 2r)
  const double2* in;
  double2* out;
  uint32_t r, ga, pa;    // rank, level-A geometry
  uint32_t k;            // right-hand sides (row length of in / out)
  uint32_t kc, nch;      // right-hand sides per item and chunks per pair (items = pairs x nch)
  int adjoint;
  uint32_t nitems;       // G_A * P_A / 2 * nch
  uint32_t fld, vld;     // shared-memory row strides of block rows and vector rows
  uint32_t stage_elems;  // 8 blocks + 2 C vector rows
  // adjoint pair ending the down half: the middle factor fused into the level-A* stores
  // (remap 1 forward chain / 2 adjoint chain, as LevelArgs::remap; factors.py:180-190)
  int remap;
  uint32_t m, mr;        // middle nodes, rank of the middle vector
  const double* mid_w;
  // rank-8 fast path with the leaf factor fused (pair8_kernel<.., LEAF>): leaf blocks
  // (nb, 16, 8); adjoint pairs read `in` as the chain input g, forward pairs write `out`
  // as the chain output (16 rows per leaf)
  const double2* leaf;
};

// Destination element and weight of middle-vector entry e under the fused middle factor.
__device__ __forceinline__ size_t pair_remap(const PairArgs& a, size_t e, double* w) {
  if (!a.remap) {
    *w = 1;
    return e;
  }
  const uint32_t mrr = a.m * a.mr;
  const uint32_t e32 = static_cast<uint32_t>(e), ia = e32 / mrr;
  const uint32_t rem = e32 - ia * mrr;
  const uint32_t ib = rem / a.mr, rho = rem - ib * a.mr;
  const size_t dst = (static_cast<size_t>(ib) * a.m + ia) * a.mr + rho;
  *w = a.remap == 1 ? __ldg(a.mid_w + dst) : __ldg(a.mid_w + (static_cast<size_t>(ia) * a.m + ib) * a.mr + rho);
  return dst;
}

__device__ __forceinline__ void pair_dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// ngemm complex GEMMs Y_g (M x N) = A_g (M x K) X_g (K x N) spread over the consumer
// warps as 8 x 16 output tiles (m8n8k4 f64: 4 real products per complex step). The K
// range is nseg segments of klen (the two stacked blocks of an adjoint level), so the
// accessors get (segment, offset) without any division in the inner loop.
// GAUSS: 3 DMMAs per complex step (see consume_tile_dmma in level_kernel.cuh).
template <bool GAUSS, typename AF, typename XF, typename YF>
__device__ __forceinline__ void pair_gemms(int ngemm, int M, int nseg, int klen, int N, const AF& aload,
                                           const XF& xload, const YF& ystore, int warp, int lane, int nwarps) {
  const int mtl = (M + 7) / 8, ntl = (N + 15) / 16;
  const int items = ngemm * mtl * ntl;
  const int lr = lane >> 2, lk = lane & 3;
  for (int it = warp; it < items; it += nwarps) {
    const int gi = it / (mtl * ntl), rest = it - gi * mtl * ntl;
    const int m0 = (rest / ntl) * 8, n0 = (rest % ntl) * 16;
    const int m = m0 + lr;
    double cr[2][2] = {{0, 0}, {0, 0}}, ci[2][2] = {{0, 0}, {0, 0}}, cs[2][2] = {{0, 0}, {0, 0}};
    for (int sg = 0; sg < nseg; ++sg)
      for (int k0 = 0; k0 < klen; k0 += 4) {
        const int kk = k0 + lk;
        const bool kok = kk < klen;
        const double2 a = (kok && m < M) ? aload(gi, m, sg, kk) : make_double2(0, 0);
        double2 b[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int n = n0 + 8 * j + lr;
          b[j] = (kok && n < N) ? xload(gi, sg, kk, n) : make_double2(0, 0);
        }
        if constexpr (GAUSS) {  // cr = T1, ci = T2, cs = T3
          const double as = a.x + a.y;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            pair_dmma(cr[j][0], cr[j][1], a.x, b[j].x);
            pair_dmma(ci[j][0], ci[j][1], a.y, b[j].y);
            pair_dmma(cs[j][0], cs[j][1], as, b[j].x + b[j].y);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            pair_dmma(cr[j][0], cr[j][1], a.x, b[j].x);
            pair_dmma(ci[j][0], ci[j][1], a.x, b[j].y);
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            pair_dmma(cr[j][0], cr[j][1], -a.y, b[j].y);
            pair_dmma(ci[j][0], ci[j][1], a.y, b[j].x);
          }
        }
      }
    if constexpr (GAUSS) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double t1 = cr[j][q], t2 = ci[j][q];
          cr[j][q] = t1 - t2;
          ci[j][q] = cs[j][q] - t1 - t2;
        }
    }
    if (m < M) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = n0 + 8 * j + 2 * lk + q;
          if (n < N) ystore(gi, m, n, make_double2(cr[j][q], ci[j][q]));
        }
    }
  }
}

// Producer: the 8 blocks (level A: (t, u) = (t, p = 2q + u); level B: (t, t') of
// g' = 2g + t) and the item's input vector rows, one bulk copy per row.
// what: 1 = arm the barrier and copy the (constant) factor blocks, 2 = the vector rows,
// 3 = both (the factor part may be issued before the dependency wait on the previous level).
__device__ __forceinline__ void pair_produce(const PairArgs& a, uint32_t item_rhs, double2* st, uint64_t* full,
                                             int lane, uint64_t pol, int what = 3) {
  const uint32_t R = a.r, C = 2 * a.r, pb = a.pa / 2;
  // items are (pair, right-hand-side chunk): chunks of one pair are independent columns
  const uint32_t item = item_rhs / a.nch, k0 = (item_rhs - item * a.nch) * a.kc, kw = min(a.kc, a.k - k0);
  const uint32_t g = item / pb, q = item - g * pb;
  const uint32_t bytes = (8 * R * C + 2 * C * kw) * static_cast<uint32_t>(sizeof(double2));
  if (what & 1) {
  if (lane == 0) mbar_arrive_expect_tx(full, bytes);
  __syncwarp();
  // block rows: 8 blocks x R rows; smem block b = (level, t, u|t') at b * R * fld
  if (a.fld == C) {   // unpadded blocks: whole-block copies (level A: (g, t, 2q), (g, t, 2q + 1) adjacent)
    const uint32_t bb = R * C * static_cast<uint32_t>(sizeof(double2));
    if (lane < 2) {
      const uint32_t t = lane;
      bulk_g2s(st + static_cast<size_t>(2 * t) * R * C, a.fac_a + static_cast<size_t>((g * 2 + t) * a.pa + 2 * q) * R * C,
               2 * bb, full, pol);
    } else if (lane < 6) {
      const uint32_t b = lane + 2, t = (b >> 1) & 1, v = b & 1;
      bulk_g2s(st + static_cast<size_t>(b) * R * C, a.fac_b + static_cast<size_t>(((2 * g + t) * 2 + v) * pb + q) * R * C,
               bb, full, pol);
    }
  } else
  for (uint32_t row = lane; row < 8 * R; row += 32) {
    const uint32_t b = row / R, rr = row - b * R;
    const uint32_t lvl = b >> 2, t = (b >> 1) & 1, v = b & 1;
    const double2* src = lvl == 0 ? a.fac_a + (static_cast<size_t>((g * 2 + t) * a.pa + 2 * q + v) * R + rr) * C
                                  : a.fac_b + (static_cast<size_t>(((2 * g + t) * 2 + v) * pb + q) * R + rr) * C;
    bulk_g2s(st + static_cast<size_t>(row) * a.fld, src, C * static_cast<uint32_t>(sizeof(double2)), full, pol);
  }
  }
  if (!(what & 2)) return;
  double2* vs = st + static_cast<size_t>(8) * R * a.fld;
  if (a.vld == kw && kw == a.k) {   // unpadded whole-k rows: contiguous row runs in one copy each
    const uint32_t rb = a.k * static_cast<uint32_t>(sizeof(double2));
    if (!a.adjoint) {
      if (lane == 0)
        bulk_g2s(vs, a.in + static_cast<size_t>(g * a.pa + 2 * q) * C * a.k, 2 * C * rb, full);
    } else if (lane < 4) {
      const uint32_t t = lane >> 1, tp = lane & 1;
      bulk_g2s(vs + static_cast<size_t>(lane) * R * a.k,
               a.in + static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * R * a.k, R * rb, full);
    }
    return;
  }
  for (uint32_t row = lane; row < 2 * C; row += 32) {
    size_t grow;
    if (!a.adjoint) {  // units (g, 2q), (g, 2q + 1): 2 C contiguous rows
      grow = static_cast<size_t>(g * a.pa + 2 * q) * C + row;
    } else {           // level-B* inputs (g' = 2g + t, t', q): R rows each, order [t][t']
      const uint32_t ch = row / R, rr = row - ch * R, t = ch >> 1, tp = ch & 1;
      grow = static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * R + rr;
    }
    bulk_g2s(vs + static_cast<size_t>(row) * a.vld, a.in + grow * a.k + k0, kw * static_cast<uint32_t>(sizeof(double2)),
             full);
  }
}

template <int STAGES, int NCW, bool GAUSS>
__global__ void __launch_bounds__((NCW + 1) * 32, 2) pair_kernel(const PairArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + STAGES;
  double2* stage0 = reinterpret_cast<double2*>(smem_raw + 128);
  double2* mi = stage0 + static_cast<size_t>(STAGES) * a.stage_elems;  // 2 C x vld intermediate
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t R = a.r, C = 2 * a.r, pb = a.pa / 2, KS = a.k;
  const uint32_t fld = a.fld, vld = a.vld;
  if (warp == NCW) {
    const uint64_t pol = policy_evict_first();
    uint32_t it = 0;
    for (uint32_t item = blockIdx.x; item < a.nitems; item += gridDim.x, ++it) {
      const uint32_t s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
      pair_produce(a, item, stage0 + static_cast<size_t>(s) * a.stage_elems, &full[s], lane, pol);
    }
    return;
  }
  uint32_t it = 0;
  for (uint32_t item = blockIdx.x; item < a.nitems; item += gridDim.x, ++it) {
    const uint32_t s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const double2* st = stage0 + static_cast<size_t>(s) * a.stage_elems;
    const double2* vs = st + static_cast<size_t>(8) * R * fld;
    const uint32_t pitem = item / a.nch, k0 = (item - pitem * a.nch) * a.kc;
    const uint32_t K = min(a.kc, KS - k0);     // this item's right-hand sides
    const uint32_t g = pitem / pb, q = pitem - g * pb;
    auto blk = [&](uint32_t b) { return st + static_cast<size_t>(b) * R * fld; };
    if (!a.adjoint) {
      // level A: Y(t, u) = B_A(g, t, 2q + u) X_u  ->  mi rows t C + u R + m
      pair_gemms<GAUSS>(
          4, R, 1, C, K, [&](int gi, int m, int, int kk) { return blk(gi)[m * fld + kk]; },
          [&](int gi, int, int kk, int n) { return vs[((gi & 1) * C + kk) * vld + n]; },
          [&](int gi, int m, int n, double2 v) { mi[((gi >> 1) * C + (gi & 1) * R + m) * vld + n] = v; }, warp, lane,
          NCW);
      consumers_sync();
      // level B: Y(t, t') = B_B(2g + t, t', q) mi_t  ->  out rows ((2g + t) 2 + t') P_B + q
      pair_gemms<GAUSS>(
          4, R, 1, C, K, [&](int gi, int m, int, int kk) { return blk(4 + gi)[m * fld + kk]; },
          [&](int gi, int, int kk, int n) { return mi[((gi >> 1) * C + kk) * vld + n]; },
          [&](int gi, int m, int n, double2 v) {
            const uint32_t t = gi >> 1, tp = gi & 1;
            a.out[(static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * R + m) * KS + k0 + n] = v;
          },
          warp, lane, NCW);
    } else {
      // level B*: Y(t) = sum_t' B_B(2g + t, t', q)^H in(2g + t, t', q)  ->  mi rows t C + c
      pair_gemms<GAUSS>(
          2, C, 2, R, K,
          [&](int gi, int m, int sg, int kk) {
            const double2 v = blk(4 + 2 * gi + sg)[kk * fld + m];
            return make_double2(v.x, neg(v.y));
          },
          [&](int gi, int sg, int kk, int n) { return vs[((gi * 2 + sg) * R + kk) * vld + n]; },
          [&](int gi, int m, int n, double2 v) { mi[(gi * C + m) * vld + n] = v; }, warp, lane, NCW);
      consumers_sync();
      // level A*: Y(u) = sum_t B_A(g, t, 2q + u)^H mi_t[u R ..]  ->  out rows (g P_A + 2q + u) C + c
      pair_gemms<GAUSS>(
          2, C, 2, R, K,
          [&](int gi, int m, int sg, int kk) {
            const double2 v = blk(2 * sg + gi)[kk * fld + m];
            return make_double2(v.x, neg(v.y));
          },
          [&](int gi, int sg, int kk, int n) { return mi[(sg * C + gi * R + kk) * vld + n]; },
          [&](int gi, int m, int n, double2 v) {
            double w;
            const size_t e = pair_remap(a, static_cast<size_t>(g * a.pa + 2 * q + gi) * C + m, &w);
            a.out[e * KS + k0 + n] = make_double2(w * v.x, w * v.y);
          },
          warp, lane, NCW);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    consumers_sync();  // mi is reused by the next item's first level
  }
}


// ---------------------------------------------------------------- rank-8 fast path
// The same pair for R = 8 (C = 16: BASELINE config 1) with every consumer warp owning one
// (t, 16-column) slice of the item end to end, so the two levels need no block-wide
// barrier and all tile geometry is compile-time:
//   forward  warp (t, n): Y(t, 0), Y(t, 1) (level A, into its own rows of mi) then, after a
//            __syncwarp, out(t, 0), out(t, 1) (level B reads only mi_t);
//   adjoint  warp (t, n): mi_t (level B*, one 16 x 16 GEMM over both t'), a 64-thread named
//            barrier with the other warp of its column slice, then out(u = t) (level A*
//            reads rows u R .. of both mi_0 and mi_1), and the same barrier again before
//            mi is rewritten.
// The 4 k-steps of each GEMM are unrolled with pointer offsets only (no predicates: the
// host takes this path when kc and k are multiples of 16). 3-multiplication complex
// products as in pair_gemms. Producer and stage layout are pair_produce's.
__device__ __forceinline__ void pair_bar(int id) {   // immediate ids: a register id reserves all 16 barriers
  switch (id) {
    case 1: asm volatile("bar.sync 1, 64;" ::: "memory"); break;
    case 2: asm volatile("bar.sync 2, 64;" ::: "memory"); break;
    case 3: asm volatile("bar.sync 3, 64;" ::: "memory"); break;
    default: asm volatile("bar.sync 4, 64;" ::: "memory"); break;
  }
}

// one complex k-step of an MT x 2 warp tile (8-row tiles i, 8-column tiles j)
template <int MT>
__device__ __forceinline__ void pair8_step(double (&t1)[MT][2][2], double (&t2)[MT][2][2], double (&t3)[MT][2][2],
                                           const double (&ar)[MT], const double (&ai)[MT], const double2 b0,
                                           const double2 b1) {
  const double bs0 = b0.x + b0.y, bs1 = b1.x + b1.y;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    pair_dmma(t1[i][0][0], t1[i][0][1], ar[i], b0.x);
    pair_dmma(t2[i][0][0], t2[i][0][1], ai[i], b0.y);
    pair_dmma(t1[i][1][0], t1[i][1][1], ar[i], b1.x);
    pair_dmma(t2[i][1][0], t2[i][1][1], ai[i], b1.y);
  }
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const double as = ar[i] + ai[i];
    pair_dmma(t3[i][0][0], t3[i][0][1], as, bs0);
    pair_dmma(t3[i][1][0], t3[i][1][1], as, bs1);
  }
}

// Producer of the leaf-fused rank-8 pair: the 8 transfer blocks (unpadded, whole-block
// copies), the item's 4 leaf blocks (leaf b = ((2g + t) 2 + t') P_B + q, 16 x 8 each) and
// the input rows — adjoint: the 4 x 16 rows of g under those leaves (chunk order [t][t']),
// forward: the pair's 2 C rows as in pair_produce.
template <bool ADJ>
__device__ __forceinline__ void pair8_produce_leaf(const PairArgs& a, uint32_t item_rhs, double2* st, uint64_t* full,
                                                   int lane, uint64_t pol, int what = 3) {
  constexpr uint32_t R = 8, C = 16, N0 = 16;
  const uint32_t pb = a.pa / 2;
  const uint32_t item = item_rhs / a.nch, k0 = (item_rhs - item * a.nch) * a.kc, kw = min(a.kc, a.k - k0);
  const uint32_t g = item / pb, q = item - g * pb;
  const uint32_t nrows = ADJ ? 4 * N0 : 2 * C;
  const uint32_t bytes = (8 * R * C + 4 * N0 * R + nrows * kw) * static_cast<uint32_t>(sizeof(double2));
  if (what & 1) {
    if (lane == 0) mbar_arrive_expect_tx(full, bytes);
    __syncwarp();
    const uint32_t bb = R * C * static_cast<uint32_t>(sizeof(double2));
    if (lane < 2) {
      const uint32_t t = lane;
      bulk_g2s(st + static_cast<size_t>(2 * t) * R * C,
               a.fac_a + static_cast<size_t>((g * 2 + t) * a.pa + 2 * q) * R * C, 2 * bb, full, pol);
    } else if (lane < 6) {
      const uint32_t b = lane + 2, t = (b >> 1) & 1, v = b & 1;
      bulk_g2s(st + static_cast<size_t>(b) * R * C,
               a.fac_b + static_cast<size_t>(((2 * g + t) * 2 + v) * pb + q) * R * C, bb, full, pol);
    } else if (lane < 10) {
      const uint32_t ch = lane - 6, t = ch >> 1, tp = ch & 1;
      bulk_g2s(st + 8 * R * C + ch * N0 * R, a.leaf + static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * N0 * R,
               bb, full, pol);
    }
  }
  if (!(what & 2)) return;
  double2* vs = st + 8 * R * C + 4 * N0 * R;
  for (uint32_t row = lane; row < nrows; row += 32) {
    size_t grow;
    if (!ADJ) {
      grow = static_cast<size_t>(g * a.pa + 2 * q) * C + row;
    } else {
      const uint32_t ch = row / N0, rr = row - ch * N0, t = ch >> 1, tp = ch & 1;
      grow = static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * N0 + rr;
    }
    bulk_g2s(vs + static_cast<size_t>(row) * a.vld, a.in + grow * a.k + k0, kw * static_cast<uint32_t>(sizeof(double2)),
             full);
  }
}

template <int STAGES, bool ADJ, int NCW, bool LEAF>
__global__ void __launch_bounds__((NCW + 1) * 32, STAGES == 1 ? (NCW <= 4 ? (ADJ ? 3 : 4) : 2) : (NCW <= 4 ? 2 : 1))
    pair8_kernel(const PairArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + STAGES;
  double2* stage0 = reinterpret_cast<double2*>(smem_raw + 128);
  double2* mi = stage0 + static_cast<size_t>(STAGES) * a.stage_elems;  // 2 C x vld intermediate
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int ncw = NCW;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncw);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // programmatic dependent launch: only the (constant) factor blocks of the first stages
  // are fetched before the wait on the previous level
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr uint32_t R = 8, C = 16;
  const uint32_t pb = a.pa / 2, KS = a.k;
  const uint32_t fld = a.fld, vld = a.vld;
  if (warp == ncw) {
    const uint64_t pol = policy_evict_first();
    auto produce = [&](uint32_t item, uint32_t s, int what) {
      if constexpr (LEAF)
        pair8_produce_leaf<ADJ>(a, item, stage0 + static_cast<size_t>(s) * a.stage_elems, &full[s], lane, pol, what);
      else
        pair_produce(a, item, stage0 + static_cast<size_t>(s) * a.stage_elems, &full[s], lane, pol, what);
    };
    uint32_t pre = 0;
    for (uint32_t item = blockIdx.x; item < a.nitems && pre < STAGES; item += gridDim.x, ++pre) produce(item, pre, 1);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint32_t it = 0;
    for (uint32_t item = blockIdx.x; item < a.nitems; item += gridDim.x, ++it) {
      const uint32_t s = it % STAGES;
      if (it >= STAGES) {
        mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        produce(item, s, 3);
      } else {
        produce(item, s, 2);
      }
    }
    return;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t t = warp & 1, nn = warp >> 1, n0 = nn * 16;
  const uint32_t lr = lane >> 2, lk = lane & 3;
  uint32_t it = 0;
  for (uint32_t item = blockIdx.x; item < a.nitems; item += gridDim.x, ++it) {
    const uint32_t s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    double2* st = stage0 + static_cast<size_t>(s) * a.stage_elems;
    const double2* lf = st + static_cast<size_t>(8) * R * fld;          // LEAF: 4 leaf blocks (16 x 8)
    double2* vs = st + static_cast<size_t>(8) * R * fld + (LEAF ? 4 * 16 * R : 0);
    constexpr uint32_t CH = (LEAF && ADJ) ? 16 : R;                      // rows per input chunk (adjoint)
    const uint32_t pitem = item / a.nch, k0 = (item - pitem * a.nch) * a.kc;
    const uint32_t K = min(a.kc, KS - k0);
    const uint32_t g = pitem / pb, q = pitem - g * pb;
    const bool act = n0 < K;   // K is a multiple of 16: a slice is whole or absent
    if constexpr (!ADJ) {
      if (act) {
        // level A: Y(t, u) = B_A(g, t, 2q + u) X_u  ->  mi rows t C + u R + m
#pragma unroll
        for (uint32_t u = 0; u < 2; ++u) {
          double t1[1][2][2] = {}, t2[1][2][2] = {}, t3[1][2][2] = {};
          const double2* ap = st + static_cast<size_t>(2 * t + u) * R * fld + lr * fld + lk;
          const double2* bp = vs + (u * C + lk) * vld + n0 + lr;
#pragma unroll
          for (int sk = 0; sk < 4; ++sk) {
            const double2 av = ap[4 * sk];
            const double ar[1] = {av.x}, ai[1] = {av.y};
            pair8_step<1>(t1, t2, t3, ar, ai, bp[4 * sk * vld], bp[4 * sk * vld + 8]);
          }
          double2* mo = mi + (t * C + u * R + lr) * vld + n0 + 2 * lk;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int qq = 0; qq < 2; ++qq)
              mo[8 * j + qq] = make_double2(t1[0][j][qq] - t2[0][j][qq], t3[0][j][qq] - t1[0][j][qq] - t2[0][j][qq]);
        }
        __syncwarp();
        // level B: Y(t, t') = B_B(2g + t, t', q) mi_t  ->  out rows ((2g + t) 2 + t') P_B + q
        double2 yb[2][2][2];   // LEAF: both t' results stay in registers until mi_t is free
#pragma unroll
        for (uint32_t tp = 0; tp < 2; ++tp) {
          double t1[1][2][2] = {}, t2[1][2][2] = {}, t3[1][2][2] = {};
          const double2* ap = st + static_cast<size_t>(4 + 2 * t + tp) * R * fld + lr * fld + lk;
          const double2* bp = mi + (t * C + lk) * vld + n0 + lr;
#pragma unroll
          for (int sk = 0; sk < 4; ++sk) {
            const double2 av = ap[4 * sk];
            const double ar[1] = {av.x}, ai[1] = {av.y};
            pair8_step<1>(t1, t2, t3, ar, ai, bp[4 * sk * vld], bp[4 * sk * vld + 8]);
          }
          double2* o = a.out + (static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * R + lr) * KS + k0 + n0 + 2 * lk;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
              const double2 v = make_double2(t1[0][j][qq] - t2[0][j][qq], t3[0][j][qq] - t1[0][j][qq] - t2[0][j][qq]);
              if constexpr (LEAF)
                yb[tp][j][qq] = v;
              else
                o[8 * j + qq] = v;
            }
        }
        if constexpr (LEAF) {
          // trail leaf (factors.py:49-56): rows of leaf b = U_b (16 x 8) Y(t, t'); Y goes through
          // this warp's own rows of mi (every lane is past its level-B reads first)
          __syncwarp();
#pragma unroll
          for (uint32_t tp = 0; tp < 2; ++tp) {
            double2* mo = mi + (t * C + tp * R + lr) * vld + n0 + 2 * lk;
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int qq = 0; qq < 2; ++qq) mo[8 * j + qq] = yb[tp][j][qq];
          }
          __syncwarp();
#pragma unroll
          for (uint32_t tp = 0; tp < 2; ++tp) {
            double t1[2][2][2] = {}, t2[2][2][2] = {}, t3[2][2][2] = {};
            const double2* ap = lf + (2 * t + tp) * 16 * R + lr * R + lk;
            const double2* bp = mi + (t * C + tp * R + lk) * vld + n0 + lr;
#pragma unroll
            for (int sk = 0; sk < 2; ++sk) {
              const double2 a0 = ap[4 * sk], a1 = ap[8 * R + 4 * sk];
              const double ar[2] = {a0.x, a1.x}, ai[2] = {a0.y, a1.y};
              pair8_step<2>(t1, t2, t3, ar, ai, bp[4 * sk * vld], bp[4 * sk * vld + 8]);
            }
            const size_t b = static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              double2* o = a.out + (b * 16 + 8 * i + lr) * KS + k0 + n0 + 2 * lk;
#pragma unroll
              for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int qq = 0; qq < 2; ++qq)
                  o[8 * j + qq] = make_double2(t1[i][j][qq] - t2[i][j][qq], t3[i][j][qq] - t1[i][j][qq] - t2[i][j][qq]);
            }
          }
        }
      }
      __syncwarp();   // every lane is past its mi reads before the next item's level A
      if (lane == 0) mbar_arrive(&empty[s]);
    } else {
      if (act) {
        if constexpr (LEAF) {
          // lead leaf adjoint (factors.py:49-56): c(t, t') = V_b^H (8 x 16) g_b, in place over
          // the first 8 rows of this warp's own 16 x 16 slice of chunk (t, t')
#pragma unroll
          for (uint32_t tp = 0; tp < 2; ++tp) {
            const uint32_t ch = t * 2 + tp;
            double t1[1][2][2] = {}, t2[1][2][2] = {}, t3[1][2][2] = {};
            const double2* ap = lf + ch * 16 * R + lk * R + lr;
            const double2* bp = vs + (ch * 16 + lk) * vld + n0 + lr;
#pragma unroll
            for (int sk = 0; sk < 4; ++sk) {
              const double2 av = ap[4 * sk * R];
              const double ar[1] = {av.x}, ai[1] = {neg(av.y)};
              pair8_step<1>(t1, t2, t3, ar, ai, bp[4 * sk * vld], bp[4 * sk * vld + 8]);
            }
            __syncwarp();   // every lane has read the chunk before its first rows are overwritten
            double2* mo = vs + (ch * 16 + lr) * vld + n0 + 2 * lk;
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int qq = 0; qq < 2; ++qq)
                mo[8 * j + qq] = make_double2(t1[0][j][qq] - t2[0][j][qq], t3[0][j][qq] - t1[0][j][qq] - t2[0][j][qq]);
          }
          __syncwarp();
        }
        // level B*: mi_t = sum_t' B_B(2g + t, t', q)^H in(2g + t, t', q)
        double t1[2][2][2] = {}, t2[2][2][2] = {}, t3[2][2][2] = {};
#pragma unroll
        for (int sk = 0; sk < 4; ++sk) {
          const uint32_t tp = sk >> 1, rho = (sk & 1) * 4 + lk;
          const double2* ap = st + static_cast<size_t>(4 + 2 * t + tp) * R * fld + rho * fld + lr;
          const double2* bp = vs + ((t * 2 + tp) * CH + rho) * vld + n0 + lr;
          const double2 a0 = ap[0], a1 = ap[8];
          const double ar[2] = {a0.x, a1.x}, ai[2] = {neg(a0.y), neg(a1.y)};  // A^H
          pair8_step<2>(t1, t2, t3, ar, ai, bp[0], bp[8]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          double2* mo = mi + (t * C + 8 * i + lr) * vld + n0 + 2 * lk;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int qq = 0; qq < 2; ++qq)
              mo[8 * j + qq] = make_double2(t1[i][j][qq] - t2[i][j][qq], t3[i][j][qq] - t1[i][j][qq] - t2[i][j][qq]);
        }
      }
      pair_bar(1 + static_cast<int>(nn));
      if (act) {
        // level A*: Y(u) = sum_t2 B_A(g, t2, 2q + u)^H mi_t2[u R ..]  ->  out rows (g P_A + 2q + u) C + c
        const uint32_t u = t;
        double t1[2][2][2] = {}, t2[2][2][2] = {}, t3[2][2][2] = {};
#pragma unroll
        for (int sk = 0; sk < 4; ++sk) {
          const uint32_t tt = sk >> 1, rho = (sk & 1) * 4 + lk;
          const double2* ap = st + static_cast<size_t>(2 * tt + u) * R * fld + rho * fld + lr;
          const double2* bp = mi + (tt * C + u * R + rho) * vld + n0 + lr;
          const double2 a0 = ap[0], a1 = ap[8];
          const double ar[2] = {a0.x, a1.x}, ai[2] = {neg(a0.y), neg(a1.y)};
          pair8_step<2>(t1, t2, t3, ar, ai, bp[0], bp[8]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          double w;
          const size_t e = pair_remap(a, static_cast<size_t>(g * a.pa + 2 * q + u) * C + 8 * i + lr, &w);
          double2* o = a.out + e * KS + k0 + n0 + 2 * lk;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int qq = 0; qq < 2; ++qq)
              o[8 * j + qq] = make_double2(w * (t1[i][j][qq] - t2[i][j][qq]), w * (t3[i][j][qq] - t1[i][j][qq] - t2[i][j][qq]));
        }
      }
      if constexpr (LEAF) fence_proxy_async_smem();  // in-place leaf outputs before the next bulk copy into the stage
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      pair_bar(1 + static_cast<int>(nn));   // both warps of the slice are past their mi reads
    }
  }
}

}  // namespace bfly

namespace bfly {

// ---------------------------------------------------------------- k-chunked level pairs
// The same two-level fusion when an item's full right-hand-side range does not fit a
// stage (cfg2 k = 256, r = 16: 8 blocks + 64 rows x 256 RHS = 330 KB): the item's 8
// factor blocks are loaded once into their own buffer, and the input rows stream
// through a ring in chunks of kc right-hand sides; per chunk, level A's outputs stay
// in shared memory (mi) for level B. The chain's intermediate vectors are read and
// written once per pair instead of once per level.
struct PairChunkArgs {
  const double2* fac_a;
  const double2* fac_b;
  const double2* in;
  double2* out;
  uint32_t r, ga, pa;
  uint32_t k;            // right-hand sides (row length of in / out)
  uint32_t kc, nch;      // chunk width, chunks per item
  int adjoint;
  uint32_t nitems;
  uint32_t fld, vld;     // shared-memory row strides of block rows and chunk rows
  uint32_t stages;       // ring depth (<= 4)
  uint32_t stage_elems;  // 2 C x vld
};

__device__ __forceinline__ void pair_chunk_factors(const PairChunkArgs& a, uint32_t item, double2* fs, uint64_t* bar,
                                                   int lane, uint64_t pol) {
  const uint32_t R = a.r, C = 2 * a.r, pb = a.pa / 2;
  const uint32_t g = item / pb, q = item - g * pb;
  if (lane == 0) mbar_arrive_expect_tx(bar, 8 * R * C * static_cast<uint32_t>(sizeof(double2)));
  __syncwarp();
  for (uint32_t row = lane; row < 8 * R; row += 32) {
    const uint32_t b = row / R, rr = row - b * R;
    const uint32_t lvl = b >> 2, t = (b >> 1) & 1, v = b & 1;
    const double2* src = lvl == 0 ? a.fac_a + (static_cast<size_t>((g * 2 + t) * a.pa + 2 * q + v) * R + rr) * C
                                  : a.fac_b + (static_cast<size_t>(((2 * g + t) * 2 + v) * pb + q) * R + rr) * C;
    bulk_g2s(fs + static_cast<size_t>(row) * a.fld, src, C * static_cast<uint32_t>(sizeof(double2)), bar, pol);
  }
}

__device__ __forceinline__ void pair_chunk_vectors(const PairChunkArgs& a, uint32_t item, uint32_t c, double2* vs,
                                                   uint64_t* bar, int lane) {
  const uint32_t R = a.r, C = 2 * a.r, pb = a.pa / 2;
  const uint32_t g = item / pb, q = item - g * pb;
  const uint32_t k0 = c * a.kc, kw = min(a.kc, a.k - k0);
  if (lane == 0) mbar_arrive_expect_tx(bar, 2 * C * kw * static_cast<uint32_t>(sizeof(double2)));
  __syncwarp();
  for (uint32_t row = lane; row < 2 * C; row += 32) {
    size_t grow;
    if (!a.adjoint) {
      grow = static_cast<size_t>(g * a.pa + 2 * q) * C + row;
    } else {
      const uint32_t ch = row / R, rr = row - ch * R, t = ch >> 1, tp = ch & 1;
      grow = static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * R + rr;
    }
    bulk_g2s(vs + static_cast<size_t>(row) * a.vld, a.in + grow * a.k + k0, kw * static_cast<uint32_t>(sizeof(double2)),
             bar);
  }
}

// One warp's share of a chunk: ngemm complex GEMMs Y_g (M x 8) = A_g (M x K) X_g (K x 8)
// for the 8 right-hand-side columns n0 .. n0 + 7 (of N), all M rows (MT 8-row tiles per
// pass, 3 DMMAs per complex k-step with GAUSS), K as nseg segments of klen.
template <bool GAUSS, typename AF, typename XF, typename YF>
__device__ __forceinline__ void warp_gemm_cols(int ngemm, int M, int nseg, int klen, int n0, int N, const AF& aload,
                                               const XF& xload, const YF& ystore, int lane) {
  constexpr int MT = 2;
  const int lr = lane >> 2, lk = lane & 3;
  const int n = n0 + lr;
  for (int gi = 0; gi < ngemm; ++gi)
    for (int m0 = 0; m0 < M; m0 += 8 * MT) {
      double cr[MT][2] = {}, ci[MT][2] = {}, cs[MT][2] = {};
      for (int sg = 0; sg < nseg; ++sg)
        for (int k0 = 0; k0 < klen; k0 += 4) {
          const int kk = k0 + lk;
          const bool kok = kk < klen;
          double2 av[MT];
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const int m = m0 + 8 * i + lr;
            av[i] = (kok && m < M) ? aload(gi, m, sg, kk) : make_double2(0, 0);
          }
          const double2 b = (kok && n < N) ? xload(gi, sg, kk, n) : make_double2(0, 0);
          if constexpr (GAUSS) {
            const double bs = b.x + b.y;
#pragma unroll
            for (int i = 0; i < MT; ++i) {
              pair_dmma(cr[i][0], cr[i][1], av[i].x, b.x);
              pair_dmma(ci[i][0], ci[i][1], av[i].y, b.y);
            }
#pragma unroll
            for (int i = 0; i < MT; ++i) pair_dmma(cs[i][0], cs[i][1], av[i].x + av[i].y, bs);
          } else {
#pragma unroll
            for (int i = 0; i < MT; ++i) {
              pair_dmma(cr[i][0], cr[i][1], av[i].x, b.x);
              pair_dmma(ci[i][0], ci[i][1], av[i].x, b.y);
            }
#pragma unroll
            for (int i = 0; i < MT; ++i) {
              pair_dmma(cr[i][0], cr[i][1], neg(av[i].y), b.y);
              pair_dmma(ci[i][0], ci[i][1], av[i].y, b.x);
            }
          }
        }
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int m = m0 + 8 * i + lr;
        if (m >= M) continue;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int nn = n0 + 2 * lk + q;
          if (nn >= N) continue;
          double re = cr[i][q], im = ci[i][q];
          if constexpr (GAUSS) {
            re = cr[i][q] - ci[i][q];
            im = cs[i][q] - cr[i][q] - ci[i][q];
          }
          ystore(gi, m, nn, make_double2(re, im));
        }
      }
    }
}

// Consumers: warp w owns right-hand-side columns 8 (w % 4) .. + 7 of every chunk and one
// half of the pair's dataflow (forward: t = w / 4, whose level-B outputs depend only on
// level-A outputs with the same t; adjoint: u = w / 4, the u-half rows of both level-B*
// outputs feed exactly the level-A* output u). Each warp's intermediate (C x 8, row
// stride 9: conflict-free fragment stores and loads) is private, so the two levels are
// separated by __syncwarp only and warps never wait for each other.
template <int NCW, bool GAUSS>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) pair_chunk_kernel(const PairChunkArgs a) {
  static_assert(NCW == 8, "4 column slices x 2 halves");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [4]
  uint64_t* empty = full + 4;                               // [4]
  uint64_t* ffull = full + 8;
  uint64_t* fempty = full + 9;
  const uint32_t R = a.r, C = 2 * a.r, pb = a.pa / 2, K = a.k, S = a.stages;
  double2* fs = reinterpret_cast<double2*>(smem_raw + 128);
  double2* ring = fs + static_cast<size_t>(8) * R * a.fld;
  double2* mis = ring + static_cast<size_t>(S) * a.stage_elems;  // NCW private C x 9 intermediates
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    mbar_init(ffull, 1);
    mbar_init(fempty, NCW);
    fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t fld = a.fld, vld = a.vld;
  if (warp == NCW) {
    const uint64_t pol = policy_evict_first();
    uint32_t it = 0, ii = 0;
    for (uint32_t item = blockIdx.x; item < a.nitems; item += gridDim.x, ++ii) {
      if (ii > 0) mbar_wait(fempty, (ii - 1) & 1);
      pair_chunk_factors(a, item, fs, ffull, lane, pol);  // constant: may precede the dependency wait
      if (ii == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
      for (uint32_t c = 0; c < a.nch; ++c, ++it) {
        const uint32_t s = it % S;
        if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
        pair_chunk_vectors(a, item, c, ring + static_cast<size_t>(s) * a.stage_elems, &full[s], lane);
      }
    }
    return;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n0 = (warp & 3) * 8, half = warp >> 2;
  double2* mi = mis + static_cast<size_t>(warp) * C * 9;
  uint32_t it = 0, ii = 0;
  auto blk = [&](uint32_t b) { return fs + static_cast<size_t>(b) * R * fld; };
  for (uint32_t item = blockIdx.x; item < a.nitems; item += gridDim.x, ++ii) {
    const uint32_t g = item / pb, q = item - g * pb;
    mbar_wait(ffull, ii & 1);
    for (uint32_t c = 0; c < a.nch; ++c, ++it) {
      const uint32_t s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      const double2* vs = ring + static_cast<size_t>(s) * a.stage_elems;
      const uint32_t k0 = c * a.kc;
      const int kw = static_cast<int>(min(a.kc, K - k0));
      if (n0 < kw) {
        if (!a.adjoint) {
          const uint32_t t = half;
          // level A, t fixed: Y_u = B_A(g, t, 2q + u) X_u  ->  mi rows u R + m
          warp_gemm_cols<GAUSS>(
              2, R, 1, C, n0, kw, [&](int u, int m, int, int kk) { return blk(2 * t + u)[m * fld + kk]; },
              [&](int u, int, int kk, int n) { return vs[(u * C + kk) * vld + n]; },
              [&](int u, int m, int n, double2 v) { mi[(u * R + m) * 9 + (n - n0)] = v; }, lane);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);  // this warp's reads of the chunk are done
          // level B: Z_t' = B_B(2g + t, t', q) mi  ->  out rows ((2g + t) 2 + t') P_B + q
          warp_gemm_cols<GAUSS>(
              2, R, 1, C, n0, kw, [&](int tp, int m, int, int kk) { return blk(4 + 2 * t + tp)[m * fld + kk]; },
              [&](int, int, int kk, int n) { return mi[kk * 9 + (n - n0)]; },
              [&](int tp, int m, int n, double2 v) {
                a.out[(static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * R + m) * K + k0 + n] = v;
              },
              lane);
        } else {
          const uint32_t u = half;
          // level B*, rows u R .. u R + R of Y_t = sum_t' B_B(2g + t, t', q)^H in(2g + t, t', q)
          warp_gemm_cols<GAUSS>(
              2, R, 2, R, n0, kw,
              [&](int t, int m, int tp, int kk) {
                const double2 v = blk(4 + 2 * t + tp)[kk * fld + u * R + m];
                return make_double2(v.x, neg(v.y));
              },
              [&](int t, int tp, int kk, int n) { return vs[((t * 2 + tp) * R + kk) * vld + n]; },
              [&](int t, int m, int n, double2 v) { mi[(t * R + m) * 9 + (n - n0)] = v; }, lane);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
          // level A*: out_u = sum_t B_A(g, t, 2q + u)^H Y_t[u half]  ->  rows (g P_A + 2q + u) C + m
          warp_gemm_cols<GAUSS>(
              1, C, 2, R, n0, kw,
              [&](int, int m, int t, int kk) {
                const double2 v = blk(2 * t + u)[kk * fld + m];
                return make_double2(v.x, neg(v.y));
              },
              [&](int, int t, int kk, int n) { return mi[(t * R + kk) * 9 + (n - n0)]; },
              [&](int, int m, int n, double2 v) {
                a.out[(static_cast<size_t>(g * a.pa + 2 * q + u) * C + m) * K + k0 + n] = v;
              },
              lane);
        }
        __syncwarp();  // mi is rewritten by the next chunk
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(fempty);  // the item's factor blocks are consumed
  }
}

}  // namespace bfly
