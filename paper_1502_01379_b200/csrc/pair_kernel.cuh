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
  uint32_t k;            // right-hand sides (all in one tile)
  int adjoint;
  uint32_t nitems;       // G_A * P_A / 2
  uint32_t fld, vld;     // shared-memory row strides of block rows and vector rows
  uint32_t stage_elems;  // 8 blocks + 2 C vector rows
};

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
__device__ __forceinline__ void pair_produce(const PairArgs& a, uint32_t item, double2* st, uint64_t* full, int lane,
                                             uint64_t pol) {
  const uint32_t R = a.r, C = 2 * a.r, pb = a.pa / 2;
  const uint32_t g = item / pb, q = item - g * pb;
  const uint32_t bytes = (8 * R * C + 2 * C * a.k) * static_cast<uint32_t>(sizeof(double2));
  if (lane == 0) mbar_arrive_expect_tx(full, bytes);
  __syncwarp();
  // block rows: 8 blocks x R rows; smem block b = (level, t, u|t') at b * R * fld
  for (uint32_t row = lane; row < 8 * R; row += 32) {
    const uint32_t b = row / R, rr = row - b * R;
    const uint32_t lvl = b >> 2, t = (b >> 1) & 1, v = b & 1;
    const double2* src = lvl == 0 ? a.fac_a + (static_cast<size_t>((g * 2 + t) * a.pa + 2 * q + v) * R + rr) * C
                                  : a.fac_b + (static_cast<size_t>(((2 * g + t) * 2 + v) * pb + q) * R + rr) * C;
    bulk_g2s(st + static_cast<size_t>(row) * a.fld, src, C * static_cast<uint32_t>(sizeof(double2)), full, pol);
  }
  double2* vs = st + static_cast<size_t>(8) * R * a.fld;
  for (uint32_t row = lane; row < 2 * C; row += 32) {
    size_t grow;
    if (!a.adjoint) {  // units (g, 2q), (g, 2q + 1): 2 C contiguous rows
      grow = static_cast<size_t>(g * a.pa + 2 * q) * C + row;
    } else {           // level-B* inputs (g' = 2g + t, t', q): R rows each, order [t][t']
      const uint32_t ch = row / R, rr = row - ch * R, t = ch >> 1, tp = ch & 1;
      grow = static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * R + rr;
    }
    bulk_g2s(vs + static_cast<size_t>(row) * a.vld, a.in + grow * a.k, a.k * static_cast<uint32_t>(sizeof(double2)),
             full);
  }
}

template <int STAGES, int NCW, bool GAUSS>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) pair_kernel(const PairArgs a) {
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
  const uint32_t R = a.r, C = 2 * a.r, pb = a.pa / 2, K = a.k;
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
    const uint32_t g = item / pb, q = item - g * pb;
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
            a.out[(static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * R + m) * K + n] = v;
          },
          warp, lane, NCW);
    } else {
      // level B*: Y(t) = sum_t' B_B(2g + t, t', q)^H in(2g + t, t', q)  ->  mi rows t C + c
      pair_gemms<GAUSS>(
          2, C, 2, R, K,
          [&](int gi, int m, int sg, int kk) {
            const double2 v = blk(4 + 2 * gi + sg)[kk * fld + m];
            return make_double2(v.x, -v.y);
          },
          [&](int gi, int sg, int kk, int n) { return vs[((gi * 2 + sg) * R + kk) * vld + n]; },
          [&](int gi, int m, int n, double2 v) { mi[(gi * C + m) * vld + n] = v; }, warp, lane, NCW);
      consumers_sync();
      // level A*: Y(u) = sum_t B_A(g, t, 2q + u)^H mi_t[u R ..]  ->  out rows (g P_A + 2q + u) C + c
      pair_gemms<GAUSS>(
          2, C, 2, R, K,
          [&](int gi, int m, int sg, int kk) {
            const double2 v = blk(2 * sg + gi)[kk * fld + m];
            return make_double2(v.x, -v.y);
          },
          [&](int gi, int sg, int kk, int n) { return mi[(sg * C + gi * R + kk) * vld + n]; },
          [&](int gi, int m, int n, double2 v) {
            a.out[(static_cast<size_t>(g * a.pa + 2 * q + gi) * C + m) * K + n] = v;
          },
          warp, lane, NCW);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    consumers_sync();  // mi is reused by the next item's first level
  }
}

}  // namespace bfly
