// pair16_kernel.cuh — two adjacent splitting transfer levels of a rank-16 chain in one
// kernel for many right-hand sides (BASELINE config 2, 64..256 RHS; config 4a), with the
// factor blocks fed to the FP64 tensor pipe straight from global memory / L2.
//
// A rank-16 pair closes over 8 blocks of 16 x 32 complex128 = 64 KB. Staging them in
// shared memory next to the item's vectors (as pair_kernel / pair8_kernel do) leaves one
// CTA per SM and no double buffering, which is why the k-chunked pair kernel lost to
// single levels. Here shared memory holds only vectors: the item's 64 input
// rows x 32 right-hand sides (a ring of stages filled by the TMA bulk engine) and the
// intermediate of the pair. Every GEMM of the pair is the same shape — 16 output rows x
// 16 right-hand sides over K = 32, in two halves of 4 k-steps — and a warp loads the A
// fragments of the NEXT half (8 x 16-byte loads per lane, one block row quarter per
// quarter warp: whole 32-byte sectors) while the DMMAs of the current half run, so the
// L2 latency of the factor reads hides behind 48 DMMAs. The pair reads and writes the
// chain's vectors once instead of twice (config 2, 256 RHS: 8.6 GB less DRAM traffic
// per level).
//
// Geometry as pair_kernel.cuh (item (g, q) x 32-RHS chunk). Every GEMM of a consumer warp
// is 8 output rows x the chunk's 32 right-hand sides over K = 32 (12 DMMAs per k-step for
// ONE 16-byte A fragment per lane, so a ring of 16 k-steps' fragments — two GEMMs ahead —
// costs 64 registers), four per item:
//   forward  warp (t, row tile): rows of Y(t, 0), Y(t, 1) into mi_t, a 64-thread named
//            barrier with the other row tile of branch t, then the same rows of out(t, 0),
//            out(t, 1) (level B of branch t reads only mi_t);
//   adjoint  warp w: rows [8 w, 8 w + 8) of mi_0 and mi_1 (level B*), the barrier with warp
//            w ^ 1 (out(u) reads rows [16 u, 16 u + 16) of both, i.e. warps 2u and 2u + 1),
//            then two 8-row tiles of out(u = w / 2) (level A*).
// The barrier is taken again at the end of the item, before mi is rewritten.
// 3-multiplication (Gauss) complex products as consume_tile_dmma (level_kernel.cuh).
#pragma once

#include "pair_kernel.cuh"

namespace bfly {

// one complex k-step of an 8-row x 32-column warp tile (3-multiplication form)
__device__ __forceinline__ void p16_step(double (&t1)[4][2], double (&t2)[4][2], double (&t3)[4][2], double ar,
                                         double ai, const double2* b) {
  double br[4], bi[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double2 v = b[8 * j];
    br[j] = v.x;
    bi[j] = v.y;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    pair_dmma(t1[j][0], t1[j][1], ar, br[j]);
    pair_dmma(t2[j][0], t2[j][1], ai, bi[j]);
  }
  const double as = ar + ai;
#pragma unroll
  for (int j = 0; j < 4; ++j) pair_dmma(t3[j][0], t3[j][1], as, br[j] + bi[j]);
}

// producer: the item's 64 input rows (forward: contiguous; adjoint: 4 chunks of 16 rows,
// order [t][t']), kw right-hand sides each, one bulk copy per row
__device__ __forceinline__ void pair16_produce(const PairArgs& a, uint32_t item_rhs, double2* vs, uint64_t* full,
                                               int lane) {
  constexpr uint32_t R = 16, C = 32;
  const uint32_t pb = a.pa / 2;
  const uint32_t item = item_rhs / a.nch, k0 = (item_rhs - item * a.nch) * a.kc, kw = min(a.kc, a.k - k0);
  const uint32_t g = item / pb, q = item - g * pb;
  if (lane == 0) mbar_arrive_expect_tx(full, 2 * C * kw * static_cast<uint32_t>(sizeof(double2)));
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
             full);
  }
}

template <int STAGES, bool ADJ>
__global__ void __launch_bounds__(128, 2) pair16_kernel(const PairArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + STAGES;
  double2* stage0 = reinterpret_cast<double2*>(smem_raw + 128);
  double2* mi = stage0 + static_cast<size_t>(STAGES) * a.stage_elems;  // 64 x vld intermediate
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // four warps, all consumers (a fifth, producer-only warp would cap the kernel at 168
  // registers per thread with two CTAs per SM; 128-thread CTAs may use 255): warp 0 also
  // refills the ring, one item ahead, at the end of each item
  constexpr int NCW = 4;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr uint32_t R = 16, C = 32, BLK = R * C;
  const uint32_t pb = a.pa / 2, KS = a.k, vld = a.vld;
  const uint32_t w = warp, lr = lane >> 2, lk = lane & 3;
  const uint32_t hi = w >> 1, lo = w & 1;   // forward: (t, row tile); adjoint: (u, column-tile pair)
  const int bar_id = 1 + static_cast<int>(hi);
  // A element of global k-step kk (GEMM kk / 8, step kk % 8) of item (g, q):
  //   forward  GEMM 0/1 = A(t, u = gm), GEMM 2/3 = B(t, t' = gm - 2): (row 8 lo + lr, column 4 s + lk)
  //   adjoint  GEMM 0/1 = mi_t (t = gm): block B(t, t' = s / 4), (row 4 (s % 4) + lk, column 8 w + lr), conjugated
  //            GEMM 2/3 = out(u = hi), column tile ct = 2 lo + gm - 2: block A(t2 = s / 4, u), (row 4 (s % 4) + lk,
  //            column 8 ct + lr), conjugated
  auto a_ptr = [&](uint32_t g, uint32_t q, uint32_t kk) -> const double2* {
    const uint32_t gm = kk >> 3, s = kk & 7;
    if constexpr (!ADJ) {
      const double2* blk = gm < 2 ? a.fac_a + static_cast<size_t>((g * 2 + hi) * a.pa + 2 * q + gm) * BLK
                                  : a.fac_b + static_cast<size_t>(((2 * g + hi) * 2 + (gm - 2)) * pb + q) * BLK;
      return blk + (8 * lo + lr) * C + 4 * s + lk;
    } else {
      const uint32_t sg = s >> 2, rho = 4 * (s & 3) + lk;
      if (gm < 2) {
        const double2* blk = a.fac_b + static_cast<size_t>(((2 * g + gm) * 2 + sg) * pb + q) * BLK;
        return blk + rho * C + 8 * w + lr;
      }
      const double2* blk = a.fac_a + static_cast<size_t>((g * 2 + sg) * a.pa + 2 * q + hi) * BLK;
      return blk + rho * C + 8 * (2 * lo + gm - 2) + lr;
    }
  };
  // ring of the next 16 k-steps' A fragments (two GEMMs ahead of the DMMAs that use them)
  double2 ring[16];
  if (blockIdx.x < a.nitems) {  // constant data: before the dependency wait
    const uint32_t pitem = blockIdx.x / a.nch;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) ring[kk] = __ldg(a_ptr(pitem / pb, pitem % pb, kk));
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (warp == 0) {
    uint32_t pre = 0;
    for (uint32_t item = blockIdx.x; item < a.nitems && pre < STAGES; item += gridDim.x, ++pre)
      pair16_produce(a, item, stage0 + static_cast<size_t>(pre) * a.stage_elems, &full[pre], lane);
  }
  uint32_t it = 0;
  for (uint32_t item = blockIdx.x; item < a.nitems; item += gridDim.x, ++it) {
    const uint32_t s = it % STAGES;
    const double2* vs = stage0 + static_cast<size_t>(s) * a.stage_elems;
    const uint32_t pitem = item / a.nch, k0 = (item - pitem * a.nch) * a.kc;
    const uint32_t g = pitem / pb, q = pitem - g * pb;
    const uint32_t nitem = item + gridDim.x;
    const uint32_t npitem = (nitem < a.nitems ? nitem : item) / a.nch;   // next item's pair (prefetch target)
    const uint32_t ng = npitem / pb, nq = npitem - ng * pb;
    double t1[4][2], t2[4][2], t3[4][2];
    // B rows of k-step s of GEMM gm (shared memory), this lane's first column
    auto b_ptr = [&](uint32_t gm, uint32_t s) -> const double2* {
      if constexpr (!ADJ) {
        const double2* base = gm < 2 ? vs + (gm * C) * vld : mi + (hi * C) * vld;
        return base + (4 * s + lk) * vld + lr;
      } else {
        const uint32_t sg = s >> 2, rho = 4 * (s & 3) + lk;
        const double2* base = gm < 2 ? vs + (gm * C + 16 * sg) * vld : mi + (sg * C + hi * 16) * vld;
        return base + rho * vld + lr;
      }
    };
    auto gemm = [&](uint32_t gm) {   // 8 k-steps; each consumed ring slot is refilled 16 k-steps ahead
#pragma unroll
      for (int j = 0; j < 4; ++j) t1[j][0] = t1[j][1] = t2[j][0] = t2[j][1] = t3[j][0] = t3[j][1] = 0.0;
#pragma unroll
      for (uint32_t s8 = 0; s8 < 8; ++s8) {
        const uint32_t kk = gm * 8 + s8, slot = kk & 15;
        const double2 av = ring[slot];
        ring[slot] = kk + 16 < 32 ? __ldg(a_ptr(g, q, kk + 16)) : __ldg(a_ptr(ng, nq, kk + 16 - 32));
        p16_step(t1, t2, t3, av.x, ADJ ? neg(av.y) : av.y, b_ptr(gm, s8));
      }
    };
    auto store_mi = [&](uint32_t row0) {  // 8 rows starting at row0 of mi, all 32 columns
      double2* mo = mi + (row0 + lr) * vld + 2 * lk;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int qq = 0; qq < 2; ++qq)
          mo[8 * j + qq] = make_double2(t1[j][qq] - t2[j][qq], t3[j][qq] - t1[j][qq] - t2[j][qq]);
    };
    auto store_out = [&](size_t e, double wgt) {
      double2* o = a.out + e * KS + k0 + 2 * lk;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const double re = t1[j][qq] - t2[j][qq], im = t3[j][qq] - t1[j][qq] - t2[j][qq];
          o[8 * j + qq] = ADJ ? make_double2(wgt * re, wgt * im) : make_double2(re, im);
        }
    };
    mbar_wait(&full[s], (it / STAGES) & 1);
    // ---- first level of the pair in apply order: GEMMs 0, 1 (inputs in the stage)
    gemm(0);
    store_mi(ADJ ? 0 * C + 8 * w : hi * C + 0 * R + 8 * lo);
    gemm(1);
    store_mi(ADJ ? 1 * C + 8 * w : hi * C + 1 * R + 8 * lo);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);   // the stage is consumed
    pair_bar(bar_id);                        // the partner warp's rows of mi
    // ---- second level: GEMMs 2, 3 (inputs in mi)
    gemm(2);
    if constexpr (!ADJ) {
      store_out(static_cast<size_t>(((2 * g + hi) * 2 + 0) * pb + q) * R + 8 * lo + lr, 1.0);
    } else {
      double wgt;
      const size_t e = pair_remap(a, static_cast<size_t>(g * a.pa + 2 * q + hi) * C + 8 * (2 * lo) + lr, &wgt);
      store_out(e, wgt);
    }
    gemm(3);
    if constexpr (!ADJ) {
      store_out(static_cast<size_t>(((2 * g + hi) * 2 + 1) * pb + q) * R + 8 * lo + lr, 1.0);
    } else {
      double wgt;
      const size_t e = pair_remap(a, static_cast<size_t>(g * a.pa + 2 * q + hi) * C + 8 * (2 * lo + 1) + lr, &wgt);
      store_out(e, wgt);
    }
    if (warp == 0) {   // refill this item's stage (released by every warp after GEMM 1) for item it + STAGES
      const uint32_t fill = item + STAGES * gridDim.x;
      if (fill < a.nitems) {
        mbar_wait(&empty[s], (it / STAGES) & 1);
        pair16_produce(a, fill, stage0 + static_cast<size_t>(s) * a.stage_elems, &full[s], lane);
      }
    }
    pair_bar(bar_id);   // both warps of the pair are past their mi reads
  }
}

}  // namespace bfly
