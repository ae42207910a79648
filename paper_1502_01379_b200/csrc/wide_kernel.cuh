// wide_kernel.cuh — many-RHS complex128 levels whose units are too wide for one
// shared-memory stage (quadtree rank 25: a unit is 4 blocks x 25 x 100 = 160 KB),
// as a K-pipelined FP64 tensor-core GEMM.
//
// A unit of a split transfer factor (factors.py:120-142, branching nt) is the GEMM
//   forward  Y (nt R x kc) = A (nt R x C) X (C x kc)       A rows t R + rho = block q(u, t)
//   adjoint  X (C x kc)    = A^H (C x nt R) Y (nt R x kc)  Y rows t R + rho at q(u, t) R + rho
// with q(u, t) = ((g nt + t) << lgP) + p for u = g P + p (level_kernel.cuh). Instead of
// staging a whole unit (single-buffered, every load exposed) the K dimension — the
// block columns forward, the concatenated (t, rho) block rows adjoint — is cut into
// KT-wide tiles: each stage holds one K tile of all nt blocks plus the matching KT
// vector rows, a producer warp streams the stages through an S-deep ring with the TMA
// bulk engine (one copy per staged row, rows padded for conflict-free DMMA fragment
// reads), and the consumer warps keep the unit's accumulators in registers across the
// unit's K tiles. Consumer warp w owns output rows 8w .. 8w + 7 (m_out <= 8 NCW) and
// every right-hand side of the item (NT 8-column DMMA tiles), 3-multiplication (Gauss)
// complex products as in consume_tile_dmma. Outputs go straight from registers to
// global memory; the middle factor (remap 1/2) is fused into the adjoint epilogue.
#pragma once

#include <cuda.h>

#include "level_kernel.cuh"  // dmma()

namespace bfly {

struct WideArgs {
  double2* out;
  const double* mid_w;  // middle weights (m, m, r) when remap != 0
  uint32_t R, C, nt, lgP;
  uint32_t k;           // row length of in / out
  uint32_t kc;          // right-hand sides per item (<= 8 NT)
  uint32_t nkc;         // items per unit (right-hand-side chunks)
  uint32_t items;       // units * nkc
  uint32_t KT;          // K tile per stage: block columns forward (multiple of 4), R adjoint
  uint32_t nks;         // stages per item: ceil(C / KT) forward, nt adjoint
  uint32_t fst;         // shared-memory row stride (elements) of staged factor rows
  uint32_t fslot;       // forward: elements per staged block (128-byte aligned slots)
  uint32_t vst;         // shared-memory row stride of staged vector rows (the vector box width)
  uint32_t voff;        // offset of the vector rows in a stage (elements, 128-byte aligned)
  uint32_t stage_elems;
  uint32_t stage_bytes; // transaction bytes of one stage (full boxes, out-of-bounds fill included)
  uint32_t stages;      // ring depth (<= 8)
  int adjoint, remap;
  uint32_t m, r;        // middle geometry (remap)
};

// TMA tensor copy (2-D tile box) global -> shared, completion as tx bytes on bar.
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int32_t c0, int32_t c1, uint64_t* bar,
                                       uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int32_t c0, int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Factor part of stage (item, j), one lane: arm the stage barrier with the stage's whole
// byte count and start the block copies (tensor map tmA over the factor's block rows:
// 2C doubles x all rows). Factors are constant across the chain, so this may run before
// the dependency wait on the previous level.
//   forward: the K tile (columns kb .. kb + KT) of each of the unit's nt blocks, one box
//            {2 KT, R} per block into 128-byte aligned slots (row stride KT)
//   adjoint: block t = j whole, one box {2 fst, R} (columns past C fill with zeros)
__device__ __forceinline__ void wide_factors(const WideArgs& a, const CUtensorMap* tmA, uint32_t item, uint32_t j,
                                             double2* st, uint64_t* full, uint64_t pol) {
  const uint32_t u = item / a.nkc;
  const uint32_t g = u >> a.lgP, p = u & ((1u << a.lgP) - 1);
  mbar_arrive_expect_tx(full, a.stage_bytes);
  if (!a.adjoint) {
    for (uint32_t t = 0; t < a.nt; ++t) {
      const uint32_t b = ((g * a.nt + t) << a.lgP) + p;
      tma_2d(st + static_cast<size_t>(t) * a.fslot, tmA, static_cast<int32_t>(2 * j * a.KT),
             static_cast<int32_t>(b * a.R), full, pol);
    }
  } else {
    const uint32_t b = ((g * a.nt + j) << a.lgP) + p;
    tma_2d(st, tmA, 0, static_cast<int32_t>(b * a.R), full, pol);
  }
}

// Vector part of stage (item, j): the K tile's input rows (the previous level's output),
// one box {2 vst, KT} of the tensor map tmV over the input vector (2k doubles x rows).
__device__ __forceinline__ void wide_vectors(const WideArgs& a, const CUtensorMap* tmV, uint32_t item, uint32_t j,
                                             double2* st, uint64_t* full) {
  const uint32_t u = item / a.nkc, k0 = (item - u * a.nkc) * a.kc;
  uint32_t row;
  if (!a.adjoint) {
    row = u * a.C + j * a.KT;
  } else {
    const uint32_t g = u >> a.lgP, p = u & ((1u << a.lgP) - 1);
    row = (((g * a.nt + j) << a.lgP) + p) * a.R;
  }
  tma_2d(st + a.voff, tmV, static_cast<int32_t>(2 * k0), static_cast<int32_t>(row), full);
}

template <int NCW, int NT, bool ADJ>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    wide_kernel(const WideArgs a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + 8;
  double2* stage0 = reinterpret_cast<double2*>(smem_raw + 128);
  const uint32_t S = a.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // programmatic dependent launch (see level_kernel): only constant factor rows are
  // fetched before the wait on the previous level
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == NCW) {
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    uint32_t pre = 0;
    for (uint32_t item = blockIdx.x; item < a.items && pre < S; item += gridDim.x)
      for (uint32_t j = 0; j < a.nks && pre < S; ++j, ++pre)
        wide_factors(a, &tmA, item, j, stage0 + static_cast<size_t>(pre) * a.stage_elems, &full[pre], pol);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint32_t cnt = 0;
    for (uint32_t item = blockIdx.x; item < a.items; item += gridDim.x)
      for (uint32_t j = 0; j < a.nks; ++j, ++cnt) {
        const uint32_t s = cnt % S;
        double2* st = stage0 + static_cast<size_t>(s) * a.stage_elems;
        if (cnt >= pre) {
          if (cnt >= S) mbar_wait(&empty[s], ((cnt / S) - 1) & 1);
          wide_factors(a, &tmA, item, j, st, &full[s], pol);
        }
        wide_vectors(a, &tmV, item, j, st, &full[s]);
      }
    return;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t m_out = ADJ ? a.C : a.nt * a.R;
  const uint32_t K = ADJ ? a.nt * a.R : a.C;
  const uint32_t lr = lane >> 2, lk = lane & 3;
  const bool act = static_cast<uint32_t>(warp) * 8 < m_out;
  const uint32_t mrow = static_cast<uint32_t>(warp) * 8 + lr;   // this lane's A row / output row
  const uint32_t mc = min(mrow, m_out - 1);
  // forward: this lane's A row (block t = mc / R, row rho) in the stage's block slots
  const uint32_t arow = ADJ ? 0 : (mc / a.R) * a.fslot + (mc - (mc / a.R) * a.R) * a.fst;
  uint32_t cnt = 0;
  for (uint32_t item = blockIdx.x; item < a.items; item += gridDim.x) {
    // T1, T2, T3 of the Gauss form per 8-column tile (two accumulator registers each)
    double t1[NT][2], t2[NT][2], t3[NT][2];
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) t1[jn][0] = t1[jn][1] = t2[jn][0] = t2[jn][1] = t3[jn][0] = t3[jn][1] = 0;
    for (uint32_t j = 0; j < a.nks; ++j, ++cnt) {
      const uint32_t s = cnt % S;
      mbar_wait(&full[s], (cnt / S) & 1);
      const double2* fs = stage0 + static_cast<size_t>(s) * a.stage_elems;
      const double2* vs = fs + a.voff;
      const uint32_t kv = min(a.KT, K - j * a.KT);
      if (act) {
        const double2* ab = ADJ ? fs + mc : fs + arow;
        for (uint32_t k0 = 0; k0 < kv; k0 += 4) {
          const uint32_t kr = k0 + lk;
          const bool kok = kr < kv;
          const uint32_t kk = kok ? kr : kv - 1;   // clamped (finite) reads, zero A past the tile
          double2 av = ADJ ? ab[kk * a.fst] : ab[kk];
          if (ADJ) av.y = neg(av.y);  // A^H
          const double ar = kok ? av.x : 0.0, ai = kok ? av.y : 0.0;
          const double as = ar + ai;
          const double2* bp = vs + kk * a.vst + lr;
          double br[NT], bi[NT];
#pragma unroll
          for (int jn = 0; jn < NT; ++jn) {
            const double2 v = bp[8 * jn];
            br[jn] = v.x;
            bi[jn] = v.y;
          }
#pragma unroll
          for (int jn = 0; jn < NT; ++jn) {
            dmma(t1[jn][0], t1[jn][1], ar, br[jn]);
            dmma(t2[jn][0], t2[jn][1], ai, bi[jn]);
          }
#pragma unroll
          for (int jn = 0; jn < NT; ++jn) dmma(t3[jn][0], t3[jn][1], as, br[jn] + bi[jn]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (!act || mrow >= m_out) continue;
    const uint32_t u = item / a.nkc, k0 = (item - u * a.nkc) * a.kc;
    const uint32_t kcn = min(a.kc, a.k - k0);
    double2* orow;
    double w = 1;
    if (!ADJ) {
      const uint32_t g = u >> a.lgP, p = u & ((1u << a.lgP) - 1);
      const uint32_t t = mrow / a.R, rho = mrow - t * a.R;
      const uint32_t b = ((g * a.nt + t) << a.lgP) + p;
      orow = a.out + (static_cast<size_t>(b) * a.R + rho) * a.k + k0;
    } else {
      size_t e = static_cast<size_t>(u) * a.C + mrow;
      if (a.remap) {  // fused middle factor (factors.py:180-190), as remap_row
        const uint32_t mr = a.m * a.r;
        const uint32_t e32 = static_cast<uint32_t>(e), ia = e32 / mr;
        const uint32_t rem = e32 - ia * mr;
        const uint32_t ib = rem / a.r, rho = rem - ib * a.r;
        const size_t dst = (static_cast<size_t>(ib) * a.m + ia) * a.r + rho;
        w = a.remap == 1 ? __ldg(a.mid_w + dst) : __ldg(a.mid_w + (static_cast<size_t>(ia) * a.m + ib) * a.r + rho);
        e = dst;
      }
      orow = a.out + e * a.k + k0;
    }
#pragma unroll
    for (int jn = 0; jn < NT; ++jn)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t n = 8 * jn + 2 * lk + q;
        if (n < kcn) {
          const double re = t1[jn][q] - t2[jn][q], im = t3[jn][q] - t1[jn][q] - t2[jn][q];
          orow[n] = make_double2(w * re, w * im);
        }
      }
  }
}

}  // namespace bfly
