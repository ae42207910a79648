// level_kernel.cuh — one factor of the butterfly chain as a persistent,
// TMA-bulk-pipelined streaming kernel (the k <= ~64 regime, HBM-bound).
//
// Every factor of the chain (reference factors.py) is the same shape of work:
// a "unit" u owns nt blocks A[u, t] (R x C complex each). Its C-side vector
// chunk (C rows x k) is contiguous at row u*C; its R-side chunk for block t
// (R rows x k) sits at row q(u, t)*R with q = (g*nt + t)*P + p, u = g*P + p.
//
//   forward  (factors.py:49-51, 120-129):  Rside[u, t] = A[u, t]   @ Cside[u]
//   adjoint  (factors.py:53-56, 131-142):  Cside[u]    = sum_t A[u, t]^H @ Rside[u, t]
//
//   leaf U^L / V^L   : R = n0, C = r,  nt = 1, P = 1      (BlockDiagonalFactor)
//   split transfer   : R = r,  C = 2r, nt = 2, P = pairs  (TransferFactor, ndim 5)
//   merge transfer   : R = r,  C = 2r, nt = 1, P = pairs  (TransferFactor, ndim 4)
//
// The reshape between consecutive levels is the identity on memory
// (SURVEY.md §8(a) a3), so the chain is a sequence of these launches. The
// middle factor M (factors.py:180-190) is fused into the epilogue of the last
// adjoint level as an index remap + real scale (remap = 1: forward chain,
// remap = 2: adjoint chain).
//
// Pipeline: warp NCW (the producer) streams tiles — U consecutive units x kt
// right-hand sides — into a STAGES-deep shared-memory ring with the TMA bulk
// engine (cp.async.bulk + mbarrier complete_tx; L2 evict_first on factor
// bytes, which are read exactly once). NCW consumer warps compute each tile
// from shared memory and write the result straight to global memory.
#pragma once

#include "common.cuh"

namespace bfly {

struct LevelArgs {
  const void* fac;    // blocks of this factor, reference layout
  const void* in;     // input vector (rows x k)
  void* out;          // output vector
  const void* mid_w;  // middle weights (m, m, r) in plan real type, when remap != 0
  uint32_t R, C, nt;
  uint64_t P;         // units per group (pairs)
  uint64_t units;
  uint32_t k;         // total right-hand sides (row length of in/out)
  uint32_t kt;        // right-hand sides per tile
  uint32_t ktiles;    // ceil(k / kt)
  uint32_t U;         // units per tile (power of two)
  uint32_t S;         // lanes cooperating on one output
  uint64_t ntiles;    // (units / U) * ktiles
  uint32_t stage_elems;
  int adjoint;
  int remap;          // 0 none, 1 middle forward, 2 middle adjoint
  uint32_t m, r;      // middle geometry (remap)
  int bulk;           // 1: 16-byte aligned, use the TMA bulk engine
};

template <typename E>
struct TileGeo {
  uint64_t u0;        // first unit
  uint32_t k0, kc;    // first rhs, rhs count in this tile
  uint32_t Pe;        // min(P, U): slot stride
  uint32_t segs;      // factor / R-side segments (nt if U <= P else 1)
  uint32_t seg_blocks;
  uint64_t seg_start[2];  // first global block index of each segment
};

template <typename E>
__device__ __forceinline__ TileGeo<E> tile_geo(const LevelArgs& a, uint64_t tile) {
  TileGeo<E> t;
  const uint64_t ut = tile / a.ktiles;
  const uint32_t kti = static_cast<uint32_t>(tile - ut * a.ktiles);
  t.u0 = ut * a.U;
  t.k0 = kti * a.kt;
  t.kc = min(a.kt, a.k - t.k0);
  const uint64_t g0 = t.u0 / a.P, p0 = t.u0 % a.P;
  if (a.U <= a.P) {
    t.Pe = a.U;
    t.segs = a.nt;
    t.seg_blocks = a.U;
    t.seg_start[0] = (g0 * a.nt + 0) * a.P + p0;
    t.seg_start[1] = (g0 * a.nt + 1) * a.P + p0;
  } else {
    t.Pe = static_cast<uint32_t>(a.P);
    t.segs = 1;
    t.seg_blocks = a.nt * a.U;
    t.seg_start[0] = g0 * a.nt * a.P;
    t.seg_start[1] = 0;
  }
  return t;
}

// Copy `rows` rows of `kc` elements (source row stride k) into contiguous smem.
template <typename E>
__device__ __forceinline__ void stage_rows(E* dst, const E* src, uint64_t rows, uint32_t kc, uint32_t k,
                                           uint64_t* bar, int lane, int bulk, int lane_base) {
  if (bulk) {
    if (kc == k) {
      if (lane == lane_base) bulk_g2s(dst, src, static_cast<uint32_t>(rows * kc * sizeof(E)), bar);
    } else {
      for (uint64_t i = lane; i < rows; i += 32)
        bulk_g2s(dst + i * kc, src + i * k, kc * sizeof(E), bar);
    }
  } else {
    for (uint64_t i = 0; i < rows; ++i)
      for (uint32_t j = lane; j < kc; j += 32) dst[i * kc + j] = src[i * k + j];
  }
}

template <typename E>
__device__ __forceinline__ void produce_tile(const LevelArgs& a, uint64_t tile, E* st, uint64_t* full, int lane,
                                             uint64_t pol) {
  const TileGeo<E> t = tile_geo<E>(a, tile);
  const uint32_t blk = a.R * a.C;
  const E* fac = static_cast<const E*>(a.fac);
  const E* in = static_cast<const E*>(a.in);
  E* vs = st + static_cast<uint64_t>(a.nt) * a.U * blk;
  const uint64_t vec_rows = a.adjoint ? static_cast<uint64_t>(a.nt) * a.U * a.R : static_cast<uint64_t>(a.U) * a.C;
  if (a.bulk) {
    const uint32_t bytes = static_cast<uint32_t>((static_cast<uint64_t>(a.nt) * a.U * blk + vec_rows * t.kc) * sizeof(E));
    if (lane == 0) mbar_arrive_expect_tx(full, bytes);
    __syncwarp();
    if (lane < static_cast<int>(t.segs))
      bulk_g2s(st + static_cast<uint64_t>(lane) * t.seg_blocks * blk, fac + t.seg_start[lane] * blk,
               t.seg_blocks * blk * sizeof(E), full, pol);
  } else {
    for (uint32_t s = 0; s < t.segs; ++s) {
      const E* src = fac + t.seg_start[s] * blk;
      E* dst = st + static_cast<uint64_t>(s) * t.seg_blocks * blk;
      for (uint32_t i = lane; i < t.seg_blocks * blk; i += 32) dst[i] = src[i];
    }
  }
  if (!a.adjoint) {  // C-side chunk of the U units: contiguous rows u0*C ..
    stage_rows(vs, in + t.u0 * a.C * a.k + t.k0, static_cast<uint64_t>(a.U) * a.C, t.kc, a.k, full, lane, a.bulk, 2);
  } else {           // R-side chunks, same segment structure as the blocks
    for (uint32_t s = 0; s < t.segs; ++s)
      stage_rows(vs + static_cast<uint64_t>(s) * t.seg_blocks * a.R * t.kc, in + t.seg_start[s] * a.R * a.k + t.k0,
                 static_cast<uint64_t>(t.seg_blocks) * a.R, t.kc, a.k, full, lane, a.bulk, 2 + s);
  }
  if (!a.bulk) {
    __syncwarp();
    if (lane == 0) mbar_arrive(full);
  }
}

template <typename E>
__device__ __forceinline__ void consume_tile(const LevelArgs& a, uint64_t tile, const E* st, int ct, int nct) {
  using Rl = typename Cx<E>::R;
  const TileGeo<E> t = tile_geo<E>(a, tile);
  const uint32_t blk = a.R * a.C;
  const E* fs = st;
  const E* vs = st + static_cast<uint64_t>(a.nt) * a.U * blk;
  E* out = static_cast<E*>(a.out);
  const uint32_t S = a.S;
  const uint32_t s = ct % S;
  const uint32_t stride = nct / S;
  const uint32_t kc = t.kc;
  if (!a.adjoint) {
    const uint32_t n_out = a.U * a.nt * a.R * kc;
    const uint32_t CS = a.C / S;
    for (uint32_t base = 0; base < n_out; base += stride) {
      const uint32_t o = base + ct / S;
      E acc = Cx<E>::make(0, 0);
      uint32_t kk = 0, rho = 0, tt = 0, ul = 0;
      if (o < n_out) {
        kk = o % kc;
        uint32_t tmp = o / kc;
        rho = tmp % a.R;
        tmp /= a.R;
        tt = tmp % a.nt;
        ul = tmp / a.nt;
        const uint32_t slot = ((ul / t.Pe) * a.nt + tt) * t.Pe + ul % t.Pe;
        const E* arow = fs + (static_cast<uint64_t>(slot) * a.R + rho) * a.C;
        const E* x = vs + static_cast<uint64_t>(ul) * a.C * kc + kk;
        uint32_t idx = rho % CS;   // rotate the column start: lanes hit distinct banks
        for (uint32_t j = 0; j < CS; ++j) {
          const uint32_t c = s + S * idx;
          cmac(acc, arow[c], x[static_cast<uint64_t>(c) * kc]);
          if (++idx == CS) idx = 0;
        }
      }
      for (uint32_t w = 1; w < S; w <<= 1) {
        const E oth = shfl_xor(acc, w);
        acc.x += oth.x;
        acc.y += oth.y;
      }
      if (o < n_out && s == 0) {
        const uint64_t u = t.u0 + ul;
        const uint64_t g = u / a.P, p = u - g * a.P;
        const uint64_t q = (g * a.nt + tt) * a.P + p;
        out[(q * a.R + rho) * a.k + t.k0 + kk] = acc;
      }
    }
  } else {
    const uint32_t n_out = a.U * a.C * kc;
    const uint32_t terms = a.nt * a.R;
    const uint32_t TS = terms / S;
    for (uint32_t base = 0; base < n_out; base += stride) {
      const uint32_t o = base + ct / S;
      E acc = Cx<E>::make(0, 0);
      uint32_t kk = 0, c = 0, ul = 0;
      if (o < n_out) {
        kk = o % kc;
        uint32_t tmp = o / kc;
        c = tmp % a.C;
        ul = tmp / a.C;
        for (uint32_t j = 0; j < TS; ++j) {
          const uint32_t term = s * TS + j;
          const uint32_t tt = term / a.R, rho = term - tt * a.R;
          const uint32_t slot = ((ul / t.Pe) * a.nt + tt) * t.Pe + ul % t.Pe;
          const uint64_t row = static_cast<uint64_t>(slot) * a.R + rho;
          cmac_conj(acc, fs[row * a.C + c], vs[row * kc + kk]);
        }
      }
      for (uint32_t w = 1; w < S; w <<= 1) {
        const E oth = shfl_xor(acc, w);
        acc.x += oth.x;
        acc.y += oth.y;
      }
      if (o < n_out && s == 0) {
        const uint64_t e = (t.u0 + ul) * a.C + c;
        if (a.remap == 0) {
          out[e * a.k + t.k0 + kk] = acc;
        } else {
          const uint64_t mr = static_cast<uint64_t>(a.m) * a.r;
          const uint64_t ia = e / mr, ib = (e / a.r) % a.m, rho = e % a.r;
          const uint64_t dst = (ib * a.m + ia) * a.r + rho;
          const Rl* W = static_cast<const Rl*>(a.mid_w);
          const Rl w = a.remap == 1 ? W[dst] : W[(ia * a.m + ib) * a.r + rho];
          out[dst * a.k + t.k0 + kk] = Cx<E>::make(w * acc.x, w * acc.y);
        }
      }
    }
  }
}

template <typename E, int STAGES, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32) level_kernel(const LevelArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + STAGES;
  E* stage0 = reinterpret_cast<E*>(smem_raw + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == NCW) {
    const uint64_t pol = policy_evict_first();
    uint32_t it = 0;
    for (uint64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
      const uint32_t s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
      produce_tile<E>(a, tile, stage0 + static_cast<uint64_t>(s) * a.stage_elems, &full[s], lane, pol);
    }
  } else {
    uint32_t it = 0;
    for (uint64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
      const uint32_t s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      consume_tile<E>(a, tile, stage0 + static_cast<uint64_t>(s) * a.stage_elems, threadIdx.x, NCW * 32);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

}  // namespace bfly
