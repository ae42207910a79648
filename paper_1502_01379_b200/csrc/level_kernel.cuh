// level_kernel.cuh — one factor of the butterfly chain as a persistent,
// TMA-bulk-pipelined streaming kernel (the small-k, HBM-bound regime).
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
// adjoint-direction level as an index remap + real scale (remap = 1: forward
// chain, remap = 2: adjoint chain).
//
// Pipeline: warp NCW (the producer) streams tiles — U consecutive units x kt
// right-hand sides — into a STAGES-deep shared-memory ring with the TMA bulk
// engine (cp.async.bulk + mbarrier complete_tx; L2 evict_first on factor
// bytes, which are read exactly once). NCW consumer warps compute each tile
// from shared memory — one output per thread, a full-length dot product with
// 8 independent FP64 accumulation chains, bank-conflict-free (rotated column
// order when lanes walk rows of a block) — and store straight to global.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace bfly {

struct LevelArgs {
  const void* fac;    // blocks of this factor, reference layout
  const void* in;     // input vector (rows x k)
  void* out;          // output vector
  const void* mid_w;  // middle weights (m, m, r) in plan real type, when remap != 0
  uint32_t R, C, nt;  // nt: blocks of a unit held per tile (a t-range of ntot)
  uint32_t ntot, t0;  // blocks per unit (2 in 1-D, 4 on quadtrees) and the first t of this launch
  int accumulate;     // adjoint with a t-range split: add into out instead of storing
  uint32_t lgP;       // log2(units per group)
  uint32_t units;
  uint32_t k;         // total right-hand sides (row length of in/out)
  uint32_t kt;        // right-hand sides per tile
  uint32_t ktiles;    // ceil(k / kt)
  uint32_t lgU;       // log2(units per tile)
  uint32_t ntiles;    // (units / U) * ktiles
  uint32_t stage_elems;
  int adjoint;
  int remap;          // 0 none, 1 middle forward, 2 middle adjoint, 3/4 the same pushed to peers
  uint32_t m, r;      // middle geometry (remap)
  uint32_t part, mp;  // remap 3/4: this part and middle nodes per part
  int bulk;           // 1: 16-byte aligned, use the TMA bulk engine
  int use_dmma;       // many-RHS complex128: FP64 tensor-core (mma.sync f64) consumer; 2 = 3-mult (Gauss) products
  // shared-memory row strides (elements) of the staged factor rows (fld, default C)
  // and vector rows (vld, 0 = the tile's kc). The DMMA consumer pads them so its
  // fragment loads hit 8 distinct 16-byte bank groups per quarter warp.
  uint32_t fld, vld;
  // MRHS = 3 (DMMA consumer, outputs in place of the stage's vector rows, TMA-stored by
  // the producer): row stride of the output rows in shared memory
  uint32_t old;
  uint32_t stages;    // pipeline depth when the kernel's STAGES template argument is 0 (<= 8)
  uint32_t dtile;     // DMMA warp tile: 0 = 2 x 4, 1 = 2 x 2, 2 = 1 x 2 (8 x 8 tiles)
  int dbg_nomath;     // BF_DBG_NOMATH=1 (diagnostics only): many-RHS consumers skip their k loops
  int dbg_noload;     // BF_DBG_NOLOAD=1 (diagnostics only): the producer moves no data (compute + stores only)
  int inplace;        // MRHS = 3: outputs overwrite the stage's vector rows (one warp item per warp)
  uint32_t tsplit;    // forward levels: t-ranges of a unit as separate tiles of one launch (1 = off)
};

// remap 3/4 receive buffers of every part ([sender][own][other local][rho][k]); a
// separate kernel parameter read only by the PUSH instantiation — inside LevelArgs
// the 64 bytes cost the many-RHS kernels a register spill and ~8%
struct PeerArgs {
  void* peers[8];
};


// Destination row (the element for right-hand side 0) and middle weight of
// output e of the last adjoint-direction level. remap 1/2 fuse the middle
// factor (factors.py:180-190): e = (a, b, rho) -> (b, a, rho), weight W[b,a] /
// W[a,b]. remap 3/4 do the same for one part of a sharded chain and store
// straight into the owning part's receive buffer (peer memory over NVLink on a
// multi-GPU box): a = own local node, b = global other node, receiver part
// b / mp, slot [sender][own][b mod mp][rho] — the layout bf_middle_pack + an
// all-to-all would produce, with no pack kernel and no collective.
template <typename E, bool PUSH>
__device__ __forceinline__ E* remap_row(const LevelArgs& a, const PeerArgs& pa, size_t e, typename Cx<E>::R* w) {
  using Rl = typename Cx<E>::R;
  E* out = static_cast<E*>(a.out);
  if (a.remap == 0) {
    *w = 1;
    return out + e * a.k;
  }
  const Rl* W = static_cast<const Rl*>(a.mid_w);
  const uint32_t mr = a.m * a.r;
  const uint32_t e32 = static_cast<uint32_t>(e), ia = e32 / mr;
  const uint32_t rem = e32 - ia * mr;
  const uint32_t ib = rem / a.r, rho = rem - ib * a.r;
  if (a.remap <= 2) {
    const size_t dst = (static_cast<size_t>(ib) * a.m + ia) * a.r + rho;
    *w = a.remap == 1 ? __ldg(W + dst) : __ldg(W + (static_cast<size_t>(ia) * a.m + ib) * a.r + rho);
    return out + dst * a.k;
  }
  if constexpr (!PUSH) {
    return out;  // remap 3/4 only run in the PUSH instantiation
  } else {
  const uint32_t own = a.part * a.mp + ia, d = ib / a.mp, bl = ib - d * a.mp;
  *w = a.remap == 3 ? __ldg(W + (static_cast<size_t>(ib) * a.m + own) * a.r + rho)
                    : __ldg(W + (static_cast<size_t>(own) * a.m + ib) * a.r + rho);
  // select the peer pointer without a dynamic index into the parameter block (which
  // would force a local-memory copy of it)
  E* base = nullptr;
#pragma unroll
  for (uint32_t q = 0; q < 8; ++q)
    if (q == d) base = static_cast<E*>(pa.peers[q]);
  return base + ((static_cast<size_t>(own) * a.mp + bl) * a.r + rho) * a.k;
  }
}

struct TileGeo {
  uint32_t u0;        // first unit
  uint32_t k0, kc;    // first rhs, rhs count in this tile
  uint32_t lgPe;      // log2(min(P, U)): slot stride
  uint32_t segs;      // factor / R-side segments (nt if U <= P else 1)
  uint32_t seg_blocks;
  uint32_t seg0;      // first global block index of segment 0
  uint32_t seg_step;  // block distance between segments
  uint32_t t0;        // first t of this tile's t-range
};

__device__ __forceinline__ TileGeo tile_geo(const LevelArgs& a, uint32_t tile) {
  TileGeo t;
  uint32_t ut = tile, kti = 0;
  t.t0 = a.t0;
  if (a.tsplit > 1) {   // forward levels: the t-ranges of a unit are consecutive tiles
    const uint32_t ts = ut % a.tsplit;
    ut /= a.tsplit;
    t.t0 += ts * a.nt;
  }
  if (a.ktiles > 1) {
    ut = tile / a.ktiles;
    kti = tile - ut * a.ktiles;
  }
  t.u0 = ut << a.lgU;
  t.k0 = kti * a.kt;
  t.kc = min(a.kt, a.k - t.k0);
  const uint32_t g0 = t.u0 >> a.lgP, p0 = t.u0 & ((1u << a.lgP) - 1);
  if (a.lgU <= a.lgP) {
    t.lgPe = a.lgU;
    t.segs = a.nt;
    t.seg_blocks = 1u << a.lgU;
    t.seg0 = ((g0 * a.ntot + t.t0) << a.lgP) + p0;
    t.seg_step = 1u << a.lgP;
  } else {
    t.lgPe = a.lgP;
    t.segs = 1;
    t.seg_blocks = a.nt << a.lgU;
    t.seg0 = (g0 * a.ntot) << a.lgP;  // (only with nt == ntot, t0 == 0)
    t.seg_step = 0;
  }
  return t;
}

// Copy `rows` rows of `kc` elements (source row stride k) into smem rows of stride ld.
template <typename E>
__device__ __forceinline__ void stage_rows(E* dst, const E* src, uint32_t rows, uint32_t kc, uint32_t k, uint32_t ld,
                                           uint64_t* bar, int lane, int bulk, int lane_base) {
  if (bulk) {
    if (kc == k && ld == kc) {
      if (lane == lane_base) bulk_g2s(dst, src, rows * kc * static_cast<uint32_t>(sizeof(E)), bar);
    } else {
      for (uint32_t i = lane; i < rows; i += 32)
        bulk_g2s(dst + static_cast<size_t>(i) * ld, src + static_cast<size_t>(i) * k, kc * sizeof(E), bar);
    }
  } else {
    const uint32_t total = rows * kc;
    for (uint32_t idx = lane; idx < total; idx += 32) {
      const uint32_t i = kc == 1 ? idx : idx / kc, j = kc == 1 ? 0 : idx - (idx / kc) * kc;
      dst[static_cast<size_t>(i) * ld + j] = src[static_cast<size_t>(i) * k + j];
    }
  }
}

// Factor part of a tile (bulk path): arm the stage barrier with the whole tile's
// byte count and start the block copies. Factors are constant across the chain,
// so this may run before the dependency wait on the previous level.
template <typename E>
__device__ __forceinline__ void produce_factors(const LevelArgs& a, const TileGeo& t, E* st, uint64_t* full, int lane,
                                                uint64_t pol) {
  const uint32_t blk = a.R * a.C;
  const E* fac = static_cast<const E*>(a.fac);
  const uint32_t U = 1u << a.lgU;
  const uint32_t vec_rows = a.adjoint ? a.nt * U * a.R : U * a.C;
  const uint32_t bytes = (a.nt * U * blk + vec_rows * t.kc) * static_cast<uint32_t>(sizeof(E));
  if (lane == 0) mbar_arrive_expect_tx(full, bytes);
  __syncwarp();
  if (a.fld == a.C) {
    if (lane < static_cast<int>(t.segs))
      bulk_g2s(st + static_cast<size_t>(lane) * t.seg_blocks * blk,
               fac + static_cast<size_t>(t.seg0 + lane * t.seg_step) * blk, t.seg_blocks * blk * sizeof(E), full, pol);
  } else {  // padded rows: one copy per block row
    const uint32_t seg_rows = t.seg_blocks * a.R;
    for (uint32_t row = lane; row < t.segs * seg_rows; row += 32) {
      const uint32_t sg = row / seg_rows, rr = row - sg * seg_rows;
      bulk_g2s(st + static_cast<size_t>(row) * a.fld,
               fac + static_cast<size_t>(t.seg0 + sg * t.seg_step) * blk + static_cast<size_t>(rr) * a.C,
               a.C * static_cast<uint32_t>(sizeof(E)), full, pol);
    }
  }
}

// Vector part of a tile: the input rows the tile's blocks multiply (the previous
// level's output).
template <typename E>
__device__ __forceinline__ void produce_vectors(const LevelArgs& a, const TileGeo& t, E* st, uint64_t* full,
                                                int lane) {
  const E* in = static_cast<const E*>(a.in);
  const uint32_t U = 1u << a.lgU;
  E* vs = st + static_cast<size_t>(a.nt) * U * a.R * a.fld;
  const uint32_t ld = a.vld ? a.vld : t.kc;
  if (!a.adjoint) {  // C-side chunk of the U units: contiguous rows u0*C ..
    stage_rows(vs, in + static_cast<size_t>(t.u0) * a.C * a.k + t.k0, U * a.C, t.kc, a.k, ld, full, lane, a.bulk, 2);
  } else {           // R-side chunks, same segment structure as the blocks
    for (uint32_t s = 0; s < t.segs; ++s)
      stage_rows(vs + static_cast<size_t>(s) * t.seg_blocks * a.R * ld,
                 in + static_cast<size_t>(t.seg0 + s * t.seg_step) * a.R * a.k + t.k0, t.seg_blocks * a.R, t.kc,
                 a.k, ld, full, lane, a.bulk, 2 + s);
  }
}

template <typename E>
__device__ __forceinline__ void produce_tile(const LevelArgs& a, uint32_t tile, E* st, uint64_t* full, int lane,
                                             uint64_t pol) {
  const TileGeo t = tile_geo(a, tile);
  const uint32_t blk = a.R * a.C;
  if (a.bulk) {
    produce_factors<E>(a, t, st, full, lane, pol);
  } else {
    const E* fac = static_cast<const E*>(a.fac);
    for (uint32_t s = 0; s < t.segs; ++s) {
      const E* src = fac + static_cast<size_t>(t.seg0 + s * t.seg_step) * blk;
      E* dst = st + static_cast<size_t>(s) * t.seg_blocks * blk;
      for (uint32_t i = lane; i < t.seg_blocks * blk; i += 32) dst[i] = src[i];
    }
  }
  produce_vectors<E>(a, t, st, full, lane);
  if (!a.bulk) {
    __syncwarp();
    if (lane == 0) mbar_arrive(full);
  }
}

// Eight independent accumulation chains (even/odd term x {rr, ii, ri, ir}).
template <typename E>
struct Acc8 {
  using Rl = typename Cx<E>::R;
  Rl rr[2] = {0, 0}, ii[2] = {0, 0}, ri[2] = {0, 0}, ir[2] = {0, 0};
  __device__ __forceinline__ void mac(int h, const E a, const E b) {  // += a b
    rr[h] = fma(a.x, b.x, rr[h]);
    ii[h] = fma(a.y, b.y, ii[h]);
    ri[h] = fma(a.x, b.y, ri[h]);
    ir[h] = fma(a.y, b.x, ir[h]);
  }
  __device__ __forceinline__ E sum() const {  // a b
    return Cx<E>::make((rr[0] - ii[0]) + (rr[1] - ii[1]), (ri[0] + ir[0]) + (ri[1] + ir[1]));
  }
  __device__ __forceinline__ E sum_conj() const {  // conj(a) b
    return Cx<E>::make((rr[0] + ii[0]) + (rr[1] + ii[1]), (ri[0] - ir[0]) + (ri[1] - ir[1]));
  }
};

template <typename E, bool PUSH>
__device__ __forceinline__ void consume_tile(const LevelArgs& a, const PeerArgs& pa, uint32_t tile, const E* st, int ct, int nct) {
  using Rl = typename Cx<E>::R;
  const TileGeo t = tile_geo(a, tile);
  const uint32_t blk = a.R * a.C;
  const uint32_t U = 1u << a.lgU;
  const uint32_t Pe_mask = (1u << t.lgPe) - 1;
  const E* fs = st;
  const E* vs = st + static_cast<size_t>(a.nt) * U * blk;
  E* out = static_cast<E*>(a.out);
  const uint32_t kc = t.kc;
  const uint32_t P_mask = (1u << a.lgP) - 1;
  if (!a.adjoint) {
    const uint32_t n_out = U * a.nt * a.R * kc;
    for (uint32_t o = ct; o < n_out; o += nct) {
      uint32_t kk = 0, rest = o;
      if (kc > 1) {
        kk = o % kc;
        rest = o / kc;
      }
      const uint32_t rho = rest % a.R;
      rest /= a.R;
      const uint32_t tt = rest % a.nt;
      const uint32_t ul = rest / a.nt;
      const uint32_t slot = ((((ul >> t.lgPe) * a.nt) + tt) << t.lgPe) + (ul & Pe_mask);
      const E* arow = fs + (static_cast<size_t>(slot) * a.R + rho) * a.C;
      const E* x = vs + static_cast<size_t>(ul) * a.C * kc + kk;
      Acc8<E> acc;
      // kc == 1: lanes walk rows of one block — rotate the start column so a
      // quarter-warp touches 8 distinct 16-byte bank groups.
      uint32_t c = kc == 1 ? rho % a.C : 0;
      uint32_t j = 0;
      for (; j + 1 < a.C; j += 2) {
        acc.mac(0, arow[c], x[static_cast<size_t>(c) * kc]);
        if (++c == a.C) c = 0;
        acc.mac(1, arow[c], x[static_cast<size_t>(c) * kc]);
        if (++c == a.C) c = 0;
      }
      if (j < a.C) acc.mac(0, arow[c], x[static_cast<size_t>(c) * kc]);
      const uint32_t u = t.u0 + ul;
      const uint32_t q = ((((u >> a.lgP) * a.ntot) + t.t0 + tt) << a.lgP) + (u & P_mask);
      out[(static_cast<size_t>(q) * a.R + rho) * a.k + t.k0 + kk] = acc.sum();
    }
  } else {
    const uint32_t n_out = U * a.C * kc;
    for (uint32_t o = ct; o < n_out; o += nct) {
      uint32_t kk = 0, rest = o;
      if (kc > 1) {
        kk = o % kc;
        rest = o / kc;
      }
      const uint32_t c = rest % a.C;
      const uint32_t ul = rest / a.C;
      // destination (and, with the fused middle factor, its weight) first: the weight's
      // global load then overlaps the dot product instead of trailing it
      Rl w;
      E* orow = remap_row<E, PUSH>(a, pa, static_cast<size_t>(t.u0 + ul) * a.C + c, &w);
      const uint32_t base = (((ul >> t.lgPe) * a.nt) << t.lgPe) + (ul & Pe_mask);
      Acc8<E> acc;
      for (uint32_t tt = 0; tt < a.nt; ++tt) {
        const uint32_t row0 = (base + (tt << t.lgPe)) * a.R;
        const E* acol = fs + static_cast<size_t>(row0) * a.C + c;
        const E* y = vs + static_cast<size_t>(row0) * kc + kk;
        uint32_t rho = 0;
        for (; rho + 1 < a.R; rho += 2) {
          acc.mac(0, acol[static_cast<size_t>(rho) * a.C], y[static_cast<size_t>(rho) * kc]);
          acc.mac(1, acol[static_cast<size_t>(rho + 1) * a.C], y[static_cast<size_t>(rho + 1) * kc]);
        }
        if (rho < a.R) acc.mac(0, acol[static_cast<size_t>(rho) * a.C], y[static_cast<size_t>(rho) * kc]);
      }
      const E v = acc.sum_conj();
      E& o_ = orow[t.k0 + kk];
      // explicit branch: a select would let the compiler load o_ on every store
      if (a.accumulate)
        o_ = Cx<E>::make(o_.x + w * v.x, o_.y + w * v.y);
      else
        o_ = Cx<E>::make(w * v.x, w * v.y);
    }
  }
}

// Many-RHS consumer (k >= 8): each unit is a small complex GEMM
//   forward  Y (nt R x kc) = A (nt R x C) X (C x kc)
//   adjoint  X (C x kc)    = A^H (C x nt R) Y (nt R x kc)
// A warp owns (32/LC)*TM output rows x LC*TN right-hand sides; lane (lr, lc)
// holds a TM x TN register tile whose TN columns are strided by LC, so each
// operand load of the warp is a contiguous, bank-conflict-free span and the A
// operand is (nearly) a broadcast. Per inner step: TM + TN shared loads feed
// 4*TM*TN FP64 FMAs — FMA-pipe bound, not shared-memory bound.
template <typename E, int TM, int TN, int LC, bool PUSH>
__device__ __forceinline__ void consume_tile_mrhs(const LevelArgs& a, const PeerArgs& pa, uint32_t tile, const E* st, int warp, int lane,
                                                  int nwarps) {
  using Rl = typename Cx<E>::R;
  constexpr int LR = 32 / LC;
  const TileGeo t = tile_geo(a, tile);
  const uint32_t blk = a.R * a.C;
  const uint32_t U = 1u << a.lgU;
  const uint32_t Pe_mask = (1u << t.lgPe) - 1;
  const E* fs = st;
  const E* vs = st + static_cast<size_t>(a.nt) * U * blk;
  E* out = static_cast<E*>(a.out);
  const uint32_t kc = t.kc;
  const uint32_t P_mask = (1u << a.lgP) - 1;
  const uint32_t m_out = a.adjoint ? a.C : a.nt * a.R;
  const uint32_t nrg = (m_out + LR * TM - 1) / (LR * TM), ncg = (kc + LC * TN - 1) / (LC * TN);
  const uint32_t items = U * nrg * ncg;
  const uint32_t lr = lane / LC, lc = lane % LC;
  for (uint32_t it = warp; it < items; it += nwarps) {
    const uint32_t cg = it % ncg;
    const uint32_t rest = it / ncg;
    const uint32_t rg = rest % nrg, ul = rest / nrg;
    // rows of this lane: rb + lr + LR*i (interleaved, so the LR row groups of a warp read
    // adjacent A columns / rows and land in different banks)
    const uint32_t col0 = cg * LC * TN + lc, rb = rg * LR * TM + lr;
    const uint32_t base = (((ul >> t.lgPe) * a.nt) << t.lgPe) + (ul & Pe_mask);
    bool colok[TN];
#pragma unroll
    for (int j = 0; j < TN; ++j) colok[j] = col0 + j * LC < kc;
    const bool colfull = (kc % (LC * TN)) == 0;
    Rl re[TM][TN], im[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) re[i][j] = im[i][j] = 0;
    if (!a.adjoint) {
      // output row o = tt*R + rho of unit ul reads factor row (slot(ul,tt)*R + rho)
      const E* arow[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const uint32_t o = min(rb + LR * i, m_out - 1);
        const uint32_t tt = o / a.R, rho = o - tt * a.R;
        arow[i] = fs + (static_cast<size_t>(base + (tt << t.lgPe)) * a.R + rho) * a.C;
      }
      const E* x = vs + static_cast<size_t>(ul) * a.C * kc + col0;
      const uint32_t ce = a.dbg_nomath ? 0 : a.C;
      if (colfull) {  // every column of the warp tile in range: no predicates, pointer steps
        const E* xp = x;
#pragma unroll 4
        for (uint32_t c = 0; c < ce; ++c, xp += kc) {
          E xv[TN];
#pragma unroll
          for (int j = 0; j < TN; ++j) xv[j] = xp[j * LC];
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const E av = arow[i][c];
#pragma unroll
            for (int j = 0; j < TN; ++j) {
              re[i][j] = fma(av.x, xv[j].x, re[i][j]);
              re[i][j] = fma(-av.y, xv[j].y, re[i][j]);
              im[i][j] = fma(av.x, xv[j].y, im[i][j]);
              im[i][j] = fma(av.y, xv[j].x, im[i][j]);
            }
          }
        }
      } else {
        for (uint32_t c = 0; c < ce; ++c) {
          E xv[TN];
#pragma unroll
          for (int j = 0; j < TN; ++j) xv[j] = colok[j] ? x[static_cast<size_t>(c) * kc + j * LC] : Cx<E>::make(0, 0);
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const E av = arow[i][c];
#pragma unroll
            for (int j = 0; j < TN; ++j) {
              re[i][j] = fma(av.x, xv[j].x, re[i][j]);
              re[i][j] = fma(-av.y, xv[j].y, re[i][j]);
              im[i][j] = fma(av.x, xv[j].y, im[i][j]);
              im[i][j] = fma(av.y, xv[j].x, im[i][j]);
            }
          }
        }
      }
      const uint32_t u = t.u0 + ul;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const uint32_t o = rb + LR * i;
        if (o >= m_out) break;
        const uint32_t tt = o / a.R, rho = o - tt * a.R;
        const uint32_t q = ((((u >> a.lgP) * a.ntot) + t.t0 + tt) << a.lgP) + (u & P_mask);
        E* dst = out + (static_cast<size_t>(q) * a.R + rho) * a.k + t.k0 + col0;
#pragma unroll
        for (int j = 0; j < TN; ++j)
          if (colok[j]) dst[j * LC] = Cx<E>::make(re[i][j], im[i][j]);
      }
    } else {
      uint32_t cidx[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) cidx[i] = min(rb + LR * i, m_out - 1);
      for (uint32_t tt = 0, te = a.dbg_nomath ? 0 : a.nt; tt < te && colfull; ++tt) {
        // every column in range: no predicates, pointer steps per block row
        const uint32_t r0 = (base + (tt << t.lgPe)) * a.R;
        const E* yp = vs + static_cast<size_t>(r0) * kc + col0;
        const E* ap = fs + static_cast<size_t>(r0) * a.C;
#pragma unroll 2
        for (uint32_t rho = 0; rho < a.R; ++rho, yp += kc, ap += a.C) {
          E yv[TN];
#pragma unroll
          for (int j = 0; j < TN; ++j) yv[j] = yp[j * LC];
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const E av = ap[cidx[i]];
#pragma unroll
            for (int j = 0; j < TN; ++j) {  // conj(av) * yv
              re[i][j] = fma(av.x, yv[j].x, re[i][j]);
              re[i][j] = fma(av.y, yv[j].y, re[i][j]);
              im[i][j] = fma(av.x, yv[j].y, im[i][j]);
              im[i][j] = fma(-av.y, yv[j].x, im[i][j]);
            }
          }
        }
      }
      for (uint32_t tt = 0, te = a.dbg_nomath ? 0 : a.nt; tt < te && !colfull; ++tt) {
        const uint32_t r0 = (base + (tt << t.lgPe)) * a.R;
        for (uint32_t rho = 0; rho < a.R; ++rho) {
          const size_t row = static_cast<size_t>(r0 + rho);
          const E* y = vs + row * kc + col0;
          E yv[TN];
#pragma unroll
          for (int j = 0; j < TN; ++j) yv[j] = colok[j] ? y[j * LC] : Cx<E>::make(0, 0);
          const E* acol = fs + row * a.C;
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const E av = acol[min(rb + LR * i, m_out - 1)];
#pragma unroll
            for (int j = 0; j < TN; ++j) {  // conj(av) * yv
              re[i][j] = fma(av.x, yv[j].x, re[i][j]);
              re[i][j] = fma(av.y, yv[j].y, re[i][j]);
              im[i][j] = fma(av.x, yv[j].y, im[i][j]);
              im[i][j] = fma(-av.y, yv[j].x, im[i][j]);
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const uint32_t c = rb + LR * i;
        if (c >= m_out) break;
        Rl w;
        E* dst = remap_row<E, PUSH>(a, pa, static_cast<size_t>(t.u0 + ul) * a.C + c, &w) + t.k0 + col0;
#pragma unroll
        for (int j = 0; j < TN; ++j)
          if (colok[j]) {
            const E v = Cx<E>::make(w * re[i][j], w * im[i][j]);
            if (a.accumulate)
              dst[j * LC] = Cx<E>::make(dst[j * LC].x + v.x, dst[j * LC].y + v.y);
            else
              dst[j * LC] = v;
          }
      }
    }
  }
}

// ---------------------------------------------------------------- FP64 tensor cores
// mma.sync m8n8k4 f64 (DMMA): A fragment A[lane/4][lane%4], B fragment
// B[lane%4][lane/4], C/D fragment C[lane/4][2(lane%4) + q] (layout confirmed on
// B200 by tools/dmma_layout.cu).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Many-RHS consumer on the FP64 tensor pipe (complex128). Each unit is the
// complex GEMM of consume_tile_mrhs, split into 4 real DMMAs per k-step
// (re += Ar Xr - Ai Xi, im += Ar Xi + Ai Xr); a warp owns MT x NT 8x8 tiles.
//
// GAUSS: the 3-multiplication complex product (T1 = Ar Xr, T2 = Ai Xi, T3 = (Ar + Ai)
// (Xr + Xi); re = T1 - T2, im = T3 - T1 - T2): 3 DMMAs per complex k-step instead of
// 4, and every accumulator is updated once per k-step (no back-to-back dependent
// DMMAs). The operand sums are two DADDs on the otherwise idle FP64 pipe; the
// rounding stays O(eps |A| |X|) per term.
template <int MT, int NT, bool PUSH, bool GAUSS>
__device__ __forceinline__ void consume_tile_dmma(const LevelArgs& a, const PeerArgs& pa, uint32_t tile, const double2* st, int warp,
                                                  int lane, int nwarps, double2* ob) {
  const TileGeo t = tile_geo(a, tile);
  const uint32_t U = 1u << a.lgU;
  const uint32_t Pe_mask = (1u << t.lgPe) - 1;
  const double2* fs = st;
  const double2* vs = st + static_cast<size_t>(a.nt) * U * a.R * a.fld;
  double2* out = static_cast<double2*>(a.out);
  const uint32_t kc = t.kc;
  const uint32_t fld = a.fld, vld = a.vld ? a.vld : kc;
  const uint32_t P_mask = (1u << a.lgP) - 1;
  const uint32_t m_out = a.adjoint ? a.C : a.nt * a.R;
  const uint32_t kdim = a.dbg_nomath ? 0 : a.adjoint ? a.nt * a.R : a.C;
  const uint32_t nmt = (m_out + MT * 8 - 1) / (MT * 8), nnt = (kc + NT * 8 - 1) / (NT * 8);
  const uint32_t items = U * nmt * nnt;
  const uint32_t lr = lane >> 2, lk = lane & 3;
  // in place (MRHS = 3): one round, every consumer warp (items <= warps, host-checked)
  // meets the barrier that ends all reads of the stage before any output overwrites it
  const bool inplace = ob != nullptr && a.inplace;
  for (uint32_t it = warp; inplace ? it == static_cast<uint32_t>(warp) : it < items; it += nwarps) {
    const bool act = it < items;
    const uint32_t ntile = it % nnt;
    const uint32_t rest = it / nnt;
    const uint32_t mt = rest % nmt, ul = rest / nmt;
    const uint32_t m0 = mt * MT * 8, n0 = ntile * NT * 8;
    const uint32_t base = (((ul >> t.lgPe) * a.nt) << t.lgPe) + (ul & Pe_mask);
    // GAUSS: cr = T1, ci = T2, cs = T3; else cr = re, ci = im (cs unused)
    double cr[MT][NT][2], ci[MT][NT][2], cs[GAUSS ? MT : 1][GAUSS ? NT : 1][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0;
    if constexpr (GAUSS) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) cs[i][j][0] = cs[i][j][1] = 0;
    }
    // forward: the A rows this lane reads are fixed (m = m0 + 8i + lane/4)
    uint32_t arow[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const uint32_t m = min(m0 + 8 * i + lr, m_out - 1);
      const uint32_t tt = m / a.R, rho = m - tt * a.R;
      arow[i] = (base + (tt << t.lgPe)) * a.R + rho;
    }
    const uint32_t kd = act ? kdim : 0;
    // one complex k-step from fragments (ar + i ai of A, br + i bi of X)
    auto mma_step = [&](const double (&ar)[MT], const double (&ai)[MT], const double (&br)[NT],
                        const double (&bi)[NT]) {
      if constexpr (GAUSS) {
        double as[MT], bs[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) as[i] = ar[i] + ai[i];
#pragma unroll
        for (int j = 0; j < NT; ++j) bs[j] = br[j] + bi[j];
        // T1, T2 of every tile first: the operand sums (DADD, which waits for the FP64
        // datapath behind queued DMMAs) are not needed until 2 MT NT DMMAs later
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            dmma(cr[i][j][0], cr[i][j][1], ar[i], br[j]);
            dmma(ci[i][j][0], ci[i][j][1], ai[i], bi[j]);
          }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(cs[i][j][0], cs[i][j][1], as[i], bs[j]);
      } else {
        double nai[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) nai[i] = neg(ai[i]);
        // two passes over the tiles: the two products accumulated into one register pair
        // are 2 MT NT instructions apart, not back to back
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            dmma(cr[i][j][0], cr[i][j][1], ar[i], br[j]);
            dmma(ci[i][j][0], ci[i][j][1], ar[i], bi[j]);
          }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            dmma(cr[i][j][0], cr[i][j][1], nai[i], bi[j]);
            dmma(ci[i][j][0], ci[i][j][1], ai[i], br[j]);
          }
      }
    };
    // Full tiles (every fragment in range, k steps inside one block for the adjoint):
    // no predicates, pointer increments only (cfg2: m_out = 32, kc = 128, k = 32).
    const bool full = (m_out % (8 * MT)) == 0 && (kc % (8 * NT)) == 0 && (a.R % 4) == 0 && (a.C % 4) == 0;
    if (full && !a.adjoint) {
      const double2* ap[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) ap[i] = fs + static_cast<size_t>(arow[i]) * fld + lk;
      const double2* bp = vs + (static_cast<size_t>(ul) * a.C + lk) * vld + n0 + lr;
      const size_t bstep = 4 * static_cast<size_t>(vld);
      for (uint32_t k0 = 0; k0 < kd; k0 += 4, bp += bstep) {
        double ar[MT], ai[MT], br[NT], bi[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const double2 v = ap[i][k0];
          ar[i] = v.x;
          ai[i] = v.y;
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const double2 v = bp[8 * j];
          br[j] = v.x;
          bi[j] = v.y;
        }
        mma_step(ar, ai, br, bi);
      }
    } else if (full) {  // adjoint: k runs over block rows (t, rho)
      const uint32_t ntk = kd ? a.nt : 0;
      for (uint32_t tt = 0; tt < ntk; ++tt) {
        const size_t row0 = static_cast<size_t>(base + (tt << t.lgPe)) * a.R + lk;
        const double2* ap = fs + row0 * fld + m0 + lr;
        const double2* bp = vs + row0 * vld + n0 + lr;
        const size_t astep = 4 * static_cast<size_t>(fld), bstep = 4 * static_cast<size_t>(vld);
        for (uint32_t rho0 = 0; rho0 < a.R; rho0 += 4, ap += astep, bp += bstep) {
          double ar[MT], ai[MT], br[NT], bi[NT];
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const double2 v = ap[8 * i];
            ar[i] = v.x;
            ai[i] = neg(v.y);  // A^H
          }
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const double2 v = bp[8 * j];
            br[j] = v.x;
            bi[j] = v.y;
          }
          mma_step(ar, ai, br, bi);
        }
      }
    } else {
      for (uint32_t k0 = 0; k0 < kd; k0 += 4) {
        const uint32_t kk = k0 + lk;
        const bool kok = kk < kdim;
        // adjoint: the k index runs over block rows j = (t, rho)
        uint32_t jrow = 0;
        if (a.adjoint) {
          const uint32_t kj = kok ? kk : 0;
          const uint32_t tt = (kj >= a.R) + (kj >= 2 * a.R) + (kj >= 3 * a.R);  // nt <= 4: no division
          jrow = (base + (tt << t.lgPe)) * a.R + (kj - tt * a.R);
        }
        double ar[MT], ai[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const uint32_t m = m0 + 8 * i + lr;
          double2 v = make_double2(0, 0);
          if (kok && m < m_out) {
            if (!a.adjoint) {
              v = fs[static_cast<size_t>(arow[i]) * fld + kk];
            } else {
              v = fs[static_cast<size_t>(jrow) * fld + m];
              v.y = neg(v.y);  // A^H
            }
          }
          ar[i] = v.x;
          ai[i] = v.y;
        }
        double br[NT], bi[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const uint32_t n = n0 + 8 * j + lr;
          double2 v = make_double2(0, 0);
          if (kok && n < kc) {
            const size_t row = a.adjoint ? jrow : static_cast<size_t>(ul) * a.C + kk;
            v = vs[row * vld + n];
          }
          br[j] = v.x;
          bi[j] = v.y;
        }
        mma_step(ar, ai, br, bi);
      }
    }
    if constexpr (GAUSS) {  // (T1, T2, T3) -> (re, im)
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double t1 = cr[i][j][q], t2 = ci[i][j][q];
            cr[i][j][q] = t1 - t2;
            ci[i][j][q] = cs[i][j][q] - t1 - t2;
          }
    }
    // epilogue: element (m0 + 8i + lane/4, n0 + 8j + 2(lane%4) + q)
    if (inplace) asm volatile("bar.sync 1, %0;" ::"r"(nwarps * 32) : "memory");
    if (ob && !act) continue;
    if (ob) {  // into the shared-memory output tile (row ul * m_out + m); TMA stores it
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const uint32_t m = m0 + 8 * i + lr;
        if (m >= m_out) continue;
        double w = 1;
        if (a.adjoint && a.remap) remap_row<double2, false>(a, pa, static_cast<size_t>(t.u0 + ul) * a.C + m, &w);
        double2* orow = ob + static_cast<size_t>(ul * m_out + m) * a.old;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint32_t n = n0 + 8 * j + 2 * lk + q;
            if (n < kc) orow[n] = make_double2(w * cr[i][j][q], w * ci[i][j][q]);
          }
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const uint32_t m = m0 + 8 * i + lr;
      if (m >= m_out) continue;
      double2* orow;
      double w = 1;
      if (!a.adjoint) {
        const uint32_t u = t.u0 + ul;
        const uint32_t tt = m / a.R, rho = m - tt * a.R;
        const uint32_t q = ((((u >> a.lgP) * a.ntot) + t.t0 + tt) << a.lgP) + (u & P_mask);
        orow = out + (static_cast<size_t>(q) * a.R + rho) * a.k + t.k0;
      } else if (a.remap >= 3) {
        orow = remap_row<double2, PUSH>(a, pa, static_cast<size_t>(t.u0 + ul) * a.C + m, &w) + t.k0;
      } else {
        size_t e = static_cast<size_t>(t.u0 + ul) * a.C + m;
        if (a.remap != 0) {
          const uint32_t mr = a.m * a.r;
          const uint32_t e32 = static_cast<uint32_t>(e), ia = e32 / mr;
          const uint32_t rem = e32 - ia * mr;
          const uint32_t ib = rem / a.r, rho = rem - ib * a.r;
          const size_t dst = (static_cast<size_t>(ib) * a.m + ia) * a.r + rho;
          const double* W = static_cast<const double*>(a.mid_w);
          w = a.remap == 1 ? W[dst] : W[(static_cast<size_t>(ia) * a.m + ib) * a.r + rho];
          e = dst;
        }
        orow = out + e * a.k + t.k0;
      }
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint32_t n = n0 + 8 * j + 2 * lk + q;
          if (n >= kc) continue;
          const double2 v = make_double2(w * cr[i][j][q], w * ci[i][j][q]);
          double2& o = orow[n];
          if (a.adjoint && a.accumulate)
            o = make_double2(o.x + v.x, o.y + v.y);
          else
            o = v;
        }
    }
  }
}

// Register-tile shapes of the many-RHS consumer, picked by right-hand sides per tile.
// DT >= 0: a complex128 instantiation with only the 3-multiplication DMMA consumer of
// warp tile DT (0 = 2 x 4, 1 = 2 x 2, 2 = 1 x 2), so the register allocation is that
// variant's alone; DT = -1 dispatches at run time (4-product DMMA, FFMA, complex64).
template <typename E, bool PUSH, int DT = -1>
__device__ __forceinline__ void consume_tile_mrhs_any(const LevelArgs& a, const PeerArgs& pa, uint32_t tile, const E* st, int warp,
                                                      int lane, int nwarps, E* ob = nullptr) {
  if constexpr (DT >= 0 && std::is_same<E, double2>::value) {
    constexpr int MT = DT == 2 ? 1 : 2, NT = DT == 0 ? 4 : 2;
    consume_tile_dmma<MT, NT, PUSH, true>(a, pa, tile, st, warp, lane, nwarps, ob);
    return;
  }
  if constexpr (std::is_same<E, double2>::value) {
    if (a.use_dmma == 2) {  // complex128: the FP64 tensor pipe, 3-multiplication products
      if (a.dtile == 0)
        consume_tile_dmma<2, 4, PUSH, true>(a, pa, tile, st, warp, lane, nwarps, ob);
      else if (a.dtile == 1)
        consume_tile_dmma<2, 2, PUSH, true>(a, pa, tile, st, warp, lane, nwarps, ob);
      else
        consume_tile_dmma<1, 2, PUSH, true>(a, pa, tile, st, warp, lane, nwarps, ob);
      return;
    }
    if (a.use_dmma) {  // complex128: the FP64 tensor pipe, 4 real products per complex step
      if (a.dtile == 0)
        consume_tile_dmma<2, 4, PUSH, false>(a, pa, tile, st, warp, lane, nwarps, ob);
      else if (a.dtile == 1)
        consume_tile_dmma<2, 2, PUSH, false>(a, pa, tile, st, warp, lane, nwarps, ob);
      else
        consume_tile_dmma<1, 2, PUSH, false>(a, pa, tile, st, warp, lane, nwarps, ob);
      return;
    }
  }
  if (a.kt >= 256 && !PUSH)
    consume_tile_mrhs<E, 4, 8, 32, PUSH>(a, pa, tile, st, warp, lane, nwarps);
  else if (a.kt >= 128)
    consume_tile_mrhs<E, 4, 4, 32, PUSH>(a, pa, tile, st, warp, lane, nwarps);
  else if (a.kt >= 64)
    consume_tile_mrhs<E, 8, 2, 32, PUSH>(a, pa, tile, st, warp, lane, nwarps);
  else if (a.kt >= 32)
    consume_tile_mrhs<E, 16, 1, 32, PUSH>(a, pa, tile, st, warp, lane, nwarps);
  else if (a.kt >= 16 && (a.adjoint ? a.C : a.nt * a.R) > 64)  // wide quadtree blocks: more, shorter items
    consume_tile_mrhs<E, 4, 1, 16, PUSH>(a, pa, tile, st, warp, lane, nwarps);
  else if (a.kt >= 16)
    consume_tile_mrhs<E, 8, 1, 16, PUSH>(a, pa, tile, st, warp, lane, nwarps);
  else
    consume_tile_mrhs<E, 4, 1, 8, PUSH>(a, pa, tile, st, warp, lane, nwarps);
}

// MRHS = 3: the output tile of `tile` (rows ul * m_out + m in shared memory, stride
// a.old) to its global rows, one TMA bulk store per row, issued by the lanes of
// one warp; each lane commits its own bulk group.
template <typename E>
__device__ __forceinline__ void store_tile_rows(const LevelArgs& a, const PeerArgs& pa, uint32_t tile, const E* ob, int lane) {
  const TileGeo t = tile_geo(a, tile);
  const uint32_t U = 1u << a.lgU;
  const uint32_t m_out = a.adjoint ? a.C : a.nt * a.R;
  const uint32_t P_mask = (1u << a.lgP) - 1;
  E* out = static_cast<E*>(a.out);
  for (uint32_t row = lane; row < U * m_out; row += 32) {
    const uint32_t ul = row / m_out, m = row - ul * m_out;
    E* dst;
    if (!a.adjoint) {
      const uint32_t u = t.u0 + ul;
      const uint32_t tt = m / a.R, rho = m - tt * a.R;
      const uint32_t q = ((((u >> a.lgP) * a.ntot) + t.t0 + tt) << a.lgP) + (u & P_mask);
      dst = out + (static_cast<size_t>(q) * a.R + rho) * a.k + t.k0;
    } else {
      typename Cx<E>::R w;
      dst = remap_row<E, false>(a, pa, static_cast<size_t>(t.u0 + ul) * a.C + m, &w) + t.k0;
    }
    bulk_s2g(dst, ob + static_cast<size_t>(row) * a.old, t.kc * static_cast<uint32_t>(sizeof(E)));
  }
  bulk_commit();
}

// MRHS = 0: streaming consumer (one output per thread); MRHS = 1: register-tiled GEMM
// consumer; MRHS = 3: the DMMA consumer writing its outputs over the tile's consumed
// vector rows, which the producer warp stores with TMA bulk copies before refilling the
// stage (the consumer warps issue no global stores).
template <typename E, int STAGES, int NCW, int MINB, int MRHS, bool PUSH, int DT = -1>
__global__ void __launch_bounds__((NCW + 1) * 32, MINB) level_kernel(const LevelArgs a, const PeerArgs pa) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  // STAGES = 0: the depth is a launch argument (a.stages <= 8; 16 barriers fit the 128-byte header)
  const uint32_t S = STAGES ? STAGES : a.stages;
  uint64_t* empty = full + (STAGES ? STAGES : 8);
  E* stage0 = reinterpret_cast<E*>(smem_raw + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // programmatic dependent launch: let the next level's CTAs launch as ours retire,
  // and wait for the previous level to finish and flush before touching its output
  // (our input) or its input (our output buffer); only constant factor blocks are
  // fetched before the wait. No-ops without the programmatic-serialization attribute.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == NCW) {
    const uint64_t pol = policy_evict_first();
    // the first S tiles' factor blocks are constant: start them before the wait
    uint32_t pre = 0;
    if (a.bulk)
      for (uint32_t tile = blockIdx.x; tile < a.ntiles && pre < S; tile += gridDim.x, ++pre)
        produce_factors<E>(a, tile_geo(a, tile), stage0 + static_cast<size_t>(pre) * a.stage_elems, &full[pre], lane,
                           pol);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
      const uint32_t s = it % S;
      E* st = stage0 + static_cast<size_t>(s) * a.stage_elems;
      if (it < pre) {
        produce_vectors<E>(a, tile_geo(a, tile), st, &full[s], lane);
        continue;
      }
      if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
      if constexpr (MRHS == 3) {
        // tile it - S left its outputs in this stage's vector rows: store them (TMA), and
        // reuse the stage once the engine has read them
        if (it >= S) {
          const uint32_t prev = tile - S * gridDim.x;
          store_tile_rows<E>(a, pa, prev, st + static_cast<size_t>(a.nt) * (1u << a.lgU) * a.R * a.fld, lane);
          bulk_wait_read<0>();
        }
      }
      if (a.dbg_noload) {
        if (lane == 0) mbar_arrive(&full[s]);
        continue;
      }
      produce_tile<E>(a, tile, st, &full[s], lane, pol);
    }
    if constexpr (MRHS == 3) {  // the last S tiles' outputs
      const uint32_t first = it > S ? it - S : 0;
      for (uint32_t j = first; j < it; ++j) {
        const uint32_t s = j % S;
        mbar_wait(&empty[s], (j / S) & 1);
        store_tile_rows<E>(a, pa, blockIdx.x + j * gridDim.x,
                           stage0 + static_cast<size_t>(s) * a.stage_elems +
                               static_cast<size_t>(a.nt) * (1u << a.lgU) * a.R * a.fld,
                           lane);
      }
      bulk_wait_all();
    }
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
      const uint32_t s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      if constexpr (MRHS == 3) {
        E* stg = stage0 + static_cast<size_t>(s) * a.stage_elems;
        consume_tile_mrhs_any<E, PUSH, DT>(a, pa, tile, stg, warp, lane, NCW,
                                           stg + static_cast<size_t>(a.nt) * (1u << a.lgU) * a.R * a.fld);
        fence_proxy_async_smem();  // the outputs (generic proxy) are read by the TMA store (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        continue;
      } else if (MRHS) {
        consume_tile_mrhs_any<E, PUSH, DT>(a, pa, tile, stage0 + static_cast<size_t>(s) * a.stage_elems, warp, lane,
                                           NCW);
      } else {
        consume_tile<E, PUSH>(a, pa, tile, stage0 + static_cast<size_t>(s) * a.stage_elems, threadIdx.x, NCW * 32);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

}  // namespace bfly
