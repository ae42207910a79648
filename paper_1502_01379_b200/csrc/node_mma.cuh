// node_mma.cuh — the many-RHS node kernel with staged factor groups.
//
// Same decomposition as node_kernel.cuh (one CTA per middle node and chunk of
// right-hand sides, the node vector resident in shared memory), for chains whose
// per-node factor slabs do not all fit in shared memory (BASELINE config 1: 131 KB
// per level and node). Each step's blocks are split into groups; the TMA bulk
// engine copies group g + 2 into the half of a two-half staging buffer that group
// g just released while the warps multiply group g + 1, so the DMMA operands come
// from shared memory and the factor stream overlaps the math. Block rows land with
// a padded stride (lda) chosen on the host so a DMMA fragment's 8 lanes per phase
// hit distinct banks.
#pragma once

#include "node_kernel.cuh"

namespace bfly {

struct NodeStage {
  uint32_t half_elems;     // complex values per staging half
  uint32_t gl_dn, gu, gl_up;   // leaves / units / leaves per group (LeafDown, levels, LeafUp)
  uint32_t lda_dn, lda_up, lda_ldn, lda_lup;   // padded row strides (levels down/up, leaves down/up)
};

// A of the staged group (local gemm index ql).
template <int KIND>
__device__ __forceinline__ double2 stg_a(const NodeArgs& a, const double2* S, uint32_t lda, int ql, int m, int seg,
                                         int kk) {
  const uint32_t r = a.r;
  if constexpr (KIND == kLeafDown) {
    const double2 v = S[(ql * a.n0 + kk) * lda + m];
    return make_double2(v.x, -v.y);
  } else if constexpr (KIND == kLevDown) {
    const double2 v = S[((ql * 2 + seg) * r + kk) * lda + m];
    return make_double2(v.x, -v.y);
  } else if constexpr (KIND == kLevUp) {
    return S[(ql * r + m) * lda + kk];
  } else {
    return S[(ql * a.n0 + m) * lda + kk];
  }
}

// Copy group rows into a staging half with 16-byte cp.async by every thread (one commit
// group per call): leaves [q0, q0 + cnt) of the node's leaf slab, or units [q0, q0 + cnt)
// of a level slab (both blocks t = 0, 1 of each unit), rows at the padded stride lda.
__device__ __forceinline__ void stg_issue(const NodeArgs& a, bool leaf, const double2* slab, uint32_t lgP, uint32_t q0,
                                          uint32_t cnt, double2* dst, uint32_t lda) {
  const uint32_t r = a.r;
  const uint32_t rows = leaf ? cnt * a.n0 : cnt * 2 * r;
  const uint32_t rl = leaf ? r : 2 * r;                 // complex values per row
  const uint32_t P = 1u << lgP;
  for (uint32_t e = threadIdx.x; e < rows * rl; e += blockDim.x) {
    const uint32_t row = e / rl, col = e - row * rl;
    const double2* src;
    if (leaf) {
      src = slab + (static_cast<size_t>(q0) * a.n0 + row) * r + col;
    } else {
      const uint32_t ul = row / (2 * r), rem = row - ul * 2 * r, t = rem / r, rho = rem - t * r;
      const uint32_t u = q0 + ul, g = u >> lgP, p = u & (P - 1);
      src = slab + ((static_cast<size_t>((g * 2 + t) * P + p)) * r + rho) * 2 * r + col;
    }
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + static_cast<size_t>(row) * lda + col)),
                 "l"(src)
                 : "memory");
  }
}

__device__ __forceinline__ void stg_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// One group of one step: items (gemm, m-tile, n-tile) of gemms [q0, q0 + gq), A staged.
template <int KIND, int STORE, int NT>
__device__ __forceinline__ void stg_group(const NodeArgs& a, const NodeCtx& c, const double2* S, uint32_t lda, int q0,
                                          int gq, int warp, int lane, int nwarps, double2 (*res)[2]) {
  int ngemm, M, nseg, klen;
  node_geom<KIND>(a, c, ngemm, M, nseg, klen);
  const int mtl = (M + 7) >> 3, ntl = (static_cast<int>(c.nc) + 8 * NT - 1) / (8 * NT);
  const int items = gq * mtl * ntl;
  const int lr = lane >> 2, lk = lane & 3;
  for (int it = warp; it < items; it += nwarps) {
    const int ql = it / (mtl * ntl), rest = it - ql * mtl * ntl;
    const int m0 = (rest / ntl) * 8, n0 = (rest % ntl) * (8 * NT);
    const int m = m0 + lr, q = q0 + ql;
    double t1[NT][2], t2[NT][2], t3[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) t1[j][0] = t1[j][1] = t2[j][0] = t2[j][1] = t3[j][0] = t3[j][1] = 0;
    for (int sg = 0; sg < nseg; ++sg) {
#pragma unroll 4
      for (int k0 = 0; k0 < klen; k0 += 4) {
        const int kk = k0 + lk;
        const bool kok = kk < klen;
        const double2 av = (kok && m < M) ? stg_a<KIND>(a, S, lda, ql, m, sg, kk) : make_double2(0, 0);
        const double as = av.x + av.y;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int n = n0 + 8 * j + lr;
          const double2 bv = (kok && n < static_cast<int>(c.nc)) ? node_x<KIND>(a, c, q, sg, kk, n)
                                                                 : make_double2(0, 0);
          node_dmma(t1[j][0], t1[j][1], av.x, bv.x);
          node_dmma(t2[j][0], t2[j][1], av.y, bv.y);
          node_dmma(t3[j][0], t3[j][1], as, bv.x + bv.y);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const double2 y = make_double2(t1[j][qq] - t2[j][qq], t3[j][qq] - t1[j][qq] - t2[j][qq]);
        if constexpr (STORE == kStoreDeferred) {
          res[j][qq] = y;          // at most one item per warp and group (host-checked)
        } else {
          const int n = n0 + 8 * j + 2 * lk + qq;
          if (m < M && n < static_cast<int>(c.nc)) node_store<KIND, STORE>(a, c, q, m, n, y);
        }
      }
  }
}

template <int KIND, int NT>
__device__ __forceinline__ void stg_deferred_store(const NodeArgs& a, const NodeCtx& c, int q0, int gq, int warp,
                                                   int lane, const double2 (*res)[2]) {
  int ngemm, M, nseg, klen;
  node_geom<KIND>(a, c, ngemm, M, nseg, klen);
  const int mtl = (M + 7) >> 3, ntl = (static_cast<int>(c.nc) + 8 * NT - 1) / (8 * NT);
  const int it = warp;
  if (it >= gq * mtl * ntl) return;
  const int lr = lane >> 2, lk = lane & 3;
  const int ql = it / (mtl * ntl), rest = it - ql * mtl * ntl;
  const int m = (rest / ntl) * 8 + lr, n0 = (rest % ntl) * (8 * NT);
  if (m >= M) return;
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int qq = 0; qq < 2; ++qq) {
      const int n = n0 + 8 * j + 2 * lk + qq;
      if (n < static_cast<int>(c.nc)) node_store<KIND, kStoreDeferred>(a, c, q0 + ql, m, n, res[j][qq]);
    }
}

// Group sequence of a half: down = LeafDown groups, then levels D-1 .. 0; up = levels
// 0 .. D-1, then LeafUp groups. Decodes running group index G into (step, first index).
struct StgSeq {
  uint32_t ng_leaf, ng_lev, D;
  bool up;
  __device__ __forceinline__ uint32_t total() const { return ng_leaf + D * ng_lev; }
  // step kind: 0 leaf, 1 level; li: level index; idx: group within the step
  __device__ __forceinline__ void decode(uint32_t G, int& leaf, uint32_t& li, uint32_t& idx) const {
    if (!up) {
      if (G < ng_leaf) { leaf = 1; li = 0; idx = G; return; }
      const uint32_t g = G - ng_leaf;
      leaf = 0; li = D - 1 - g / ng_lev; idx = g % ng_lev;
    } else {
      if (G < D * ng_lev) { leaf = 0; li = G / ng_lev; idx = G % ng_lev; return; }
      leaf = 1; li = 0; idx = G - D * ng_lev;
    }
  }
};

template <int UP, int NT, int MAXG>
__global__ void __launch_bounds__(512, 1) node_mma_kernel(const NodeArgs a, const NodeStage sg) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  NodeCtx c;
  c.node = blockIdx.x / a.nch;
  const uint32_t chunk = blockIdx.x - c.node * a.nch;
  c.c0 = chunk * a.kc;
  c.nc = min(a.kc, a.k - c.c0);
  c.NL = 1u << a.D;
  c.vs = reinterpret_cast<double2*>(smem_raw + 256);
  const uint32_t vbytes = ((c.NL * a.r * a.vld * static_cast<uint32_t>(sizeof(double2))) + 127u) & ~127u;
  double2* halves = reinterpret_cast<double2*>(smem_raw + 256 + vbytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const double2* leaf_g = a.leaf + static_cast<size_t>(c.node) * c.NL * a.n0 * a.r;
  const size_t lev_off = static_cast<size_t>(c.node) * c.NL * 2 * a.r * a.r;
  const uint32_t gl = UP ? sg.gl_up : sg.gl_dn;
  StgSeq seq{c.NL / gl, (c.NL / 2) / sg.gu, a.D, UP != 0};
  const uint32_t lda_lev = UP ? sg.lda_up : sg.lda_dn, lda_leaf = UP ? sg.lda_lup : sg.lda_ldn;
  // every call commits one cp.async group (empty past the end), so "all but the newest
  // group complete" (wait_group 1) always means the group about to be consumed has landed
  auto issue = [&](uint32_t G) {
    if (G < seq.total()) {
      int leaf;
      uint32_t li, idx;
      seq.decode(G, leaf, li, idx);
      double2* dst = halves + static_cast<size_t>(G & 1) * sg.half_elems;
      if (leaf)
        stg_issue(a, true, leaf_g, 0, idx * gl, gl, dst, lda_leaf);
      else
        stg_issue(a, false, a.lev[li] + lev_off, a.D - 1 - li, idx * sg.gu, sg.gu, dst, lda_lev);
    }
    stg_commit();
  };
  (void)bars;
  issue(0);   // factors are constant: stage them before waiting on the previous kernel
  issue(1);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  c.xin = a.in + static_cast<size_t>(c.node) * c.NL * a.n0 * a.k + c.c0;
  c.xld = a.k;
  uint32_t G = 0;
  auto wait_stage = [&](uint32_t g) -> const double2* {
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();      // every thread's copies of group g have landed
    return halves + static_cast<size_t>(g & 1) * sg.half_elems;
  };
  auto release = [&](uint32_t g) {
    __syncthreads();      // every warp is done with this half (and, for deferred steps, with its reads)
    issue(g + 2);
  };
  double2 res[MAXG][NT][2];
  if constexpr (!UP) {
    c.li = 0;
    c.lgP = 0;
    for (uint32_t i = 0; i < seq.ng_leaf; ++i, ++G) {
      const double2* S = wait_stage(G);
      stg_group<kLeafDown, kStoreNow, NT>(a, c, S, lda_leaf, static_cast<int>(i * gl), static_cast<int>(gl), warp,
                                          lane, nwarps, res[0]);
      release(G);
    }
    for (int li = static_cast<int>(a.D) - 1; li >= 0; --li) {
      c.li = static_cast<uint32_t>(li);
      c.lgP = a.D - 1 - c.li;
      if (li > 0) {
#pragma unroll
        for (int gi = 0; gi < MAXG; ++gi) {
          if (gi >= static_cast<int>(seq.ng_lev)) break;
          const double2* S = wait_stage(G);
          stg_group<kLevDown, kStoreDeferred, NT>(a, c, S, lda_lev, gi * static_cast<int>(sg.gu),
                                                  static_cast<int>(sg.gu), warp, lane, nwarps, res[gi]);
          release(G);
          ++G;
        }
#pragma unroll
        for (int gi = 0; gi < MAXG; ++gi) {
          if (gi >= static_cast<int>(seq.ng_lev)) break;
          stg_deferred_store<kLevDown, NT>(a, c, gi * static_cast<int>(sg.gu), static_cast<int>(sg.gu), warp, lane,
                                           res[gi]);
        }
        __syncthreads();
      } else {
        for (uint32_t gi = 0; gi < seq.ng_lev; ++gi, ++G) {
          const double2* S = wait_stage(G);
          stg_group<kLevDown, kStoreRemap, NT>(a, c, S, lda_lev, static_cast<int>(gi * sg.gu),
                                               static_cast<int>(sg.gu), warp, lane, nwarps, res[0]);
          release(G);
        }
      }
    }
  } else {
    const uint32_t rows = c.NL * a.r;
    const double2* src = a.in + static_cast<size_t>(c.node) * rows * a.k + c.c0;
    for (uint32_t e = threadIdx.x; e < rows * c.nc; e += blockDim.x) {
      const uint32_t row = e / c.nc, n = e - row * c.nc;
      c.vs[row * a.vld + n] = __ldg(src + static_cast<size_t>(row) * a.k + n);
    }
    __syncthreads();
    for (uint32_t li = 0; li < a.D; ++li) {
      c.li = li;
      c.lgP = a.D - 1 - li;
#pragma unroll
      for (int gi = 0; gi < MAXG; ++gi) {
        if (gi >= static_cast<int>(seq.ng_lev)) break;
        const double2* S = wait_stage(G);
        // units [gi gu, (gi + 1) gu) = gemms [2 gi gu, 2 (gi + 1) gu)
        stg_group<kLevUp, kStoreDeferred, NT>(a, c, S, lda_lev, 2 * gi * static_cast<int>(sg.gu),
                                              2 * static_cast<int>(sg.gu), warp, lane, nwarps, res[gi]);
        release(G);
        ++G;
      }
#pragma unroll
      for (int gi = 0; gi < MAXG; ++gi) {
        if (gi >= static_cast<int>(seq.ng_lev)) break;
        stg_deferred_store<kLevUp, NT>(a, c, 2 * gi * static_cast<int>(sg.gu), 2 * static_cast<int>(sg.gu), warp,
                                       lane, res[gi]);
      }
      __syncthreads();
    }
    for (uint32_t i = 0; i < seq.ng_leaf; ++i, ++G) {
      const double2* S = wait_stage(G);
      stg_group<kLeafUp, kStoreNow, NT>(a, c, S, lda_leaf, static_cast<int>(i * gl), static_cast<int>(gl), warp, lane,
                                        nwarps, res[0]);
      release(G);
    }
  }
}

}  // namespace bfly
