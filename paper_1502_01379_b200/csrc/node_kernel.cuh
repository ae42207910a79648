// node_kernel.cuh — one half of the apply chain per middle node, in ONE launch
// (the "subtree" kernels for the latency-bound chains).
//
// The V^L*/H* side of the chain is block-diagonal per middle column node and
// the G/U^L side per middle row node; every level keeps a
// node's m r vector rows contiguous (factors.py:217-237 with the reshape
// identities of §8(a) a3). So a node's whole half — leaf factor plus the
// L - h transfer levels — runs inside one CTA with its vector resident in
// shared memory:
//
//   down (forward chain: V^L*, H^{L-1}* .. H^h*, then M fused into the stores;
//         adjoint chain: U^L*, G^{L-1}* .. G^h*, M* fused)
//   up   (forward chain: G^h .. G^{L-1}, U^L; adjoint chain: H^h .. H^{L-1}, V^L)
//
// Two launches per apply instead of 2 + 2(L - h): cfg0 (N = 1024, 8 launches)
// and cfg1 (N = 2^16, 64 RHS, 14 levels) are latency bound on the per-level
// launches and on the intermediate vectors' round trips through HBM.
//
// A CTA owns (node, chunk of kc right-hand sides). Every step is a set of small
// complex GEMMs Y (M x kc) = A (M x K) X (K x kc) with A a factor block (read
// from global / L2; the chain's factors are L2-resident at these sizes) and X
// node vector rows in shared memory. Steps that rewrite the vector in place
// keep their outputs in registers until every warp has read its inputs (one
// barrier), then store. Many RHS (kc >= 8): FP64 tensor cores (mma.sync
// m8n8k4 DMMA, 3-multiplication complex form); few RHS: one output per thread
// on the FMA pipe.
#pragma once

#include "common.cuh"

namespace bfly {

constexpr int kNodeMaxLev = 16;

struct NodeArgs {
  const double2* leaf;              // (nb, n0, r) leaf factor of this half
  const double2* lev[kNodeMaxLev];  // transfer factors (G, 2, P, r, 2r), index = level - h
  const double2* in;                // down: chain input (n, k); up: middle vector (m m r, k)
  double2* out;                     // down: middle vector; up: chain output (n, k)
  const double* mid_w;              // (m, m, r) middle weights (down half: fused M / M*)
  uint32_t n0, r, D, k, kc, nch;    // leaf rows, rank, levels per side (= h), rhs, rhs per CTA, chunks
  uint32_t vld;                     // shared-memory row stride of the node vector (elements)
  uint32_t ksplit;                  // FMA path: threads per output (power of two <= 32)
  int xstage;                       // down half with PF: stage the node's input rows in shared memory
  unsigned long long* trace;        // diagnostics (bf_debug_node_trace): per-CTA %globaltimer stamps
  int remap;                        // down half: 1 forward-chain M, 2 adjoint-chain M*
};

enum NodeStepKind { kLeafDown = 0, kLevDown = 1, kLevUp = 2, kLeafUp = 3 };
enum NodeStore { kStoreNow = 0, kStoreDeferred = 1, kStoreRemap = 2 };

struct NodeCtx {
  uint32_t node, c0, nc;   // middle node, first rhs column, rhs columns of this CTA
  uint32_t NL, li, lgP;    // leaves (= middle nodes) per node, level index, log2 P of the level
  const double2* fac;      // this step's factor (level or leaf)
  double2* vs;             // node vector in shared memory (NL r rows x vld)
  const double2* xin;      // down half: this CTA's input rows (global, or staged in shared memory)
  uint32_t xld;            // row stride of xin
};

// GEMM shapes of a step: ngemm GEMMs of M rows, K = nseg x klen.
template <int KIND>
__device__ __forceinline__ void node_geom(const NodeArgs& a, const NodeCtx& c, int& ngemm, int& M, int& nseg,
                                          int& klen) {
  const int r = static_cast<int>(a.r);
  if constexpr (KIND == kLeafDown) {
    ngemm = c.NL; M = r; nseg = 1; klen = a.n0;
  } else if constexpr (KIND == kLevDown) {
    ngemm = c.NL / 2; M = 2 * r; nseg = 2; klen = r;
  } else if constexpr (KIND == kLevUp) {
    ngemm = c.NL; M = r; nseg = 1; klen = 2 * r;
  } else {
    ngemm = c.NL; M = a.n0; nseg = 1; klen = r;
  }
}

// A[q][m][seg, kk] of step KIND (complex, conjugated where the step is an adjoint).
// c.fac is the node's slab of the step's factor — contiguous in the reference layout:
// leaf blocks [node NL, (node + 1) NL), level groups [node 2^li, (node + 1) 2^li) —
// in global memory (SM = false) or prefetched into shared memory (SM = true).
template <bool SM>
__device__ __forceinline__ double2 node_ld(const double2* p) {
  if constexpr (SM) return *p;
  else return __ldg(p);
}

template <int KIND, bool SM>
__device__ __forceinline__ double2 node_a(const NodeArgs& a, const NodeCtx& c, int q, int m, int seg, int kk) {
  const uint32_t r = a.r;
  if constexpr (KIND == kLeafDown) {  // conj(V[b, kk, m])            factors.py:53-56
    const double2 v = node_ld<SM>(c.fac + (static_cast<size_t>(q) * a.n0 + kk) * r + m);
    return make_double2(v.x, -v.y);
  } else if constexpr (KIND == kLevDown) {  // conj(B[g, seg, p][kk][m])   factors.py:131-139
    const uint32_t P = 1u << c.lgP, g = q >> c.lgP, p = q & (P - 1);
    const double2 v = node_ld<SM>(c.fac + ((static_cast<size_t>(g * 2 + seg) * P + p) * r + kk) * (2 * r) + m);
    return make_double2(v.x, -v.y);
  } else if constexpr (KIND == kLevUp) {  // B[g, t, p][m][kk], q = 2u + t  factors.py:120-126
    const uint32_t u = q >> 1, t = q & 1, P = 1u << c.lgP, g = u >> c.lgP, p = u & (P - 1);
    return node_ld<SM>(c.fac + ((static_cast<size_t>(g * 2 + t) * P + p) * r + m) * (2 * r) + kk);
  } else {  // U[b, m, kk]                                                factors.py:49-51
    return node_ld<SM>(c.fac + (static_cast<size_t>(q) * a.n0 + m) * r + kk);
  }
}

// X[q][seg, kk][n] of step KIND
template <int KIND>
__device__ __forceinline__ double2 node_x(const NodeArgs& a, const NodeCtx& c, int q, int seg, int kk, int n) {
  const uint32_t r = a.r;
  if constexpr (KIND == kLeafDown) {
    return c.xin[(static_cast<size_t>(q) * a.n0 + kk) * c.xld + n];
  } else if constexpr (KIND == kLevDown) {
    const uint32_t P = 1u << c.lgP, g = q >> c.lgP, p = q & (P - 1);
    return c.vs[(((g * 2 + seg) * P + p) * r + kk) * a.vld + n];
  } else if constexpr (KIND == kLevUp) {
    return c.vs[((q >> 1) * 2 * r + kk) * a.vld + n];
  } else {
    return c.vs[(q * r + kk) * a.vld + n];
  }
}

// Destination of output (q, m, n); STORE kStoreRemap applies the middle factor.
template <int KIND, int STORE>
__device__ __forceinline__ void node_store(const NodeArgs& a, const NodeCtx& c, int q, int m, int n, double2 y) {
  const uint32_t r = a.r;
  if constexpr (KIND == kLeafUp) {
    a.out[(static_cast<size_t>(c.node * c.NL + q) * a.n0 + m) * a.k + c.c0 + n] = y;
  } else if constexpr (KIND == kLeafDown) {
    c.vs[(q * r + m) * a.vld + n] = y;
  } else if constexpr (KIND == kLevUp) {
    const uint32_t u = q >> 1, t = q & 1, P = 1u << c.lgP, g = u >> c.lgP, p = u & (P - 1);
    c.vs[(((g * 2 + t) * P + p) * r + m) * a.vld + n] = y;
  } else if constexpr (STORE == kStoreRemap) {
    // local row e = (other node ib, rho) of node a; w'[ib, node] = W x w[node, ib] (factors.py:180-190)
    const uint32_t e = q * 2 * r + m, ib = e / r, rho = e - ib * r;
    const size_t dst = (static_cast<size_t>(ib) * c.NL + c.node) * r + rho;
    const double w = a.remap == 1 ? __ldg(a.mid_w + dst)
                                  : __ldg(a.mid_w + (static_cast<size_t>(c.node) * c.NL + ib) * r + rho);
    a.out[dst * a.k + c.c0 + n] = make_double2(w * y.x, w * y.y);
  } else {
    c.vs[(q * 2 * r + m) * a.vld + n] = y;
  }
}

__device__ __forceinline__ void node_dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// One step on the FP64 tensor pipe: items of 8 rows x 8 NT columns over the warps.
// Deferred steps (in-place on the node vector) hold up to MAXIT items per warp in
// registers across one barrier.
template <int KIND, int STORE, int NT, int MAXIT, bool SM>
__device__ __forceinline__ void node_step_mma(const NodeArgs& a, const NodeCtx& c, int warp, int lane, int nwarps) {
  int ngemm, M, nseg, klen;
  node_geom<KIND>(a, c, ngemm, M, nseg, klen);
  const int mtl = (M + 7) >> 3, ntl = (static_cast<int>(c.nc) + 8 * NT - 1) / (8 * NT);
  const int items = ngemm * mtl * ntl;
  const int lr = lane >> 2, lk = lane & 3;
  constexpr int SLOTS = STORE == kStoreDeferred ? MAXIT : 1;
  double2 res[SLOTS][NT][2];
  const int nrounds = STORE == kStoreDeferred ? MAXIT : (items + nwarps - 1) / nwarps;
#pragma unroll
  for (int s = 0; s < (STORE == kStoreDeferred ? MAXIT : 1); ++s) {
    for (int rr = (STORE == kStoreDeferred ? s : 0); rr < (STORE == kStoreDeferred ? s + 1 : nrounds); ++rr) {
      const int it = warp + rr * nwarps;
      if (it >= items) break;
      const int gi = it / (mtl * ntl), rest = it - gi * mtl * ntl;
      const int m0 = (rest / ntl) * 8, n0 = (rest % ntl) * (8 * NT);
      const int m = m0 + lr;
      double t1[NT][2], t2[NT][2], t3[NT][2];
#pragma unroll
      for (int j = 0; j < NT; ++j) t1[j][0] = t1[j][1] = t2[j][0] = t2[j][1] = t3[j][0] = t3[j][1] = 0;
      for (int sg = 0; sg < nseg; ++sg) {
#pragma unroll 2
        for (int k0 = 0; k0 < klen; k0 += 4) {
          const int kk = k0 + lk;
          const bool kok = kk < klen;
          const double2 av = (kok && m < M) ? node_a<KIND, SM>(a, c, gi, m, sg, kk) : make_double2(0, 0);
          const double as = av.x + av.y;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const int n = n0 + 8 * j + lr;
            const double2 bv = (kok && n < static_cast<int>(c.nc)) ? node_x<KIND>(a, c, gi, sg, kk, n)
                                                                   : make_double2(0, 0);
            node_dmma(t1[j][0], t1[j][1], av.x, bv.x);
            node_dmma(t2[j][0], t2[j][1], av.y, bv.y);
            node_dmma(t3[j][0], t3[j][1], as, bv.x + bv.y);
          }
        }
      }
      const int sl = STORE == kStoreDeferred ? s : 0;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q)
          res[sl][j][q] = make_double2(t1[j][q] - t2[j][q], t3[j][q] - t1[j][q] - t2[j][q]);
      if constexpr (STORE != kStoreDeferred) {
        if (m < M) {
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int n = n0 + 8 * j + 2 * lk + q;
              if (n < static_cast<int>(c.nc)) node_store<KIND, STORE>(a, c, gi, m, n, res[0][j][q]);
            }
        }
      }
    }
  }
  if constexpr (STORE == kStoreDeferred) {
    __syncthreads();  // every warp has read the step's inputs
#pragma unroll
    for (int s = 0; s < MAXIT; ++s) {
      const int it = warp + s * nwarps;
      if (it >= items) break;
      const int gi = it / (mtl * ntl), rest = it - gi * mtl * ntl;
      const int m = (rest / ntl) * 8 + lr, n0 = (rest % ntl) * (8 * NT);
      if (m < M) {
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = n0 + 8 * j + 2 * lk + q;
            if (n < static_cast<int>(c.nc)) node_store<KIND, STORE>(a, c, gi, m, n, res[s][j][q]);
          }
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void node_stamp(const NodeArgs& a, int i) {
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    if (i >= 23) t = clock64();   // intra-step: SM cycles
    else asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[blockIdx.x * 32 + i] = t;
  }
}

// Row pointers of output (q, m, n): A element (seg, kk) at ap[kk * as] (conjugated for
// the adjoint steps), X element at xp[kk * xs].
template <int KIND>
__device__ __forceinline__ void node_rows(const NodeArgs& a, const NodeCtx& c, int q, int m, int seg, int n,
                                          const double2*& ap, uint32_t& as, const double2*& xp, uint32_t& xs) {
  const uint32_t r = a.r;
  if constexpr (KIND == kLeafDown) {
    ap = c.fac + static_cast<size_t>(q) * a.n0 * r + m;
    as = r;
    xp = c.xin + static_cast<size_t>(q) * a.n0 * c.xld + n;
    xs = c.xld;
  } else if constexpr (KIND == kLevDown) {
    const uint32_t P = 1u << c.lgP, g = q >> c.lgP, p = q & (P - 1), blk = (g * 2 + seg) * P + p;
    ap = c.fac + static_cast<size_t>(blk) * r * 2 * r + m;
    as = 2 * r;
    xp = c.vs + blk * r * a.vld + n;
    xs = a.vld;
  } else if constexpr (KIND == kLevUp) {
    const uint32_t u = q >> 1, t = q & 1, P = 1u << c.lgP, g = u >> c.lgP, p = u & (P - 1);
    ap = c.fac + (static_cast<size_t>((g * 2 + t) * P + p) * r + m) * 2 * r;
    as = 1;
    xp = c.vs + u * 2 * r * a.vld + n;
    xs = a.vld;
  } else {
    ap = c.fac + (static_cast<size_t>(q) * a.n0 + m) * r;
    as = 1;
    xp = c.vs + q * r * a.vld + n;
    xs = a.vld;
  }
}

// One step on the FMA pipe: each output (q, m, n) is a dot product split over KS
// consecutive threads (strided k, shuffle reduction), so the dependent FMA chains
// are K / KS long; up to MAXO outputs per thread group held for deferred stores.
template <int KIND, int STORE, int MAXO, bool SM>
__device__ __forceinline__ void node_step_fma(const NodeArgs& a, const NodeCtx& c, int tid, int nthr) {
  int ngemm, M, nseg, klen;
  node_geom<KIND>(a, c, ngemm, M, nseg, klen);
  const int nc = static_cast<int>(c.nc);
  const int outs = ngemm * M * nc;
  const int KS = static_cast<int>(a.ksplit), sub = tid & (KS - 1), ngrp = nthr / KS;
  constexpr bool CONJ = KIND == kLeafDown || KIND == kLevDown;
  constexpr int SLOTS = STORE == kStoreDeferred ? MAXO : 1;
  if constexpr (STORE == kStoreDeferred) node_stamp(a, 23);
  double2 res[SLOTS];
  const int nrounds = STORE == kStoreDeferred ? MAXO : (outs + ngrp - 1) / ngrp;
#pragma unroll
  for (int s = 0; s < (STORE == kStoreDeferred ? MAXO : 1); ++s) {
    for (int rr = (STORE == kStoreDeferred ? s : 0); rr < (STORE == kStoreDeferred ? s + 1 : nrounds); ++rr) {
      const int o0 = tid / KS + rr * ngrp;
      if (o0 - tid / KS >= outs) break;           // uniform across the CTA
      const bool valid = o0 < outs;
      const int o = valid ? o0 : 0;
      const int q = o / (M * nc), rest = o - q * M * nc, m = rest / nc, n = rest - m * nc;
      double2 acc = make_double2(0, 0);
      if constexpr (STORE == kStoreDeferred) node_stamp(a, 26);
      if (valid) {
        for (int sg = 0; sg < nseg; ++sg) {
          const double2* ap;
          const double2* xp;
          uint32_t as, xs;
          node_rows<KIND>(a, c, q, m, sg, n, ap, as, xp, xs);
#pragma unroll 1
          for (int kk = sub; kk < klen; kk += KS) {
            const double2 av = node_ld<SM>(ap + kk * as);
            const double2 xv = xp[kk * xs];
            if constexpr (CONJ) cmac_conj(acc, av, xv);
            else cmac(acc, av, xv);
          }
        }
      }
      if constexpr (STORE == kStoreDeferred) node_stamp(a, 27);
      for (int w = KS >> 1; w > 0; w >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, w);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, w);
      }
      if constexpr (STORE == kStoreDeferred) node_stamp(a, 28);
      if constexpr (STORE == kStoreDeferred) res[s] = acc;
      else if (valid && sub == 0) node_store<KIND, STORE>(a, c, q, m, n, acc);
    }
  }
  if constexpr (STORE == kStoreDeferred) {
    node_stamp(a, 24);
    __syncthreads();
    node_stamp(a, 25);
    if (sub == 0) {
#pragma unroll
      for (int s = 0; s < MAXO; ++s) {
        const int o = tid / KS + s * ngrp;
        if (o >= outs) break;
        const int q = o / (M * nc), rest = o - q * M * nc, m = rest / nc, n = rest - m * nc;
        node_store<KIND, STORE>(a, c, q, m, n, res[s]);
      }
    }
    __syncthreads();
  }
}

template <bool MMA, int KIND, int STORE, int NT, int MAXIT, bool SM>
__device__ __forceinline__ void node_step(const NodeArgs& a, const NodeCtx& c) {
  if constexpr (MMA)
    node_step_mma<KIND, STORE, NT, MAXIT, SM>(a, c, threadIdx.x >> 5, threadIdx.x & 31, blockDim.x >> 5);
  else
    node_step_fma<KIND, STORE, MAXIT, SM>(a, c, threadIdx.x, blockDim.x);
}

// Bytes of one step's node slab: leaf NL n0 r, level NL 2 r^2 complex values.
__device__ __forceinline__ uint32_t node_slab_bytes(const NodeArgs& a, bool leaf) {
  const uint32_t NL = 1u << a.D;
  return (leaf ? NL * a.n0 * a.r : NL * 2 * a.r * a.r) * static_cast<uint32_t>(sizeof(double2));
}

// UP = 0: the down half of one node (leaf adjoint, levels L-1 .. h adjoint, middle
// factor fused into the stores of the last level). UP = 1: the up half (levels h ..
// L-1 forward, leaf forward). grid = nodes x chunks. Dynamic shared memory: 256 B of
// mbarriers, the node vector (NL r rows x vld), and with PF every step's factor slab,
// prefetched by the TMA bulk engine at kernel start (before the wait on the previous
// kernel: factors are constant), so the steps read their blocks at shared-memory latency.
template <int UP, bool MMA, int NT, int MAXIT, bool PF>
__global__ void __launch_bounds__(512, 1) node_kernel(const NodeArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  node_stamp(a, 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  NodeCtx c;
  c.node = blockIdx.x / a.nch;
  const uint32_t chunk = blockIdx.x - c.node * a.nch;
  c.c0 = chunk * a.kc;
  c.nc = min(a.kc, a.k - c.c0);
  c.NL = 1u << a.D;
  c.vs = reinterpret_cast<double2*>(smem_raw + 256);
  const uint32_t vbytes = ((c.NL * a.r * a.vld * static_cast<uint32_t>(sizeof(double2))) + 127u) & ~127u;
  double2* slabs = reinterpret_cast<double2*>(smem_raw + 256 + vbytes);
  const uint32_t lbytes = node_slab_bytes(a, true), tbytes = node_slab_bytes(a, false);
  const double2* leaf_g = a.leaf + static_cast<size_t>(c.node) * c.NL * a.n0 * a.r;
  const size_t lev_off = static_cast<size_t>(c.node) * c.NL * 2 * a.r * a.r;
  // slab of step s in consumption order: down: leaf, lev D-1 .. 0; up: lev 0 .. D-1, leaf
  auto slab_smem = [&](uint32_t s) -> double2* {
    const bool leaf_first = !UP;
    if (leaf_first) return s == 0 ? slabs : slabs + (lbytes + (s - 1) * tbytes) / sizeof(double2);
    return slabs + static_cast<size_t>(s) * tbytes / sizeof(double2);
  };
  if constexpr (PF) {
    if (threadIdx.x == 0) {
      for (uint32_t s = 0; s <= a.D + 1; ++s) mbar_init(&bars[s], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (uint32_t s = 0; s <= a.D; ++s) {
        const bool is_leaf = UP ? s == a.D : s == 0;
        const uint32_t li = UP ? s : a.D - s;   // down: step s >= 1 is level D - s
        const double2* src = is_leaf ? leaf_g : a.lev[li] + lev_off;
        const uint32_t bytes = is_leaf ? lbytes : tbytes;
        mbar_arrive_expect_tx(&bars[s], bytes);
        bulk_g2s(slab_smem(s), src, bytes, &bars[s]);
      }
    }
  }
  node_stamp(a, 1);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous kernel's outputs / readers
  node_stamp(a, 2);
  c.xin = a.in + static_cast<size_t>(c.node) * c.NL * a.n0 * a.k + c.c0;
  c.xld = a.k;
  if constexpr (!UP && PF) {
    // one chunk per node: the node's input rows are contiguous; stage them with one bulk copy
    const uint32_t xbytes = c.NL * a.n0 * a.k * static_cast<uint32_t>(sizeof(double2));
    if (a.nch == 1 && a.xstage) {
      double2* xs = slab_smem(a.D + 1);
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bars[a.D + 1], xbytes);
        bulk_g2s(xs, c.xin, xbytes, &bars[a.D + 1]);
      }
      mbar_wait(&bars[a.D + 1], 0);
      c.xin = xs;
    }
  }
  node_stamp(a, 3);
  if constexpr (!UP) {
    if constexpr (PF) {
      mbar_wait(&bars[0], 0);
      c.fac = slab_smem(0);
    } else {
      c.fac = leaf_g;
    }
    node_stamp(a, 15);
    c.li = 0;
    c.lgP = 0;
    node_step<MMA, kLeafDown, kStoreNow, NT, MAXIT, PF>(a, c);
    __syncthreads();
    node_stamp(a, 4);
    for (int li = static_cast<int>(a.D) - 1; li >= 0; --li) {
      const uint32_t s = a.D - static_cast<uint32_t>(li);
      if constexpr (PF) {
        mbar_wait(&bars[s], 0);
        c.fac = slab_smem(s);
      } else {
        c.fac = a.lev[li] + lev_off;
      }
      node_stamp(a, 15 + static_cast<int>(s));
      c.li = static_cast<uint32_t>(li);
      c.lgP = a.D - 1 - c.li;
      if (li > 0)
        node_step<MMA, kLevDown, kStoreDeferred, NT, MAXIT, PF>(a, c);
      else
        node_step<MMA, kLevDown, kStoreRemap, NT, MAXIT, PF>(a, c);
      node_stamp(a, 5 + static_cast<int>(s) - 1);
    }
  } else {
    const uint32_t rows = c.NL * a.r;
    const double2* src = a.in + static_cast<size_t>(c.node) * rows * a.k + c.c0;
    for (uint32_t e = threadIdx.x; e < rows * c.nc; e += blockDim.x) {
      const uint32_t row = e / c.nc, n = e - row * c.nc;
      c.vs[row * a.vld + n] = __ldg(src + static_cast<size_t>(row) * a.k + n);
    }
    __syncthreads();
    node_stamp(a, 4);
    for (uint32_t li = 0; li < a.D; ++li) {
      if constexpr (PF) {
        mbar_wait(&bars[li], 0);
        c.fac = slab_smem(li);
      } else {
        c.fac = a.lev[li] + lev_off;
      }
      node_stamp(a, 15 + static_cast<int>(li));
      c.li = li;
      c.lgP = a.D - 1 - li;
      node_step<MMA, kLevUp, kStoreDeferred, NT, MAXIT, PF>(a, c);
      node_stamp(a, 5 + static_cast<int>(li));
    }
    if constexpr (PF) {
      mbar_wait(&bars[a.D], 0);
      c.fac = slab_smem(a.D);
    } else {
      c.fac = leaf_g;
    }
    node_step<MMA, kLeafUp, kStoreNow, NT, MAXIT, PF>(a, c);
    node_stamp(a, 5 + static_cast<int>(a.D));
  }
}

}  // namespace bfly
