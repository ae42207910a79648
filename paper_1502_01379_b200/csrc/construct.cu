// construct.cu — the sampling construction on B200: batched randomized
// sampling SVD of middle-level blocks (lowrank.py:219-258 via
// construct.py:43-68) and the recursive block SVDs (construct.py:127-163).
//
// One CTA owns one middle block (or one recursion problem). The random draws
// of every block are made on the host with the reference's own generator
// (SeedSequence(seed, spawn_key=(0, i, j)), construct.py:31-33) and uploaded
// as tables: the draws never depend on pivot results, so
// the device consumes exactly the index sets the reference would.
//
// Stage kernels, per sweep s of `iters`:
//   k_union      rows = union1d(draw, skeleton)             (lowrank.py:280-281)
//   k_fill_wide  K(rows, :) or K(:, cols)^H  ->  (|set| x side)
//   k_pivot_wide greedy pivoted Gram-Schmidt, r picks       (lowrank.py:102-129)
// then the bases (k_fill_tall, k_pivot_tall, k_fill_sel, k_cgs2 — lowrank.py:
// 132-154), the floored least-squares middle matrix and its SVD (k_mid,
// lowrank.py:90-94, 257, 284-293) and the scaled factors (k_assemble).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include <cooperative_groups.h>

#include "entry_eval.cuh"
#include "linalg.cuh"
#include "plan.h"

namespace bfly {

constexpr int kSetCap = 128;  // |rows|, |cols| <= r*q + r (r <= 32 at q = 3)
constexpr int kSmemSet = 64;  // small matrices live in shared memory when the set size S <= 64

struct BlockState {
  int64_t r0, c0;
  int32_t nrows, ncols, nskr, nskc, tc, tr, t, pad;
  int32_t rows[kSetCap], cols[kSetCap];
  int32_t skr[kSetCap], skc[kSetCap];
  int32_t pivc[kSetCap], pivr[kSetCap];
};

// construct.py MiddleSampler._STATE decodes this layout for the staged-parity traces
static_assert(sizeof(BlockState) == 3120, "BlockState layout is mirrored on the host");

struct MidArgs {
  EntrySrc src;
  int64_t side;
  int r, rqs, iters, nblocks;
  int S;                  // set capacity of this launch (64 or 128); strides of the per-block buffers
  BlockState* st;
  const int32_t* draws;   // (nblocks, 2*(iters+1), rqs)
  double2* wide;          // (nblocks, S, side)
  double2* tall;          // (nblocks, S, side)  column-major side x S
  double2* qc;            // (nblocks, S, side)
  double2* qr;            // (nblocks, S, side)
  double2* qbuf;          // (nblocks, side)
  double2* scr;           // (nblocks, 6, S, S) small-matrix scratch
  double* sig;            // (nblocks, S)
  double2* u_out;         // (nblocks, side, r)  u0 * sigma0
  double2* v_out;         // (nblocks, side, r)  v0 * sigma0
  double* w_out;          // (nblocks, r)        floored_inverse(sigma0)
  // matvec mode (bf_middle_probes): probe width (0 = sampling mode) and the products
  int probe_w;
  const double2* kc;      // (n, ldc)  K @ col_probe
  const double2* kr;      // (n, ldr)  K^H @ row_probe
  const double2* rprobe;  // (m, side, probe_w) row-probe diagonal blocks
  int64_t ldc, ldr;
};

enum { kRows = 0, kCols = 1 };

__global__ void k_init(MidArgs a, const int32_t* ij) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.nblocks) return;
  BlockState& s = a.st[b];
  s.r0 = static_cast<int64_t>(ij[2 * b]) * a.side;
  s.c0 = static_cast<int64_t>(ij[2 * b + 1]) * a.side;
  s.nrows = s.ncols = s.nskr = s.nskc = s.tc = s.tr = s.t = 0;
}

// set = sorted unique(draw[slot] U skeleton)  (np.union1d)
__global__ void k_union(MidArgs a, int slot, int which) {
  BlockState& s = a.st[blockIdx.x];
  __shared__ int32_t vals[2 * kSetCap];
  const int32_t* d = a.draws + (static_cast<int64_t>(blockIdx.x) * 2 * (a.iters + 1) + slot) * a.rqs;
  const int nsk = which == kRows ? s.nskr : s.nskc;
  const int32_t* sk = which == kRows ? s.skr : s.skc;
  const int tot = a.rqs + nsk;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) vals[i] = i < a.rqs ? d[i] : sk[i - a.rqs];
  __syncthreads();
  int32_t* out = which == kRows ? s.rows : s.cols;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    const int32_t v = vals[i];
    bool dup = false;
    int rank = 0;
    for (int k = 0; k < tot; ++k) {
      const int32_t w = vals[k];
      if (w == v && k < i) dup = true;
      // distinct values smaller than v: count each value once (its first occurrence)
      if (w < v) {
        bool first = true;
        for (int q = 0; q < k; ++q) first &= vals[q] != w;
        rank += first;
      }
    }
    if (!dup) out[rank] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int cnt = 0;
    for (int i = 0; i < tot; ++i) {
      bool first = true;
      for (int q = 0; q < i; ++q) first &= vals[q] != vals[i];
      cnt += first;
    }
    if (which == kRows)
      s.nrows = cnt;
    else
      s.ncols = cnt;
  }
}

// rows mode: W[a][c] = K(r0 + rows[a], c0 + c)            (entry(rows, all))
// cols mode: W[a][c] = conj(K(r0 + c, c0 + cols[a]))      (entry(all, cols)^H)
__global__ void k_fill_wide(MidArgs a, int which) {
  const BlockState& s = a.st[blockIdx.x];
  const int nr = which == kRows ? s.nrows : s.ncols;
  double2* W = a.wide + static_cast<int64_t>(blockIdx.x) * a.S * a.side;
  const int64_t total = nr * a.side;
  for (int64_t x = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int ai = static_cast<int>(x / a.side);
    const int64_t c = x - ai * a.side;
    W[x] = which == kRows ? entry_eval(a.src, s.r0 + s.rows[ai], s.c0 + c)
                          : cconj(entry_eval(a.src, s.r0 + c, s.c0 + s.cols[ai]));
  }
}

// Greedy column pivoting (select_pivot_columns, lowrank.py:102-129) on W
// (nr x ncols, row-major, nr <= kSetCap), k picks, CTA-cooperative. Initial
// norms sum over rows in the reference's order: sequential when the
// reference's matrix is C-ordered, numpy pairwise when it is F-ordered.
// Residual norms are downdated, never recomputed; ties within 2*PIVOT_TIE
// go to the lowest index. Returns the pick count; picks in pick order.
// Shared: norms (ncols doubles), q (kSetCap), red (32 doubles), redi (32 ints).
__device__ int pivot_rows_core(const double2* W, int nr, int ncols, int k, double rel_tol, bool pairwise,
                               double* norms, double2* q, double* red, int* redi, int* picks, double2* Rm) {
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    auto get = [&](int i) { return abs2(W[static_cast<int64_t>(i) * ncols + c]); };
    norms[c] = pairwise ? pairwise_sum(get, 0, nr) : sequential_sum(get, nr);
  }
  __syncthreads();
  k = min(k, min(nr, ncols));
  double lm0 = 0.0;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) lm0 = fmax(lm0, norms[c]);
  const double floor_v = rel_tol * rel_tol * block_max(lm0, red);
  int npick = 0;
  for (int it = 0; it < k; ++it) {
    double lm = 0.0;
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) lm = fmax(lm, norms[c]);
    const double best = block_max(lm, red);
    if (best <= floor_v || best <= 0.0) break;
    const double thr = __dmul_rn(best, 1.0 - 2.0 * kPivotTie);
    int li = INT_MAX;
    for (int c = threadIdx.x; c < ncols; c += blockDim.x)
      if (norms[c] >= thr) li = min(li, c);
    const int j = block_min_int(li, redi);
    const double sq = sqrt(norms[j]);
    for (int i = threadIdx.x; i < nr; i += blockDim.x) q[i] = W[static_cast<int64_t>(i) * ncols + j];
    if (threadIdx.x == 0) picks[npick] = j;
    __syncthreads();
    // left-looking form of the Gram-Schmidt step: with q = work_j / sqrt(norms_j),
    // q^H work_c = (w_j^H w_c - sum_l conj(P_lj) P_lc) / sqrt(norms_j), so W stays
    // read-only and only the projection rows P (k x ncols) are written
    double2* prow = Rm + static_cast<int64_t>(npick) * ncols;
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
      double2 g = make_double2(0, 0);
#pragma unroll 8
      for (int i = 0; i < nr; ++i) {  // unrolled: 8 independent loads in flight per thread
        const double2 t = cmulc(q[i], W[static_cast<int64_t>(i) * ncols + c]);
        g.x += t.x;
        g.y += t.y;
      }
      for (int l = 0; l < npick; ++l) {
        const double2 t = cmulc(Rm[static_cast<int64_t>(l) * ncols + j], Rm[static_cast<int64_t>(l) * ncols + c]);
        g.x -= t.x;
        g.y -= t.y;
      }
      const double2 pr = make_double2(__ddiv_rn(g.x, sq), __ddiv_rn(g.y, sq));
      prow[c] = pr;
      norms[c] = fmax(__dsub_rn(norms[c], abs2(pr)), 0.0);
    }
    ++npick;
    __syncthreads();
    if (threadIdx.x == 0) norms[j] = 0.0;
    __syncthreads();
  }
  return npick;
}

// Sweep pivots: rows mode picks columns of K(rows, :) -> column skeleton;
// cols mode picks columns of K(:, cols)^H -> row skeleton (lowrank.py:237-243).
__global__ void k_pivot_wide(MidArgs a, int which) {
  extern __shared__ double smem_d[];
  double* norms = smem_d;                                       // side
  double2* q = reinterpret_cast<double2*>(norms + a.side);      // kSetCap
  double* red = reinterpret_cast<double*>(q + kSetCap);         // 32
  int* redi = reinterpret_cast<int*>(red + 32);                 // 32
  int* picks = redi + 32;                                       // kSetCap
  BlockState& s = a.st[blockIdx.x];
  const int nr = which == kRows ? s.nrows : s.ncols;
  double2* W = a.wide + static_cast<int64_t>(blockIdx.x) * a.S * a.side;
  double2* Rm = a.tall + static_cast<int64_t>(blockIdx.x) * a.S * a.side;  // projection rows (r x side)
  const int npick = pivot_rows_core(W, nr, static_cast<int>(a.side), a.r, 0.0, which == kCols, norms, q, red, redi,
                                    picks, Rm);
  // skeleton = sorted(picks)
  if (threadIdx.x == 0) {
    int32_t* sk = which == kRows ? s.skc : s.skr;
    for (int i = 0; i < npick; ++i) {
      int rank = 0;
      for (int m = 0; m < npick; ++m) rank += picks[m] < picks[i];
      sk[rank] = picks[i];
    }
    if (which == kRows)
      s.nskc = npick;
    else
      s.nskr = npick;
  }
}

// Cluster form of k_pivot_wide for wide samples (side >= 1024): a cluster of CL CTAs
// shares one block, CTA c owning columns [c side/CL, (c+1) side/CL). With one CTA per SM
// only 148/CL blocks are in flight, so their samples (|rows| x side complex: 4 MB at
// cfg2) stay L2-resident across the r passes of the greedy loop instead of streaming
// from HBM on every pick. Per pick the column maximum and the first index above the
// tie threshold are exchanged through distributed shared memory: max and min are
// exact, and every column's arithmetic is the single-CTA kernel's, so the picks (and
// the construction) are bitwise identical to k_pivot_wide.
template <int CL>
__global__ void __launch_bounds__(512, 1) k_pivot_wide_cl(MidArgs a, int which) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double smem_d[];
  const int cr = static_cast<int>(cluster.block_rank());
  const int blk = blockIdx.x / CL;
  const int ncols = static_cast<int>(a.side);
  const int c0 = cr * ncols / CL, c1 = (cr + 1) * ncols / CL, nloc = c1 - c0;
  double* norms = smem_d;                                             // nloc (own columns)
  double2* q = reinterpret_cast<double2*>(norms + ((nloc + 1) & ~1));  // kSetCap
  double* red = reinterpret_cast<double*>(q + kSetCap);               // 32
  int* redi = reinterpret_cast<int*>(red + 32);                       // 32
  __shared__ double cl_val[CL];                                       // per-CTA maxima
  __shared__ int cl_idx[CL];                                          // per-CTA first index >= thr
  __shared__ double cl_nrm[CL];                                       // and its norm
  __shared__ int picks[kSetCap];
  BlockState& s = a.st[blk];
  const int nr = which == kRows ? s.nrows : s.ncols;
  const bool pairwise = which == kCols;
  const double2* W = a.wide + static_cast<int64_t>(blk) * a.S * a.side;
  double2* Rm = a.tall + static_cast<int64_t>(blk) * a.S * a.side;
  auto put_val = [&](double v) {  // every CTA gets this CTA's value in slot cr
    if (threadIdx.x < CL) *cluster.map_shared_rank(&cl_val[cr], threadIdx.x) = v;
  };
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    auto get = [&](int i) { return abs2(W[static_cast<int64_t>(i) * ncols + c]); };
    norms[c - c0] = pairwise ? pairwise_sum(get, 0, nr) : sequential_sum(get, nr);
  }
  const int k = min(a.r, min(nr, ncols));
  cluster.sync();  // every CTA of the cluster is running before any DSMEM store
  int npick = 0;
  // two cluster barriers per pick: the maxima are read before a CTA arrives at the second,
  // the first indices before it arrives at the next pick's first, so single buffers do
  for (int it = 0; it < k; ++it) {
    double lm = 0.0;
    for (int c = threadIdx.x; c < nloc; c += blockDim.x) lm = fmax(lm, norms[c]);
    lm = block_max(lm, red);
    put_val(lm);
    cluster.sync();
    double best = 0.0;
    for (int x = 0; x < CL; ++x) best = fmax(best, cl_val[x]);
    if (best <= 0.0) break;  // rel_tol = 0 in the sweeps (lowrank.py:237-243); identical in every CTA
    const double thr = __dmul_rn(best, 1.0 - 2.0 * kPivotTie);
    int li = INT_MAX;
    for (int c = threadIdx.x; c < nloc; c += blockDim.x)
      if (norms[c] >= thr) li = min(li, c);
    li = block_min_int(li, redi);
    if (threadIdx.x < CL) {
      *cluster.map_shared_rank(&cl_idx[cr], threadIdx.x) = li == INT_MAX ? INT_MAX : c0 + li;
      *cluster.map_shared_rank(&cl_nrm[cr], threadIdx.x) = li == INT_MAX ? 0.0 : norms[li];
    }
    cluster.sync();  // also orders the previous picks' projection rows (global) before their reads
    int j = INT_MAX;
    double nj = 0.0;
    for (int x = 0; x < CL; ++x)
      if (cl_idx[x] < j) {
        j = cl_idx[x];
        nj = cl_nrm[x];
      }
    const double sq = sqrt(nj);
    for (int i = threadIdx.x; i < nr; i += blockDim.x) q[i] = W[static_cast<int64_t>(i) * ncols + j];
    if (threadIdx.x == 0) picks[npick] = j;
    __syncthreads();
    double2* prow = Rm + static_cast<int64_t>(npick) * ncols;
    for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
      double2 g = make_double2(0, 0);
#pragma unroll 8
      for (int i = 0; i < nr; ++i) {
        const double2 t = cmulc(q[i], W[static_cast<int64_t>(i) * ncols + c]);
        g.x += t.x;
        g.y += t.y;
      }
      for (int l = 0; l < npick; ++l) {
        const double2 t = cmulc(Rm[static_cast<int64_t>(l) * ncols + j], Rm[static_cast<int64_t>(l) * ncols + c]);
        g.x -= t.x;
        g.y -= t.y;
      }
      const double2 pr = make_double2(__ddiv_rn(g.x, sq), __ddiv_rn(g.y, sq));
      prow[c] = pr;
      norms[c - c0] = fmax(__dsub_rn(norms[c - c0], abs2(pr)), 0.0);
    }
    ++npick;
    __syncthreads();
    if (threadIdx.x == 0 && j >= c0 && j < c1) norms[j - c0] = 0.0;
    __syncthreads();
  }
  cluster.sync();  // projection rows complete before any CTA exits (DSMEM lifetime)
  if (cr == 0 && threadIdx.x == 0) {
    int32_t* sk = which == kRows ? s.skc : s.skr;
    for (int i = 0; i < npick; ++i) {
      int rank = 0;
      for (int m = 0; m < npick; ++m) rank += picks[m] < picks[i];
      sk[rank] = picks[i];
    }
    if (which == kRows)
      s.nskc = npick;
    else
      s.nskr = npick;
  }
}

// Register form of k_pivot_wide_cl for r <= 16 and at most one column per thread
// (side / CL <= 512: every cluster shape launch_pivot_wide uses): the projection rows
// never touch global memory — a thread keeps its own column's projections P_lc in
// registers, the pivot column's P_lj travel with the pick through distributed shared
// memory — and a pick costs ONE cluster barrier: every CTA publishes its maximum, its
// first column within the tie threshold of that maximum, that column's norm and
// projections; with thr = best (1 - 2 tie) the global pick is the first published column
// of a CTA whose maximum reaches thr. Only when some CTA's maximum reaches thr but its
// published column does not (a near-tie between different columns of one CTA) does that
// pick fall back to the two-barrier exchange with the global threshold. With no global
// stores inside the loop the barrier's release fence has nothing to flush (ncu:
// membar + barrier stalls 22% of k_pivot_wide_cl). The arithmetic of every column is
// k_pivot_wide's, term for term, so picks are bitwise identical.
constexpr int kPivReg = 16;

template <int CL>
__global__ void __launch_bounds__(512, 1) k_pivot_wide_cl2(MidArgs a, int which) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = static_cast<int>(cluster.block_rank());
  const int blk = blockIdx.x / CL;
  const int ncols = static_cast<int>(a.side);
  const int c0 = cr * ncols / CL, c1 = (cr + 1) * ncols / CL, nloc = c1 - c0;
  extern __shared__ double2 pcs[];               // own columns' projections P_lc: [l][thread]
  __shared__ double2 q[kSetCap];
  __shared__ double red[32];
  __shared__ int redi[32];
  __shared__ double cl_val[2][CL];               // per-CTA maxima (double-buffered by pick parity)
  __shared__ int cl_idx[2][CL];                  // per-CTA first column within the tie of its maximum
  __shared__ double cl_nrm[2][CL];               // its norm
  __shared__ double2 cl_pc[2][CL][kPivReg];      // and its projections
  __shared__ double2 mypc[kPivReg];
  __shared__ int picks[kSetCap];
  __shared__ double s_norm;
  BlockState& s = a.st[blk];
  const int nr = which == kRows ? s.nrows : s.ncols;
  const bool pairwise = which == kCols;
  const double2* W = a.wide + static_cast<int64_t>(blk) * a.S * a.side;
  const int tid = threadIdx.x;
  const bool own = tid < nloc;
  const int c = c0 + tid;
  double norm = 0.0;
  if (own) {
    auto get = [&](int i) { return abs2(W[static_cast<int64_t>(i) * ncols + c]); };
    norm = pairwise ? pairwise_sum(get, 0, nr) : sequential_sum(get, nr);
  }
  double2* pc = pcs + tid;                       // pc[l * 512]
  const int k = min(a.r, min(nr, ncols));
  cluster.sync();  // every CTA of the cluster is running before any DSMEM store
  int npick = 0;
  // publish this CTA's candidate for a threshold factor: maximum, first column >= thr_of(max)
  auto publish = [&](int par, double thr_in, bool use_thr_in) {
    const double lm = block_max(own ? norm : 0.0, red);
    const double thr = use_thr_in ? thr_in : __dmul_rn(lm, 1.0 - 2.0 * kPivotTie);
    int li = (own && norm >= thr && lm > 0.0) ? tid : INT_MAX;
    li = block_min_int(li, redi);
    if (tid == li) s_norm = norm;
    if (li != INT_MAX && tid < npick) mypc[tid] = pcs[tid * 512 + li];
    __syncthreads();
    if (tid < CL) {
      *cluster.map_shared_rank(&cl_val[par][cr], tid) = lm;
      *cluster.map_shared_rank(&cl_idx[par][cr], tid) = li == INT_MAX ? INT_MAX : c0 + li;
      *cluster.map_shared_rank(&cl_nrm[par][cr], tid) = li == INT_MAX ? 0.0 : s_norm;
    }
    if (li != INT_MAX && tid >= 32 && tid < 32 + CL * kPivReg) {
      const int d = (tid - 32) / kPivReg, l = (tid - 32) % kPivReg;
      if (l < npick) *cluster.map_shared_rank(&cl_pc[par][cr][l], d) = mypc[l];
    }
  };
  int par = 0;
  for (int it = 0; it < k; ++it) {
    publish(par, 0.0, false);
    cluster.sync();
    double best = 0.0;
#pragma unroll
    for (int x = 0; x < CL; ++x) best = fmax(best, cl_val[par][x]);
    if (best <= 0.0) break;  // rel_tol = 0 in the sweeps (lowrank.py:237-243); identical in every CTA
    const double thr = __dmul_rn(best, 1.0 - 2.0 * kPivotTie);
    bool ambiguous = false;
#pragma unroll
    for (int x = 0; x < CL; ++x) ambiguous |= cl_val[par][x] >= thr && !(cl_nrm[par][x] >= thr);
    int usepar = par;
    if (ambiguous) {  // (uniform across the cluster) republish with the global threshold
      usepar = par ^ 1;
      cluster.sync();   // every CTA has read this pick's first round before the other buffer is rewritten
      publish(usepar, thr, true);
      cluster.sync();
    }
    int j = INT_MAX, xo = 0;
#pragma unroll
    for (int x = 0; x < CL; ++x)
      if (cl_val[usepar][x] >= thr && cl_idx[usepar][x] < j) {
        j = cl_idx[usepar][x];
        xo = x;
      }
    const double nj = cl_nrm[usepar][xo];
    const double sq = sqrt(nj);
    for (int i = tid; i < nr; i += blockDim.x) q[i] = W[static_cast<int64_t>(i) * ncols + j];
    if (tid == 0) picks[npick] = j;
    __syncthreads();
    if (own) {
      double2 g = make_double2(0, 0);
#pragma unroll 8
      for (int i = 0; i < nr; ++i) {
        const double2 t = cmulc(q[i], W[static_cast<int64_t>(i) * ncols + c]);
        g.x += t.x;
        g.y += t.y;
      }
      for (int l = 0; l < npick; ++l) {
        const double2 t = cmulc(cl_pc[usepar][xo][l], pc[l * 512]);
        g.x -= t.x;
        g.y -= t.y;
      }
      const double2 pr = make_double2(__ddiv_rn(g.x, sq), __ddiv_rn(g.y, sq));
      pc[npick * 512] = pr;
      norm = fmax(__dsub_rn(norm, abs2(pr)), 0.0);
      if (c == j) norm = 0.0;
    }
    ++npick;
    if (ambiguous) {
      // both buffers were used by this pick: resynchronise before either is rewritten
      cluster.sync();
    } else {
      par ^= 1;
    }
    __syncthreads();   // q and the candidate buffers are free for the next pick
  }
  cluster.sync();  // no CTA exits while its shared memory may still be written
  if (cr == 0 && tid == 0) {
    int32_t* sk = which == kRows ? s.skc : s.skr;
    for (int i = 0; i < npick; ++i) {
      int rank = 0;
      for (int m = 0; m < npick; ++m) rank += picks[m] < picks[i];
      sk[rank] = picks[i];
    }
    if (which == kRows)
      s.nskc = npick;
    else
      s.nskr = npick;
  }
}

// Standalone batched pivot selection (bf_select_pivots): matrices (batch, m, n)
// complex128 row-major, m <= kSetCap, copied to scratch then pivoted in place.
__global__ void k_select_pivots(const double2* A, double2* scratch, int m, int n, int k, double rel_tol, int pairwise,
                                int32_t* pivots, int32_t* counts) {
  extern __shared__ double smem_d[];
  double* norms = smem_d;
  double2* q = reinterpret_cast<double2*>(norms + n + (n & 1));
  double* red = reinterpret_cast<double*>(q + kSetCap);
  int* redi = reinterpret_cast<int*>(red + 32);
  int* picks = redi + 32;
  const int64_t off = static_cast<int64_t>(blockIdx.x) * m * n;
  double2* Rm = scratch + static_cast<int64_t>(blockIdx.x) * min(k, m) * n;
  const int np = pivot_rows_core(A + off, m, n, k, rel_tol, pairwise != 0, norms, q, red, redi, picks, Rm);
  for (int i = threadIdx.x; i < np; i += blockDim.x) pivots[static_cast<int64_t>(blockIdx.x) * k + i] = picks[i];
  if (threadIdx.x == 0) counts[blockIdx.x] = np;
}

// Tall column-major fill: column p of T (side rows) is
//   cols mode: K(r0 + :, c0 + cols[sel(p)])           (entry(all, cols))
//   rows mode: conj(K(r0 + rows[sel(p)], c0 + :))     (entry(rows, all)^H)
// with sel = identity (ncols/nrows columns) or the basis pivots (tc/tr columns).
__global__ void k_fill_tall(MidArgs a, int which, int use_piv, double2* dst_base) {
  const BlockState& s = a.st[blockIdx.x];
  const int ncol = use_piv ? (which == kCols ? s.tc : s.tr) : (which == kCols ? s.ncols : s.nrows);
  double2* T = dst_base + static_cast<int64_t>(blockIdx.x) * a.S * a.side;
  const int64_t total = ncol * a.side;
  for (int64_t x = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int p = static_cast<int>(x / a.side);
    const int64_t i = x - p * a.side;
    const int sel = use_piv ? (which == kCols ? s.pivc[p] : s.pivr[p]) : p;
    T[x] = which == kCols ? entry_eval(a.src, s.r0 + i, s.c0 + s.cols[sel])
                          : cconj(entry_eval(a.src, s.r0 + s.rows[sel], s.c0 + i));
  }
}

// Greedy pivoting on the tall T (side x nc, column-major), up to kmax picks,
// rel_tol = BASIS_TRIM; pick order kept (orthonormal_columns, lowrank.py:132-154).
// Greedy pivoting of the tall T (side x nc, column-major; orthonormal_columns,
// lowrank.py:132-154) through its Gram matrix: G = T^H T in one pass over T
// (row chunks staged in shared memory), then the pivoted Cholesky recurrence
// on G, which reproduces select_pivot_columns' (lowrank.py:102-129) Gram-Schmidt
// step for step: with q = work_j / sqrt(norms_j), the projections are
// proj_c = (G_jc - sum_l conj(P_lj) P_lc) / sqrt(norms_j) and the norms are
// downdated by |proj_c|^2. The initial norms keep the reference's exact
// summation order; the first pick is therefore bitwise the reference's.
// Past the numerical rank both this and the reference pick rounding noise.
constexpr int kGramChunk = 32;
constexpr int kGramTiles = 3;     // 8 x 8 Gram tiles per warp and pass (64 columns: 36 tiles, 16 warps)
constexpr int kPivotTallThreads = 512;

__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kPivotTallThreads) k_pivot_tall(MidArgs a, int which) {
  extern __shared__ double2 tsm[];
  __shared__ double norms[kSetCap];
  __shared__ int picks[kSetCap];
  __shared__ int s_j, s_stop;
  __shared__ double s_sq;
  BlockState& s = a.st[blockIdx.x];
  const int nc = which == kCols ? s.ncols : s.nrows;
  const int side = static_cast<int>(a.side);
  const int S = a.S;
  const double2* T = a.tall + static_cast<int64_t>(blockIdx.x) * S * a.side;
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    const double2* col = T + static_cast<int64_t>(c) * side;
    auto get = [&](int i) { return abs2(col[i]); };
    // np.sum over axis 0: sequential for C-ordered copies (entry(all, cols), and the
    // probe products in matvec mode), pairwise for the F-ordered entry(rows, all)^H
    norms[c] = (which == kCols || a.probe_w > 0) ? sequential_sum(get, side) : pairwise_sum(get, 0, side);
  }
  const int Sp = S + 2;   // chunk row stride: a DMMA fragment's 4 k-rows land on distinct banks
  double2* chunk = tsm;                                           // kGramChunk x Sp
  const int64_t SS = static_cast<int64_t>(S) * S;
  double2* gscr = a.scr + static_cast<int64_t>(blockIdx.x) * 9 * SS;
  double2* G = S <= kSmemSet ? tsm + kGramChunk * Sp : gscr;      // S x S
  double2* Rm = S <= kSmemSet ? G + SS : gscr + SS;               // picks x S
  // ---- Gram matrix T^H T on the FP64 tensor pipe (mma.sync m8n8k4, DMMA): 8 x 8 tiles of
  // the upper block triangle, up to kGramTiles per warp, accumulated over row chunks
  // staged through registers one chunk ahead (the next chunk's global loads are in
  // flight while this one is multiplied); complex products in the 3-multiplication form
  // (T1 = Re a Re b, T2 = Im a' Im b, T3 = (Re + Im a')(Re + Im b), a' = conj(a)).
  const int nct = (nc + 7) / 8;
  const int ntiles = nct * (nct + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  for (int tbase = 0; tbase < ntiles; tbase += nw * kGramTiles) {
  int tta[kGramTiles], ttb[kGramTiles];
#pragma unroll
  for (int q = 0; q < kGramTiles; ++q) {
    int rem = tbase + warp + q * nw, ta = 0;
    if (rem < ntiles)
      while (rem >= nct - ta) {
        rem -= nct - ta;
        ++ta;
      }
    tta[q] = rem < ntiles ? ta : -1;
    ttb[q] = ta + rem;
  }
  double t1[kGramTiles][2], t2[kGramTiles][2], t3[kGramTiles][2];
#pragma unroll
  for (int q = 0; q < kGramTiles; ++q) t1[q][0] = t1[q][1] = t2[q][0] = t2[q][1] = t3[q][0] = t3[q][1] = 0;
  {
    constexpr int kPre = (kSetCap * kGramChunk + kPivotTallThreads - 1) / kPivotTallThreads;
    const int nel = nct * 8 * kGramChunk;
    double2 pre[kPre];
    auto fetch = [&](int r0) {
#pragma unroll
      for (int q = 0; q < kPre; ++q) {
        const int x = threadIdx.x + q * static_cast<int>(blockDim.x);
        const int c = x / kGramChunk, i = x % kGramChunk;
        pre[q] = (x < nel && r0 + i < side && c < nc) ? T[static_cast<int64_t>(c) * side + r0 + i]
                                                       : make_double2(0, 0);
      }
    };
    fetch(0);
    for (int r0 = 0; r0 < side; r0 += kGramChunk) {
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kPre; ++q) {
        const int x = threadIdx.x + q * static_cast<int>(blockDim.x);
        if (x < nel) chunk[(x % kGramChunk) * Sp + x / kGramChunk] = pre[q];
      }
      __syncthreads();
      if (r0 + kGramChunk < side) fetch(r0 + kGramChunk);
#pragma unroll 2
      for (int k0 = 0; k0 < kGramChunk; k0 += 4) {
        const double2* row = chunk + (k0 + lk) * Sp + lr;
#pragma unroll
        for (int q = 0; q < kGramTiles; ++q) {
          if (tta[q] < 0) break;
          const double2 av = row[tta[q] * 8], bv = row[ttb[q] * 8];
          const double ar = av.x, ai = -av.y;
          dmma_f64(t1[q][0], t1[q][1], ar, bv.x);
          dmma_f64(t2[q][0], t2[q][1], ai, bv.y);
          dmma_f64(t3[q][0], t3[q][1], ar + ai, bv.x + bv.y);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kGramTiles; ++q) {
    if (tta[q] < 0) break;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ra = tta[q] * 8 + lr, cb = ttb[q] * 8 + 2 * lk + h;
      const double2 g = make_double2(t1[q][h] - t2[q][h], t3[q][h] - t1[q][h] - t2[q][h]);
      if (ra < nc && cb < nc && (tta[q] < ttb[q] || ra <= cb)) {
        G[ra * S + cb] = g;
        G[cb * S + ra] = cconj(g);
      }
    }
  }
  }   // tile batches
  __syncthreads();
  // ---- pivoted Cholesky recurrence == the greedy Gram-Schmidt pivoting
  // sampling mode: k = min(width, side), rel_tol = BASIS_TRIM (lowrank.py:252-256);
  // matvec mode: k = probe width, rel_tol = 0 (svd_from_probes, lowrank.py:213-214)
  const int width = a.probe_w > 0 ? a.probe_w : max(a.r, min(s.nrows, s.ncols) - a.r);
  const int kmax = min(min(width, side), min(side, nc));
  double mx0 = 0.0;
  for (int c = 0; c < nc; ++c) mx0 = fmax(mx0, norms[c]);
  const double floor_v = a.probe_w > 0 ? 0.0 : kBasisTrim * kBasisTrim * mx0;
  int npick = 0;
  for (int it = 0; it < kmax; ++it) {
    if (threadIdx.x == 0) {
      double best = 0.0;
      for (int c = 0; c < nc; ++c) best = fmax(best, norms[c]);
      s_stop = (best <= floor_v || best <= 0.0);
      if (!s_stop) {
        const double thr = __dmul_rn(best, 1.0 - 2.0 * kPivotTie);
        int j = 0;
        while (norms[j] < thr) ++j;
        s_j = j;
        s_sq = sqrt(norms[j]);
        picks[npick] = j;
      }
    }
    __syncthreads();
    if (s_stop) break;
    const int j = s_j;
    const double sq = s_sq;
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
      double2 v = G[j * S + c];
      for (int l = 0; l < it; ++l) {
        const double2 d = cmulc(Rm[l * S + j], Rm[l * S + c]);
        v.x -= d.x;
        v.y -= d.y;
      }
      Rm[it * S + c] = make_double2(__ddiv_rn(v.x, sq), __ddiv_rn(v.y, sq));
    }
    ++npick;
    __syncthreads();
    for (int c = threadIdx.x; c < nc; c += blockDim.x)
      norms[c] = fmax(__dsub_rn(norms[c], abs2(Rm[it * S + c])), 0.0);
    __syncthreads();
    if (threadIdx.x == 0) norms[j] = 0.0;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int32_t* piv = which == kCols ? s.pivc : s.pivr;
    for (int i = 0; i < npick; ++i) piv[i] = picks[i];
    if (which == kCols)
      s.tc = npick;
    else
      s.tr = npick;
  }
}

// Classical Gram-Schmidt, two passes: an orthonormal basis of the selected
// columns (the reference uses np.linalg.qr; only span(Q) reaches the factors,
// see DESIGN.md "Construction parity").
__global__ void k_cgs2(MidArgs a, int which) {
  __shared__ double2 coef[kSetCap];
  __shared__ double red[32];
  const BlockState& s = a.st[blockIdx.x];
  const int t = which == kCols ? s.tc : s.tr;
  const int side = static_cast<int>(a.side);
  double2* Q = (which == kCols ? a.qc : a.qr) + static_cast<int64_t>(blockIdx.x) * a.S * a.side;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int p = 0; p < t; ++p) {
    double2* x = Q + static_cast<int64_t>(p) * side;
    for (int pass = 0; pass < 2; ++pass) {
      for (int l = warp; l < p; l += nw) {
        const double2* ql = Q + static_cast<int64_t>(l) * side;
        double2 acc = make_double2(0, 0);
        for (int i = lane; i < side; i += 32) {
          const double2 g = cmulc(ql[i], x[i]);
          acc.x += g.x;
          acc.y += g.y;
        }
        acc = warp_sum2(acc);
        if (lane == 0) coef[l] = acc;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < side; i += blockDim.x) {
        double2 v = x[i];
        for (int l = 0; l < p; ++l) {
          const double2 d = cmul(Q[static_cast<int64_t>(l) * side + i], coef[l]);
          v.x -= d.x;
          v.y -= d.y;
        }
        x[i] = v;
      }
      __syncthreads();
    }
    double part = 0;
    for (int i = threadIdx.x; i < side; i += blockDim.x) part += x[i].x * x[i].x + x[i].y * x[i].y;
    const double nrm = sqrt(block_sum(part, red));
    const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
    for (int i = threadIdx.x; i < side; i += blockDim.x) x[i] = make_double2(x[i].x * inv, x[i].y * inv);
    __syncthreads();
  }
}

// Block classical Gram-Schmidt with reorthogonalisation (BCGS2): the same
// orthonormal basis as k_cgs2 up to rounding (only span(Q) reaches the
// factors), with the columns processed in panels of `pw` held in shared memory.
// Per panel, twice: project the panel against all previous columns (one pass
// over Q[:, :j0] computes every panel column's coefficients, one more applies
// them), then classical Gram-Schmidt inside the panel. k_cgs2 reads each
// previous column ~6 times per new column from global memory; here each previous
// column is read 4 times per panel.
constexpr int kPanelMax = 8;

__global__ void __launch_bounds__(1024) k_bcgs2(MidArgs a, int which, int pw, int nseg) {
  extern __shared__ double2 pan[];  // pw columns of length side, then S * nseg * pw partial coefficients
  __shared__ double2 coef[kSetCap][kPanelMax];
  __shared__ double red[2 * 32];
  const BlockState& s = a.st[blockIdx.x];
  const int t = which == kCols ? s.tc : s.tr;
  const int side = static_cast<int>(a.side);
  double2* Q = (which == kCols ? a.qc : a.qr) + static_cast<int64_t>(blockIdx.x) * a.S * a.side;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j0 = 0; j0 < t; j0 += pw) {
    const int nb = min(pw, t - j0);
    for (int x = threadIdx.x; x < nb * side; x += blockDim.x) pan[x] = Q[static_cast<int64_t>(j0) * side + x];
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      if (j0 > 0) {
        // C = Q[:, :j0]^H pan: one warp per (previous column, row segment) unit — with whole
        // columns per warp only j0 of the 32 warps work (and 33..45 columns leave a second,
        // mostly empty round); the segments' partial sums are added in segment order
        double2* cpart = pan + static_cast<int64_t>(pw) * side;
        const int seglen = (((side + nseg - 1) / nseg) + 31) & ~31;
        for (int u = warp; u < j0 * nseg; u += nw) {
          const int l = u % j0, sg = u / j0;
          const double2* ql = Q + static_cast<int64_t>(l) * side;
          const int i1 = min(side, (sg + 1) * seglen);
          double2 acc[kPanelMax];
#pragma unroll
          for (int b = 0; b < kPanelMax; ++b) acc[b] = make_double2(0, 0);
#pragma unroll 4
          for (int i = sg * seglen + lane; i < i1; i += 32) {
            const double2 q = ql[i];
#pragma unroll
            for (int b = 0; b < kPanelMax; ++b)
              if (b < nb) {
                const double2 g = cmulc(q, pan[b * side + i]);
                acc[b].x += g.x;
                acc[b].y += g.y;
              }
          }
#pragma unroll
          for (int b = 0; b < kPanelMax; ++b)
            if (b < nb) {
              const double2 v = warp_sum2(acc[b]);
              if (lane == 0) {
                if (nseg == 1) coef[l][b] = v;
                else cpart[(l * nseg + sg) * pw + b] = v;
              }
            }
        }
        __syncthreads();
        if (nseg > 1) {
          for (int x = threadIdx.x; x < j0 * nb; x += blockDim.x) {
            const int l = x / nb, b = x % nb;
            double2 v = cpart[(l * nseg) * pw + b];
            for (int sg = 1; sg < nseg; ++sg) {
              const double2 w2 = cpart[(l * nseg + sg) * pw + b];
              v.x += w2.x;
              v.y += w2.y;
            }
            coef[l][b] = v;
          }
          __syncthreads();
        }
        // pan -= Q[:, :j0] C, one thread per row
        for (int i = threadIdx.x; i < side; i += blockDim.x) {
          double2 v[kPanelMax];
#pragma unroll
          for (int b = 0; b < kPanelMax; ++b) v[b] = b < nb ? pan[b * side + i] : make_double2(0, 0);
#pragma unroll 4
          for (int l = 0; l < j0; ++l) {
            const double2 q = Q[static_cast<int64_t>(l) * side + i];
#pragma unroll
            for (int b = 0; b < kPanelMax; ++b) {
              const double2 d = cmul(q, coef[l][b]);
              v[b].x -= d.x;
              v[b].y -= d.y;
            }
          }
#pragma unroll
          for (int b = 0; b < kPanelMax; ++b)
            if (b < nb) pan[b * side + i] = v[b];
        }
        __syncthreads();
      }
      // classical Gram-Schmidt inside the panel
      for (int c = 0; c < nb; ++c) {
        double2* xc = pan + c * side;
        for (int cc = 0; cc < c; ++cc) {
          const double2* xq = pan + cc * side;
          double2 acc = make_double2(0, 0);
          for (int i = threadIdx.x; i < side; i += blockDim.x) {
            const double2 g = cmulc(xq[i], xc[i]);
            acc.x += g.x;
            acc.y += g.y;
          }
          acc = warp_sum2(acc);
          __syncthreads();
          if (lane == 0) {
            red[warp] = acc.x;
            red[32 + warp] = acc.y;
          }
          __syncthreads();
          double2 cf = make_double2(0, 0);
          for (int w2 = 0; w2 < nw; ++w2) {
            cf.x += red[w2];
            cf.y += red[32 + w2];
          }
          for (int i = threadIdx.x; i < side; i += blockDim.x) {
            const double2 d = cmul(xq[i], cf);
            xc[i].x -= d.x;
            xc[i].y -= d.y;
          }
        }
        __syncthreads();
        double part = 0;
        for (int i = threadIdx.x; i < side; i += blockDim.x) part += xc[i].x * xc[i].x + xc[i].y * xc[i].y;
        const double nrm = sqrt(block_sum(part, red));
        const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
        for (int i = threadIdx.x; i < side; i += blockDim.x) xc[i] = make_double2(xc[i].x * inv, xc[i].y * inv);
        __syncthreads();
      }
    }
    for (int x = threadIdx.x; x < nb * side; x += blockDim.x) Q[static_cast<int64_t>(j0) * side + x] = pan[x];
    __syncthreads();
  }
}

// BCGS2 over a thread-block cluster (round 2): the CL CTAs of a cluster own row slices
// [cr side/CL, (cr + 1) side/CL) of one block's basis, so a panel of pw columns fits
// in shared memory with pw CL times wider than one CTA could hold (cfg2: 12 columns
// instead of 3), and every previous column is re-read from memory once per panel
// and pass — 4x fewer passes over Q. Panel coefficients (Q^H pan over the slices)
// are summed across the cluster through distributed shared memory in a fixed rank
// order (deterministic); the in-panel classical Gram-Schmidt reads the other CTAs'
// panel slices directly, so every CTA computes the identical coefficients itself.
constexpr int kPanelMaxCl = 12;

template <int CL>
__global__ void __launch_bounds__(512, 1) k_bcgs2_cl(MidArgs a, int which, int pw) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double2 cl_smem[];
  __shared__ double red[2 * 32];
  const int cr = static_cast<int>(cluster.block_rank());
  const int blk = blockIdx.x / CL;
  const BlockState& s = a.st[blk];
  const int t = which == kCols ? s.tc : s.tr;
  const int side = static_cast<int>(a.side);
  const int nloc = side / CL, r0 = cr * nloc;
  double2* cl_pan = cl_smem;                                // pw x nloc (own rows)
  double2* part = cl_pan + static_cast<size_t>(pw) * nloc;  // own partial coefficients
  double2* coef = part + kSetCap * kPanelMaxCl;             // summed over the cluster
  double2* Q = (which == kCols ? a.qc : a.qr) + static_cast<int64_t>(blk) * a.S * a.side;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  auto sum_over_cluster = [&](int n) {   // coef[x] = sum over ranks of part[x], rank order
    cluster.sync();
    for (int x = threadIdx.x; x < n; x += blockDim.x) {
      double2 v = make_double2(0, 0);
      for (int rk = 0; rk < CL; ++rk) {
        const double2 w = *cluster.map_shared_rank(&part[x], rk);
        v.x += w.x;
        v.y += w.y;
      }
      coef[x] = v;
    }
    cluster.sync();                      // partials are consumed before they are rewritten
  };
  for (int j0 = 0; j0 < t; j0 += pw) {
    const int nb = min(pw, t - j0);
    for (int x = threadIdx.x; x < nb * nloc; x += blockDim.x) {
      const int b = x / nloc, i = x - b * nloc;
      cl_pan[x] = Q[static_cast<int64_t>(j0 + b) * side + r0 + i];
    }
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      if (j0 > 0) {
        // own rows of C = Q[:, :j0]^H pan, one warp per previous column
        for (int l = warp; l < j0; l += nw) {
          const double2* ql = Q + static_cast<int64_t>(l) * side + r0;
          double2 acc[kPanelMaxCl];
#pragma unroll
          for (int b = 0; b < kPanelMaxCl; ++b) acc[b] = make_double2(0, 0);
#pragma unroll 2
          for (int i = lane; i < nloc; i += 32) {
            const double2 q = ql[i];
#pragma unroll
            for (int b = 0; b < kPanelMaxCl; ++b)
              if (b < nb) {
                const double2 g = cmulc(q, cl_pan[b * nloc + i]);
                acc[b].x += g.x;
                acc[b].y += g.y;
              }
          }
#pragma unroll
          for (int b = 0; b < kPanelMaxCl; ++b)
            if (b < nb) {
              const double2 v = warp_sum2(acc[b]);
              if (lane == 0) part[l * kPanelMaxCl + b] = v;
            }
        }
        sum_over_cluster(j0 * kPanelMaxCl);
        // pan -= Q[:, :j0] C on own rows, one thread per row
        for (int i = threadIdx.x; i < nloc; i += blockDim.x) {
          double2 v[kPanelMaxCl];
#pragma unroll
          for (int b = 0; b < kPanelMaxCl; ++b) v[b] = b < nb ? cl_pan[b * nloc + i] : make_double2(0, 0);
#pragma unroll 2
          for (int l = 0; l < j0; ++l) {
            const double2 q = Q[static_cast<int64_t>(l) * side + r0 + i];
#pragma unroll
            for (int b = 0; b < kPanelMaxCl; ++b) {
              const double2 d = cmul(q, coef[l * kPanelMaxCl + b]);
              v[b].x -= d.x;
              v[b].y -= d.y;
            }
          }
#pragma unroll
          for (int b = 0; b < kPanelMaxCl; ++b)
            if (b < nb) cl_pan[b * nloc + i] = v[b];
        }
        __syncthreads();
      }
      // classical Gram-Schmidt inside the panel: column c against columns cc < c, the
      // dot products over all rows read through distributed shared memory
      for (int c = 0; c < nb; ++c) {
        cluster.sync();                  // every CTA's slice of columns <= c is current
        // coefficients of column c on columns cc < c (warp cc), then its norm (after update)
        for (int cc = warp; cc < c; cc += nw) {
          double2 acc = make_double2(0, 0);
          for (int rk = 0; rk < CL; ++rk) {
            const double2* rp = cluster.map_shared_rank(cl_pan, rk);
            for (int i = lane; i < nloc; i += 32) {
              const double2 g = cmulc(rp[cc * nloc + i], rp[c * nloc + i]);
              acc.x += g.x;
              acc.y += g.y;
            }
          }
          acc = warp_sum2(acc);
          if (lane == 0) coef[cc] = acc;
        }
        cluster.sync();                  // every CTA has read column c everywhere before updates
        for (int i = threadIdx.x; i < nloc; i += blockDim.x) {
          double2 v = cl_pan[c * nloc + i];
          for (int cc = 0; cc < c; ++cc) {
            const double2 d = cmul(cl_pan[cc * nloc + i], coef[cc]);
            v.x -= d.x;
            v.y -= d.y;
          }
          cl_pan[c * nloc + i] = v;
        }
        cluster.sync();                  // updated column c visible to every CTA
        double partn = 0;
        for (int rk = 0; rk < CL; ++rk) {
          const double2* rp = cluster.map_shared_rank(cl_pan, rk);
          double pr = 0;
          for (int i = threadIdx.x; i < nloc; i += blockDim.x) pr += rp[c * nloc + i].x * rp[c * nloc + i].x +
                                                                    rp[c * nloc + i].y * rp[c * nloc + i].y;
          partn += block_sum(pr, red);
        }
        const double nrm = sqrt(partn);
        const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
        cluster.sync();                  // all norms read before any CTA rescales its slice
        for (int i = threadIdx.x; i < nloc; i += blockDim.x)
          cl_pan[c * nloc + i] = make_double2(cl_pan[c * nloc + i].x * inv, cl_pan[c * nloc + i].y * inv);
        __syncthreads();
      }
    }
    for (int x = threadIdx.x; x < nb * nloc; x += blockDim.x) {
      const int b = x / nloc, i = x - b * nloc;
      Q[static_cast<int64_t>(j0 + b) * side + r0 + i] = cl_pan[x];
    }
    __syncthreads();
  }
  cluster.sync();                        // no CTA exits while others may read its slices
}

// pinv_floored (lowrank.py:90-94) of M (m x n) into P (n x m, row-major, ld S).
__device__ void pinv_small(const double2* M, int m, int n, int ld, double2* P, double2* U, double2* V, double* sig,
                           double2* W, double2* Vt, int* flag, int* perm, double* ssc, int S) {
  svd_small(M, m, n, ld, U, S, V, S, sig, W, Vt, flag, perm, ssc);
  const int sn = min(m, n);
  double smax = 0;
  for (int k = 0; k < sn; ++k) smax = fmax(smax, sig[k]);
  // P = V diag(finv) U^H  : P[c][a] = sum_k V[c][k] finv_k conj(U[a][k])
  for (int x = threadIdx.x; x < n * m; x += blockDim.x) {
    const int c = x / m, aa = x % m;
    double2 acc = make_double2(0, 0);
    for (int k = 0; k < sn; ++k) {
      const double fi = floored_inv(sig[k], smax);
      if (fi == 0.0) continue;
      const double2 g = cmul(V[c * S + k], cconj(U[aa * S + k]));
      acc.x += fi * g.x;
      acc.y += fi * g.y;
    }
    P[c * S + aa] = acc;
  }
  __syncthreads();
}

// Per-block small-matrix scratch (global): svd U, svd V, P1, P2, U_M, V_M, and — when the
// set capacity S exceeds 64 — the three work matrices that otherwise live in shared memory.
struct SmallBufs {
  double2 *sU, *sV, *P1, *P2, *UM, *VM, *Mb, *W, *Vt;
};
__device__ __forceinline__ SmallBufs small_bufs(const MidArgs& a, double2* smem) {
  const int64_t SS = static_cast<int64_t>(a.S) * a.S;
  double2* scr = a.scr + static_cast<int64_t>(blockIdx.x) * 9 * SS;
  SmallBufs b;
  b.sU = scr;
  b.sV = scr + SS;
  b.P1 = scr + 2 * SS;
  b.P2 = scr + 3 * SS;
  b.UM = scr + 4 * SS;
  b.VM = scr + 5 * SS;
  const bool sh = a.S <= kSmemSet;
  b.Mb = sh ? smem : scr + 6 * SS;
  b.W = sh ? smem + SS : scr + 7 * SS;
  b.Vt = sh ? smem + 2 * SS : scr + 8 * SS;
  return b;
}

// mid = pinv(qc[rows, :tc]) @ K(rows, cols) @ pinv(qr[cols, :tr]^H); SVD(mid)
// (lowrank.py:257, 284-293). Results: U_M (tc x s), V_M (tr x s), sigma, and the
// kept rank t = min(r, s) in the block state.
__global__ void __launch_bounds__(768) k_mid(MidArgs a) {
  extern __shared__ double2 sm2[];
  __shared__ int flag, perm[kSetCap];
  __shared__ double ssc[kSetCap], sg[kSetCap];
  BlockState& s = a.st[blockIdx.x];
  const int side = static_cast<int>(a.side), S = a.S;
  const int nrw = s.nrows, ncl = s.ncols, tc = s.tc, tr = s.tr;
  const SmallBufs bb = small_bufs(a, sm2);
  double2 *Mb = bb.Mb, *W = bb.W, *Vt = bb.Vt, *P1 = bb.P1, *P2 = bb.P2;
  const double2* QC = a.qc + static_cast<int64_t>(blockIdx.x) * S * a.side;
  const double2* QR = a.qr + static_cast<int64_t>(blockIdx.x) * S * a.side;
  if (tc == 0 || tr == 0) {
    if (threadIdx.x == 0) s.t = 0;
    return;
  }
  // P1 = pinv(qc[rows, :])
  for (int x = threadIdx.x; x < nrw * tc; x += blockDim.x) {
    const int i = x / tc, l = x % tc;
    Mb[i * S + l] = QC[static_cast<int64_t>(l) * side + s.rows[i]];
  }
  __syncthreads();
  pinv_small(Mb, nrw, tc, S, P1, bb.sU, bb.sV, sg, W, Vt, &flag, perm, ssc, S);
  // P2 = pinv(qr[cols, :]^H)   (tr x ncols) -> (ncols x tr)
  for (int x = threadIdx.x; x < tr * ncl; x += blockDim.x) {
    const int l = x / ncl, c = x % ncl;
    Mb[l * S + c] = cconj(QR[static_cast<int64_t>(l) * side + s.cols[c]]);
  }
  __syncthreads();
  pinv_small(Mb, tr, ncl, S, P2, bb.sU, bb.sV, sg, W, Vt, &flag, perm, ssc, S);
  // Er = K(rows, cols) into Mb ; T1 = P1 @ Er (tc x ncols) into W
  for (int x = threadIdx.x; x < nrw * ncl; x += blockDim.x) {
    const int i = x / ncl, c = x % ncl;
    Mb[i * S + c] = entry_eval(a.src, s.r0 + s.rows[i], s.c0 + s.cols[c]);
  }
  __syncthreads();
  for (int x = threadIdx.x; x < tc * ncl; x += blockDim.x) {
    const int l = x / ncl, c = x % ncl;
    double2 acc = make_double2(0, 0);
    for (int i = 0; i < nrw; ++i) {
      const double2 g = cmul(P1[l * S + i], Mb[i * S + c]);
      acc.x += g.x;
      acc.y += g.y;
    }
    W[l * S + c] = acc;
  }
  __syncthreads();
  // mid = T1 @ P2 (tc x tr) into Mb
  for (int x = threadIdx.x; x < tc * tr; x += blockDim.x) {
    const int l = x / tr, m2 = x % tr;
    double2 acc = make_double2(0, 0);
    for (int c = 0; c < ncl; ++c) {
      const double2 g = cmul(W[l * S + c], P2[c * S + m2]);
      acc.x += g.x;
      acc.y += g.y;
    }
    Mb[l * S + m2] = acc;
  }
  __syncthreads();
  svd_small(Mb, tc, tr, S, bb.UM, S, bb.VM, S, sg, W, Vt, &flag, perm, ssc);
  double* sig = a.sig + static_cast<int64_t>(blockIdx.x) * S;
  const int sn = min(tc, tr);
  for (int k = threadIdx.x; k < sn; k += blockDim.x) sig[k] = sg[k];
  if (threadIdx.x == 0) s.t = min(a.r, sn);
}

// Dense branch (r*q >= side, lowrank.py:231-234): truncated SVD of the whole block.
__global__ void k_dense(MidArgs a) {
  extern __shared__ double2 sm2[];
  __shared__ int flag, perm[kSetCap];
  __shared__ double ssc[kSetCap], sg[kSetCap];
  BlockState& s = a.st[blockIdx.x];
  const int side = static_cast<int>(a.side), S = a.S;
  const SmallBufs bb = small_bufs(a, sm2);
  for (int x = threadIdx.x; x < side * side; x += blockDim.x) {
    const int i = x / side, j = x % side;
    bb.Mb[i * S + j] = entry_eval(a.src, s.r0 + i, s.c0 + j);
  }
  __syncthreads();
  svd_small(bb.Mb, side, side, S, bb.UM, S, bb.VM, S, sg, bb.W, bb.Vt, &flag, perm, ssc);
  double* sig = a.sig + static_cast<int64_t>(blockIdx.x) * S;
  for (int k = threadIdx.x; k < side; k += blockDim.x) sig[k] = sg[k];
  if (threadIdx.x == 0) {
    s.t = a.r;
    s.tc = s.tr = -1;  // marks the dense branch for k_assemble
  }
}

// u0 sigma0 = (qc @ U_M[:, :t]) sigma, v0 sigma0 = (qr @ V_M[:, :t]) sigma, zero past t
// (_assemble, lowrank.py:284-293; the _pad_orthonormal columns meet sigma = 0 and
// vanish from u0*sigma0 / v0*sigma0, construct.py:63-65), and W = floored_inverse(sigma0).
__global__ void k_assemble(MidArgs a) {
  const BlockState& s = a.st[blockIdx.x];
  const int side = static_cast<int>(a.side), S = a.S;
  const int r = a.r, t = s.t;
  const bool dense = s.tc < 0;
  const int64_t SS = static_cast<int64_t>(S) * S;
  const double2* scr = a.scr + static_cast<int64_t>(blockIdx.x) * 9 * SS;
  const double2* UM = scr + 4 * SS;
  const double2* VM = scr + 5 * SS;
  const double* sig = a.sig + static_cast<int64_t>(blockIdx.x) * S;
  const double2* QC = a.qc + static_cast<int64_t>(blockIdx.x) * S * a.side;
  const double2* QR = a.qr + static_cast<int64_t>(blockIdx.x) * S * a.side;
  double2* uo = a.u_out + static_cast<int64_t>(blockIdx.x) * a.side * r;
  double2* vo = a.v_out + static_cast<int64_t>(blockIdx.x) * a.side * r;
  const int64_t total = static_cast<int64_t>(side) * r;
  for (int64_t x = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int i = static_cast<int>(x / r), rho = static_cast<int>(x % r);
    double2 u = make_double2(0, 0), v = make_double2(0, 0);
    if (rho < t) {
      if (dense) {
        u = UM[i * S + rho];
        v = VM[i * S + rho];
      } else {
        for (int l = 0; l < s.tc; ++l) {
          const double2 g = cmul(QC[static_cast<int64_t>(l) * side + i], UM[l * S + rho]);
          u.x += g.x;
          u.y += g.y;
        }
        for (int l = 0; l < s.tr; ++l) {
          const double2 g = cmul(QR[static_cast<int64_t>(l) * side + i], VM[l * S + rho]);
          v.x += g.x;
          v.y += g.y;
        }
      }
      const double sg = sig[rho];
      u = make_double2(u.x * sg, u.y * sg);
      v = make_double2(v.x * sg, v.y * sg);
    }
    uo[x] = u;
    vo[x] = v;
  }
  if (blockIdx.y == 0 && threadIdx.x < r) {
    double smax = 0;
    for (int k = 0; k < t; ++k) smax = fmax(smax, sig[k]);
    const int rho = threadIdx.x;
    a.w_out[static_cast<int64_t>(blockIdx.x) * r + rho] = rho < t ? floored_inv(sig[rho], smax) : 0.0;
  }
}

// k_assemble with one thread per row of the block: the basis columns are read coalesced
// (consecutive threads, consecutive rows of a column), the middle factors U_M, V_M sit in
// shared memory (broadcast reads) and each thread keeps its row's R outputs in registers.
// Same sums in the same order as k_assemble. Grid (blocks, ceil(side / 256)).
template <int R>
__global__ void __launch_bounds__(256, R <= 16 ? 2 : 1) k_assemble_rows(MidArgs a) {
  extern __shared__ double2 sm2[];
  const BlockState& s = a.st[blockIdx.x];
  const int side = static_cast<int>(a.side), S = a.S;
  const int r = a.r, t = s.t;
  const bool dense = s.tc < 0;
  const int tc = dense ? 0 : s.tc, tr = dense ? 0 : s.tr;
  const int64_t SS = static_cast<int64_t>(S) * S;
  const double2* scr = a.scr + static_cast<int64_t>(blockIdx.x) * 9 * SS;
  const double2* UM = scr + 4 * SS;
  const double2* VM = scr + 5 * SS;
  const double* sig = a.sig + static_cast<int64_t>(blockIdx.x) * S;
  double2* Us = sm2;
  double2* Vs = sm2 + static_cast<int64_t>(tc) * R;
  for (int x = threadIdx.x; x < tc * R; x += blockDim.x) {
    const int l = x / R, rho = x % R;
    Us[x] = rho < t ? UM[l * S + rho] : make_double2(0, 0);
  }
  for (int x = threadIdx.x; x < tr * R; x += blockDim.x) {
    const int l = x / R, rho = x % R;
    Vs[x] = rho < t ? VM[l * S + rho] : make_double2(0, 0);
  }
  __syncthreads();
  if (blockIdx.y == 0 && threadIdx.x < r) {
    double smax = 0;
    for (int k = 0; k < t; ++k) smax = fmax(smax, sig[k]);
    const int rho = threadIdx.x;
    a.w_out[static_cast<int64_t>(blockIdx.x) * r + rho] = rho < t ? floored_inv(sig[rho], smax) : 0.0;
  }
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= side) return;
#pragma unroll 1
  for (int which = 0; which < 2; ++which) {
    const double2* Q = (which == 0 ? a.qc : a.qr) + static_cast<int64_t>(blockIdx.x) * S * a.side + i;
    const double2* Ms = which == 0 ? Us : Vs;
    const double2* Md = which == 0 ? UM : VM;
    const int tl = which == 0 ? tc : tr;
    double2 acc[R];
#pragma unroll
    for (int rho = 0; rho < R; ++rho) acc[rho] = make_double2(0, 0);
    if (dense) {
#pragma unroll
      for (int rho = 0; rho < R; ++rho)
        if (rho < t) acc[rho] = Md[i * S + rho];
    } else {
      // eight basis values in flight per thread (the loop is bound by load latency otherwise)
      constexpr int kAhead = R <= 16 ? 8 : 4;
      for (int l0 = 0; l0 < tl; l0 += kAhead) {
        double2 q[kAhead];
#pragma unroll
        for (int j = 0; j < kAhead; ++j)
          q[j] = l0 + j < tl ? __ldcs(Q + static_cast<int64_t>(l0 + j) * side) : make_double2(0, 0);
#pragma unroll
        for (int j = 0; j < kAhead; ++j) {
          if (l0 + j >= tl) break;
          const double2* m = Ms + (l0 + j) * R;
#pragma unroll
          for (int rho = 0; rho < R; ++rho) {
            const double2 g = cmul(q[j], m[rho]);
            acc[rho].x += g.x;
            acc[rho].y += g.y;
          }
        }
      }
    }
    double2* o = (which == 0 ? a.u_out : a.v_out) + (static_cast<int64_t>(blockIdx.x) * a.side + i) * r;
#pragma unroll
    for (int rho = 0; rho < R; ++rho)
      if (rho < r) {
        const double sg = rho < t ? sig[rho] : 0.0;
        o[rho] = rho < t ? make_double2(acc[rho].x * sg, acc[rho].y * sg) : make_double2(0, 0);
      }
  }
}

// ---------------------------------------------------------------- matvec mode
// Probe product slices of block (i, j) into the tall buffer (side x width,
// column-major): kCols y_col = k_cols[i side + row, j w + c], kRows y_row =
// k_rows[j side + row, i w + c] (construct.py:114-118).
__global__ void k_fill_probe(MidArgs a, int which) {
  BlockState& s = a.st[blockIdx.x];
  const int w = a.probe_w;
  const int64_t bi = s.r0 / a.side, bj = s.c0 / a.side;
  double2* T = a.tall + static_cast<int64_t>(blockIdx.x) * a.S * a.side;
  const int64_t total = static_cast<int64_t>(w) * a.side;
  for (int64_t x = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int c = static_cast<int>(x / a.side);
    const int64_t row = x - c * a.side;
    T[x] = which == kCols ? a.kc[(bi * a.side + row) * a.ldc + bj * w + c]
                          : a.kr[(bj * a.side + row) * a.ldr + bi * w + c];
  }
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    if (which == kCols)
      s.ncols = w;
    else
      s.nrows = w;
  }
}

// Basis input of orthonormal_columns(y, width) (lowrank.py:143-154): the pivot
// columns in pick order, then canonical columns e_0, e_1, ... up to `width`.
__global__ void k_sel_probe(MidArgs a, int which) {
  BlockState& s = a.st[blockIdx.x];
  const int w = a.probe_w;
  const int npick = which == kCols ? s.tc : s.tr;
  const int32_t* piv = which == kCols ? s.pivc : s.pivr;
  const double2* T = a.tall + static_cast<int64_t>(blockIdx.x) * a.S * a.side;
  double2* Q = (which == kCols ? a.qc : a.qr) + static_cast<int64_t>(blockIdx.x) * a.S * a.side;
  const int64_t total = static_cast<int64_t>(w) * a.side;
  for (int64_t x = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int c = static_cast<int>(x / a.side);
    const int64_t row = x - c * a.side;
    Q[x] = c < npick ? T[static_cast<int64_t>(piv[c]) * a.side + row]
                     : make_double2(row == c - npick ? 1.0 : 0.0, 0.0);
  }
}

__global__ void k_set_probe_counts(MidArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.nblocks) return;
  a.st[b].tc = a.st[b].tr = a.probe_w;
}

// mid = pinv_floored(R* Q_col) (y_row* Q_row) and its SVD (svd_from_probes,
// lowrank.py:215; _assemble 284-293). The tall buffer still holds y_row.
__global__ void k_mid_probe(MidArgs a) {
  extern __shared__ double2 sm2[];
  __shared__ int flag, perm[kSetCap];
  __shared__ double ssc[kSetCap], sg[kSetCap];
  BlockState& s = a.st[blockIdx.x];
  const int side = static_cast<int>(a.side), S = a.S, w = a.probe_w;
  const int64_t bi = s.r0 / a.side;
  const SmallBufs bb = small_bufs(a, sm2);
  double2 *Mb = bb.Mb, *W = bb.W, *Vt = bb.Vt, *P1 = bb.P1;
  const double2* QC = a.qc + static_cast<int64_t>(blockIdx.x) * S * a.side;
  const double2* QR = a.qr + static_cast<int64_t>(blockIdx.x) * S * a.side;
  const double2* YR = a.tall + static_cast<int64_t>(blockIdx.x) * S * a.side;
  const double2* R = a.rprobe + bi * a.side * w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // A1 = R^H Q_col into Mb, A2 = y_row^H Q_row into P2 (both w x w, ld S)
  for (int pq = warp; pq < 2 * w * w; pq += nw) {
    const bool second = pq >= w * w;
    const int x = second ? pq - w * w : pq, ra = x / w, cb = x % w;
    double2 acc = make_double2(0, 0);
    for (int row = lane; row < side; row += 32) {
      const double2 l = second ? YR[static_cast<int64_t>(ra) * side + row] : R[static_cast<int64_t>(row) * w + ra];
      const double2 g = cmulc(l, second ? QR[static_cast<int64_t>(cb) * side + row]
                                        : QC[static_cast<int64_t>(cb) * side + row]);
      acc.x += g.x;
      acc.y += g.y;
    }
    acc = warp_sum2(acc);
    if (lane == 0) (second ? bb.P2 : Mb)[ra * S + cb] = acc;
  }
  __syncthreads();
  pinv_small(Mb, w, w, S, P1, bb.sU, bb.sV, sg, W, Vt, &flag, perm, ssc, S);
  // mid = P1 @ A2 into Mb
  for (int x = threadIdx.x; x < w * w; x += blockDim.x) {
    const int l = x / w, c = x % w;
    double2 acc = make_double2(0, 0);
    for (int k = 0; k < w; ++k) {
      const double2 g = cmul(P1[l * S + k], bb.P2[k * S + c]);
      acc.x += g.x;
      acc.y += g.y;
    }
    Mb[l * S + c] = acc;
  }
  __syncthreads();
  svd_small(Mb, w, w, S, bb.UM, S, bb.VM, S, sg, W, Vt, &flag, perm, ssc);
  double* sig = a.sig + static_cast<int64_t>(blockIdx.x) * S;
  for (int k = threadIdx.x; k < w; k += blockDim.x) sig[k] = sg[k];
  if (threadIdx.x == 0) s.t = min(a.r, w);
}

// ---------------------------------------------------------------- recursion
// One level of _recurse (construct.py:127-163) for problems [p0, p0 + np):
// splitting levels factor (part x b r) stacks (b = branching: 2, or 4 on
// quadtrees), merge-only levels (1 x b r) rows.
struct RecArgs {
  const double2* cur;   // (nb, rows, groups, r)
  double2* nxt;         // next cur
  double2* g;           // transfer blocks of this level
  double2* scr;         // per-problem scratch
  double2* rbuf;        // tall stacks up to 32 wide: R (w x w, row-major) per problem of the chunk
  int64_t nb, rows, pairs;
  int r, b, S;          // rank, branching, small-matrix capacity (64: shared memory; 128: global)
  int64_t p0;
};

__device__ void householder_r(double2* A, int m, int n, double2* R, int ldr, double* red) {
  // A (m x n) row-major in global scratch, overwritten by reflectors; R (n x n), ld ldr.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __shared__ double2 s_beta;
  __shared__ double s_vn2;
  for (int i = threadIdx.x; i < n * ldr; i += blockDim.x) R[i] = make_double2(0, 0);
  for (int p = 0; p < n; ++p) {
    double part = 0;
    for (int i = p + threadIdx.x; i < m; i += blockDim.x) part += A[i * n + p].x * A[i * n + p].x + A[i * n + p].y * A[i * n + p].y;
    const double nx2 = block_sum(part, red);
    if (threadIdx.x == 0) {
      const double2 al = A[p * n + p];
      const double nx = sqrt(nx2), aa = hypot(al.x, al.y);
      const double2 beta = aa > 0 ? make_double2(-al.x / aa * nx, -al.y / aa * nx) : make_double2(-nx, 0);
      const double2 v0 = make_double2(al.x - beta.x, al.y - beta.y);
      s_beta = beta;
      s_vn2 = nx2 - aa * aa + v0.x * v0.x + v0.y * v0.y;
      A[p * n + p] = v0;
    }
    __syncthreads();
    const double vn2 = s_vn2;
    if (vn2 > 0) {
      for (int j = p + 1 + warp; j < n; j += nw) {
        double2 w = make_double2(0, 0);
        for (int i = p + lane; i < m; i += 32) {
          const double2 g = cmulc(A[i * n + p], A[i * n + j]);
          w.x += g.x;
          w.y += g.y;
        }
        w = warp_sum2(w);
        const double f = 2.0 / vn2;
        w = make_double2(w.x * f, w.y * f);
        for (int i = p + lane; i < m; i += 32) {
          const double2 d = cmul(A[i * n + p], w);
          A[i * n + j].x -= d.x;
          A[i * n + j].y -= d.y;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) R[p * ldr + p] = vn2 > 0 ? s_beta : A[p * n + p];
    for (int j = p + 1 + threadIdx.x; j < n; j += blockDim.x) R[p * ldr + j] = A[p * n + j];
    __syncthreads();
  }
}


// One warp: Householder QR of B (rows x n) in shared memory, COLUMN-major with
// an odd leading dimension ldb (element (i, c) at B[c * ldb + i]): the norm of
// column p is a lane-strided reduction over contiguous elements, and the
// reflector is applied with one lane per trailing column (lane j walks rows of
// column j at stride 1 while v_i is a broadcast) — no shuffles in the update
// and no bank conflicts (odd ldb). On return rows 0..n-1 hold R.
__device__ void warp_householder(double2* B, int ldb, int rows, int n) {
  const int lane = threadIdx.x & 31;
  for (int p = 0; p < n && p < rows; ++p) {
    double2* vp = B + p * ldb;
    double s2 = 0;
    for (int i = p + lane; i < rows; i += 32) s2 += vp[i].x * vp[i].x + vp[i].y * vp[i].y;
    s2 = warp_sum(s2);
    const double2 al = vp[p];
    const double nx = sqrt(s2), aa = hypot(al.x, al.y);
    const double2 beta = aa > 0 ? make_double2(-al.x / aa * nx, -al.y / aa * nx) : make_double2(-nx, 0);
    const double2 v0 = make_double2(al.x - beta.x, al.y - beta.y);
    const double vn2 = s2 - aa * aa + v0.x * v0.x + v0.y * v0.y;
    __syncwarp();
    if (lane == 0) vp[p] = v0;
    __syncwarp();
    if (vn2 > 0) {
      const double f = 2.0 / vn2;
      for (int j = p + 1 + lane; j < n; j += 32) {
        double2* cj = B + j * ldb;
        double2 w0 = make_double2(0, 0), w1 = make_double2(0, 0);
        int i = p;
        for (; i + 1 < rows; i += 2) {
          const double2 g0 = cmulc(vp[i], cj[i]), g1 = cmulc(vp[i + 1], cj[i + 1]);
          w0.x += g0.x;
          w0.y += g0.y;
          w1.x += g1.x;
          w1.y += g1.y;
        }
        if (i < rows) {
          const double2 g0 = cmulc(vp[i], cj[i]);
          w0.x += g0.x;
          w0.y += g0.y;
        }
        const double2 w = make_double2((w0.x + w1.x) * f, (w0.y + w1.y) * f);
        for (i = p; i < rows; ++i) {
          const double2 d = cmul(vp[i], w);
          cj[i].x -= d.x;
          cj[i].y -= d.y;
        }
      }
    }
    __syncwarp();
    for (int i = p + 1 + lane; i < rows; i += 32) vp[i] = make_double2(0, 0);
    if (lane == 0) vp[p] = vn2 > 0 ? beta : al;
    __syncwarp();
  }
}

// Register-resident TSQR for stacks up to 32 columns wide: lane j of a warp
// keeps column j of its running R in registers (R[p][j] for p = 0..31, p
// unrolled), the incoming row chunk sits in shared memory (column-major, odd
// leading dimension: conflict-free). Reflector p acts on [R[p][:]; chunk]
// only — the rows of R below p are zero in column p — so a chunk of `ch` rows
// costs ~2 ch complex FMAs per column per step instead of ~2 (n + ch). Every
// warp of the CTA streams its own chunks; the warps' R's are then merged
// pairwise by treating one R as the next warp's chunk.
constexpr int kTsqrCh = 32;

// Fold the chunk C (rows x n, column-major, leading dimension ldc, in shared
// memory) into the lane-distributed R.
__device__ __forceinline__ void tsqr_fold(double2 (&Rc)[32], double2* C, int ldc, int rows, int n) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    if (p >= n) break;
    const double2* cp = C + p * ldc;
    double s2 = 0;
    for (int i = lane; i < rows; i += 32) s2 += cp[i].x * cp[i].x + cp[i].y * cp[i].y;
    s2 = warp_sum(s2);
    double2 al;
    al.x = __shfl_sync(0xffffffffu, Rc[p].x, p);
    al.y = __shfl_sync(0xffffffffu, Rc[p].y, p);
    if (s2 == 0.0) continue;  // the chunk column is already zero: nothing to reflect
    const double aa = hypot(al.x, al.y), nx = sqrt(aa * aa + s2);
    const double2 beta = aa > 0 ? make_double2(-al.x / aa * nx, -al.y / aa * nx) : make_double2(-nx, 0);
    const double2 v0 = make_double2(al.x - beta.x, al.y - beta.y);
    const double f = 2.0 / (v0.x * v0.x + v0.y * v0.y + s2);
    if (lane > p && lane < n) {
      double2* cj = C + lane * ldc;
      double2 d0 = cmulc(v0, Rc[p]), d1 = make_double2(0, 0);
      int i = 0;
      for (; i + 1 < rows; i += 2) {
        const double2 g0 = cmulc(cp[i], cj[i]), g1 = cmulc(cp[i + 1], cj[i + 1]);
        d0.x += g0.x;
        d0.y += g0.y;
        d1.x += g1.x;
        d1.y += g1.y;
      }
      if (i < rows) {
        const double2 g0 = cmulc(cp[i], cj[i]);
        d0.x += g0.x;
        d0.y += g0.y;
      }
      const double2 wj = make_double2((d0.x + d1.x) * f, (d0.y + d1.y) * f);
      const double2 u = cmul(v0, wj);
      Rc[p].x -= u.x;
      Rc[p].y -= u.y;
      for (i = 0; i < rows; ++i) {
        const double2 d = cmul(cp[i], wj);
        cj[i].x -= d.x;
        cj[i].y -= d.y;
      }
    }
    if (lane == p) Rc[p] = beta;
    __syncwarp();
  }
}

// R (n x n, n <= 32) of the tall (part x n) stack into Rout (row-major, ld ldr).
// smem: nwarps * (kTsqrCh + 1) * n complex values.
template <typename F>
__device__ void tsqr_reg(const F& src, int64_t part, int n, double2* smem, double2* Rout, int ldr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int ldc = kTsqrCh + 1;
  double2* C = smem + static_cast<int64_t>(warp) * ldc * n;
  double2 Rc[32];
#pragma unroll
  for (int p = 0; p < 32; ++p) Rc[p] = make_double2(0, 0);
  const int64_t nchunks = (part + kTsqrCh - 1) / kTsqrCh;
  for (int64_t cidx = warp; cidx < nchunks; cidx += nw) {
    const int64_t r0 = cidx * kTsqrCh;
    const int rows = static_cast<int>((part - r0) < kTsqrCh ? (part - r0) : kTsqrCh);
    __syncwarp();
    for (int x = lane; x < rows * n; x += 32) {
      const int i = x / n, c = x % n;
      C[c * ldc + i] = src(r0 + i, c);
    }
    __syncwarp();
    tsqr_fold(Rc, C, ldc, rows, n);
  }
  // pairwise merge: warp w + step hands its R (as an n-row chunk) to warp w
  for (int step = 1; step < nw; step *= 2) {
    __syncthreads();
    if (warp % (2 * step) == step && lane < n) {
#pragma unroll
      for (int p = 0; p < 32; ++p)
        if (p < n) C[lane * ldc + p] = Rc[p];
    }
    __syncthreads();
    if (warp % (2 * step) == 0 && warp + step < nw)
      tsqr_fold(Rc, smem + static_cast<int64_t>(warp + step) * ldc * n, ldc, n, n);
  }
  __syncthreads();
  if (warp == 0 && lane < n) {
#pragma unroll
    for (int p = 0; p < 32; ++p)
      if (p < n) Rout[p * ldr + lane] = p <= lane ? Rc[p] : make_double2(0, 0);
  }
  __syncthreads();
}

// Register TSQR, second form: the row chunk lives in registers as well (lane j: column j
// of 8 rows), reflector p's chunk column reaches every lane by shuffles and every lane
// derives the reflector itself — no shared-memory traffic, no warp reductions and no
// per-step barrier inside a fold; only the pairwise merge of the warps' R's goes through
// shared memory.
constexpr int kTsqrRows = 8;

__device__ __forceinline__ void tsqr_fold_reg(double2 (&Rc)[32], double2 (&c)[kTsqrRows], int n) {
  static_assert(kTsqrRows == 8, "the sums below are written out as trees over 8 rows");
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    if (p >= n) break;
    double2 v[kTsqrRows];
#pragma unroll
    for (int i = 0; i < kTsqrRows; ++i) {
      v[i].x = __shfl_sync(full, c[i].x, p);
      v[i].y = __shfl_sync(full, c[i].y, p);
    }
    double2 al;
    al.x = __shfl_sync(full, Rc[p].x, p);
    al.y = __shfl_sync(full, Rc[p].y, p);
    // |v|^2 and v^H c as balanced trees (the dependent-DFMA latency is the fold's critical
    // path): every product is independent, three levels of adds
    double q[kTsqrRows];
    double2 e[kTsqrRows];
#pragma unroll
    for (int i = 0; i < kTsqrRows; ++i) {
      q[i] = fma(v[i].x, v[i].x, v[i].y * v[i].y);
      e[i].x = fma(v[i].x, c[i].x, v[i].y * c[i].y);    // conj(v) * c
      e[i].y = fma(v[i].x, c[i].y, -(v[i].y * c[i].x));
    }
    const double s2 = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
    if (s2 == 0.0) continue;  // the chunk column is already zero: nothing to reflect (uniform)
    double2 d;
    d.x = ((e[0].x + e[1].x) + (e[2].x + e[3].x)) + ((e[4].x + e[5].x) + (e[6].x + e[7].x));
    d.y = ((e[0].y + e[1].y) + (e[2].y + e[3].y)) + ((e[4].y + e[5].y) + (e[6].y + e[7].y));
    // reflector: beta = -al / |al| * nx, v0 = al - beta, f = 2 / (|v0|^2 + s2) = 1 / (nx (nx + |al|))
    const double aa2 = fma(al.x, al.x, al.y * al.y);
    const double nx = sqrt(aa2 + s2);
    const double ra = aa2 > 0 ? rsqrt(aa2) : 0.0;
    const double aa = aa2 * ra;
    const double f = 1.0 / (nx * (nx + aa));
    const double sc = -nx * ra;
    const double2 beta = aa2 > 0 ? make_double2(al.x * sc, al.y * sc) : make_double2(-nx, 0);
    const double2 v0 = make_double2(al.x - beta.x, al.y - beta.y);
    if (lane > p && lane < n) {
      const double2 h = cmulc(v0, Rc[p]);
      const double2 wj = make_double2((d.x + h.x) * f, (d.y + h.y) * f);
      const double2 u = cmul(v0, wj);
      Rc[p].x -= u.x;
      Rc[p].y -= u.y;
#pragma unroll
      for (int i = 0; i < kTsqrRows; ++i) {
        c[i].x = fma(-v[i].x, wj.x, fma(v[i].y, wj.y, c[i].x));
        c[i].y = fma(-v[i].x, wj.y, fma(-v[i].y, wj.x, c[i].y));
      }
    }
    if (lane == p) Rc[p] = beta;
  }
}

// One reflector step of the register fold with R's row p in Rrow (see tsqr_fold_roll).
template <int CH>
__device__ __forceinline__ void tsqr_step_reg(double2& Rrow, double2 (&c)[CH], int p, int n) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double2 v[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    v[i].x = __shfl_sync(full, c[i].x, p);
    v[i].y = __shfl_sync(full, c[i].y, p);
  }
  double2 al;
  al.x = __shfl_sync(full, Rrow.x, p);
  al.y = __shfl_sync(full, Rrow.y, p);
  // |v|^2 and v^H c on two accumulators each
  double s2a = 0, s2b = 0;
  double2 d0 = make_double2(0, 0), d1 = make_double2(0, 0);
#pragma unroll
  for (int i = 0; i < CH; i += 2) {
    s2a = fma(v[i].x, v[i].x, fma(v[i].y, v[i].y, s2a));
    s2b = fma(v[i + 1].x, v[i + 1].x, fma(v[i + 1].y, v[i + 1].y, s2b));
    d0.x = fma(v[i].x, c[i].x, fma(v[i].y, c[i].y, d0.x));  // conj(v) * c
    d0.y = fma(v[i].x, c[i].y, fma(-v[i].y, c[i].x, d0.y));
    d1.x = fma(v[i + 1].x, c[i + 1].x, fma(v[i + 1].y, c[i + 1].y, d1.x));
    d1.y = fma(v[i + 1].x, c[i + 1].y, fma(-v[i + 1].y, c[i + 1].x, d1.y));
  }
  const double s2 = s2a + s2b;
  // reflector: beta = -al / |al| * nx, v0 = al - beta, f = 2 / (|v0|^2 + s2) = 1 / (nx (nx + |al|));
  // a zero chunk column (s2 = 0) leaves everything as it is (f = 0, beta = al)
  const bool live = s2 > 0.0;
  const double aa2 = fma(al.x, al.x, al.y * al.y);
  const double nx = sqrt(aa2 + s2);
  const double ra = aa2 > 0 ? rsqrt(aa2) : 0.0;
  const double aa = aa2 * ra;
  const double f = live ? 1.0 / (nx * (nx + aa)) : 0.0;
  const double sc = -nx * ra;
  const double2 beta = !live ? al : aa2 > 0 ? make_double2(al.x * sc, al.y * sc) : make_double2(-nx, 0);
  const double2 v0 = make_double2(al.x - beta.x, al.y - beta.y);
  if (lane > p && lane < n) {
    const double2 h = cmulc(v0, Rrow);
    const double2 wj = make_double2(((d0.x + d1.x) + h.x) * f, ((d0.y + d1.y) + h.y) * f);
    const double2 u = cmul(v0, wj);
    Rrow.x -= u.x;
    Rrow.y -= u.y;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      c[i].x = fma(-v[i].x, wj.x, fma(v[i].y, wj.y, c[i].x));
      c[i].y = fma(-v[i].x, wj.y, fma(-v[i].y, wj.x, c[i].y));
    }
  }
  if (lane == p) Rrow = beta;
}

// The fold as a rolled loop: four reflector steps on Rc[0..3], then the register R rotated
// by four rows, eight times (back in place) — a loop body of ~1k instructions instead of
// 32 unrolled steps (the unrolled fold overflows the instruction cache).
__device__ __forceinline__ void tsqr_fold_roll(double2 (&Rc)[32], double2 (&c)[kTsqrRows], int n) {
#pragma unroll 1
  for (int p0 = 0; p0 < 32; p0 += 4) {
    if (p0 < n) {
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (p0 + s < n) tsqr_step_reg<kTsqrRows>(Rc[s], c, p0 + s, n);
    }
    const double2 t0 = Rc[0], t1 = Rc[1], t2 = Rc[2], t3 = Rc[3];
#pragma unroll
    for (int k = 0; k < 28; ++k) Rc[k] = Rc[k + 4];
    Rc[28] = t0;
    Rc[29] = t1;
    Rc[30] = t2;
    Rc[31] = t3;
  }
}

// R of every tall stack (up to 32 wide) of the chunk -> a.rbuf, one warp (one 32-thread
// CTA) per problem: no merges, no barriers, uniform control flow. The running R sits in
// shared memory as a packed upper triangle (8.4 KB; lane j touches only column j, one
// load and one store per reflector), the CH-row chunk in registers: ~100 registers, so
// 16-20 problems share an SM and hide each other's sqrt / divide chains.
__device__ __host__ __forceinline__ int tri_off(int p) { return p * 32 - (p * (p - 1)) / 2 - p; }
constexpr int kTriElems = 528;

template <int CH>
__global__ void __launch_bounds__(32) k_recurse_tsqr1(RecArgs a) {
  extern __shared__ double2 sm2[];
  const int lane = threadIdx.x;
  const int64_t idx = blockIdx.x;
  const int64_t prob = a.p0 + idx;
  const int b = a.b;
  const int64_t pairs = a.pairs, part = a.rows / b;
  const int n = b * a.r;
  const int64_t gb = prob / (b * pairs), t = (prob / pairs) % b, p = prob % pairs;
  const double2* base = a.cur + ((gb * a.rows + t * part) * pairs + p) * n + lane;
  const int64_t rstride = pairs * n;
  for (int x = lane; x < kTriElems; x += 32) sm2[x] = make_double2(0, 0);
  __syncwarp();
#pragma unroll 1
  for (int64_t r0 = 0; r0 < part; r0 += CH) {
    double2 c[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i)
      c[i] = (lane < n && r0 + i < part) ? __ldcs(base + (r0 + i) * rstride) : make_double2(0, 0);
#pragma unroll 1
    for (int q = 0; q < n; ++q) {
      double2* rp = sm2 + tri_off(q) + lane;
      double2 Rrow = lane >= q ? *rp : make_double2(0, 0);
      tsqr_step_reg<CH>(Rrow, c, q, n);
      if (lane >= q) *rp = Rrow;
    }
  }
  __syncwarp();
  if (lane < n) {
    double2* Rout = a.rbuf + idx * static_cast<int64_t>(n) * n;
    for (int q = 0; q < n; ++q) Rout[q * n + lane] = q <= lane ? sm2[tri_off(q) + lane] : make_double2(0, 0);
  }
}

// R of every tall stack (up to 32 wide) of the chunk -> a.rbuf, W warps per problem
// (W = 1, 2, 4 or 8: 8 / W problems per CTA), each warp folding 8-row chunks into its
// register R; the group's R's are merged pairwise through shared memory.
__global__ void __launch_bounds__(256, 1) k_recurse_tsqr2(RecArgs a, int64_t cnt, int W) {
  extern __shared__ double2 sm2[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wl = warp % W;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * (8 / W) + warp / W;
  const bool active = idx < cnt;
  const int64_t prob = a.p0 + (active ? idx : 0);
  const int b = a.b;
  const int64_t pairs = a.pairs, part = a.rows / b;
  const int n = b * a.r;
  const int64_t gb = prob / (b * pairs), t = (prob / pairs) % b, p = prob % pairs;
  const double2* base = a.cur + ((gb * a.rows + t * part) * pairs + p) * n + lane;
  const int64_t rstride = pairs * n;
  const int ldc = 33;
  double2 Rc[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) Rc[q] = make_double2(0, 0);
  if (active) {
    const int64_t nchunks = (part + kTsqrRows - 1) / kTsqrRows;
    for (int64_t cidx = wl; cidx < nchunks; cidx += W) {
      const int64_t r0 = cidx * kTsqrRows;
      double2 c[kTsqrRows];
#pragma unroll
      for (int i = 0; i < kTsqrRows; ++i)
        c[i] = (lane < n && r0 + i < part) ? __ldcs(base + (r0 + i) * rstride) : make_double2(0, 0);
      tsqr_fold_roll(Rc, c, n);
    }
  }
  double2* mine = sm2 + static_cast<int64_t>(warp) * ldc * 32;
  for (int step = 1; step < W; step *= 2) {
    __syncthreads();
    if (wl % (2 * step) == step && lane < n) {
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q < n) mine[lane * ldc + q] = Rc[q];
    }
    __syncthreads();
    if (active && wl % (2 * step) == 0 && wl + step < W) {
      const double2* other = sm2 + static_cast<int64_t>(warp + step) * ldc * 32;
      for (int i0 = 0; i0 < n; i0 += kTsqrRows) {
        double2 c[kTsqrRows];
#pragma unroll
        for (int i = 0; i < kTsqrRows; ++i)
          c[i] = (lane < n && i0 + i < n) ? other[lane * ldc + i0 + i] : make_double2(0, 0);
        tsqr_fold_roll(Rc, c, n);
      }
    }
  }
  if (active && wl == 0 && lane < n) {
    double2* Rout = a.rbuf + idx * static_cast<int64_t>(n) * n;
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (q < n) Rout[q * n + lane] = q <= lane ? Rc[q] : make_double2(0, 0);
  }
}

// R factor of a tall (part x n) stack by TSQR in shared memory: warps stream
// row chunks into [R_acc; chunk] buffers (column-major, odd ld) and QR them (no
// block barriers), then combine their R's pairwise. Leaves R (n x n, row-major)
// in Rout (ld ldr). smem must hold nwu * tsqr_ld(n, ch) * n complex values.
__device__ __host__ __forceinline__ int tsqr_ld(int n, int ch) { return (n + ch) | 1; }

template <typename F>
__device__ void tsqr_r(const F& src, int64_t part, int n, double2* smem, int nwu, int ch, double2* Rout, int ldr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ldb = tsqr_ld(n, ch);
  double2* B = smem + static_cast<int64_t>(warp) * ldb * n;
  const int64_t nchunks = (part + ch - 1) / ch;
  if (warp < nwu) {
    for (int x = lane; x < ldb * n; x += 32) B[x] = make_double2(0, 0);
    for (int64_t cidx = warp; cidx < nchunks; cidx += nwu) {
      const int64_t r0 = cidx * ch;
      const int rows = static_cast<int>((part - r0) < ch ? (part - r0) : ch);
      __syncwarp();
      for (int x = lane; x < rows * n; x += 32) {
        const int i = x / n, c = x % n;
        B[c * ldb + n + i] = src(r0 + i, c);
      }
      __syncwarp();
      warp_householder(B, ldb, n + rows, n);
    }
  }
  __syncthreads();
  for (int step = 1; step < nwu; step *= 2) {
    if (warp < nwu && warp % (2 * step) == 0 && warp + step < nwu) {
      const double2* B2 = smem + static_cast<int64_t>(warp + step) * ldb * n;
      for (int x = lane; x < n * n; x += 32) {
        const int c = x / n, i = x % n;
        B[c * ldb + n + i] = B2[c * ldb + i];
      }
      __syncwarp();
      warp_householder(B, ldb, 2 * n, n);
    }
    __syncthreads();
  }
  // R of warp 0 -> Rout (through registers: Rout may overlap the warp buffers)
  double2 vals[16];
  int cnt = 0;
  const int ldb0 = tsqr_ld(n, ch);
  for (int x = threadIdx.x; x < n * n && cnt < 16; x += blockDim.x) vals[cnt++] = smem[(x % n) * ldb0 + x / n];
  __syncthreads();
  cnt = 0;
  for (int x = threadIdx.x; x < n * n && cnt < 16; x += blockDim.x) {
    const int i = x / n, c = x % n;
    Rout[i * ldr + c] = i <= c ? vals[cnt] : make_double2(0, 0);
    ++cnt;
  }
  __syncthreads();
}

// Per-problem global scratch: [Ac: max(part, S) x w][Ug: S x S][Vg: S x S][Mb, W, Vt: S x S each when S > 64].
__device__ __host__ __forceinline__ int64_t rec_scratch_elems(int64_t part, int w, int S) {
  // shared-memory problems (S <= kSmemSet) keep only U and V in global scratch
  return S <= kSmemSet ? 2ll * S * S : (part > S ? part : S) * w + 5ll * S * S;
}

// dynamic shared memory of k_recurse_split when S <= kSmemSet (see its layout)
__device__ __host__ __forceinline__ int64_t rec_smem_elems(int w, int S) {
  return static_cast<int64_t>(S) * (w + 1) + static_cast<int64_t>(S) * w + static_cast<int64_t>(w) * (w + 1);
}

// Register TSQR of every tall stack (up to 32 wide) of the chunk: R -> a.rbuf.
// Its own kernel: the 128-register R columns would otherwise cap the SVD kernel
// at one CTA per SM; here all 8 warps stream chunks, there the Jacobi runs 2 per SM.
__global__ void k_recurse_tsqr(RecArgs a) {
  extern __shared__ double2 sm2[];
  const int64_t prob = a.p0 + blockIdx.x;
  const int b = a.b;
  const int64_t pairs = a.pairs, part = a.rows / b;
  const int w = b * a.r;
  const int64_t gb = prob / (b * pairs), t = (prob / pairs) % b, p = prob % pairs;
  auto src = [&](int64_t row, int c) { return a.cur[((gb * a.rows + t * part + row) * pairs + p) * w + c]; };
  tsqr_reg(src, part, w, sm2, a.rbuf + static_cast<int64_t>(blockIdx.x) * w * w, w);
}

// TALL = false: stacks of at most S rows (direct Jacobi); TALL = true: taller stacks
// (R from k_recurse_tsqr when the stack is at most 32 wide, else a TSQR / Householder
// pass here).
template <bool TALL>
__global__ void __launch_bounds__(TALL ? 256 : 512, 2) k_recurse_split(RecArgs a) {
  extern __shared__ double2 sm2[];
  __shared__ int flag, perm[kSetCap];
  __shared__ double ssc[kSetCap], sg[kSetCap], red[32];
  const int64_t prob = a.p0 + blockIdx.x;
  const int b = a.b, S = a.S;
  const int64_t pairs = a.pairs, part = a.rows / b;
  const int w = b * a.r, r = a.r;
  const int64_t gb = prob / (b * pairs), t = (prob / pairs) % b, p = prob % pairs;
  // paired = cur.reshape(nb, rows, pairs, b r); stack t takes rows [t*part, (t+1)*part)
  auto src = [&](int64_t row, int c) { return a.cur[((gb * a.rows + t * part + row) * pairs + p) * w + c]; };
  const int keep = static_cast<int>(part < r ? part : r);
  const int64_t SS = static_cast<int64_t>(S) * S;
  double2* Ac = a.scr + static_cast<int64_t>(blockIdx.x) * rec_scratch_elems(part, w, S);
  double2* Ug = S <= kSmemSet ? Ac : Ac + (part > S ? part : S) * w;
  double2* Vg = Ug + SS;
  const bool sh = S <= kSmemSet;
  // shared layout (S <= 64): Mb (S x (w+1)) | W (S x w) | Vt (w x (w+1)), odd row
  // strides (rec_smem_elems); global scratch (S = 128) keeps stride S
  const int ldm = sh ? w + 1 : S;
  double2* Mb = sh ? sm2 : Vg + SS;
  double2* W = sh ? sm2 + S * ldm : Vg + 2 * SS;
  double2* Vt = sh ? W + S * w : Vg + 3 * SS;
  const int64_t out_base = ((gb * b + t) * part) * pairs + p;  // new_u.transpose(0,1,3,2,4): row (gb,t,row=0,p)
  // stacks up to S rows go straight to the Jacobi SVD; taller ones through a TSQR first
  // (the register TSQR for stacks up to 32 columns wide)
  const bool wreg = sh && w <= 32;
  if constexpr (!TALL) {
    for (int x = threadIdx.x; x < part * w; x += blockDim.x) Mb[(x / w) * ldm + x % w] = src(x / w, x % w);
    __syncthreads();
    svd_small(Mb, static_cast<int>(part), w, ldm, Ug, S, Vg, S, sg, W, Vt, &flag, perm, ssc);
    for (int x = threadIdx.x; x < part * r; x += blockDim.x) {
      const int row = x / r, rho = x % r;
      double2 u = make_double2(0, 0);
      if (rho < keep) u = make_double2(Ug[row * S + rho].x * sg[rho], Ug[row * S + rho].y * sg[rho]);
      a.nxt[(out_base + row * pairs) * r + rho] = u;
    }
  } else {
    // tall stack: R factor (TSQR in shared memory when the stack width fits, else a
    // Householder pass in global memory); the SVD of R gives sigma and V; new_u = A V[:, :keep]
    if (wreg) {
      const double2* R = a.rbuf + static_cast<int64_t>(blockIdx.x) * w * w;
      for (int x = threadIdx.x; x < w * w; x += blockDim.x) Mb[(x / w) * ldm + x % w] = R[x];
      __syncthreads();
    } else if (sh) {
      const int ch = 32;
      const int per = tsqr_ld(w, ch) * w;
      int nwu = static_cast<int>(rec_smem_elems(w, S) / per);
      nwu = nwu < 1 ? 1 : (nwu > static_cast<int>(blockDim.x >> 5) ? static_cast<int>(blockDim.x >> 5) : nwu);
      tsqr_r(src, part, w, sm2, nwu, ch, Mb, ldm);
    } else {
      for (int64_t x = threadIdx.x; x < part * w; x += blockDim.x) Ac[x] = src(x / w, static_cast<int>(x % w));
      __syncthreads();
      householder_r(Ac, static_cast<int>(part), w, Mb, ldm, red);
      __syncthreads();
    }
    svd_small(Mb, w, w, ldm, Ug, S, Vg, S, sg, W, Vt, &flag, perm, ssc);
    for (int x = threadIdx.x; x < w * w; x += blockDim.x) Vt[(x / w) * ldm + x % w] = Vg[(x / w) * S + x % w];
    __syncthreads();
    for (int64_t x = threadIdx.x; x < part * r; x += blockDim.x) {
      const int64_t row = x / r;
      const int rho = static_cast<int>(x % r);
      double2 u = make_double2(0, 0);
      if (rho < keep)
        for (int c = 0; c < w; ++c) {
          const double2 g = cmul(src(row, c), Vt[c * ldm + rho]);
          u.x += g.x;
          u.y += g.y;
        }
      a.nxt[(out_base + row * pairs) * r + rho] = u;
    }
  }
  __syncthreads();
  // transfer block G = vh[:keep] zero-padded to (r x b r): G[rho][c] = conj(V[c][rho])
  double2* G = a.g + prob * static_cast<int64_t>(r) * w;
  for (int x = threadIdx.x; x < r * w; x += blockDim.x) {
    const int rho = x / w, c = x % w;
    G[x] = rho < keep ? cconj(Vg[c * S + rho]) : make_double2(0, 0);
  }
}

// Stacks up to 32 columns wide, one warp per problem: Jacobi on the columns of R^H (R from
// k_recurse_tsqr, or the stack itself when it has at most 32 rows — zero rows below), held
// one column per lane in registers. R^H J = V Sigma gives sigma and the right singular
// vectors of the stack directly; no rotation matrix is accumulated and nothing lives in
// shared memory, so 12 problems share an SM. Writes the transfer block G = vh[:keep]
// (zero-padded rows); new_u = A conj(G)^T follows in k_recurse_av.
template <int RR, int MINB>
__global__ void __launch_bounds__(128, MINB) k_recurse_wsvd(RecArgs a, int64_t cnt, int from_r) {
  const int lane = threadIdx.x & 31;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * 4 + (threadIdx.x >> 5);
  if (idx >= cnt) return;
  const int64_t prob = a.p0 + idx;
  const int b = a.b, r = a.r, w = b * a.r;
  const int64_t pairs = a.pairs, part = a.rows / b;
  const int64_t gb = prob / (b * pairs), t = (prob / pairs) % b, p = prob % pairs;
  const int keep = static_cast<int>(part < r ? part : r);
  const int cc = from_r ? w : static_cast<int>(part);  // rows of R (or of the short stack) = columns of its adjoint
  const double2* rowp = from_r ? a.rbuf + idx * static_cast<int64_t>(w) * w + static_cast<int64_t>(lane) * w
                               : a.cur + ((gb * a.rows + t * part + lane) * pairs + p) * w;
  double2 col[RR];
#pragma unroll
  for (int k = 0; k < RR; ++k) col[k] = (lane < cc && k < w) ? cconj(rowp[k]) : make_double2(0, 0);
  warp_jacobi_reg<RR>(col, cc, static_cast<int>(blockIdx.z));
  double nrm = 0;
#pragma unroll
  for (int k = 0; k < RR; ++k) nrm += col[k].x * col[k].x + col[k].y * col[k].y;
  nrm = lane < cc ? sqrt(nrm) : -1.0;
  int rank = 0;
  for (int d = 0; d < cc; ++d) {
    const double o = __shfl_sync(0xffffffffu, nrm, d);
    rank += (o > nrm) || (o == nrm && d < lane);
  }
  // G[rho][c] = conj(V[c][rho]), V[:, rho] = column / sigma of the lane ranked rho
  double2* G = a.g + prob * static_cast<int64_t>(r) * w;
  if (lane < cc && rank < keep) {
    double2* row = G + static_cast<int64_t>(rank) * w;
    const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
#pragma unroll
    for (int k = 0; k < RR; ++k)
      if (k < w) row[k] = make_double2(col[k].x * inv, -col[k].y * inv);
  }
  for (int x = keep * w + lane; x < r * w; x += 32) G[x] = make_double2(0, 0);
}

// new_u = A V[:, :keep] = A conj(G)^T for the problems of a chunk: one CTA per (problem,
// 128-row tile), each thread two rows by four ranks.
__global__ void __launch_bounds__(256) k_recurse_av(RecArgs a, int tiles) {
  extern __shared__ double2 sm2[];  // Vt[c][rho], w x R4
  const int64_t idx = blockIdx.x / tiles;
  const int tile = blockIdx.x % tiles;
  const int64_t prob = a.p0 + idx;
  const int b = a.b, r = a.r, w = b * a.r;
  const int R4 = (r + 3) & ~3;
  const int64_t pairs = a.pairs, part = a.rows / b;
  const int64_t gb = prob / (b * pairs), t = (prob / pairs) % b, p = prob % pairs;
  const double2* G = a.g + prob * static_cast<int64_t>(r) * w;
  for (int x = threadIdx.x; x < R4 * w; x += blockDim.x) {
    const int rho = x / w, c = x % w;
    sm2[c * R4 + rho] = rho < r ? cconj(G[x]) : make_double2(0, 0);
  }
  __syncthreads();
  const int rho0 = (threadIdx.x & 3) * 4;
  const int64_t row0 = static_cast<int64_t>(tile) * 128 + (threadIdx.x >> 2) * 2;
  if (rho0 >= r || row0 >= part) return;
  const bool two = row0 + 1 < part;
  const double2* a0 = a.cur + ((gb * a.rows + t * part + row0) * pairs + p) * w;
  const double2* a1 = two ? a0 + pairs * w : a0;
  double2 acc[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0, 0);
#pragma unroll 4
  for (int c = 0; c < w; ++c) {
    const double2 x0 = a0[c], x1 = a1[c];
    const double2* v = sm2 + c * R4 + rho0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 vj = v[j];
      acc[0][j].x = fma(x0.x, vj.x, fma(-x0.y, vj.y, acc[0][j].x));
      acc[0][j].y = fma(x0.x, vj.y, fma(x0.y, vj.x, acc[0][j].y));
      acc[1][j].x = fma(x1.x, vj.x, fma(-x1.y, vj.y, acc[1][j].x));
      acc[1][j].y = fma(x1.x, vj.y, fma(x1.y, vj.x, acc[1][j].y));
    }
  }
  const int64_t out_base = ((gb * b + t) * part) * pairs + p;  // new_u.transpose(0,1,3,2,4): row (gb,t,row=0,p)
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (i == 1 && !two) break;
    double2* o = a.nxt + (out_base + (row0 + i) * pairs) * r + rho0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (rho0 + j < r) o[j] = acc[i][j];
  }
}

__global__ void k_recurse_merge(RecArgs a, int64_t nprob) {
  // (1 x b r) rows: sigma = |row|, vh = row / sigma; new_u = (sigma, 0, ..., 0)
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int64_t prob = a.p0 + warp;
  if (prob >= a.p0 + nprob) return;
  const int w = a.b * a.r, r = a.r;
  const double2* row = a.cur + prob * w;
  double acc = 0;
  for (int c = lane; c < w; c += 32) acc += row[c].x * row[c].x + row[c].y * row[c].y;
  const double sgm = sqrt(warp_sum(acc));
  double2* G = a.g + prob * static_cast<int64_t>(r) * w;
  for (int x = lane; x < r * w; x += 32) {
    const int rho = x / w, c = x % w;
    G[x] = (rho == 0 && sgm > 0) ? make_double2(row[c].x / sgm, row[c].y / sgm) : make_double2(0, 0);
  }
  const int64_t gb = prob / a.pairs, p = prob % a.pairs;
  for (int rho = lane; rho < r; rho += 32)
    a.nxt[(gb * a.pairs + p) * r + rho] = make_double2(rho == 0 ? sgm : 0.0, 0);
}

}  // namespace bfly

using namespace bfly;

namespace {

// Set capacity for a launch: |rows|, |cols| <= r q + r (or side in the dense branch).
int set_capacity(uint64_t side, uint32_t rank, uint32_t q_over) {
  const uint64_t rq = static_cast<uint64_t>(rank) * q_over;
  const uint64_t need = rq >= side ? side : rq + rank;
  return need <= static_cast<uint64_t>(kSmemSet) ? kSmemSet : (need <= static_cast<uint64_t>(kSetCap) ? kSetCap : -1);
}

uint64_t mid_ws_layout(uint64_t side, uint32_t nblocks, int S, uint64_t* off) {
  uint64_t o = 0;
  auto take = [&](uint64_t bytes) {
    const uint64_t r = o;
    o += (bytes + 255) / 256 * 256;
    return r;
  };
  off[0] = take(sizeof(BlockState) * nblocks);
  off[1] = take(16ull * nblocks * S * side);  // wide
  off[2] = take(16ull * nblocks * S * side);  // tall
  off[3] = take(16ull * nblocks * S * side);  // qc
  off[4] = take(16ull * nblocks * S * side);  // qr
  off[5] = take(16ull * nblocks * side);      // qbuf
  off[6] = take(16ull * nblocks * 9 * S * S); // small-matrix scratch
  off[7] = take(8ull * nblocks * S);          // sig
  return o;
}

// Orthonormal bases of the selected columns: BCGS2 with a shared-memory panel of up to
// kPanelMax columns when at least two fit, else column-by-column CGS2.
int env_int_c(const char* name, int dflt);

template <int CL>
cudaError_t launch_bcgs2_cl(const MidArgs& a, uint32_t nblocks, int which, cudaStream_t st) {
  auto* kern = k_bcgs2_cl<CL>;
  const int64_t slice_bytes = (a.side / CL) * static_cast<int64_t>(sizeof(double2));
  const int pw = static_cast<int>(std::min<int64_t>(kPanelMaxCl, (150 * 1024) / slice_bytes));
  const size_t smem = static_cast<size_t>(pw) * slice_bytes + 2ull * kSetCap * kPanelMaxCl * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nblocks * CL);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, which, pw);
}

void launch_basis(const MidArgs& a, uint32_t nblocks, int which, cudaStream_t st) {
  // the cluster form is opt-in (BF_BCGS2_CL=1): at cfg2 it reads Q 4x less but measures a
  // 66.4 ms block-row against 38.2 ms — a quarter of the blocks in flight, and four cluster
  // barriers plus distributed-shared-memory dot products per panel column
  static const bool cl_on = env_int_c("BF_BCGS2_CL", 0) != 0;
  if (cl_on && a.side >= 4096 && launch_bcgs2_cl<4>(a, nblocks, which, st) == cudaSuccess) return;
  if (cl_on && a.side >= 2048 && a.side < 4096 && launch_bcgs2_cl<2>(a, nblocks, which, st) == cudaSuccess) return;
  const int64_t col_bytes = a.side * static_cast<int64_t>(sizeof(double2));
  int pw = static_cast<int>(std::min<int64_t>(kPanelMax, (200 * 1024) / col_bytes));
  if (getenv("BF_CGS2")) pw = 0;
  if (pw >= 2) {
    allow_max_dyn_smem(k_bcgs2);
    // coefficient sweeps split into row segments while the partial sums fit next to the panel
    static const int seg_env = env_int_c("BF_BCGS2_SEG", 4);
    int nseg = std::max(1, std::min(8, seg_env));
    size_t smem = static_cast<size_t>(pw) * col_bytes + static_cast<size_t>(a.S) * nseg * pw * sizeof(double2);
    if (nseg == 1 || smem > 207 * 1024) {
      nseg = 1;
      smem = static_cast<size_t>(pw) * col_bytes;
    }
    k_bcgs2<<<nblocks, 1024, smem, st>>>(a, which, pw, nseg);
  } else {
    k_cgs2<<<nblocks, 512, 0, st>>>(a, which);
  }
}

bool tree_geometry(uint64_t n, uint32_t levels, uint32_t branching, uint64_t* m, uint64_t* side) {
  if (branching != 2 && branching != 4) return false;
  const uint32_t lb = branching == 4 ? 2 : 1;
  if (n < 4 || (n & (n - 1)) || levels < 2 || levels % 2 || levels > 40) return false;
  if (branching == 4 && ((63 - __builtin_clzll(n)) % 2)) return false;
  if (lb * (levels / 2) >= 63 || (1ull << (lb * (levels / 2))) > n) return false;
  *m = 1ull << (lb * (levels / 2));
  *side = n / *m;
  return true;
}

}  // namespace

namespace {

int env_int_c(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

// _assemble: one thread per block row with the middle factors in shared memory (ranks up
// to 32); BF_ASSEMBLE_OLD=1 or a larger rank keeps the thread-per-output kernel.
cudaError_t launch_assemble(const MidArgs& a, unsigned nblocks, cudaStream_t st) {
  static const bool old = env_int_c("BF_ASSEMBLE_OLD", 0) != 0;
  const int T = 256;
  if (old || a.r > 32) {
    const unsigned yas = static_cast<unsigned>(std::min<uint64_t>(32, (a.side * a.r + T - 1) / T));
    k_assemble<<<dim3(nblocks, yas), T, 0, st>>>(a);
    return cudaGetLastError();
  }
  const int R = a.r <= 4 ? 4 : a.r <= 8 ? 8 : a.r <= 16 ? 16 : 32;
  const size_t smem = 2ull * a.S * R * sizeof(double2);
  const dim3 grid(nblocks, static_cast<unsigned>((a.side + T - 1) / T));
  cudaError_t e = cudaSuccess;
  switch (R) {
    case 4: e = allow_max_dyn_smem(k_assemble_rows<4>); k_assemble_rows<4><<<grid, T, smem, st>>>(a); break;
    case 8: e = allow_max_dyn_smem(k_assemble_rows<8>); k_assemble_rows<8><<<grid, T, smem, st>>>(a); break;
    case 16: e = allow_max_dyn_smem(k_assemble_rows<16>); k_assemble_rows<16><<<grid, T, smem, st>>>(a); break;
    default: e = allow_max_dyn_smem(k_assemble_rows<32>); k_assemble_rows<32><<<grid, T, smem, st>>>(a); break;
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Greedy sweep pivots: the cluster kernel (k_pivot_wide_cl) for samples of >= 1024
// columns, one CTA per SM (shared-memory request above half the SM) so that only
// 148/CL blocks' samples are live in L2; BF_NO_PIVOT_CLUSTER=1 keeps one CTA per block.
template <int CL>
cudaError_t launch_pivot_cl(const MidArgs& a, int which, int nblocks, cudaStream_t st) {
  // register form (one barrier per pick, no global projection rows) when it applies;
  // BF_PIVOT_CL2=0 keeps the two-barrier kernel
  static const bool cl2 = env_int_c("BF_PIVOT_CL2", 1) != 0;
  const bool use2 = cl2 && a.r <= kPivReg && a.side / CL <= 512;
  void (*kern)(MidArgs, int) = use2 ? k_pivot_wide_cl2<CL> : k_pivot_wide_cl<CL>;
  const int per_sm = std::max(1, std::min(4, env_int_c("BF_PIVOT_CTAS_PER_SM", 1)));
  const size_t need = use2 ? static_cast<size_t>(kPivReg) * 512 * sizeof(double2)
                           : static_cast<size_t>((a.side / CL + 2) * sizeof(double) + kSetCap * sizeof(double2) + 32 * 8 + 32 * 4);
  const size_t smem = std::max(need, static_cast<size_t>(228 * 1024 / (per_sm + 1) + 1024));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(nblocks) * CL);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, which);
}

cudaError_t launch_pivot_wide(const MidArgs& a, int which, int nblocks, size_t piv_smem, cudaStream_t st) {
  static const bool off = env_int_c("BF_NO_PIVOT_CLUSTER", 0) != 0;
  if (!off && a.side >= 4096) return launch_pivot_cl<8>(a, which, nblocks, st);
  if (!off && a.side >= 2048) return launch_pivot_cl<4>(a, which, nblocks, st);
  if (!off && a.side >= 1024) return launch_pivot_cl<2>(a, which, nblocks, st);
  k_pivot_wide<<<nblocks, 512, piv_smem, st>>>(a, which);
  return cudaGetLastError();
}

}  // namespace

extern "C" {

uint64_t bf_middle_workspace_bytes(uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank, uint32_t q_over,
                                   uint32_t nblocks) {
  uint64_t m = 0, side = 0, off[8];
  if (!tree_geometry(n, levels, branching, &m, &side)) return 0;
  const int S = set_capacity(side, rank, q_over ? q_over : 1);
  if (S < 0) return 0;
  return mid_ws_layout(side, nblocks, S, off);
}

static int middle_blocks(int kernel_id, uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank,
                         uint32_t q_over, uint32_t iters, const void* dense, const int32_t* slot, uint32_t nblocks,
                         const int32_t* block_ij, const int32_t* draws, void* u_out, void* v_out, double* w_out,
                         void* workspace, uint64_t ws_bytes, void* stream);

int bf_middle_blocks(int kernel_id, uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank, uint32_t q_over,
                     uint32_t iters, const void* dense, uint32_t nblocks, const int32_t* block_ij, const int32_t* draws,
                     void* u_out, void* v_out, double* w_out, void* workspace, uint64_t ws_bytes, void* stream) {
  if (kernel_id < BF_KERNEL_FIO || kernel_id > BF_KERNEL_DFT) return fail(BF_EINVAL, "unknown entry kernel id");
  return middle_blocks(kernel_id, n, levels, branching, rank, q_over, iters, dense, nullptr, nblocks, block_ij,
                       draws, u_out, v_out, w_out, workspace, ws_bytes, stream);
}

int bf_middle_blocks_tiled(uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank, uint32_t q_over,
                           uint32_t iters, const void* tiles, const int32_t* slot, uint32_t nblocks,
                           const int32_t* block_ij, const int32_t* draws, void* u_out, void* v_out, double* w_out,
                           void* workspace, uint64_t ws_bytes, void* stream) {
  if (!tiles || !slot) return fail(BF_EINVAL, "tiled middle blocks need tiles and a slot table");
  return middle_blocks(BF_KERNEL_TILES, n, levels, branching, rank, q_over, iters, tiles, slot, nblocks, block_ij,
                       draws, u_out, v_out, w_out, workspace, ws_bytes, stream);
}

static int middle_blocks(int kernel_id, uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank,
                         uint32_t q_over, uint32_t iters, const void* dense, const int32_t* slot, uint32_t nblocks,
                         const int32_t* block_ij, const int32_t* draws, void* u_out, void* v_out, double* w_out,
                         void* workspace, uint64_t ws_bytes, void* stream) {
  if (kernel_id == BF_KERNEL_DENSE && !dense) return fail(BF_EINVAL, "dense oracle needs a matrix pointer");
  uint64_t m = 0, side = 0;
  if (!tree_geometry(n, levels, branching, &m, &side)) return fail(BF_EINVAL, "bad partition geometry");
  if (kernel_id == BF_KERNEL_RADON2D && branching != 4) return fail(BF_EINVAL, "the 2-D kernel needs a quadtree");
  if (rank < 1 || q_over < 1 || iters < 1) return fail(BF_EINVAL, "bad rank / oversampling parameters");
  if (side < rank) return fail(BF_EINVAL, "middle blocks are narrower than the rank");
  const uint64_t rq = static_cast<uint64_t>(rank) * q_over;
  const bool dense_branch = rq >= side;  // lowrank.py:231-234
  const uint64_t rqs = rq < side ? rq : side;
  const int S = set_capacity(side, rank, q_over);
  if (S < 0) return fail(BF_EINVAL, "rank too large for the batched sampling kernels (need r*(q+1) <= 128)");
  if (!nblocks) return BF_OK;
  if (!block_ij || (!dense_branch && !draws) || !u_out || !v_out || !w_out || !workspace)
    return fail(BF_EINVAL, "null pointer");
  uint64_t off[8];
  if (ws_bytes < mid_ws_layout(side, nblocks, S, off)) return fail(BF_EINVAL, "middle workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(workspace);
  MidArgs a{};
  a.src.kind = kernel_id;
  a.src.n = n;
  a.src.dense = static_cast<const double2*>(dense);
  a.src.tab = nullptr;
  a.src.slot = slot;
  a.src.side = side;
  a.src.m = m;
  if (kernel_id == BF_KERNEL_FIO || kernel_id == BF_KERNEL_RADON2D) {
    a.src.tab = row_table(kernel_id, n, static_cast<cudaStream_t>(stream));
    if (!a.src.tab) return BF_ECUDA;
  }
  a.side = static_cast<int64_t>(side);
  a.r = static_cast<int>(rank);
  a.rqs = static_cast<int>(rqs);
  a.iters = static_cast<int>(iters);
  a.nblocks = static_cast<int>(nblocks);
  a.S = S;
  a.st = reinterpret_cast<BlockState*>(base + off[0]);
  a.draws = draws;
  a.wide = reinterpret_cast<double2*>(base + off[1]);
  a.tall = reinterpret_cast<double2*>(base + off[2]);
  a.qc = reinterpret_cast<double2*>(base + off[3]);
  a.qr = reinterpret_cast<double2*>(base + off[4]);
  a.qbuf = reinterpret_cast<double2*>(base + off[5]);
  a.scr = reinterpret_cast<double2*>(base + off[6]);
  a.sig = reinterpret_cast<double*>(base + off[7]);
  a.u_out = static_cast<double2*>(u_out);
  a.v_out = static_cast<double2*>(v_out);
  a.w_out = w_out;
  const int T = 256;
  const unsigned yfill = static_cast<unsigned>(std::min<uint64_t>(64, (S * side + T - 1) / T));
  const size_t small_smem = S <= kSmemSet ? 3ull * S * S * sizeof(double2) : 0;
  BF_CUDA(allow_max_dyn_smem(k_mid));
  BF_CUDA(allow_max_dyn_smem(k_dense));
  k_init<<<(nblocks + 127) / 128, 128, 0, st>>>(a, block_ij);
  if (dense_branch) {
    k_dense<<<nblocks, T, small_smem, st>>>(a);
  } else {
    const size_t piv_smem = side * sizeof(double) + kSetCap * sizeof(double2) + 32 * 8 + 32 * 4 + kSetCap * 4;
    if (piv_smem > 227 * 1024) return fail(BF_EINVAL, "middle blocks too wide for the pivot kernel");
    BF_CUDA(allow_max_dyn_smem(k_pivot_wide));
    for (uint32_t sw = 0; sw < iters; ++sw) {
      k_union<<<nblocks, 128, 0, st>>>(a, 2 * sw, kRows);
      k_fill_wide<<<dim3(nblocks, yfill), T, 0, st>>>(a, kRows);
      BF_CUDA(launch_pivot_wide(a, kRows, nblocks, piv_smem, st));
      k_union<<<nblocks, 128, 0, st>>>(a, 2 * sw + 1, kCols);
      k_fill_wide<<<dim3(nblocks, yfill), T, 0, st>>>(a, kCols);
      BF_CUDA(launch_pivot_wide(a, kCols, nblocks, piv_smem, st));
    }
    k_union<<<nblocks, 128, 0, st>>>(a, 2 * iters, kRows);
    k_union<<<nblocks, 128, 0, st>>>(a, 2 * iters + 1, kCols);
    const size_t tall_smem = (static_cast<size_t>(kGramChunk) * (S + 2) + (S <= kSmemSet ? 2ull * S * S : 0)) * 16;
    BF_CUDA(allow_max_dyn_smem(k_pivot_tall));
    for (int which : {kCols, kRows}) {
      k_fill_tall<<<dim3(nblocks, yfill), T, 0, st>>>(a, which, 0, a.tall);
      k_pivot_tall<<<nblocks, kPivotTallThreads, tall_smem, st>>>(a, which);
      k_fill_tall<<<dim3(nblocks, yfill), T, 0, st>>>(a, which, 1, which == kCols ? a.qc : a.qr);
      launch_basis(a, nblocks, which, st);
    }
    k_mid<<<nblocks, 768, small_smem, st>>>(a);  // 24 warps: a 48-column Jacobi round in one pass
  }
  BF_CUDA(launch_assemble(a, nblocks, st));
  BF_CUDA(cudaGetLastError());
  return BF_OK;
}

uint64_t bf_probe_workspace_bytes(uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank, uint32_t width,
                                  uint32_t nblocks) {
  uint64_t m = 0, side = 0, off[8];
  if (!tree_geometry(n, levels, branching, &m, &side)) return 0;
  if (width < 1 || width > static_cast<uint32_t>(kSetCap)) return 0;
  const int S = width <= static_cast<uint32_t>(kSmemSet) ? kSmemSet : kSetCap;
  return mid_ws_layout(side, nblocks, S, off);
}

int bf_middle_probes(uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank, uint32_t width,
                     uint32_t nblocks, const int32_t* block_ij, const void* k_cols, uint64_t ldc,
                     const void* k_rows, uint64_t ldr, const void* row_probe, void* u_out, void* v_out,
                     double* w_out, void* workspace, uint64_t ws_bytes, void* stream) {
  uint64_t m = 0, side = 0;
  if (!tree_geometry(n, levels, branching, &m, &side)) return fail(BF_EINVAL, "bad partition geometry");
  if (rank < 1 || side < rank) return fail(BF_EINVAL, "middle blocks are narrower than the rank");
  if (width < rank || width > side || width > static_cast<uint32_t>(kSetCap))
    return fail(BF_EINVAL, "probe width must satisfy r <= width <= min(side, 128)");
  if (ldc < m * width || ldr < m * width) return fail(BF_EINVAL, "probe products narrower than m * width");
  if (!nblocks) return BF_OK;
  if (!block_ij || !k_cols || !k_rows || !row_probe || !u_out || !v_out || !w_out || !workspace)
    return fail(BF_EINVAL, "null pointer");
  const int S = width <= static_cast<uint32_t>(kSmemSet) ? kSmemSet : kSetCap;
  uint64_t off[8];
  if (ws_bytes < mid_ws_layout(side, nblocks, S, off)) return fail(BF_EINVAL, "probe workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(workspace);
  MidArgs a{};
  a.side = static_cast<int64_t>(side);
  a.r = static_cast<int>(rank);
  a.nblocks = static_cast<int>(nblocks);
  a.S = S;
  a.st = reinterpret_cast<BlockState*>(base + off[0]);
  a.wide = reinterpret_cast<double2*>(base + off[1]);
  a.tall = reinterpret_cast<double2*>(base + off[2]);
  a.qc = reinterpret_cast<double2*>(base + off[3]);
  a.qr = reinterpret_cast<double2*>(base + off[4]);
  a.qbuf = reinterpret_cast<double2*>(base + off[5]);
  a.scr = reinterpret_cast<double2*>(base + off[6]);
  a.sig = reinterpret_cast<double*>(base + off[7]);
  a.u_out = static_cast<double2*>(u_out);
  a.v_out = static_cast<double2*>(v_out);
  a.w_out = w_out;
  a.probe_w = static_cast<int>(width);
  a.kc = static_cast<const double2*>(k_cols);
  a.kr = static_cast<const double2*>(k_rows);
  a.rprobe = static_cast<const double2*>(row_probe);
  a.ldc = static_cast<int64_t>(ldc);
  a.ldr = static_cast<int64_t>(ldr);
  const int T = 256;
  const unsigned yfill = static_cast<unsigned>(std::min<uint64_t>(64, (width * side + T - 1) / T));
  const size_t small_smem = S <= kSmemSet ? 3ull * S * S * sizeof(double2) : 0;
  const size_t tall_smem = (static_cast<size_t>(kGramChunk) * (S + 2) + (S <= kSmemSet ? 2ull * S * S : 0)) * 16;
  BF_CUDA(allow_max_dyn_smem(k_mid_probe));
  BF_CUDA(allow_max_dyn_smem(k_pivot_tall));
  k_init<<<(nblocks + 127) / 128, 128, 0, st>>>(a, block_ij);
  for (int which : {kCols, kRows}) {
    k_fill_probe<<<dim3(nblocks, yfill), T, 0, st>>>(a, which);
    k_pivot_tall<<<nblocks, kPivotTallThreads, tall_smem, st>>>(a, which);
    k_sel_probe<<<dim3(nblocks, yfill), T, 0, st>>>(a, which);
  }
  k_set_probe_counts<<<(nblocks + 127) / 128, 128, 0, st>>>(a);
  for (int which : {kCols, kRows}) launch_basis(a, nblocks, which, st);
  k_mid_probe<<<nblocks, T, small_smem, st>>>(a);
  BF_CUDA(launch_assemble(a, nblocks, st));
  BF_CUDA(cudaGetLastError());
  return BF_OK;
}

// One level of the recursive refactorisation (construct.py:127-163) with
// branching b (2, or 4 on quadtrees): cur (nb, rows, groups, r) complex128 ->
// blocks (nb, b, groups/b, r, b r) [rows >= b] or (nb, groups/b, r, b r)
// [rows < b] and the next cur. With workspace == NULL, *ws_bytes receives the
// scratch size.
int bf_recurse_level(uint32_t rank, uint32_t branching, uint64_t nb, uint64_t rows, uint64_t groups, const void* cur,
                     void* blocks, void* next, void* workspace, uint64_t* ws_bytes, void* stream) {
  if (!ws_bytes) return fail(BF_EINVAL, "null ws_bytes");
  if (branching != 2 && branching != 4) return fail(BF_EINVAL, "branching must be 2 or 4");
  const uint32_t w = branching * rank;
  if (rank < 1 || w > static_cast<uint32_t>(kSetCap)) return fail(BF_EINVAL, "rank must satisfy 1 <= b r <= 128");
  if (groups % branching || groups == 0 || rows == 0) return fail(BF_EINVAL, "bad recursion geometry");
  const int S = w <= static_cast<uint32_t>(kSmemSet) ? kSmemSet : kSetCap;
  const int64_t pairs = groups / branching;
  const int64_t part = rows / branching;
  // stacks up to 32 wide: R by the register TSQR (stacks taller than 32 rows), warp-per-problem
  // Jacobi on R^H, new_u = A V in its own kernel; BF_NO_WSVD=1 restores the CTA-per-problem SVD
  static const bool wsvd_on = env_int_c("BF_NO_WSVD", 0) == 0;
  const bool wsvd = wsvd_on && rows >= branching && w <= 32;
  // problems per launch: the warp-per-problem kernels keep no per-problem scratch besides R,
  // so one launch takes up to 8,192 (the block scheduler back-fills finished warps; 2,048
  // problems are only 1.2 machine-fills of 12 warps per SM)
  static const int64_t chunk_env = env_int_c("BF_RECURSE_CHUNK", 0);
  const int64_t nprob_all = static_cast<int64_t>(nb) * (rows >= branching ? branching : 1) * pairs;
  const int64_t chunk = std::min<int64_t>(chunk_env > 0 ? chunk_env : (wsvd ? 8192 : 2048), std::max<int64_t>(nprob_all, 1));
  const bool reg_tsqr = rows >= branching && S <= kSmemSet && w <= 32 && part > (wsvd ? static_cast<int64_t>(w) : static_cast<int64_t>(S));
  const uint64_t scr_bytes =
      rows >= branching && !wsvd ? static_cast<uint64_t>(chunk) * rec_scratch_elems(part, w, S) * 16 : 0;
  // never 0: a NULL workspace is the size query, so a caller must always have a buffer to pass
  const uint64_t need = std::max<uint64_t>(16, scr_bytes + (reg_tsqr ? static_cast<uint64_t>(chunk) * w * w * 16 : 0));
  if (!workspace) {
    *ws_bytes = need;
    return BF_OK;
  }
  if (*ws_bytes < need) return fail(BF_EINVAL, "recursion workspace too small");
  if (!cur || !blocks || !next) return fail(BF_EINVAL, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  RecArgs a{};
  a.cur = static_cast<const double2*>(cur);
  a.nxt = static_cast<double2*>(next);
  a.g = static_cast<double2*>(blocks);
  a.scr = static_cast<double2*>(workspace);
  a.nb = static_cast<int64_t>(nb);
  a.rows = static_cast<int64_t>(rows);
  a.pairs = pairs;
  a.r = static_cast<int>(rank);
  a.b = static_cast<int>(branching);
  a.S = S;
  if (rows >= branching) {
    const int64_t nprob = static_cast<int64_t>(nb) * branching * pairs;
    const size_t smem = S <= kSmemSet ? rec_smem_elems(static_cast<int>(w), S) * sizeof(double2) : 0;
    const size_t tsqr_smem = 8ull * (kTsqrCh + 1) * w * sizeof(double2);  // every warp streams its own chunk
    a.rbuf = reg_tsqr ? reinterpret_cast<double2*>(static_cast<char*>(workspace) + scr_bytes) : nullptr;
    if (reg_tsqr) BF_CUDA(allow_max_dyn_smem(k_recurse_tsqr));
    if (reg_tsqr) BF_CUDA(allow_max_dyn_smem(k_recurse_tsqr2));
    static const int tsqr_w_env = env_int_c("BF_TSQR_W", 0);
    const int tsqr_w = (tsqr_w_env == 1 || tsqr_w_env == 2 || tsqr_w_env == 4 || tsqr_w_env == 8) ? tsqr_w_env : 0;
    const bool tall = part > S;
    void (*kern)(RecArgs) = tall ? k_recurse_split<true> : k_recurse_split<false>;
    BF_CUDA(allow_max_dyn_smem(kern));
    const int av_tiles = static_cast<int>((part + 127) / 128);
    const size_t av_smem = static_cast<size_t>((rank + 3) & ~3u) * w * sizeof(double2);
    for (int64_t p0 = 0; p0 < nprob; p0 += chunk) {
      a.p0 = p0;
      const int64_t cnt = std::min<int64_t>(chunk, nprob - p0);
      if (reg_tsqr && wsvd) {
        // warps per problem: about four 8-row chunks each before the pairwise merge
        const int64_t nch = (part + kTsqrRows - 1) / kTsqrRows;
        // one warp per problem once the chunk fills the machine (8 warps per SM); fewer problems
        // spread over W warps each (about four 8-row chunks per warp before the pairwise merge)
        int W = nch >= 32 ? 8 : nch >= 16 ? 4 : nch >= 8 ? 2 : 1;
        while (W > 1 && cnt * W > 2 * 148 * 8) W /= 2;
        if (tsqr_w > 0) W = tsqr_w;
        if (W == 1) {
          static const int tsqr_ch = env_int_c("BF_TSQR_CH", 16);
          const size_t tri = kTriElems * sizeof(double2);
          if (tsqr_ch == 16) k_recurse_tsqr1<16><<<static_cast<unsigned>(cnt), 32, tri, st>>>(a);
          else k_recurse_tsqr1<8><<<static_cast<unsigned>(cnt), 32, tri, st>>>(a);
        } else {
          const unsigned gt = static_cast<unsigned>((cnt * W + 7) / 8);
          k_recurse_tsqr2<<<gt, 256, 8 * 33 * 32 * sizeof(double2), st>>>(a, cnt, W);
        }
      } else if (reg_tsqr) {
        k_recurse_tsqr<<<static_cast<unsigned>(cnt), 256, tsqr_smem, st>>>(a);
      }
      if (wsvd) {
        const unsigned g4 = static_cast<unsigned>((cnt + 3) / 4);
        // 32-row columns: 255 registers and no spills at 8 warps per SM, or 168 registers with
        // the column partly in local memory at 12 (BF_WSVD_OCC=3)
        static const int occ = env_int_c("BF_WSVD_OCC", 2);
        if (w <= 16) k_recurse_wsvd<16, 4><<<g4, 128, 0, st>>>(a, cnt, reg_tsqr ? 1 : 0);
        else if (occ == 3) k_recurse_wsvd<32, 3><<<g4, 128, 0, st>>>(a, cnt, reg_tsqr ? 1 : 0);
        else k_recurse_wsvd<32, 2><<<g4, 128, 0, st>>>(a, cnt, reg_tsqr ? 1 : 0);
        k_recurse_av<<<static_cast<unsigned>(cnt * av_tiles), 256, av_smem, st>>>(a, av_tiles);
        continue;
      }
      kern<<<static_cast<unsigned>(cnt), tall ? 256 : 512, smem, st>>>(a);  // short stacks: 16 warps, one pass per Jacobi round
    }
  } else {
    const int64_t nprob = static_cast<int64_t>(nb) * pairs;
    a.p0 = 0;
    k_recurse_merge<<<static_cast<unsigned>((nprob + 7) / 8), 256, 0, st>>>(a, nprob);
  }
  BF_CUDA(cudaGetLastError());
  return BF_OK;
}

// Greedy pivoted column selection (select_pivot_columns, lowrank.py:102-129)
// on a batch of device matrices a (batch, m, n) complex128 row-major, m <= 64,
// n <= 16384: up to k picks each (pick order) into pivots (batch, k), pick
// counts into counts (batch). pairwise = 1 sums the initial column norms in
// numpy's pairwise order (the reference's matrix is F-ordered), 0 sequentially.
int bf_select_pivots(const void* a, uint32_t batch, uint32_t m, uint32_t n, uint32_t k, double rel_tol, int pairwise,
                     int32_t* pivots, int32_t* counts, void* workspace, uint64_t ws_bytes, void* stream) {
  if (m > static_cast<uint32_t>(kSetCap) || n > 16384 || k > 1024) return fail(BF_EINVAL, "pivot matrix too large");
  if (!batch || !m || !n || !k) return BF_OK;
  if (!a || !pivots || !counts || !workspace) return fail(BF_EINVAL, "null pointer");
  const uint64_t kk = k < m ? k : m;
  if (ws_bytes < 16ull * batch * kk * n) return fail(BF_EINVAL, "pivot workspace too small (16*batch*min(k,m)*n bytes)");
  const size_t smem = (n + (n & 1)) * 8 + kSetCap * 16 + 32 * 8 + 32 * 4 + 1024 * 4;
  BF_CUDA(allow_max_dyn_smem(k_select_pivots));
  k_select_pivots<<<batch, 512, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const double2*>(a), static_cast<double2*>(workspace), static_cast<int>(m), static_cast<int>(n),
      static_cast<int>(k), rel_tol, pairwise, pivots, counts);
  BF_CUDA(cudaGetLastError());
  return BF_OK;
}

}  // extern "C"
