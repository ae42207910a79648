// tc_kernel.cuh — complex64 many-RHS levels on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in tensor memory), 3xTF32-split for FP32
// accuracy (the north star's optional c64 mode, <= 1e-5).
//
// One tile = one unit of a level (factors.py:120-139; a2/a3 of SURVEY.md §8(a)) and 128
// right-hand sides, computed transposed so the 128 RHS fill the MMA's M dimension:
//   forward  Y^T (128 x nt R) = X^T (128 x C)    . B^T      (B: nt blocks R x C)
//   adjoint  Y^T (128 x C)    = X^T (128 x nt R) . conj(B)  (the nt blocks stacked)
// Complex operands are split into real planes and each plane into a TF32 pair hi + lo
// (hi = rna(x), lo = rna(x - hi)); every real product is hi.hi + hi.lo + lo.hi, so a
// complex tile is 12 MMA products per K step: Re += Xr Br - Xi Bi, Im += Xr Bi + Xi Br
// (the subtraction through the instruction descriptor's negate-A bit). Both operands
// are staged K-major in the canonical no-swizzle layout (8-row x 16-byte core matrices:
// LBO = 128 B along K, SBO = K/4 x 128 B along rows; tools/tcgen05_probe.cu checks the
// encoding on the B200). One thread issues the MMAs; tcgen05.commit signals an
// mbarrier; four warps read their 32 TMEM lanes each (tcgen05.ld 32x32b) and store the
// outputs, the middle factor fused when the level ends the down half.
//
// Status: correct (tests/test_apply_gpu.py::test_c64_tensor_core_levels) but opt-in
// (BF_TC=1). At cfg2 with 256 RHS it measures 46.7 ms per apply against 29.4 ms for the
// FFMA consumer, with a relative error of 7.7e-6 against 6.1e-7 — the split warps (raw
// tile -> 4 tf32 planes per operand, ~6k cycles per 128-RHS tile) set the pace while the
// MMAs take ~100 cycles, and the three-term TF32 products accumulate an order of magnitude
// more error over the chain's 18 levels than FP32 FMAs (close to the 1e-5 bound).
#pragma once

#include "level_kernel.cuh"

namespace bfly {

struct TcArgs {
  const float2* fac;
  const float2* in;
  float2* out;
  const float* mid_w;
  uint32_t R, C, nt, lgP, units, k, ktiles;
  uint32_t N, K, Kp;     // output columns (of Y^T), contraction length, padded to a multiple of 8
  int adjoint, remap;
  uint32_t m, r;         // middle geometry (remap)
  uint32_t tmem_cols;    // power of two >= max(2 N, N + 32): the epilogue reads 32 columns at a time
  unsigned long long* trace;  // diagnostics (bf_debug_node_trace): CTA 0's clock64 per tile phase
};

__device__ __forceinline__ void tc_stamp(const TcArgs& a, uint32_t it, int i) {
  if (a.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && it < 16) a.trace[it * 8 + i] = clock64();
}

__device__ __forceinline__ uint32_t tc_canon(uint32_t row, uint32_t k, uint32_t Kp) {
  return (k >> 2) * 128 + (row >> 3) * (Kp >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4;  // bytes
}

__device__ __forceinline__ uint64_t tc_sdesc(uint32_t saddr, uint32_t Kp) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(128 >> 4) << 16;                       // LBO: next core matrix along K
  d |= static_cast<uint64_t>(((Kp >> 2) * 128) >> 4) << 32;         // SBO: next 8-row group
  d |= 1ull << 46;                                                  // descriptor version (sm_100)
  return d;                                                         // layout type 0: no swizzle
}

__device__ __forceinline__ uint32_t tc_idesc(uint32_t n, int neg_a) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(neg_a) << 13) | ((n >> 3) << 17) |
         ((128u >> 4) << 24);   // D f32, A/B tf32, K-major, M = 128
}

// hi = rna(x) to TF32, lo = rna(x - hi). (Truncating hi with a mask instead measured no
// faster and doubled the error: cfg2 256 RHS 1.5e-5 against 7.7e-6.)
__device__ __forceinline__ void tc_split(float x, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - hi));
  lo = __uint_as_float(l);
}

__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

template <int NC>
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t u[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
        "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
        "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]),
        "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(u[i]);
}

__device__ __forceinline__ void tc_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t u[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(u[i]);
}

// Row of the level's input / output vector for contraction index kk / output column n of unit u.
__device__ __forceinline__ uint32_t tc_chunk_row(const TcArgs& a, uint32_t u, uint32_t idx) {
  const uint32_t P = 1u << a.lgP, g = u >> a.lgP, p = u & (P - 1);
  const uint32_t t = idx / a.R, rho = idx - t * a.R;
  return ((g * a.nt + t) * P + p) * a.R + rho;
}

// (A plane, B plane) of the six MMAs per K step. A planes: Xr_hi, Xr_lo, Xi_hi, Xi_lo.
// B planes (2N rows each): B1 = [Br; Bi] hi, lo and B2 = [-Bi; Br] hi, lo, so one N = 2N
// product accumulates Re (columns [0, N)) and Im ([N, 2N)) together:
//   [Re | Im] += Xr [Br | Bi] + Xi [-Bi | Br], each real product as hi.hi + hi.lo + lo.hi
__constant__ uint8_t kTcProd[6][2] = {{0, 0}, {0, 1}, {1, 0}, {2, 2}, {2, 3}, {3, 2}};

// Warp roles: 4 split warps (raw X tile -> tf32 planes, B from global), 4 epilogue warps
// (TMEM lane quarter = warp % 4), 1 MMA warp (allocates TMEM; lane 0 issues).
constexpr int kTcSplitWarps = 8, kTcEpiWarps = 4;
constexpr int kTcThreads = (kTcSplitWarps + kTcEpiWarps + 1) * 32;

__device__ __forceinline__ void split_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// The unit's X rows (kc RHS each) into the raw buffer with 16-byte cp.async by the split
// warps (one commit group).
__device__ __forceinline__ void tc_issue_x(const TcArgs& a, uint32_t tile, uint32_t ntiles, float2* rx) {
  if (tile < ntiles) {
    const uint32_t u = tile / a.ktiles, k0 = (tile - u * a.ktiles) * 128;
    const uint32_t kc = min(128u, a.k - k0), q = kc / 2;     // 16-byte pieces per row
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t kk = warp; kk < a.K; kk += kTcSplitWarps) {   // one row per warp, pieces per lane
      const uint32_t row = a.adjoint ? tc_chunk_row(a, u, kk) : u * a.C + kk;
      const float2* src = a.in + static_cast<size_t>(row) * a.k + k0;
      for (uint32_t j = lane; j < q; j += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(rx + kk * 128 + 2 * j)),
                     "l"(src + 2 * j)
                     : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// This thread's B elements of a tile (n, 4 consecutive kk per item, items e = tid + 256 i),
// loaded ahead of their split so the global latency overlaps the X split.
constexpr int kTcBItems = 2;
__device__ __forceinline__ void tc_load_b(const TcArgs& a, uint32_t tile, uint32_t ntiles, float2 (&bv)[kTcBItems][4]) {
  if (tile >= ntiles) return;
  const uint32_t u = tile / a.ktiles;
  const uint32_t P = 1u << a.lgP, g = u >> a.lgP, p = u & (P - 1);
#pragma unroll
  for (int i = 0; i < kTcBItems; ++i) {
    const uint32_t e = threadIdx.x + i * kTcSplitWarps * 32;
    const uint32_t n = e % a.N, kq = e / a.N;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t kk = kq * 4 + j;
      float2 v = make_float2(0.f, 0.f);
      if (e < a.N * (a.Kp / 4) && kk < a.K) {
        const uint32_t tr = a.adjoint ? kk : n, c = a.adjoint ? n : kk;
        const uint32_t t = tr / a.R, rho = tr - t * a.R;
        v = __ldg(a.fac + (static_cast<size_t>((g * a.nt + t) * P + p) * a.R + rho) * a.C + c);
        if (a.adjoint) v.y = -v.y;
      }
      bv[i][j] = v;
    }
  }
}

// Dynamic shared memory: two sets of tf32 planes (A: 4 x 128 x Kp, B: 4 x 2N x Kp) and one
// raw X tile (K x 128 float2). Tile i's planes are multiplied (TMEM accumulator i % 2) and
// tile i - 1's accumulator drained to global while the split warps convert tile i + 1.
__global__ void __launch_bounds__(kTcThreads, 1) tc_level_kernel(const TcArgs a) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t planes_full[2], mma_done[2], tmem_empty[2];
  const uint32_t Kp = a.Kp, N = a.N;
  const uint32_t aplane = 128 * Kp * 4, bplane = 2 * N * Kp * 4;   // bytes per tf32 plane
  const uint32_t setb = 4 * aplane + 4 * bplane;                   // bytes per plane set
  float2* rx = reinterpret_cast<float2*>(tsm + 2 * setb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mma_warp = kTcSplitWarps + kTcEpiWarps;
  if (warp == mma_warp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base))), "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&planes_full[s], kTcSplitWarps);
      mbar_init(&mma_done[s], 1);
      mbar_init(&tmem_empty[s], kTcEpiWarps);
    }
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t ntiles = a.units * a.ktiles;
  const uint32_t step = gridDim.x;
  if (warp < kTcSplitWarps) {
    // ================= split warps
    tc_issue_x(a, blockIdx.x, ntiles, rx);
    float2 bv[kTcBItems][4];
    tc_load_b(a, blockIdx.x, ntiles, bv);
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += step, ++it) {
      const uint32_t s = it & 1;
      unsigned char* sA = tsm + s * setb;
      unsigned char* sB = sA + 4 * aplane;
      const uint32_t u = tile / a.ktiles, k0 = (tile - u * a.ktiles) * 128;
      const uint32_t kc = min(128u, a.k - k0);
      const uint32_t P = 1u << a.lgP, g = u >> a.lgP, p = u & (P - 1);
      if (it >= 2) mbar_wait(&mma_done[s], ((it >> 1) - 1) & 1);   // the MMAs of tile it - 2 read planes s
      (void)g;
      (void)p;
      tc_stamp(a, it, 0);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      split_bar();                                                // every split thread's copies landed
      tc_stamp(a, it, 1);
      for (uint32_t e = threadIdx.x; e < 128 * (Kp / 4); e += kTcSplitWarps * 32) {
        const uint32_t m = e & 127, kq = e >> 7;
        float hr[4], lr[4], hi[4], li[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t kk = kq * 4 + j;
          const float2 x = (kk < a.K && m < kc) ? rx[kk * 128 + m] : make_float2(0.f, 0.f);
          tc_split(x.x, hr[j], lr[j]);
          tc_split(x.y, hi[j], li[j]);
        }
        const uint32_t off = tc_canon(m, kq * 4, Kp);
        *reinterpret_cast<float4*>(sA + off) = make_float4(hr[0], hr[1], hr[2], hr[3]);
        *reinterpret_cast<float4*>(sA + aplane + off) = make_float4(lr[0], lr[1], lr[2], lr[3]);
        *reinterpret_cast<float4*>(sA + 2 * aplane + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<float4*>(sA + 3 * aplane + off) = make_float4(li[0], li[1], li[2], li[3]);
      }
      split_bar();                                                // raw tile consumed
      tc_issue_x(a, tile + step, ntiles, rx);                     // next tile's X streams in now
      // B^T (loaded one tile ahead): forward B[t][rho][c] (n = t R + rho, kk = c); adjoint
      // conj(B[t][rho][c]) (n = c, kk = t R + rho)
#pragma unroll
      for (int i = 0; i < kTcBItems; ++i) {
        const uint32_t e = threadIdx.x + i * kTcSplitWarps * 32;
        if (e < N * (Kp / 4)) {
          const uint32_t n = e % N, kq = e / N;
          float hr[4], lr[4], hi[4], li[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            tc_split(bv[i][j].x, hr[j], lr[j]);
            tc_split(bv[i][j].y, hi[j], li[j]);
          }
          const uint32_t o0 = tc_canon(n, kq * 4, Kp), o1 = tc_canon(n + N, kq * 4, Kp);
          const float4 rh = make_float4(hr[0], hr[1], hr[2], hr[3]), rl = make_float4(lr[0], lr[1], lr[2], lr[3]);
          const float4 ih = make_float4(hi[0], hi[1], hi[2], hi[3]), il = make_float4(li[0], li[1], li[2], li[3]);
          *reinterpret_cast<float4*>(sB + o0) = rh;                 // B1 = [Br; Bi]
          *reinterpret_cast<float4*>(sB + o1) = ih;
          *reinterpret_cast<float4*>(sB + bplane + o0) = rl;
          *reinterpret_cast<float4*>(sB + bplane + o1) = il;
          *reinterpret_cast<float4*>(sB + 2 * bplane + o0) = make_float4(-hi[0], -hi[1], -hi[2], -hi[3]);  // B2 = [-Bi; Br]
          *reinterpret_cast<float4*>(sB + 2 * bplane + o1) = rh;
          *reinterpret_cast<float4*>(sB + 3 * bplane + o0) = make_float4(-li[0], -li[1], -li[2], -li[3]);
          *reinterpret_cast<float4*>(sB + 3 * bplane + o1) = rl;
        }
      }
      tc_load_b(a, tile + step, ntiles, bv);                      // next tile's blocks in flight
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy writes -> tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(&planes_full[s]);
      tc_stamp(a, it, 2);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else if (warp == mma_warp) {
    // ================= MMA issuer
    const uint32_t idn2 = tc_idesc(2 * N, 0);
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += step, ++it) {
      const uint32_t s = it & 1;
      mbar_wait(&planes_full[s], (it >> 1) & 1);
      if (it >= 2) mbar_wait(&tmem_empty[s], ((it >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(tsm + s * setb));
        const uint64_t adesc0 = tc_sdesc(base, Kp), bdesc0 = tc_sdesc(base + 4 * aplane, Kp);
        const uint32_t acc = tbase + s * 2 * N;
        for (uint32_t ks = 0; ks < Kp / 8; ++ks)
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const uint64_t ad = adesc0 + ((kTcProd[q][0] * aplane + ks * 256) >> 4);
            const uint64_t bd = bdesc0 + ((kTcProd[q][1] * bplane + ks * 256) >> 4);
            tc_mma(acc, ad, bd, idn2, (ks == 0 && q == 0) ? 0u : 1u);
          }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&mma_done[s]))
                     : "memory");
      }
      __syncwarp();
    }
  } else {
    // ================= epilogue warps: TMEM lane quarter q4 (rhs 32 q4 + lane), all columns
    const uint32_t q4 = warp & 3, m = q4 * 32 + lane;
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += step, ++it) {
      const uint32_t s = it & 1;
      const uint32_t u = tile / a.ktiles, k0 = (tile - u * a.ktiles) * 128;
      const uint32_t kc = min(128u, a.k - k0);
      const uint32_t P = 1u << a.lgP, g = u >> a.lgP, p = u & (P - 1);
      mbar_wait(&mma_done[s], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t lane_addr = tbase + s * 2 * N + ((q4 * 32) << 16);
      for (uint32_t c0 = 0; c0 < N; c0 += 8) {
        float re[8], im[8];
        tc_ld8(lane_addr + c0, re);
        tc_ld8(lane_addr + N + c0, im);
        if (m < kc) {
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j) {
            const uint32_t n = c0 + j;
            float w = 1.f;
            size_t row;
            if (!a.adjoint) {
              const uint32_t t = n / a.R, rho = n - t * a.R;
              row = static_cast<size_t>((g * a.nt + t) * P + p) * a.R + rho;
            } else if (!a.remap) {
              row = static_cast<size_t>(u) * a.C + n;
            } else {  // the middle factor fused (factors.py:180-190): e = (ia, ib, rho) -> (ib, ia, rho)
              const uint32_t e = u * a.C + n, mr = a.m * a.r, ia = e / mr, rem = e - ia * mr;
              const uint32_t ib = rem / a.r, rho = rem - ib * a.r;
              row = (static_cast<size_t>(ib) * a.m + ia) * a.r + rho;
              w = a.remap == 1 ? __ldg(a.mid_w + row)
                               : __ldg(a.mid_w + (static_cast<size_t>(ia) * a.m + ib) * a.r + rho);
            }
            a.out[row * a.k + k0 + m] = make_float2(w * re[j], w * im[j]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[s]);
      if (q4 == 0) tc_stamp(a, it, 3);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == mma_warp)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(a.tmem_cols));
}

}  // namespace bfly
