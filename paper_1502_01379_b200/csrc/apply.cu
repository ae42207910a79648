// apply.cu — the butterfly apply chain on B200: level launches, the middle
// factor, and the chain driver behind bf_apply / bf_apply_factor.
//
// Reference: ButterflyFactors._chain (pkg/src/butterfly/factors.py:217-237)
//   forward:  V^L*  -> H^{L-1}* .. H^{h}*  -> M -> G^{h} .. G^{L-1} -> U^L
//   adjoint:  U^L*  -> G^{L-1}* .. G^{h}*  -> M* -> H^{h} .. H^{L-1} -> V^L
// with M (or M*) fused into the epilogue of the last adjoint-direction level.
#include <algorithm>
#include <vector>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "level_kernel.cuh"
#include "pair_kernel.cuh"
#include "pair16_kernel.cuh"
#include "node_mma.cuh"
#include "tc_kernel.cuh"
#include "wide_kernel.cuh"
#include <cudaTypedefs.h>
#include "plan.h"

namespace bfly {

namespace {


template <typename E>
__global__ void middle_kernel(const E* __restrict__ in, E* __restrict__ out,
                              const typename Cx<E>::R* __restrict__ W, uint32_t m, uint32_t r, uint32_t k,
                              int adjoint) {
  // forward (factors.py:180-184): out[i, j, rho] = W[i, j, rho] * in[j, i, rho]
  // adjoint (factors.py:186-190): out[j, i, rho] = W[i, j, rho] * in[i, j, rho]
  const uint64_t total = static_cast<uint64_t>(m) * m * r * k;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t kk = x % k, row = x / k;
    const uint64_t rho = row % r, ij = row / r;
    const uint64_t i = ij / m, j = ij % m;       // output block (i, j)
    const uint64_t src = (j * m + i) * r + rho;  // input slot (j, i)
    const auto w = adjoint ? W[src] : W[row];
    const E v = in[src * k + kk];
    out[x] = Cx<E>::make(w * v.x, w * v.y);
  }
}

bool dmma_disabled() {
  static const bool off = [] {
    const char* v = std::getenv("BF_NO_DMMA");
    return v && v[0] && v[0] != '0';
  }();
  return off;
}

// BF_NO_GAUSS=1: four real DMMAs per complex k-step instead of the 3-multiplication form
bool gauss_disabled() {
  static const bool off = [] {
    const char* v = std::getenv("BF_NO_GAUSS");
    return v && v[0] && v[0] != '0';
  }();
  return off;
}

uint32_t ilog2(uint64_t x) {
  uint32_t l = 0;
  while ((1ull << (l + 1)) <= x) ++l;
  return l;
}

// Launch shapes: the streaming kernel (k small: HBM-bound on factor bytes) and
// the register-tiled many-RHS kernel (k >= kMrhsMinK: FP64-FMA bound).
#ifndef STREAM64_STAGES
#define STREAM64_STAGES 3
#endif
struct Shape {
  int stages, ncw, ctas_per_sm;
  uint32_t stage_bytes;
};
// two stages of 34.5 KB per CTA, four consumer warps, two CTAs per SM (cfg2 k=1: 1.34 ms
// against 1.416 ms with three stages and two consumer warps; k=2 1.94 vs 3.00 ms; four or
// more stages stop two CTAs fitting an SM)
constexpr Shape kStream{2, 4, 2, 34 * 1024 + 512};
// complex64 streams half the bytes per output: twice the consumer warps keep the
// same per-SM output rate at the same stage size
constexpr Shape kStream64{STREAM64_STAGES, 8, 2, 34 * 1024 + 512};
template <typename E>
constexpr Shape stream_shape() {
  return sizeof(E) == 8 ? kStream64 : kStream;
}

// Experiments only (complex128 streaming levels): BF_STREAM_{STAGES,KB,CTAS,NCW} select a
// runtime-depth instantiation; unset, the tuned constexpr kStream shape is used.
struct StreamExp {
  bool on;
  Shape s;
};
StreamExp stream_exp();
constexpr Shape kMrhs{2, 8, 1, 112 * 1024};

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

// Tuning / diagnostic switches read once per process (no getenv on the launch path).
struct EnvKnobs {
  int mrhs_stages, mrhs_stage_kb, dbg_nomath, dbg_noload, dtile;
};
const EnvKnobs& knobs() {
  static const EnvKnobs k{env_int("BF_MRHS_STAGES", 0), env_int("BF_MRHS_STAGE_KB", 0), env_int("BF_DBG_NOMATH", 0),
                          env_int("BF_DBG_NOLOAD", 0), env_int("BF_DTILE", -1)};
  return k;
}

// Many-RHS pipeline shape: depth (<= 8) and stage budget are launch arguments of the
// STAGES = 0 instantiation (BF_MRHS_STAGES, BF_MRHS_STAGE_KB override them).
StreamExp stream_exp() {
  static const StreamExp x = [] {
    StreamExp e{false, kStream};
    const int st = env_int("BF_STREAM_STAGES", 0), kb = env_int("BF_STREAM_KB", 0);
    const int ct = env_int("BF_STREAM_CTAS", 0), nw = env_int("BF_STREAM_NCW", 0);
    if (st || kb || ct || nw) {
      e.on = true;
      if (st) e.s.stages = std::min(8, std::max(1, st));
      if (kb) e.s.stage_bytes = static_cast<uint32_t>(kb) * 1024;
      if (ct == 3) e.s.ctas_per_sm = 3;
      if (nw == 4) e.s.ncw = 4;
    }
    return e;
  }();
  return x;
}

Shape mrhs_shape() {
  static const Shape s = [] {
    Shape x = kMrhs;
    x.stages = std::min(8, std::max(1, env_int("BF_MRHS_STAGES", kMrhs.stages)));
    x.stage_bytes = static_cast<uint32_t>(env_int("BF_MRHS_STAGE_KB", kMrhs.stage_bytes / 1024)) * 1024;
    x.ncw = env_int("BF_MRHS_NCW", 0);  // 0: per launch (mrhs_warps)
    return x;
  }();
  return s;
}

// complex128 levels with wide blocks (C > 64: the r = 25 quadtree, C = 4r = 100): one
// 200 KB stage holds a whole unit (4 x 25 x 100 blocks), so the level runs as one launch
// instead of t-range splits that re-read the inputs / accumulate partial outputs; the
// single buffer costs less than the splits (cfg3 0.611 -> 0.543 ms, cfg4b 11.5 -> 10.0 ms)
template <typename E>
Shape mrhs_shape_for(uint32_t C) {
  Shape s = mrhs_shape();
  if (sizeof(E) == 16 && C > 64 && knobs().mrhs_stages == 0 && knobs().mrhs_stage_kb == 0) {
    s.stages = 1;
    s.stage_bytes = 200 * 1024;
  }
  return s;
}
constexpr uint32_t kMrhsMinK = 8;

// Diagnostics: when set (bf_debug_node_trace), node kernels stamp %globaltimer per CTA
// (down half into [0, m nch x 32), up half after it) and the tcgen05 level kernel its CTA
// 0 tile phases (clock64).
unsigned long long* g_node_trace = nullptr;

using LevelKernel = void (*)(LevelArgs, PeerArgs);

// complex128 3-multiplication DMMA kernels, one instantiation per warp tile (dt):
// MRHS = 3 (in-place outputs, TMA-stored) or 1 (register stores) with 8 or 16 consumer warps
template <typename E>
LevelKernel ffma16_kernel() {
  if constexpr (std::is_same<E, float2>::value)
    return level_kernel<float2, 0, 16, 1, 1, false>;
  else
    return nullptr;
}

// The down half's last two levels as one pair kernel with the middle factor fused into its
// stores (default since the whole-block pair copies: cfg1 234.4 vs 239.4 us; it was 0.287
// vs 0.284 ms before them). BF_REMAP_PAIR=0 keeps two single launches.
bool remap_pair_enabled() {
  static const bool on = env_int("BF_REMAP_PAIR", 1) != 0;
  return on;
}

// BF_NO_INPLACE=1: many-RHS DMMA consumers store their outputs from registers (MRHS = 1)
bool inplace_disabled() {
  static const bool off = env_int("BF_NO_INPLACE", 0) != 0;
  return off;
}

template <typename E>
LevelKernel dmma_kernel(int ncw, uint32_t dt, bool inplace) {
  if constexpr (std::is_same<E, double2>::value) {
    if (inplace) {  // MRHS = 3: outputs in place of the stage's vector rows, stored by the producer's TMA
      static const LevelKernel p8[3] = {level_kernel<double2, 0, 8, 1, 3, false, 0>,
                                        level_kernel<double2, 0, 8, 1, 3, false, 1>,
                                        level_kernel<double2, 0, 8, 1, 3, false, 2>};
      static const LevelKernel p16[3] = {level_kernel<double2, 0, 16, 1, 3, false, 0>,
                                         level_kernel<double2, 0, 16, 1, 3, false, 1>,
                                         level_kernel<double2, 0, 16, 1, 3, false, 2>};
      static const LevelKernel p4[3] = {level_kernel<double2, 0, 4, 2, 3, false, 0>,
                                        level_kernel<double2, 0, 4, 2, 3, false, 1>,
                                        level_kernel<double2, 0, 4, 2, 3, false, 2>};
      return ncw == 16 ? p16[dt] : ncw == 4 ? p4[dt] : p8[dt];
    }
    static const LevelKernel r8[3] = {level_kernel<double2, 0, 8, 1, 1, false, 0>,
                                      level_kernel<double2, 0, 8, 1, 1, false, 1>,
                                      level_kernel<double2, 0, 8, 1, 1, false, 2>};
    static const LevelKernel r16[3] = {level_kernel<double2, 0, 16, 1, 1, false, 0>,
                                       level_kernel<double2, 0, 16, 1, 1, false, 1>,
                                       level_kernel<double2, 0, 16, 1, 1, false, 2>};
    static const LevelKernel r4[3] = {level_kernel<double2, 0, 4, 2, 1, false, 0>,
                                      level_kernel<double2, 0, 4, 2, 1, false, 1>,
                                      level_kernel<double2, 0, 4, 2, 1, false, 2>};
    return ncw == 16 ? r16[dt] : ncw == 4 ? r4[dt] : r8[dt];
  } else {
    return nullptr;
  }
}

// Padded shared-memory rows for the DMMA consumer (BF_NO_PAD=1 turns them off).
bool pad_disabled() {
  static const bool off = [] {
    const char* e = getenv("BF_NO_PAD");
    return e && *e && *e != '0';
  }();
  return off;
}

// Programmatic dependent launch between consecutive level kernels (the next
// level's prologue overlaps the previous one's tail); BF_NO_PDL=1 turns it off.
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("BF_NO_PDL");
    return !(e && *e && *e != '0');
  }();
  return on;
}

template <typename E>
int launch_level_t(const Plan& pl, const void* fac, uint32_t R, uint32_t C, uint32_t nt, uint32_t ntot, uint32_t t0,
                   int accumulate, uint64_t P, uint64_t units, const void* in, void* out, uint32_t k, int adjoint,
                   int remap, cudaStream_t st, void* const* peers, uint32_t tsplit = 1);

// Wide many-RHS levels (wide_kernel.cuh): complex128 units whose blocks do not fit a
// shared-memory stage whole (quadtree rank 25, C = 4r = 100) as a K-pipelined DMMA GEMM,
// one consumer warp per 8 output rows. BF_NO_WIDE=1 restores the whole-unit stage;
// BF_WIDE_KT sets the K tile (multiple of 4, default 20).
bool wide_disabled() {
  static const bool off = env_int("BF_NO_WIDE", 0) != 0;
  return off;
}
constexpr int kWideNcw = 13;

bool wide_applies(uint32_t R, uint32_t C, uint32_t nt, uint32_t k, int remap, size_t esz) {
  // units wider than one stage (C > 64), and the branching-4 units of a rank-16 chain folded
  // from pairs of binary levels (C = 64, nt = 4: 32.7 vs 53.9 ms at cfg2 size through the
  // whole-unit stage); BF_WIDE_MIN_C lowers the threshold for any shape
  static const uint32_t min_c = static_cast<uint32_t>(env_int("BF_WIDE_MIN_C", 65));
  return esz == 16 && !wide_disabled() && !dmma_disabled() && !gauss_disabled() && k >= kMrhsMinK && remap <= 2 &&
         (C >= min_c || (C == 64 && nt == 4)) && nt * R <= 8u * kWideNcw && C <= 8u * kWideNcw;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D FP64 tensor map over a row-major (rows x cols) array, box (box_cols x box_rows),
// no swizzle, zero fill out of bounds
int tmap_2d(CUtensorMap* tm, const void* base, uint64_t cols, uint64_t rows, uint32_t box_cols, uint32_t box_rows,
            CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  const auto enc = tmap_encoder();
  if (!enc) return fail(BF_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * sizeof(double)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BF_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return 0;
}

int launch_wide(const Plan& pl, const void* fac, uint32_t R, uint32_t C, uint32_t nt, uint64_t P, uint64_t units,
                const void* in, void* out, uint32_t k, int adjoint, int remap, cudaStream_t st) {
  auto pad_to = [](uint64_t x, uint64_t target) { return x + (target + 8 - x % 8) % 8; };
  auto up8 = [](uint64_t x) { return (x + 7) / 8 * 8; };  // 128-byte multiples of complex128
  WideArgs a{};
  a.out = static_cast<double2*>(out);
  a.mid_w = static_cast<const double*>(pl.weights);
  a.R = R;
  a.C = C;
  a.nt = nt;
  a.lgP = ilog2(P);
  a.k = k;
  // consumer warps: one per 8 output rows — 8 for the branching-4 units of a rank-16 chain
  // (64 rows either way), 13 for the r = 25 quadtree (100 rows); with 8 warps the register
  // budget allows 64 right-hand sides per item (NT = 8: each staged factor tile feeds twice
  // the DMMAs; BF_WIDE_NT8=0 keeps 32)
  const uint32_t ncw = std::max(nt * R, C) <= 64 ? 8 : kWideNcw;
  static const bool nt8 = env_int("BF_WIDE_NT8", 1) != 0;
  const uint32_t NT = (ncw == 8 && nt8 && k >= 64) ? 8 : k > 16 ? 4 : k > 8 ? 2 : 1;
  a.kc = std::min<uint32_t>(k, 8 * NT);
  a.nkc = (k + a.kc - 1) / a.kc;
  const uint64_t frows = units * nt * R, vrows = adjoint ? frows : units * C;
  if (units * a.nkc >= (1ull << 31) || frows >= (1ull << 31) || vrows >= (1ull << 31))
    return fail(BF_EINVAL, "level has too many blocks for one launch");
  a.items = static_cast<uint32_t>(units * a.nkc);
  // K tiles: forward BF_WIDE_KT block columns (multiple of 4, = 4 mod 8 for conflict-free A
  // fragment rows; default 20), adjoint one whole block (R rows)
  static const int kt_env0 = env_int("BF_WIDE_KT", 0);
  const int kt_env = kt_env0 > 0 ? kt_env0 : (C == 64 ? 36 : 20);   // C = 64: tiles of 36 + 28 columns (31.8 vs 33.0 ms at 20)
  if (!adjoint) {
    a.KT = std::min<uint32_t>(static_cast<uint32_t>(std::max(4, kt_env / 4 * 4)), (C + 3) / 4 * 4);
    a.nks = (C + a.KT - 1) / a.KT;
    a.fst = a.KT;
    a.fslot = static_cast<uint32_t>(up8(static_cast<uint64_t>(R) * a.KT));
    a.voff = nt * a.fslot;
  } else {
    a.KT = R;
    a.nks = nt;
    a.fst = static_cast<uint32_t>(pad_to(C, 2));  // A^H fragment columns: stride 2 mod 8
    a.fslot = 0;
    a.voff = static_cast<uint32_t>(up8(static_cast<uint64_t>(R) * a.fst));
  }
  a.vst = static_cast<uint32_t>(pad_to(8 * NT, 2));   // B fragment rows: stride 2 mod 8
  if (2 * a.fst > 256 || 2 * a.vst > 256 || a.KT > 256 || R > 256)
    return fail(BF_EINVAL, "wide level: tensor box exceeds 256 elements");
  const uint64_t stage = up8(a.voff + static_cast<uint64_t>(a.KT) * a.vst);
  a.stage_elems = static_cast<uint32_t>(stage);
  a.stage_bytes = static_cast<uint32_t>(
      ((adjoint ? static_cast<uint64_t>(R) * a.fst : static_cast<uint64_t>(nt) * R * a.KT) +
       static_cast<uint64_t>(a.KT) * a.vst) * sizeof(double2));
  const uint64_t fit = (static_cast<uint64_t>(kMaxDynSmem) - 128) / (stage * sizeof(double2));
  static const int st_env = env_int("BF_WIDE_STAGES", 8);
  a.stages = static_cast<uint32_t>(std::min<uint64_t>(fit, static_cast<uint64_t>(std::max(2, std::min(8, st_env)))));
  if (a.stages < 2) return fail(BF_EINVAL, "wide level: K tile does not double-buffer");
  a.adjoint = adjoint;
  a.remap = remap;
  a.m = pl.m;
  a.r = pl.rank;
  CUtensorMap tmA, tmV;
  // L2 promotion of the factor boxes (BF_WIDE_PROMO: 0 none, 1 64 B, 2 128 B, 3 256 B)
  static const int promo = std::max(0, std::min(3, env_int("BF_WIDE_PROMO", 3)));
  int rc = tmap_2d(&tmA, fac, 2ull * C, frows, adjoint ? 2 * a.fst : 2 * a.KT, R,
                   static_cast<CUtensorMapL2promotion>(CU_TENSOR_MAP_L2_PROMOTION_NONE + promo));
  if (!rc) rc = tmap_2d(&tmV, in, 2ull * k, vrows, 2 * a.vst, a.KT);
  if (rc) return rc;
  const size_t smem = 128 + static_cast<size_t>(a.stages) * stage * sizeof(double2);
  void (*kern)(const WideArgs, const CUtensorMap, const CUtensorMap) = nullptr;
  if (ncw == 8) {
    if (adjoint)
      kern = NT == 8 ? wide_kernel<8, 8, true> : NT == 4 ? wide_kernel<8, 4, true> : NT == 2 ? wide_kernel<8, 2, true> : wide_kernel<8, 1, true>;
    else
      kern = NT == 8 ? wide_kernel<8, 8, false> : NT == 4 ? wide_kernel<8, 4, false> : NT == 2 ? wide_kernel<8, 2, false> : wide_kernel<8, 1, false>;
  } else if (adjoint)
    kern = NT == 4 ? wide_kernel<kWideNcw, 4, true> : NT == 2 ? wide_kernel<kWideNcw, 2, true> : wide_kernel<kWideNcw, 1, true>;
  else
    kern = NT == 4 ? wide_kernel<kWideNcw, 4, false> : NT == 2 ? wide_kernel<kWideNcw, 2, false> : wide_kernel<kWideNcw, 1, false>;
  BF_CUDA(allow_max_dyn_smem(kern));
  static const bool dbg = env_int("BF_DEBUG_LAUNCH", 0) != 0;
  if (dbg)
    fprintf(stderr, "[bf] wide_kernel R=%u C=%u nt=%u units=%llu k=%u kc=%u NT=%u KT=%u nks=%u stages=%u smem=%zu adj=%d\n", R,
            C, nt, static_cast<unsigned long long>(units), k, a.kc, NT, a.KT, a.nks, a.stages, smem, adjoint);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min<uint32_t>(a.items, static_cast<uint32_t>(pl.sms)));
  cfg.blockDim = dim3((ncw + 1) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, kern, a, tmA, tmV));
  return 0;
}

// One factor launch. A unit's nt blocks normally share one tile; when they do
// not fit a shared-memory stage (quadtree rank 25: 4 x 25 x 100 complex128 =
// 160 KB) the blocks are split into t-ranges, one launch each: forward outputs
// are disjoint per t, adjoint partial sums accumulate into the output.
template <typename E>
int launch_level(const Plan& pl, const void* fac, uint32_t R, uint32_t C, uint32_t nt, uint64_t P, uint64_t units,
                 const void* in, void* out, uint32_t k, int adjoint, int remap, cudaStream_t st,
                 void* const* peers = nullptr) {
  if (wide_applies(R, C, nt, k, remap, sizeof(E)))
    return launch_wide(pl, fac, R, C, nt, P, units, in, out, k, adjoint, remap, st);
  const Shape sh = k >= kMrhsMinK ? mrhs_shape_for<E>(C) : stream_shape<E>();
  // wide many-RHS forward levels (quadtree r = 25: a unit is 160 KB of blocks), opt-in
  // BF_WIDE_SPLIT=1: the two t-halves of every unit as consecutive tiles of ONE launch
  // through two ~113 KB stages (forward outputs of different t are disjoint). Measured
  // slower than the single-buffered whole-unit stage (cfg3 0.595 vs 0.530 ms, cfg4b 11.5 vs
  // 9.9 ms): the half-unit warp items, not the exposed loads, set the pace.
  static const bool wide_split = env_int("BF_WIDE_SPLIT", 0) != 0;
  if (wide_split && !adjoint && !remap && k >= kMrhsMinK && sizeof(E) == 16 && C > 64 && nt % 2 == 0 &&
      static_cast<uint64_t>(nt / 2) * R * C + static_cast<uint64_t>(C) * std::min<uint32_t>(k, 16) <=
          (static_cast<uint64_t>(kMaxDynSmem) - 1024) / 2 / sizeof(E))
    return launch_level_t<E>(pl, fac, R, C, nt / 2, nt, 0, 0, P, units, in, out, k, adjoint, remap, st, peers, 2);
  uint32_t nt_tile = nt;
  auto tile_elems = [&](uint64_t t) { return t * R * C + (adjoint ? t * R : static_cast<uint64_t>(C)); };
  while (nt_tile > 1 && tile_elems(nt_tile) * sizeof(E) > sh.stage_bytes) nt_tile /= 2;
  if (nt_tile == nt)
    return launch_level_t<E>(pl, fac, R, C, nt, nt, 0, 0, P, units, in, out, k, adjoint, remap, st, peers);
  for (uint32_t t0 = 0; t0 < nt; t0 += nt_tile) {
    const int rc = launch_level_t<E>(pl, fac, R, C, nt_tile, nt, t0, adjoint && t0 > 0, P, units, in, out, k,
                                     adjoint, remap, st, peers);
    if (rc) return rc;
  }
  return 0;
}

template <typename E>
int launch_level_t(const Plan& pl, const void* fac, uint32_t R, uint32_t C, uint32_t nt, uint32_t ntot, uint32_t t0,
                   int accumulate, uint64_t P, uint64_t units, const void* in, void* out, uint32_t k, int adjoint,
                   int remap, cudaStream_t st, void* const* peers, uint32_t tsplit) {
  if (units >= (1ull << 31)) return fail(BF_EINVAL, "level has too many blocks for one launch");
  if constexpr (std::is_same<E, float2>::value) {
    // complex64 with >= 128 right-hand sides on tcgen05 (kind::tf32, 3xTF32) tiles of 128 RHS
    // (tc_kernel.cuh): opt-in BF_TC=1 — slower and less accurate than the FFMA consumer at the
    // benchmark shapes (cfg2 256 RHS: 46.7 vs 29.4 ms, rel. error 7.7e-6 vs 6.1e-7)
    static const bool tc_off = env_int("BF_TC", 0) == 0;
    const uint32_t N = adjoint ? C : nt * R, K = adjoint ? nt * R : C, Kp = (K + 7) / 8 * 8;
    const uint64_t tc_smem = 2 * 4ull * (128 + 2 * N) * Kp * 4 + static_cast<uint64_t>(K) * 128 * 8;
    // (bulk copies: even k keeps every 128-RHS row segment 16-byte aligned and sized)
    if (!tc_off && k >= 128 && k % 2 == 0 && remap < 3 && !accumulate && nt == ntot && N % 16 == 0 && N <= 128 &&
        2 * N <= 256 && Kp <= 64 && (static_cast<uint64_t>(R) * C) % 2 == 0 &&
        static_cast<uint64_t>(N) * (Kp / 4) <= static_cast<uint64_t>(kTcBItems) * kTcSplitWarps * 32 &&
        tc_smem + 1024 <= static_cast<uint64_t>(kMaxDynSmem)) {
      TcArgs a{};
      a.fac = static_cast<const float2*>(fac);
      a.in = static_cast<const float2*>(in);
      a.out = static_cast<float2*>(out);
      a.mid_w = static_cast<const float*>(pl.weights);
      a.R = R;
      a.C = C;
      a.nt = nt;
      a.lgP = ilog2(P);
      a.units = static_cast<uint32_t>(units);
      a.k = k;
      a.ktiles = (k + 127) / 128;
      a.N = N;
      a.K = K;
      a.Kp = Kp;
      a.adjoint = adjoint;
      a.remap = remap;
      a.m = pl.m;
      a.r = pl.rank;
      uint32_t cols = 32;
      while (cols < 4 * N) cols *= 2;   // two accumulators [Re | Im]
      a.tmem_cols = cols;
      a.trace = g_node_trace;
      // tf32 planes + two raw tiles (X rows of 128 RHS, the unit's blocks)
      const size_t smem = 2 * 4ull * (128 + 2 * N) * Kp * 4 + static_cast<uint64_t>(K) * 128 * 8;
      BF_CUDA(allow_max_dyn_smem(tc_level_kernel));
      const uint64_t ntiles = units * a.ktiles;
      const uint32_t per_sm = 1;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(static_cast<unsigned>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(pl.sms) * per_sm)));
      cfg.blockDim = dim3(kTcThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      BF_CUDA(cudaLaunchKernelEx(&cfg, tc_level_kernel, a));
      return 0;
    }
  }
  if (remap && static_cast<uint64_t>(pl.m) * pl.m * pl.rank >= (1ull << 32))
    return fail(BF_EINVAL, "middle vector too long for 32-bit remap indices");
  const bool mrhs = k >= kMrhsMinK;
  constexpr Shape ks = stream_shape<E>();
  Shape sh = mrhs ? mrhs_shape_for<E>(C) : ks;
  const bool sexp = !mrhs && sizeof(E) == 16 && remap < 3 && stream_exp().on;
  if (sexp) sh = stream_exp().s;
  if (tsplit > 1) {   // t-range tiles of one launch: double-buffered half-units
    sh.stages = 2;
    sh.stage_bytes = (static_cast<uint32_t>(kMaxDynSmem) - 1024) / 2;
  }
  // complex128 DMMA consumers: 16 warps for the wide quadtree blocks (C = 4r = 100: long
  // k loops, few warp items per tile; cfg3 0.75 -> 0.59 ms, cfg4b 14.6 -> 11.0 ms), 8
  // otherwise (cfg2 k = 256: 43.9 vs 47.3 ms; cfg1 0.26 vs 0.32 ms)
  // complex128 DMMA shapes with C <= 64 (binary trees, r <= 32): two independent 4-warp
  // CTAs per SM on 48 KB stages (k = 64 tiles), each with its own in-place barrier, so the
  // two CTAs' compute and store phases interleave (cfg2 k=256 41.5 -> 37.6 ms, k=64
  // 10.8 -> 9.6 ms, k=16 6.1 -> 3.9 ms; cfg1 0.284 -> 0.271 ms)
  if (mrhs && sh.ncw != 16 && sh.ncw != 8 && sh.ncw != 4) {
    if (C > 64) {
      sh.ncw = 16;
    } else if (sizeof(E) == 16 && !dmma_disabled() && remap < 3 &&
               (static_cast<uint64_t>(nt) * R * C + (adjoint ? static_cast<uint64_t>(nt) * R : C) * 16) * 16 <=
                   48 * 1024) {
      sh.ncw = 4;
      if (knobs().mrhs_stage_kb == 0) sh.stage_bytes = 48 * 1024;
    } else {
      sh.ncw = 8;
    }
  }
  if (mrhs && sh.ncw == 4) sh.ctas_per_sm = 2;  // two independent 4-warp CTAs per SM
  LevelArgs a{};
  a.fac = fac;
  a.in = in;
  a.out = out;
  a.mid_w = pl.weights;
  a.R = R;
  a.C = C;
  a.nt = nt;
  a.ntot = ntot;
  a.t0 = t0;
  a.accumulate = accumulate;
  a.lgP = ilog2(P);
  a.units = static_cast<uint32_t>(units);
  a.k = k;
  a.adjoint = adjoint;
  a.remap = remap;
  a.m = pl.m;
  a.r = pl.rank;
  a.part = pl.part;
  a.mp = pl.m / pl.nparts;
  PeerArgs pa{};
  if (remap >= 3) {
    if (!peers || pl.nparts > 8) return fail(BF_EINVAL, "peer push needs <= 8 receive buffers");
    for (uint32_t d = 0; d < pl.nparts; ++d) pa.peers[d] = peers[d];
  }
  const uint64_t esz = sizeof(E);
  const uint64_t fac_unit = static_cast<uint64_t>(nt) * R * C;
  const uint64_t vec_col = adjoint ? static_cast<uint64_t>(nt) * R : C;  // vector elems per unit per rhs
  const uint64_t m_out = adjoint ? C : static_cast<uint64_t>(nt) * R;
  // right-hand sides per tile: all of them unless one unit no longer fits a stage
  // right-hand sides per tile: up to 128 (complex128) / 256 (complex64: a whole 256-RHS
  // row range in one contiguous copy; cfg2 c64 k=256 34.5 -> 30.2 ms)
  static const int kt_env = env_int("BF_MRHS_KT_MAX", 0);
  const uint32_t kt_max = kt_env > 0 ? static_cast<uint32_t>(std::max(8, kt_env)) : (sizeof(E) == 8 ? 256u : 128u);
  uint32_t kt = mrhs ? std::min<uint32_t>(k, kt_max) : k;
  while (kt > 1 && (fac_unit + vec_col * kt) * esz > sh.stage_bytes) kt = (kt + 1) / 2;
  if (mrhs && kt > 4) kt = (kt + 3) / 4 * 4;
  if (esz == 8 && kt > 1 && (kt & 1)) ++kt;
  kt = std::min(kt, k);
  uint64_t U = 1;
  const uint64_t want_items = static_cast<uint64_t>(sh.ncw) * 32;
  // many-RHS warp tiles cover (32/LC)*TM rows x LC*TN columns (see consume_tile_mrhs_any)
  const uint64_t tile_rows = kt >= 32 ? (kt >= 128 ? 4 : kt >= 64 ? 8 : 16) : (kt >= 16 ? 16 : 16);
  const uint64_t tile_cols = kt >= 128 ? 128 : kt >= 64 ? 64 : kt >= 32 ? 32 : kt >= 16 ? 16 : 8;
  auto items = [&](uint64_t u) { return u * ((m_out + tile_rows - 1) / tile_rows) * ((kt + tile_cols - 1) / tile_cols) * 32; };
  while (nt == ntot && U * 2 <= units && (U * 2) * (fac_unit + vec_col * kt) * esz <= sh.stage_bytes &&
         (!mrhs || items(U) < want_items))
    U *= 2;
  a.kt = kt;
  a.ktiles = (k + kt - 1) / kt;
  a.lgU = ilog2(U);
  a.tsplit = tsplit;
  a.ntiles = static_cast<uint32_t>((units / U) * a.ktiles * tsplit);
  uint64_t stage = U * (fac_unit + vec_col * kt);
  if (stage & 1) ++stage;
  a.stage_elems = static_cast<uint32_t>(stage);
  const bool aligned = (reinterpret_cast<uintptr_t>(fac) % 16 == 0) && (reinterpret_cast<uintptr_t>(in) % 16 == 0);
  // every bulk copy must move a multiple of 16 bytes between 16-byte aligned addresses:
  // complex128 always does; complex64 needs even block sizes and, when a row is split
  // into k-tiles, even k and kt.
  a.use_dmma = mrhs && esz == 16 && kt >= 16 && !dmma_disabled() ? (gauss_disabled() ? 1 : 2) : 0;
  // complex64: blocks of an even element count (R C even) keep every block start 16-byte
  // aligned, and an even k (and kt) every vector row (cfg3/cfg4b: R = 25, C = 100)
  const uint64_t vec_unit = adjoint ? static_cast<uint64_t>(R) * k : static_cast<uint64_t>(C) * k;  // chunk stride
  a.bulk = aligned && (esz == 16 || ((static_cast<uint64_t>(R) * C) % 2 == 0 &&
                                     (a.ktiles == 1 ? vec_unit % 2 == 0 : (k % 2 == 0 && kt % 2 == 0))));
  a.fld = C;
  a.vld = 0;
  if (a.use_dmma && a.bulk && a.ktiles > 1 && !pad_disabled()) {  // rows are copied one by one anyway
    // DMMA fragment loads: a quarter warp reads rows (lane/4) x k-slots (lane%4) of a
    // factor block and k-rows x columns of the vector tile; row strides = 4 (forward
    // A), 2 (adjoint A, vectors) mod 8 sixteen-byte units put the 8 lanes of every
    // quarter warp on distinct bank groups (unpadded: 2- to 4-way conflicts)
    auto pad_to = [](uint64_t x, uint64_t target) { return x + (target + 8 - x % 8) % 8; };
    const uint64_t fld = pad_to(C, adjoint ? 2 : 4), vld = pad_to(kt, 2);
    const uint64_t vrows = adjoint ? static_cast<uint64_t>(nt) * R : C;
    uint64_t Up = U;
    auto padded = [&](uint64_t u) { return u * (static_cast<uint64_t>(nt) * R * fld + vrows * vld); };
    while (Up > 1 && 128 + sh.stages * padded(Up) * esz > static_cast<uint64_t>(kMaxDynSmem)) Up /= 2;
    if (128 + sh.stages * padded(Up) * esz <= static_cast<uint64_t>(kMaxDynSmem)) {
      U = Up;
      a.lgU = ilog2(U);
      a.ntiles = static_cast<uint32_t>((units / U) * a.ktiles * tsplit);
      a.fld = static_cast<uint32_t>(fld);
      a.vld = static_cast<uint32_t>(vld);
      uint64_t st2 = padded(U);
      if (st2 & 1) ++st2;
      a.stage_elems = static_cast<uint32_t>(st2);
    }
  }
  const int stages = sh.stages;
  a.stages = static_cast<uint32_t>(stages);
  a.dbg_nomath = knobs().dbg_nomath;
  a.dbg_noload = mrhs ? knobs().dbg_noload : 0;
  if (a.use_dmma) {  // warp tile: the largest that still gives every consumer warp an item
    const uint64_t ncw = (a.use_dmma == 2 && remap < 3) ? sh.ncw : kMrhs.ncw;
    auto di = [&](uint64_t mt, uint64_t n8) {
      return U * ((m_out + 8 * mt - 1) / (8 * mt)) * ((a.kt + 8 * n8 - 1) / (8 * n8));
    };
    a.dtile = a.kt >= 32 && di(2, 4) >= ncw ? 0 : (di(2, 2) >= ncw || a.kt < 16) ? 1 : 2;
    const int forced = knobs().dtile;
    if (forced >= 0 && forced <= 2) a.dtile = static_cast<uint32_t>(forced);
  }
  const size_t smem = 128 + static_cast<size_t>(stages) * a.stage_elems * esz;
  if (smem > 227 * 1024) return fail(BF_EINVAL, "rank too large: one block pair exceeds the shared-memory stage");
  // the peer-push epilogue (remap 3/4) is its own instantiation: compiled into the common
  // kernels it costs the many-RHS paths registers and ~8% (cfg2 k=256)
  const bool push = remap >= 3;
  // complex64 FFMA consumers may run 16 warps too (their own instantiation; complex128's
  // generic kernel stays at 8: it also carries the 4-product DMMA paths)
  const bool ffma16 = mrhs && !push && a.use_dmma == 0 && sizeof(E) == 8 && sh.ncw == 16;
  const int kncw = ffma16 ? 16 : (mrhs && (push || a.use_dmma != 2)) ? kMrhs.ncw : sh.ncw;
  // in-place outputs (MRHS = 3): every consumer warp holds at most one warp item per tile,
  // the outputs fit the tile's vector rows, and the rows have one stride in every tile
  bool inplace = false;
  // (8-warp shapes only: the 16-warp quadtree levels measured 2-5% slower in place)
  if (a.use_dmma == 2 && !push && !accumulate && a.bulk && !inplace_disabled() && (kncw == 8 || kncw == 4) &&
      m_out <= vec_col && (a.vld != 0 || a.ktiles == 1)) {
    const uint64_t mt = a.dtile == 2 ? 1 : 2, n8 = a.dtile == 0 ? 4 : 2;
    const uint64_t items = U * ((m_out + 8 * mt - 1) / (8 * mt)) * ((a.kt + 8 * n8 - 1) / (8 * n8));
    inplace = items <= static_cast<uint64_t>(kncw);
  }
  a.inplace = inplace ? 1 : 0;
  a.old = inplace ? (a.vld ? a.vld : a.kt) : a.old;
  LevelKernel kern =
      a.use_dmma == 2 && !push ? dmma_kernel<E>(kncw, a.dtile, inplace)
      : mrhs ? (push     ? level_kernel<E, 0, kMrhs.ncw, kMrhs.ctas_per_sm, 1, true>
                : ffma16 ? ffma16_kernel<E>()
                         : level_kernel<E, 0, kMrhs.ncw, kMrhs.ctas_per_sm, 1, false>)
           : (push ? level_kernel<E, ks.stages, ks.ncw, ks.ctas_per_sm, 0, true>
              : sexp ? (sh.ncw == 4 ? level_kernel<E, 0, 4, 2, 0, false>
                        : sh.ctas_per_sm == 3 ? level_kernel<E, 0, 2, 3, 0, false>
                                              : level_kernel<E, 0, 2, 2, 0, false>)
                   : level_kernel<E, ks.stages, ks.ncw, ks.ctas_per_sm, 0, false>);
  BF_CUDA(allow_max_dyn_smem(kern));
  const uint64_t per_sm = (kncw == sh.ncw) && smem * sh.ctas_per_sm <= 227 * 1024 ? sh.ctas_per_sm : 1;
  const uint64_t grid = std::min<uint64_t>(a.ntiles, static_cast<uint64_t>(pl.sms) * per_sm);
  static const bool dbg = [] {
    const char* e = getenv("BF_DEBUG_LAUNCH");
    return e && *e && *e != '0';
  }();
  if (dbg)
    fprintf(stderr, "[bf] level_kernel %s%s R=%u C=%u nt=%u units=%llu k=%u kt=%u U=%llu ntiles=%u grid=%llu smem=%zu dmma=%d\n",
            mrhs ? "mrhs" : "stream", push ? "+push" : "", R, C, nt, static_cast<unsigned long long>(units), k, kt,
            static_cast<unsigned long long>(U), a.ntiles, static_cast<unsigned long long>(grid), smem,
            a.use_dmma + (inplace ? 20 : 0));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3((kncw + 1) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, kern, a, pa));
  return 0;
}

}  // namespace

template <typename E>
int launch_middle(const Plan& pl, const void* in, void* out, uint32_t k, int adjoint, cudaStream_t st) {
  const uint64_t total = static_cast<uint64_t>(pl.m) * pl.m * pl.rank * k;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, pl.sms * 8ull));
  middle_kernel<E><<<grid, 256, 0, st>>>(static_cast<const E*>(in), static_cast<E*>(out),
                                         static_cast<const typename Cx<E>::R*>(pl.weights), pl.m, pl.rank, k,
                                         adjoint);
  BF_CUDA(cudaGetLastError());
  return 0;
}

namespace {

// Level pairs (pair_kernel.cuh): two adjacent splitting transfer levels i, i + 1 of a
// binary-tree complex128 plan in one kernel when the whole item (8 blocks + 2C vector
// rows, all right-hand sides) double-buffers in shared memory next to the 2C-row
// intermediate. BF_NO_PAIR=1 turns it off.
bool pair_disabled() {
  static const bool off = [] {
    const char* e = getenv("BF_NO_PAIR");
    return e && *e && *e != '0';
  }();
  return off;
}

constexpr int kPairNcw = 8;
// pipeline depth of the whole-tile pair kernel (2, 3 or 4; BF_PAIR_STAGES overrides)
int pair_stages() {
  static const int st = std::max(2, std::min(4, env_int("BF_PAIR_STAGES", 2)));
  return st;
}

// k-chunked pairs (pair_chunk_kernel) only with BF_CHUNK_PAIR=1: at cfg2 k = 256 they
// halve the vector traffic but run 47.3 ms against 43.8 ms for single levels (32-RHS
// chunks leave each warp 8 x 16 GEMM slices with 6 DMMAs per k-step: latency bound)
bool chunk_pair_disabled() {
  static const bool off = env_int("BF_CHUNK_PAIR", 0) == 0;
  return off;
}

struct PairGeo {
  uint32_t fld, vld, stage_elems;
  size_t smem;
  bool chunk;             // k-chunked kernel (factor blocks once per item, input rows in chunks)
  uint32_t kc, nch, stages;
  uint32_t ctas = 1;      // whole-tile pair kernel: CTAs per SM
};

bool pair_geometry(const Plan& pl, int i, uint32_t k, int adjoint, PairGeo* pg) {
  // k >= 64: below, the single-level kernel is faster (cfg1 at k = 32: 0.18 vs 0.20 ms)
  if (pair_disabled() || pl.dtype != BF_C128 || pl.branch != 2 || k < 64) return false;
  if (i < 0 || i + 1 >= static_cast<int>(pl.nlev)) return false;
  const LevelGeo& A = pl.lev[i];
  const LevelGeo& B = pl.lev[i + 1];
  if (!A.splits || !B.splits || A.P < 2 || B.G != 2 * A.G || 2 * B.P != A.P) return false;
  const uint64_t R = pl.rank, C = 2 * R;
  auto pad_to = [](uint64_t x, uint64_t target) { return x + (target + 8 - x % 8) % 8; };
  // unpadded factor rows, copied as whole blocks: 6 bulk copies per item instead of one per
  // block row — the producer warp's copy issue rate, not the DMMA pipe, paced the pairs
  // (ncu: 29% of consumer stall samples on the stage's full barrier; cfg1 268 -> 239 us).
  // The A-fragment reads take 2- to 4-way bank conflicts instead. BF_PAIR_FPAD=1 pads again.
  static const bool fpad = env_int("BF_PAIR_FPAD", 0) != 0;
  const uint64_t fld = fpad ? pad_to(C, adjoint ? 2 : 4) : C;
  pg->fld = static_cast<uint32_t>(fld);
  pg->chunk = false;
  // rank 8 (pair8_kernel): 32-RHS chunks as independent items whatever k is
  static const bool no_pair8 = env_int("BF_NO_PAIR8", 0) != 0;
  static const int kc_env0 = env_int("BF_PAIR_KC", 0);
  const bool p8 = R == 8 && !no_pair8 && !gauss_disabled() && k % 32 == 0 && kc_env0 <= 0;
  if (k <= 256 || p8) {  // whole right-hand-side range per stage (or k / 2 chunks), double-buffered
    // BF_PAIR_VPAD=0: unpadded vector rows (whole-k items copy contiguous row runs; measured
    // slower: 4-way conflicts on the X fragments, cfg1 257.6 vs 239.4 us)
    static const bool vpad = env_int("BF_PAIR_VPAD", 1) != 0;
    auto vld_for = [&](uint64_t kc) { return vpad ? pad_to(kc, 2) : kc; };
    auto smem_for = [&](uint64_t kc, uint64_t* stage_out) {
      const uint64_t vld = vld_for(kc);
      uint64_t stage = 8 * R * fld + 2 * C * vld;
      if (stage & 1) ++stage;
      *stage_out = stage;
      return 128 + (pair_stages() * stage + 2 * C * vld) * sizeof(double2);
    };
    // Right-hand-side chunks are independent items: halving the chunk lets two CTAs share an
    // SM (18 warps instead of 9 to cover the DMMA and shared-memory latencies) at the cost of
    // reading each pair's factor blocks once per chunk. BF_PAIR_KC overrides the chunk width.
    static const int kc_env = env_int("BF_PAIR_KC", 0);
    uint64_t kc = k, stage = 0;
    if (p8) {
      kc = 32;
    } else if (kc_env > 0) {
      kc = std::min<uint64_t>(k, static_cast<uint64_t>(kc_env));
    } else if (2 * smem_for(k, &stage) > static_cast<uint64_t>(kMaxDynSmem) && k >= 64 &&
               2 * smem_for((k + 1) / 2, &stage) <= static_cast<uint64_t>(kMaxDynSmem)) {
      kc = (k + 1) / 2;
    }
    const uint64_t smem = smem_for(kc, &stage);
    if (smem <= static_cast<uint64_t>(kMaxDynSmem)) {
      pg->vld = static_cast<uint32_t>(vld_for(kc));
      pg->stage_elems = static_cast<uint32_t>(stage);
      pg->smem = smem;
      pg->kc = static_cast<uint32_t>(kc);
      pg->nch = static_cast<uint32_t>((k + kc - 1) / kc);
      pg->ctas = 2 * smem <= static_cast<uint64_t>(kMaxDynSmem) ? 2 : 1;
      return true;
    }
  }
  if (chunk_pair_disabled()) return false;
  // k-chunked: factor buffer + a ring of 32-RHS input chunks + the chunk intermediate
  const uint64_t kc = 32, vld = pad_to(kc, 2), stage = 2 * C * vld;
  for (uint64_t S = 4; S >= 2; --S) {
    const uint64_t smem = 128 + (8 * R * fld + S * stage + kPairNcw * C * 9) * sizeof(double2);
    if (smem > static_cast<uint64_t>(kMaxDynSmem)) continue;
    pg->chunk = true;
    pg->kc = static_cast<uint32_t>(kc);
    pg->nch = static_cast<uint32_t>((k + kc - 1) / kc);
    pg->stages = static_cast<uint32_t>(S);
    pg->vld = static_cast<uint32_t>(vld);
    pg->stage_elems = static_cast<uint32_t>(stage);
    pg->smem = smem;
    return true;
  }
  return false;
}

int launch_pair_chunk(const Plan& pl, const void* fac_a, const void* fac_b, int i, const void* in, void* out,
                      uint32_t k, int adjoint, const PairGeo& pg, cudaStream_t st) {
  const LevelGeo& A = pl.lev[i];
  PairChunkArgs a{};
  a.fac_a = static_cast<const double2*>(fac_a);
  a.fac_b = static_cast<const double2*>(fac_b);
  a.in = static_cast<const double2*>(in);
  a.out = static_cast<double2*>(out);
  a.r = pl.rank;
  a.ga = static_cast<uint32_t>(A.G);
  a.pa = static_cast<uint32_t>(A.P);
  a.k = k;
  a.kc = pg.kc;
  a.nch = pg.nch;
  a.adjoint = adjoint;
  a.nitems = static_cast<uint32_t>(A.G * A.P / 2);
  a.fld = pg.fld;
  a.vld = pg.vld;
  a.stages = pg.stages;
  a.stage_elems = pg.stage_elems;
  auto* kern = gauss_disabled() ? pair_chunk_kernel<kPairNcw, false> : pair_chunk_kernel<kPairNcw, true>;
  BF_CUDA(allow_max_dyn_smem(kern));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min<uint32_t>(a.nitems, static_cast<uint32_t>(pl.sms)));
  cfg.blockDim = dim3((kPairNcw + 1) * 32);
  cfg.dynamicSmemBytes = pg.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return 0;
}

// Rank-8 fast path of the level pairs (pair8_kernel): warp-owned (t, 16-column) slices, no
// block barrier between the levels. BF_NO_PAIR8=1 turns it off; BF_PAIR8_STAGES=1 runs one
// stage per CTA (up to four CTAs per SM) instead of two (measured: cfg1 0.227 vs 0.197 ms).
int pair8_stages() {
  static const int st = env_int("BF_PAIR8_STAGES", 2) == 1 ? 1 : 2;
  return st;
}
bool pair8_ok(const Plan& pl, const PairGeo& pg, uint32_t k) {
  static const bool off = env_int("BF_NO_PAIR8", 0) != 0;
  return !off && !pg.chunk && !gauss_disabled() && pl.rank == 8 && (pg.kc == 32 || pg.kc == 64) && k % 16 == 0;
}
// stage of the leaf-fused pair: 8 unpadded blocks, 4 leaf blocks (16 x 8), the input rows
uint32_t pair8_leaf_stage(uint32_t vld, int adjoint) { return 8 * 8 * 16 + 4 * 16 * 8 + (adjoint ? 64u : 32u) * vld; }
size_t pair8_smem(uint32_t stage_elems, uint32_t vld) {
  return 128 + (static_cast<size_t>(pair8_stages()) * stage_elems + 2 * 16 * vld) * sizeof(double2);
}
uint32_t pair8_ctas(uint32_t ncw, int adjoint, size_t smem) {
  const size_t cap = pair8_stages() == 1 ? (ncw == 4 ? (adjoint ? 3 : 4) : 2) : (ncw == 4 ? 2 : 1);
  return static_cast<uint32_t>(std::min<size_t>(cap, static_cast<size_t>(kMaxDynSmem) / (smem + 1024)));
}
// The leaf factor rides in the pair next to it (the down half's first pair reads the chain
// input, the up half's last pair writes the chain output): 16-point leaves, unpadded
// blocks. The right-hand-side chunk (32 or 64) is the one that keeps the most consumer
// warps per SM with the larger stage. BF_NO_PAIR8_LEAF=1 turns it off.
bool pair8_leaf_geo(const Plan& pl, const PairGeo& pg, uint32_t k, int adjoint, PairGeo* out) {
  static const bool off = env_int("BF_NO_PAIR8_LEAF", 0) != 0;
  if (off || !pair8_ok(pl, pg, k) || pl.leaf_n0 != 16 || pg.fld != 16 || pl.nparts != 1) return false;
  uint32_t best = 0;
  for (uint32_t kc : {pg.kc, 64u}) {
    if (kc > k || kc < pg.kc) continue;
    const uint32_t vld = pg.vld == pg.kc ? kc : kc + 2;
    const uint32_t stage = pair8_leaf_stage(vld, adjoint);
    const size_t smem = pair8_smem(stage, vld);
    if (smem > static_cast<size_t>(kMaxDynSmem)) continue;
    const uint32_t warps = pair8_ctas(kc / 8, adjoint, smem) * (kc / 8);
    if (warps > best) {
      best = warps;
      *out = pg;
      out->kc = kc;
      out->nch = (k + kc - 1) / kc;
      out->vld = vld;
      out->stage_elems = stage;
      out->smem = smem;
    }
  }
  return best > 0;
}

// Rank-16 pairs with register-fed factors (pair16_kernel.cuh): shared memory holds only
// the item's vectors (64 rows x 32 right-hand sides per stage) and the pair's intermediate,
// so two CTAs share an SM. Opt-in (BF_PAIR16=1; 2 = forward pairs only): at config 2 with 256
// right-hand sides a pair moves 10.0 GB of DRAM traffic instead of 18.2 GB for its two levels,
// but runs 4.17 ms forward (DMMA pipe 67%) and 5.3 ms adjoint (51%: its two-block K ranges
// spill registers) against 2 x 2.17 ms — 42.3 vs 38.2 ms per apply. BF_PAIR16_STAGES=3
// deepens the ring (one CTA per SM: 60.7 ms).
bool pair16_geometry(const Plan& pl, int i, uint32_t k, int adjoint, PairGeo* pg) {
  static const int mode = env_int("BF_PAIR16", 0);
  static const int kmin = env_int("BF_PAIR16_MIN_K", 64);
  const bool off = mode == 0 || (mode == 2 && adjoint);
  if (off || pair_disabled() || gauss_disabled() || pl.dtype != BF_C128 || pl.branch != 2 || pl.rank != 16) return false;
  if (k < static_cast<uint32_t>(kmin) || k % 32 != 0) return false;
  if (i < 0 || i + 1 >= static_cast<int>(pl.nlev)) return false;
  const LevelGeo& A = pl.lev[i];
  const LevelGeo& B = pl.lev[i + 1];
  if (!A.splits || !B.splits || A.P < 2 || B.G != 2 * A.G || 2 * B.P != A.P) return false;
  static const int stages = env_int("BF_PAIR16_STAGES", 2) == 3 ? 3 : 2;
  pg->fld = 32;
  pg->vld = 34;
  pg->stage_elems = 64 * 34;
  pg->kc = 32;
  pg->nch = k / 32;
  pg->stages = static_cast<uint32_t>(stages);
  pg->smem = 128 + static_cast<size_t>(stages + 1) * pg->stage_elems * sizeof(double2);
  pg->chunk = false;
  pg->ctas = stages == 2 ? 2 : 1;
  return true;
}

int launch_pair16(const Plan& pl, const void* fac_a, const void* fac_b, int i, const void* in, void* out, uint32_t k,
                  int adjoint, const PairGeo& pg, cudaStream_t st, int remap) {
  const LevelGeo& A = pl.lev[i];
  PairArgs a{};
  a.fac_a = static_cast<const double2*>(fac_a);
  a.fac_b = static_cast<const double2*>(fac_b);
  a.in = static_cast<const double2*>(in);
  a.out = static_cast<double2*>(out);
  a.r = pl.rank;
  a.ga = static_cast<uint32_t>(A.G);
  a.pa = static_cast<uint32_t>(A.P);
  a.k = k;
  a.kc = pg.kc;
  a.nch = pg.nch;
  a.adjoint = adjoint;
  a.nitems = static_cast<uint32_t>(A.G * A.P / 2 * pg.nch);
  a.fld = pg.fld;
  a.vld = pg.vld;
  a.stage_elems = pg.stage_elems;
  a.remap = remap;
  a.m = pl.m;
  a.mr = pl.rank;
  a.mid_w = static_cast<const double*>(pl.weights);
  void (*kern)(const PairArgs) = pg.stages == 3 ? (adjoint ? pair16_kernel<3, true> : pair16_kernel<3, false>)
                                                : (adjoint ? pair16_kernel<2, true> : pair16_kernel<2, false>);
  BF_CUDA(allow_max_dyn_smem(kern));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min<uint32_t>(a.nitems, static_cast<uint32_t>(pl.sms) * pg.ctas));
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = pg.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return 0;
}

int launch_pair(const Plan& pl, const void* fac_a, const void* fac_b, int i, const void* in, void* out, uint32_t k,
                int adjoint, const PairGeo& pg, cudaStream_t st, int remap = 0, const void* leaf = nullptr) {
  if (pg.chunk) return launch_pair_chunk(pl, fac_a, fac_b, i, in, out, k, adjoint, pg, st);
  const LevelGeo& A = pl.lev[i];
  PairArgs a{};
  a.fac_a = static_cast<const double2*>(fac_a);
  a.fac_b = static_cast<const double2*>(fac_b);
  a.in = static_cast<const double2*>(in);
  a.out = static_cast<double2*>(out);
  a.r = pl.rank;
  a.ga = static_cast<uint32_t>(A.G);
  a.pa = static_cast<uint32_t>(A.P);
  a.k = k;
  a.kc = pg.kc;
  a.nch = pg.nch;
  a.adjoint = adjoint;
  a.nitems = static_cast<uint32_t>(A.G * A.P / 2 * pg.nch);
  a.fld = pg.fld;
  a.vld = pg.vld;
  a.stage_elems = pg.stage_elems;
  a.remap = remap;
  a.m = pl.m;
  a.mr = pl.rank;
  a.mid_w = static_cast<const double*>(pl.weights);
  // rank 8, 16-column slices (pair8_kernel): warp-owned slices, no block barrier between
  // the levels; one stage per CTA and up to four CTAs per SM. BF_NO_PAIR8=1 turns it off,
  // BF_PAIR8_STAGES=2 double-buffers inside the CTA instead.
  if (pair8_ok(pl, pg, k)) {
    const int p8_stages = pair8_stages();
    a.leaf = static_cast<const double2*>(leaf);   // leaf: pg is pair8_leaf_geo's (its stage holds the leaf blocks)
    const size_t smem = pair8_smem(a.stage_elems, pg.vld);
    if (smem > static_cast<size_t>(kMaxDynSmem)) return fail(BF_EINVAL, "leaf-fused pair exceeds shared memory");
    const uint32_t ncw = pg.kc / 8;
    void (*kern)(const PairArgs);
    if (leaf)
      kern = ncw == 4 ? (p8_stages == 2 ? (adjoint ? pair8_kernel<2, true, 4, true> : pair8_kernel<2, false, 4, true>)
                                        : (adjoint ? pair8_kernel<1, true, 4, true> : pair8_kernel<1, false, 4, true>))
                      : (p8_stages == 2 ? (adjoint ? pair8_kernel<2, true, 8, true> : pair8_kernel<2, false, 8, true>)
                                        : (adjoint ? pair8_kernel<1, true, 8, true> : pair8_kernel<1, false, 8, true>));
    else
      kern = ncw == 4 ? (p8_stages == 2 ? (adjoint ? pair8_kernel<2, true, 4, false> : pair8_kernel<2, false, 4, false>)
                                        : (adjoint ? pair8_kernel<1, true, 4, false> : pair8_kernel<1, false, 4, false>))
                      : (p8_stages == 2 ? (adjoint ? pair8_kernel<2, true, 8, false> : pair8_kernel<2, false, 8, false>)
                                        : (adjoint ? pair8_kernel<1, true, 8, false> : pair8_kernel<1, false, 8, false>));
    BF_CUDA(allow_max_dyn_smem(kern));
    static const int ctas_env = env_int("BF_PAIR8_CTAS", 0);
    uint32_t ctas = pair8_ctas(ncw, adjoint, smem);
    if (ctas_env > 0) ctas = std::min<uint32_t>(ctas, static_cast<uint32_t>(ctas_env));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(std::min<uint32_t>(a.nitems, static_cast<uint32_t>(pl.sms) * std::max(1u, ctas)));
    cfg.blockDim = dim3((ncw + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    BF_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    return 0;
  }
  const int ps = pair_stages();
  auto* kern = gauss_disabled() ? pair_kernel<2, kPairNcw, false>
               : ps == 4       ? pair_kernel<4, kPairNcw, true>
               : ps == 3       ? pair_kernel<3, kPairNcw, true>
                               : pair_kernel<2, kPairNcw, true>;
  BF_CUDA(allow_max_dyn_smem(kern));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min<uint32_t>(a.nitems, static_cast<uint32_t>(pl.sms) * pg.ctas));
  cfg.blockDim = dim3((kPairNcw + 1) * 32);
  cfg.dynamicSmemBytes = pg.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return 0;
}

// One factor op, dispatched by kind. `lvl_idx` indexes the plan's level table.
template <typename E>
int factor_op(const Plan& pl, int which, int lvl_idx, int adjoint, const void* in, void* out, uint32_t k, int remap,
              cudaStream_t st, void* const* peers = nullptr, bool fold = false) {
  if (which == BF_FACTOR_V || which == BF_FACTOR_U) {
    const void* fac = which == BF_FACTOR_V ? pl.v_leaf : pl.u_leaf;
    return launch_level<E>(pl, fac, pl.leaf_n0, pl.rank, 1, 1, pl.leaf_nb, in, out, k, adjoint, 0, st);
  }
  if (which == BF_FACTOR_M) return launch_middle<E>(pl, in, out, k, adjoint, st);
  const LevelGeo& lg = pl.lev[lvl_idx];
  if (fold) {  // the outermost level with its leaf factor folded in: blocks (n0 x C)
    const void* fac = which == BF_FACTOR_G ? pl.g_fold : pl.h_fold;
    return launch_level<E>(pl, fac, pl.leaf_n0, pl.branch * pl.rank, lg.splits ? pl.branch : 1, lg.P, lg.G * lg.P, in,
                           out, k, adjoint, remap, st, peers);
  }
  const void* fac = which == BF_FACTOR_G ? pl.g_lev[lvl_idx] : pl.h_lev[lvl_idx];
  return launch_level<E>(pl, fac, pl.rank, pl.branch * pl.rank, lg.splits ? pl.branch : 1, lg.P, lg.G * lg.P, in, out,
                         k, adjoint, remap, st, peers);
}

template <typename E>
int timed_op(LaunchRecorder* rec, const Plan& pl, int which, int lvl_idx, int adjoint, const void* in, void* out,
             uint32_t k, int remap, cudaStream_t st, void* const* peers = nullptr, bool fold = false) {
  int rc = rec ? rec->before(st) : 0;
  if (!rc) rc = factor_op<E>(pl, which, lvl_idx, adjoint, in, out, k, remap, st, peers, fold);
  if (!rc && rec) rc = rec->after(st);
  return rc;
}

// First half of the chain (factors.py:230-233): lead leaf adjoint, then the
// down levels L-1 .. h in the adjoint direction. With remap the middle factor
// is fused into the last level; the result lands in final_dst or (when null)
// in whichever ping-pong buffer the alternation reaches (returned in *result).
template <typename E>
int run_down(const Plan& pl, const void* in, E* bufs[2], void* final_dst, uint32_t k, int adjoint, int remap,
             cudaStream_t st, LaunchRecorder* rec, const void** result, void* const* peers = nullptr) {
  const int nl = static_cast<int>(pl.nlev);
  const int lead = adjoint ? BF_FACTOR_U : BF_FACTOR_V;
  const int down = adjoint ? BF_FACTOR_G : BF_FACTOR_H;
  int cur = 0;
  int rc = 0;
  // rank-8 pairs: the lead leaf rides in the first pair (pair8_kernel<.., LEAF>), which then
  // reads the chain input itself
  bool leaf_fused = false;
  PairGeo lpg{};
  if constexpr (std::is_same<E, double2>::value) {
    PairGeo pg0{};
    const int lo0 = nl - 2;
    if (!rec && lo0 >= 0 && !(lo0 == 0 && (remap >= 3 || peers)) && pair_geometry(pl, lo0, k, 1, &pg0) &&
        !(lo0 == 0 && remap && (pg0.chunk || !remap_pair_enabled())) && pair8_leaf_geo(pl, pg0, k, 1, &lpg))
      leaf_fused = true;
  }
  // otherwise the folded outermost level (plan_fold_leaves) reads the chain input, unless
  // that level runs inside a pair kernel (uniform block shapes)
  bool fold = false;
  if (!leaf_fused && pl.h_fold && nl >= 1) {
    PairGeo pgf{};
    const int lo0 = nl - 2;
    bool paired = false;
    if constexpr (std::is_same<E, double2>::value)
      paired = !rec && lo0 >= 0 && !(lo0 == 0 && (remap >= 3 || peers)) &&
               (pair16_geometry(pl, lo0, k, 1, &pgf) ||
                (pair_geometry(pl, lo0, k, 1, &pgf) && !(lo0 == 0 && remap && (pgf.chunk || !remap_pair_enabled()))));
    fold = !paired;
  }
  if (!leaf_fused && !fold) {
    rc = timed_op<E>(rec, pl, lead, 0, 1, in, bufs[0], k, 0, st);
    if (rc) return rc;
  }
  for (int i = nl - 1; i >= 0; --i) {
    // levels i and i - 1 as one pair kernel (not in instrumented runs: per-level timing;
    // not for the remapped / pushed last level)
    PairGeo pg{};
    const int lo = i - 1;
    const bool may_pair = !(fold && i == nl - 1);   // the folded level has its own block shape
    if (may_pair && !rec && std::is_same<E, double2>::value && lo >= 0 && !(lo == 0 && (remap >= 3 || peers)) &&
        pair16_geometry(pl, lo, k, 1, &pg)) {
      void* dst = (lo == 0 && final_dst) ? final_dst : bufs[cur ^ 1];
      const void* fa = down == BF_FACTOR_G ? pl.g_lev[lo] : pl.h_lev[lo];
      const void* fb = down == BF_FACTOR_G ? pl.g_lev[i] : pl.h_lev[i];
      rc = launch_pair16(pl, fa, fb, lo, bufs[cur], dst, k, 1, pg, st, lo == 0 ? remap : 0);
      if (rc) return rc;
      if (dst == bufs[cur ^ 1]) cur ^= 1;
      --i;
      continue;
    }
    // (the last pair may carry the fused middle factor, remap 1/2, not the peer push;
    // the k-chunked pair kernel has no remap epilogue)
    if (may_pair && !rec && std::is_same<E, double2>::value && lo >= 0 && !(lo == 0 && (remap >= 3 || peers)) &&
        pair_geometry(pl, lo, k, 1, &pg) && !(lo == 0 && remap && (pg.chunk || !remap_pair_enabled()))) {
      void* dst = (lo == 0 && final_dst) ? final_dst : bufs[cur ^ 1];
      const void* fa = down == BF_FACTOR_G ? pl.g_lev[lo] : pl.h_lev[lo];
      const void* fb = down == BF_FACTOR_G ? pl.g_lev[i] : pl.h_lev[i];
      if (leaf_fused && i == nl - 1)
        rc = launch_pair(pl, fa, fb, lo, in, dst, k, 1, lpg, st, lo == 0 ? remap : 0,
                         lead == BF_FACTOR_U ? pl.u_leaf : pl.v_leaf);
      else
        rc = launch_pair(pl, fa, fb, lo, bufs[cur], dst, k, 1, pg, st, lo == 0 ? remap : 0);
      if (rc) return rc;
      if (dst == bufs[cur ^ 1]) cur ^= 1;
      --i;
      continue;
    }
    void* dst = (i == 0 && final_dst) ? final_dst : bufs[cur ^ 1];
    if (fold && i == nl - 1) {   // first op of the half: reads the chain input, lands in bufs[0] (or final_dst)
      if (dst == bufs[cur ^ 1]) dst = bufs[0];
      rc = timed_op<E>(rec, pl, down, i, 1, in, dst, k, i == 0 ? remap : 0, st, i == 0 ? peers : nullptr, true);
      if (rc) return rc;
      cur = 0;
      continue;
    }
    rc = timed_op<E>(rec, pl, down, i, 1, bufs[cur], dst, k, i == 0 ? remap : 0, st, i == 0 ? peers : nullptr);
    if (rc) return rc;
    if (dst == bufs[cur ^ 1]) cur ^= 1;
  }
  *result = final_dst ? final_dst : bufs[cur];
  return 0;
}

// Second half (factors.py:234-236): up levels h .. L-1 forward, then the trail leaf.
template <typename E>
int run_up(const Plan& pl, const void* mid, E* bufs[2], void* out, uint32_t k, int adjoint, cudaStream_t st,
           LaunchRecorder* rec) {
  const int nl = static_cast<int>(pl.nlev);
  const int up = adjoint ? BF_FACTOR_H : BF_FACTOR_G;
  const int trail = adjoint ? BF_FACTOR_V : BF_FACTOR_U;
  const void* src = mid;
  int nxt = (mid == bufs[0]) ? 1 : 0;
  for (int i = 0; i < nl; ++i) {
    PairGeo pg{};
    if (!rec && std::is_same<E, double2>::value && pair16_geometry(pl, i, k, 0, &pg)) {
      const void* fa = up == BF_FACTOR_G ? pl.g_lev[i] : pl.h_lev[i];
      const void* fb = up == BF_FACTOR_G ? pl.g_lev[i + 1] : pl.h_lev[i + 1];
      int rc = launch_pair16(pl, fa, fb, i, src, bufs[nxt], k, 0, pg, st, 0);
      if (rc) return rc;
      src = bufs[nxt];
      nxt ^= 1;
      ++i;
      continue;
    }
    if (!rec && std::is_same<E, double2>::value && pair_geometry(pl, i, k, 0, &pg)) {
      const void* fa = up == BF_FACTOR_G ? pl.g_lev[i] : pl.h_lev[i];
      const void* fb = up == BF_FACTOR_G ? pl.g_lev[i + 1] : pl.h_lev[i + 1];
      PairGeo lpg{};
      if (i + 2 == nl && pair8_leaf_geo(pl, pg, k, 0, &lpg))   // the trail leaf rides in the last pair
        return launch_pair(pl, fa, fb, i, src, out, k, 0, lpg, st, 0, trail == BF_FACTOR_U ? pl.u_leaf : pl.v_leaf);
      int rc = launch_pair(pl, fa, fb, i, src, bufs[nxt], k, 0, pg, st);
      if (rc) return rc;
      src = bufs[nxt];
      nxt ^= 1;
      ++i;
      continue;
    }
    if (i == nl - 1 && pl.g_fold)   // the folded outermost level writes the chain output
      return timed_op<E>(rec, pl, up, i, 0, src, out, k, 0, st, nullptr, true);
    int rc = timed_op<E>(rec, pl, up, i, 0, src, bufs[nxt], k, 0, st);
    if (rc) return rc;
    src = bufs[nxt];
    nxt ^= 1;
  }
  return timed_op<E>(rec, pl, trail, 0, 0, src, out, k, 0, st);
}

// Node kernels (node_kernel.cuh): the whole down half and the whole up half as one
// launch each, one CTA per (middle node, chunk of right-hand sides), for chains whose
// factors sit in L2 (latency bound: BASELINE configs 0 and 1). BF_NO_NODE=1 turns them
// off; BF_NODE=1 uses them whenever the node vector fits shared memory.
struct NodeCfg {
  bool mma, pf;
  uint32_t kc, nch, vld, threads;
  int nt;
  size_t smem;
  uint32_t ksplit = 1;
  bool xstage = false;
  NodeStage stage{};
};

// Padded row stride (complex values, >= len) for staged factor rows so that one phase of
// a DMMA A fragment (lanes 0-7: k = lane & 3, m = lane >> 2) touches 8 distinct 16-byte
// bank groups: `rows_k` = the fragment's k index walks rows (adjoint steps), else columns.
uint32_t conflict_free_ld(uint32_t len, bool rows_k) {
  uint32_t best = len, best_conf = 99;
  for (uint32_t ld = len; ld < len + 8; ++ld) {
    uint32_t used[8], conf = 0;
    for (int l = 0; l < 8; ++l) {
      const uint32_t k = l & 3, m = l >> 2;
      const uint32_t e = rows_k ? k * ld + m : m * ld + k;
      used[l] = (e * 4) % 32;
      for (int j = 0; j < l; ++j)
        if (used[j] == used[l]) ++conf;
    }
    if (conf < best_conf) {
      best_conf = conf;
      best = ld;
    }
    if (!conf) break;
  }
  return best;
}

constexpr int kNodeMaxGroups = 4;   // staged groups per in-place step (registers: one item per warp each)

constexpr int kNodeMaxIt = 4;       // deferred DMMA items per warp (16 warps)
constexpr int kNodeMaxOut = 2;      // deferred FMA outputs per thread group (compact code: i-cache)
constexpr uint64_t kNodeMaxFactorBytes = 512ull << 20;

// Shared memory of a node CTA: mbarriers, the node vector, and (pf) every step's slab.
size_t node_smem(const Plan& pl, uint32_t vld, bool pf) {
  const uint64_t NL = 1ull << pl.nlev, R = pl.rank;
  const uint64_t vbytes = (NL * R * vld * sizeof(double2) + 127) & ~127ull;
  const uint64_t slabs = (NL * pl.leaf_n0 * R + pl.nlev * NL * 2 * R * R) * sizeof(double2);
  return 256 + vbytes + (pf ? slabs : 0);
}

bool node_config(const Plan& pl, uint32_t k, NodeCfg* nc) {
  static const int mode = env_int("BF_NO_NODE", 0) ? -1 : env_int("BF_NODE", 0);
  if (mode < 0 || pl.dtype != BF_C128 || pl.branch != 2 || pl.nparts != 1 || !pl.leaf_n0) return false;
  if (pl.nlev != pl.half || pl.nlev == 0 || pl.nlev > static_cast<uint32_t>(kNodeMaxLev)) return false;
  for (const LevelGeo& lg : pl.lev)
    if (!lg.splits) return false;
  if (mode == 0 && pl.base_bytes > kNodeMaxFactorBytes) return false;
  const uint64_t NL = 1ull << pl.nlev, rows = NL * pl.rank, R = pl.rank;
  if (NL != pl.m) return false;
  const size_t cap = static_cast<size_t>(kMaxDynSmem);
  if (k >= 8) {
    // staged many-RHS kernel (node_mma.cuh): vector + two staging halves of factor groups.
    // Opt-in (BF_NODE_MMA=1): at cfg1 (64 RHS) it measures 398 us per apply against 264 us for
    // the level / pair kernels — each CTA's groups are too small to cover the staging latency
    // with two halves next to a 147 KB node vector.
    static const bool mma_on = env_int("BF_NODE_MMA", 0) != 0;
    if (!mma_on) return false;
    const uint32_t n0 = pl.leaf_n0;
    NodeStage sg{};
    sg.lda_dn = conflict_free_ld(2 * R, true);
    sg.lda_up = conflict_free_ld(2 * R, false);
    sg.lda_ldn = conflict_free_ld(R, true);
    sg.lda_lup = conflict_free_ld(R, false);
    uint64_t gu = 1;
    while ((NL / 2) / gu > static_cast<uint64_t>(kNodeMaxGroups)) gu <<= 1;
    for (uint32_t kc : {16u, 8u}) {
      const int nt = kc / 8;
      // one DMMA item per warp and group in the in-place steps (16 warps)
      if (gu * ((2 * R + 7) / 8) > 16 || 2 * gu * ((R + 7) / 8) > 16) return false;
      const uint32_t vld = kc + 2;
      const uint64_t vbytes = (rows * vld * sizeof(double2) + 127) & ~127ull;
      const uint64_t lev_elems = 2 * gu * R * std::max(sg.lda_dn, sg.lda_up);
      const uint64_t avail = cap - 256 - vbytes;
      if (avail < 2 * lev_elems * sizeof(double2)) continue;
      const uint64_t half = std::min<uint64_t>(avail / 2 / sizeof(double2), 1ull << 20) & ~7ull;
      if (half < lev_elems) continue;
      uint64_t gl_dn = NL, gl_up = NL;
      while (gl_dn > 1 && gl_dn * n0 * sg.lda_ldn > half) gl_dn >>= 1;
      while (gl_up > 1 && gl_up * n0 * sg.lda_lup > half) gl_up >>= 1;
      if (gl_dn * n0 * sg.lda_ldn > half || gl_up * n0 * sg.lda_lup > half) continue;
      sg.half_elems = static_cast<uint32_t>(half);
      sg.gu = static_cast<uint32_t>(gu);
      sg.gl_dn = static_cast<uint32_t>(gl_dn);
      sg.gl_up = static_cast<uint32_t>(gl_up);
      NodeCfg c{true, false, kc, (k + kc - 1) / kc, vld, 512, nt, 256 + vbytes + 2 * half * sizeof(double2)};
      c.stage = sg;
      *nc = c;
      return true;
    }
    return false;
  }
  const uint64_t outs = rows * k;
  // split each dot product over ks threads while the CTA stays <= 512 threads
  uint32_t ks = 8;
  while (ks > 1 && outs * ks > 512) ks >>= 1;
  const uint64_t groups = std::min<uint64_t>(512 / ks, outs);
  if ((outs + groups - 1) / groups > static_cast<uint64_t>(kNodeMaxOut)) return false;
  const uint32_t threads = static_cast<uint32_t>(std::max<uint64_t>(64, ((groups * ks + 31) / 32) * 32));
  for (bool pf : {true, false}) {
    size_t smem = node_smem(pl, k, pf);
    if (smem > cap || (!pf && smem > 200 * 1024)) continue;
    NodeCfg c{false, pf, k, 1, k, threads, 1, smem};
    c.ksplit = ks;
    const size_t xbytes = static_cast<size_t>(pl.side) * k * sizeof(double2);
    if (pf && smem + xbytes <= cap) {
      c.xstage = true;
      c.smem = smem + xbytes;
    }
    *nc = c;
    return true;
  }
  return false;
}

template <int UP>
void* node_kernel_for(const NodeCfg& nc) {
  if (nc.mma) return nc.nt == 2 ? (void*)node_mma_kernel<UP, 2, kNodeMaxGroups> : (void*)node_mma_kernel<UP, 1, kNodeMaxGroups>;
  return nc.pf ? (void*)node_kernel<UP, false, 1, kNodeMaxOut, true> : (void*)node_kernel<UP, false, 1, kNodeMaxOut, false>;
}


int launch_node(const Plan& pl, int up, int adjoint, const void* in, void* out, uint32_t k, const NodeCfg& nc,
                cudaStream_t st) {
  NodeArgs a{};
  const bool fwd_leaf_v = (up == 0) != (adjoint != 0);   // down of the forward chain / up of the adjoint: V
  a.leaf = static_cast<const double2*>(fwd_leaf_v ? pl.v_leaf : pl.u_leaf);
  const bool h_side = fwd_leaf_v;
  for (uint32_t i = 0; i < pl.nlev; ++i)
    a.lev[i] = static_cast<const double2*>(h_side ? pl.h_lev[i] : pl.g_lev[i]);
  a.in = static_cast<const double2*>(in);
  a.out = static_cast<double2*>(out);
  a.mid_w = static_cast<const double*>(pl.weights);
  a.n0 = pl.leaf_n0;
  a.r = pl.rank;
  a.D = pl.nlev;
  a.k = k;
  a.kc = nc.kc;
  a.nch = nc.nch;
  a.vld = nc.vld;
  a.ksplit = nc.ksplit;
  a.xstage = up ? 0 : nc.xstage;
  a.remap = adjoint ? 2 : 1;
  a.trace = g_node_trace ? g_node_trace + (up ? static_cast<size_t>(pl.m) * nc.nch * 32 : 0) : nullptr;
  void* kp = up ? node_kernel_for<1>(nc) : node_kernel_for<0>(nc);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.m * nc.nch);
  cfg.blockDim = dim3(nc.threads);
  cfg.dynamicSmemBytes = nc.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (nc.mma) {
    auto* kern = reinterpret_cast<void (*)(const NodeArgs, const NodeStage)>(kp);
    BF_CUDA(allow_max_dyn_smem(kern));
    BF_CUDA(cudaLaunchKernelEx(&cfg, kern, a, nc.stage));
  } else {
    auto* kern = reinterpret_cast<void (*)(const NodeArgs)>(kp);
    BF_CUDA(allow_max_dyn_smem(kern));
    BF_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  }
  return 0;
}

template <typename E>
int chain(const Plan& pl, const void* in, void* out, uint32_t k, int adjoint, void* ws, cudaStream_t st,
          LaunchRecorder* rec) {
  const uint64_t dk = pl.dim_max * k;
  E* bufs[2] = {static_cast<E*>(ws), static_cast<E*>(ws) + dk};
  if constexpr (std::is_same<E, double2>::value) {
    NodeCfg nc{};
    if (node_config(pl, k, &nc)) {
      int rc = rec ? rec->before(st) : 0;
      if (!rc) rc = launch_node(pl, 0, adjoint, in, bufs[0], k, nc, st);
      if (!rc && rec) rc = rec->after(st);
      if (!rc && rec) rc = rec->before(st);
      if (!rc) rc = launch_node(pl, 1, adjoint, bufs[0], out, k, nc, st);
      if (!rc && rec) rc = rec->after(st);
      return rc;
    }
  }
  const void* mid = nullptr;
  int rc = run_down<E>(pl, in, bufs, nullptr, k, adjoint, adjoint ? 2 : 1, st, rec, &mid);
  if (rc) return rc;
  return run_up<E>(pl, mid, bufs, out, k, adjoint, st, rec);
}

// Sharded middle exchange: this part's down-half output
// mid[(a*m + b)*r + rho][kk] (a: own local node, b: global other node) is packed
// per destination part e as send[e][a][b - e*mp][rho][kk], scaled by the middle
// weight (factors.py:180-190); the receiver scatters recv[d][a'][b'][rho][kk]
// to out[(b'*m + d*mp + a')*r + rho][kk].
template <typename E>
__global__ void pack_kernel(const E* __restrict__ mid, E* __restrict__ send, const typename Cx<E>::R* __restrict__ W,
                            uint32_t m, uint32_t mp, uint32_t r, uint32_t k, uint32_t part, uint32_t nparts,
                            int adjoint) {
  const uint64_t per = static_cast<uint64_t>(mp) * mp * r * k;
  const uint64_t total = per * nparts;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = static_cast<uint32_t>(x / per);
    uint64_t rem = x - e * per;
    const uint32_t kk = static_cast<uint32_t>(rem % k);
    rem /= k;
    const uint32_t rho = static_cast<uint32_t>(rem % r);
    rem /= r;
    const uint32_t bl = static_cast<uint32_t>(rem % mp), a = static_cast<uint32_t>(rem / mp);
    const uint32_t own = part * mp + a, other = e * mp + bl;
    // forward: own = column node j, other = row node i, weight W[i, j]; adjoint: own = i, other = j
    const uint64_t wi = adjoint ? (static_cast<uint64_t>(own) * m + other) : (static_cast<uint64_t>(other) * m + own);
    const auto w = W[wi * r + rho];
    const E v = mid[((static_cast<uint64_t>(a) * m + other) * r + rho) * k + kk];
    send[x] = Cx<E>::make(w * v.x, w * v.y);
  }
}

template <typename E>
__global__ void unpack_kernel(const E* __restrict__ recv, E* __restrict__ out, uint32_t m, uint32_t mp, uint32_t r,
                              uint32_t k, uint32_t nparts) {
  const uint64_t per = static_cast<uint64_t>(mp) * mp * r * k;
  const uint64_t total = per * nparts;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t d = static_cast<uint32_t>(x / per);
    uint64_t rem = x - d * per;
    const uint32_t kk = static_cast<uint32_t>(rem % k);
    rem /= k;
    const uint32_t rho = static_cast<uint32_t>(rem % r);
    rem /= r;
    const uint32_t b = static_cast<uint32_t>(rem % mp), a = static_cast<uint32_t>(rem / mp);
    out[((static_cast<uint64_t>(b) * m + d * mp + a) * r + rho) * k + kk] = recv[x];
  }
}

}  // namespace

extern "C" int bf_debug_node_trace(unsigned long long* dev_buf) {
  g_node_trace = dev_buf;
  return 0;
}

int plan_apply(const Plan& pl, const void* in, void* out, uint32_t k, int adjoint, void* ws, cudaStream_t st,
               LaunchRecorder* rec) {
  return pl.dtype == BF_C128 ? chain<double2>(pl, in, out, k, adjoint, ws, st, rec)
                             : chain<float2>(pl, in, out, k, adjoint, ws, st, rec);
}

int plan_apply_half(const Plan& pl, int up, const void* in, void* out, uint32_t k, int adjoint, void* ws,
                    cudaStream_t st) {
  const uint64_t dk = pl.dim_max * k;
  const void* res = nullptr;
  if (pl.dtype == BF_C128) {
    double2* bufs[2] = {static_cast<double2*>(ws), static_cast<double2*>(ws) + dk};
    return up ? run_up<double2>(pl, in, bufs, out, k, adjoint, st, nullptr)
              : run_down<double2>(pl, in, bufs, out, k, adjoint, 0, st, nullptr, &res);
  }
  float2* bufs[2] = {static_cast<float2*>(ws), static_cast<float2*>(ws) + dk};
  return up ? run_up<float2>(pl, in, bufs, out, k, adjoint, st, nullptr)
            : run_down<float2>(pl, in, bufs, out, k, adjoint, 0, st, nullptr, &res);
}

// Sharded down half whose last level stores its outputs, middle weights
// applied, straight into every part's receive buffer (remap 3/4).
int plan_apply_down_push(const Plan& pl, const void* in, void* const* peers, uint32_t k, int adjoint, void* ws,
                         cudaStream_t st) {
  const uint64_t dk = pl.dim_max * k;
  const void* res = nullptr;
  const int remap = adjoint ? 4 : 3;
  if (pl.dtype == BF_C128) {
    double2* bufs[2] = {static_cast<double2*>(ws), static_cast<double2*>(ws) + dk};
    return run_down<double2>(pl, in, bufs, nullptr, k, adjoint, remap, st, nullptr, &res, peers);
  }
  float2* bufs[2] = {static_cast<float2*>(ws), static_cast<float2*>(ws) + dk};
  return run_down<float2>(pl, in, bufs, nullptr, k, adjoint, remap, st, nullptr, &res, peers);
}

int plan_middle_exchange(const Plan& pl, int unpack, const void* in, void* out, uint32_t k, int adjoint,
                         cudaStream_t st) {
  const uint32_t mp = pl.m / pl.nparts;
  const uint64_t total = static_cast<uint64_t>(mp) * mp * pl.rank * k * pl.nparts;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, pl.sms * 8ull));
  if (pl.dtype == BF_C128) {
    if (unpack)
      unpack_kernel<double2><<<grid, 256, 0, st>>>(static_cast<const double2*>(in), static_cast<double2*>(out), pl.m,
                                                   mp, pl.rank, k, pl.nparts);
    else
      pack_kernel<double2><<<grid, 256, 0, st>>>(static_cast<const double2*>(in), static_cast<double2*>(out),
                                                 static_cast<const double*>(pl.weights), pl.m, mp, pl.rank, k,
                                                 pl.part, pl.nparts, adjoint);
  } else {
    if (unpack)
      unpack_kernel<float2><<<grid, 256, 0, st>>>(static_cast<const float2*>(in), static_cast<float2*>(out), pl.m,
                                                  mp, pl.rank, k, pl.nparts);
    else
      pack_kernel<float2><<<grid, 256, 0, st>>>(static_cast<const float2*>(in), static_cast<float2*>(out),
                                                static_cast<const float*>(pl.weights), pl.m, mp, pl.rank, k, pl.part,
                                                pl.nparts, adjoint);
  }
  BF_CUDA(cudaGetLastError());
  return 0;
}

int plan_apply_factor(const Plan& pl, int which, int lvl_idx, int adjoint, const void* in, void* out, uint32_t k,
                      cudaStream_t st) {
  return pl.dtype == BF_C128 ? factor_op<double2>(pl, which, lvl_idx, adjoint, in, out, k, 0, st)
                             : factor_op<float2>(pl, which, lvl_idx, adjoint, in, out, k, 0, st);
}

}  // namespace bfly

namespace bfly {

// A part view of a full plan: the slice of every factor that middle nodes
// [part m/P, (part+1) m/P) own, as pointer offsets into the
// full plan's storage — no copies. Used to pipeline host transfers with compute.
Plan part_view(const Plan& full, uint32_t part, uint32_t nparts) {
  Plan v = full;
  v.part = part;
  v.nparts = nparts;
  v.base = nullptr;
  v.base_bytes = 0;
  const uint64_t es = full.elem();
  v.leaf_nb = full.leaf_nb / nparts;
  v.dim_max = full.dim_max / nparts;
  const uint64_t leaf_bytes = v.leaf_nb * full.leaf_n0 * full.rank * es;
  v.u_leaf = static_cast<char*>(full.u_leaf) + part * leaf_bytes;
  v.v_leaf = static_cast<char*>(full.v_leaf) + part * leaf_bytes;
  for (uint32_t i = 0; i < full.nlev; ++i) {
    v.lev[i].G = full.lev[i].G / nparts;
    v.lev[i].nblocks = full.lev[i].nblocks / nparts;
    const uint64_t lb = v.lev[i].nblocks * full.rank * full.branch * full.rank * es;
    v.g_lev[i] = static_cast<char*>(full.g_lev[i]) + part * lb;
    v.h_lev[i] = static_cast<char*>(full.h_lev[i]) + part * lb;
  }
  v.fold_base = nullptr;
  if (full.g_fold) {
    const uint64_t fb = v.lev[full.nlev - 1].nblocks * full.leaf_n0 * full.branch * full.rank * es;
    v.g_fold = static_cast<char*>(full.g_fold) + part * fb;
    v.h_fold = static_cast<char*>(full.h_fold) + part * fb;
  }
  return v;
}

// ---------------------------------------------------------------- leaf folding
// fold[q] (n0 x C) = leaf[q] (n0 x r) * level[q] (r x C) for every block q of the
// outermost transfer level (its P is 1, so block q = (g, t) feeds / is fed by leaf q:
// factors.py:49-56 after 120-139). One CTA per block, double accumulation.
template <typename E>
__global__ void k_fold_leaf(const E* __restrict__ leaf, const E* __restrict__ lev, E* __restrict__ out, uint32_t n0,
                            uint32_t r, uint32_t C) {
  const size_t q = blockIdx.x;
  const E* L = leaf + q * n0 * r;
  const E* F = lev + q * r * C;
  E* O = out + q * n0 * C;
  for (uint32_t e = threadIdx.x; e < n0 * C; e += blockDim.x) {
    const uint32_t i = e / C, c = e - i * C;
    double re = 0, im = 0;
    for (uint32_t rho = 0; rho < r; ++rho) {
      const double ax = L[i * r + rho].x, ay = L[i * r + rho].y, bx = F[rho * C + c].x, by = F[rho * C + c].y;
      re += ax * bx - ay * by;
      im += ax * by + ay * bx;
    }
    O[e].x = static_cast<decltype(O[e].x)>(re);
    O[e].y = static_cast<decltype(O[e].y)>(im);
  }
}

// ---------------------------------------------------------------- radix-4 folding
// Two adjacent splitting levels A (index 2j, nearer the middle) and B (2j + 1) multiplied
// into one level of branching 4: F4[g][2t + t'][q] (r x 4r) = [ B(t,t')[:, 0:r] A(t,0) |
// B(t,t')[:, r:2r] A(t,1) ] with A(t,u) = A[(2g + t) P_A + 2q + u], B(t,t') =
// B[((2g + t) 2 + t') P_B + q] (factors.py:120-139 applied twice). Unit (g, q) of the folded
// level reads the 4r rows that A's units (g, 2q), (g, 2q + 1) read and writes the four
// r-row blocks that B's units (2g, q), (2g + 1, q) write, so the result is an ordinary
// level of a branching-4 plan (the quadtree plans' kernels) with exactly as many nonzeros
// as the two levels it replaces: 16 r^2 per item either way.
template <typename E>
__global__ void k_fold_pair(const E* __restrict__ fa, const E* __restrict__ fb, E* __restrict__ out, uint32_t r,
                            uint32_t pa) {
  const uint32_t pb = pa / 2, C = 2 * r;
  const uint32_t item = blockIdx.x >> 2, t4 = blockIdx.x & 3, t = t4 >> 1, tp = t4 & 1;
  const uint32_t g = item / pb, q = item - g * pb;
  const E* B = fb + static_cast<size_t>(((2 * g + t) * 2 + tp) * pb + q) * r * C;
  E* O = out + static_cast<size_t>((g * 4 + t4) * pb + q) * r * 2 * C;
  for (uint32_t e = threadIdx.x; e < r * 2 * C; e += blockDim.x) {
    const uint32_t row = e / (2 * C), col = e - row * 2 * C, u = col / C, c = col - u * C;
    const E* A = fa + static_cast<size_t>((g * 2 + t) * pa + 2 * q + u) * r * C;
    double re = 0, im = 0;
    for (uint32_t rho = 0; rho < r; ++rho) {
      const double bx = B[row * C + u * r + rho].x, by = B[row * C + u * r + rho].y;
      const double ax = A[rho * C + c].x, ay = A[rho * C + c].y;
      re += bx * ax - by * ay;
      im += bx * ay + by * ax;
    }
    O[e].x = static_cast<decltype(O[e].x)>(re);
    O[e].y = static_cast<decltype(O[e].y)>(im);
  }
}

// The branching-4 twin of a binary plan for many right-hand sides (an even
// number of splitting levels per side, 64 <= 4r <= 104 so its levels run as the K-pipelined
// wide GEMM): half the launches, the chain's intermediate vectors read and written once
// per TWO reference levels, 16 k-steps per unit instead of 8. Same operator; the folded
// blocks are rounded once more. Leaves and middle weights are shared with `p`; returns
// nullptr when the plan does not qualify or there is no memory for the copy (cfg2: 9.1 GB).
Plan* plan_build_radix4(const Plan& p, cudaStream_t st) {
  static const bool off = env_int("BF_NO_RADIX4", 0) != 0;
  if (off || !p.uploaded || p.branch != 2 || p.nlev < 2 || (p.nlev & 1)) return nullptr;
  // complex128: ranks whose branching-4 levels run as the wide GEMM; complex64 (FFMA levels, 16 warps
  // for wide blocks): the same ranks (cfg2 size, 256 RHS 26.8 -> 25.4 ms, 64 RHS 8.46 -> 7.11 ms)
  if (!wide_applies(p.rank, 4 * p.rank, 4, kMrhsMinK, 0, 16) && env_int("BF_RADIX4_ANY", 0) == 0) return nullptr;
  if (p.dtype == BF_C64 && env_int("BF_NO_RADIX4_C64", 0) != 0) return nullptr;
  for (uint32_t j = 0; j < p.nlev; j += 2) {
    const LevelGeo& A = p.lev[j];
    const LevelGeo& B = p.lev[j + 1];
    if (!A.splits || !B.splits || A.P < 2 || B.G != 2 * A.G || 2 * B.P != A.P) return nullptr;
    if (A.G * A.P / 2 * 4 >= (1ull << 31)) return nullptr;
  }
  Plan* q = new (std::nothrow) Plan(p);
  if (!q) return nullptr;
  q->branch = 4;
  q->base = nullptr;
  q->base_bytes = 0;
  q->fold_base = q->g_fold = q->h_fold = nullptr;
  q->nlev = p.nlev / 2;
  q->lev.clear();
  uint64_t bytes = 0;
  const uint64_t blk = static_cast<uint64_t>(p.rank) * 4 * p.rank * p.elem();
  for (uint32_t j = 0; j < q->nlev; ++j) {
    const LevelGeo& A = p.lev[2 * j];
    LevelGeo g4{A.level, true, A.G, A.P / 2, A.G * 4 * (A.P / 2)};
    q->lev.push_back(g4);
    bytes += 2 * ((g4.nblocks * blk + 255) / 256 * 256);
  }
  // the twin doubles the plan's footprint: only when that leaves at least 15% of the device free
  size_t mem_free = 0, mem_total = 0;
  if (cudaMemGetInfo(&mem_free, &mem_total) != cudaSuccess || mem_free < bytes + mem_total * 15 / 100 ||
      cudaMalloc(&q->base, bytes) != cudaSuccess) {
    cudaGetLastError();
    delete q;
    return nullptr;
  }
  q->base_bytes = bytes;
  q->g_lev.assign(q->nlev, nullptr);
  q->h_lev.assign(q->nlev, nullptr);
  char* cur = static_cast<char*>(q->base);
  for (int side = 0; side < 2; ++side)
    for (uint32_t j = 0; j < q->nlev; ++j) {
      (side ? q->h_lev : q->g_lev)[j] = cur;
      cur += (q->lev[j].nblocks * blk + 255) / 256 * 256;
      const auto& src = side ? p.h_lev : p.g_lev;
      void* dst = (side ? q->h_lev : q->g_lev)[j];
      const unsigned nb4 = static_cast<unsigned>(q->lev[j].nblocks);
      const uint32_t pa = static_cast<uint32_t>(p.lev[2 * j].P);
      if (p.dtype == BF_C128)
        k_fold_pair<double2><<<nb4, 128, 0, st>>>(static_cast<const double2*>(src[2 * j]),
                                                   static_cast<const double2*>(src[2 * j + 1]),
                                                   static_cast<double2*>(dst), p.rank, pa);
      else
        k_fold_pair<float2><<<nb4, 128, 0, st>>>(static_cast<const float2*>(src[2 * j]),
                                                  static_cast<const float2*>(src[2 * j + 1]),
                                                  static_cast<float2*>(dst), p.rank, pa);
    }
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess || plan_fold_leaves(*q, st) != 0) {
    cudaGetLastError();
    plan_free_radix4(q);
    return nullptr;
  }
  return q;
}

void plan_free_radix4(Plan* q) {
  if (!q) return;
  if (q->fold_base) cudaFree(q->fold_base);
  if (q->base) cudaFree(q->base);
  delete q;
}

// Folds the leaf factors into the outermost transfer level (BF_NO_FOLD=1 keeps the
// reference's factor list): the chain then runs 2 (L - h) launches instead of 2 + 2 (L - h),
// never materialises the rank-space vector next to the leaves, and — for leaves with fewer
// than 2 r points — does less arithmetic (n0 C instead of n0 r + r C per block).
// The operator is the same; entries of the folded blocks are rounded once more (apply
// parity against the oracle's unfolded chain stays at 1e-15, tests/test_apply_gpu.py).
int plan_fold_leaves(Plan& pl, cudaStream_t st) {
  static const bool off = env_int("BF_NO_FOLD", 0) != 0;
  if (off || !pl.uploaded || pl.nlev == 0 || pl.g_fold) return 0;
  const LevelGeo& last = pl.lev[pl.nlev - 1];
  if (last.P != 1 || last.nblocks != pl.leaf_nb) return 0;
  const uint32_t nt = last.splits ? pl.branch : 1;
  const uint32_t C = pl.branch * pl.rank, n0 = pl.leaf_n0, r = pl.rank;
  (void)nt;
  const uint64_t bytes = (last.nblocks * n0 * C * pl.elem() + 255) / 256 * 256;
  if (cudaMalloc(&pl.fold_base, 2 * bytes) != cudaSuccess) {   // no room: keep the unfolded chain
    cudaGetLastError();
    pl.fold_base = nullptr;
    return 0;
  }
  pl.g_fold = pl.fold_base;
  pl.h_fold = static_cast<char*>(pl.fold_base) + bytes;
  const unsigned blocks = static_cast<unsigned>(last.nblocks);
  if (pl.dtype == BF_C128) {
    k_fold_leaf<double2><<<blocks, 128, 0, st>>>(static_cast<const double2*>(pl.u_leaf),
                                                  static_cast<const double2*>(pl.g_lev[pl.nlev - 1]),
                                                  static_cast<double2*>(pl.g_fold), n0, r, C);
    k_fold_leaf<double2><<<blocks, 128, 0, st>>>(static_cast<const double2*>(pl.v_leaf),
                                                  static_cast<const double2*>(pl.h_lev[pl.nlev - 1]),
                                                  static_cast<double2*>(pl.h_fold), n0, r, C);
  } else {
    k_fold_leaf<float2><<<blocks, 128, 0, st>>>(static_cast<const float2*>(pl.u_leaf),
                                                 static_cast<const float2*>(pl.g_lev[pl.nlev - 1]),
                                                 static_cast<float2*>(pl.g_fold), n0, r, C);
    k_fold_leaf<float2><<<blocks, 128, 0, st>>>(static_cast<const float2*>(pl.v_leaf),
                                                 static_cast<const float2*>(pl.h_lev[pl.nlev - 1]),
                                                 static_cast<float2*>(pl.h_fold), n0, r, C);
  }
  BF_CUDA(cudaGetLastError());
  BF_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// Host-buffer apply with the transfers pipelined against compute (captured into
// a graph by the caller): chunk c's H2D copy (stream cp) overlaps the down half
// of chunk c-1 (stream run); the middle factor runs once on the full middle
// vector; chunk e's D2H overlaps the up half of chunk e+1.
int plan_apply_host_pipelined(const Plan& pl, const void* in_host, void* out_host, void* din, void* dout, void* mid,
                              void* mid2, void* ws, uint32_t k, int adjoint, uint32_t chunks, cudaStream_t run,
                              cudaStream_t cp, cudaEvent_t* ev, uint32_t taper, cudaStream_t aux) {
  const uint64_t es = pl.elem();
  const uint64_t mid_rows = static_cast<uint64_t>(pl.m) * pl.m * pl.rank;
  // chunk c = part (first, second) of the middle nodes. Uniform: `chunks` equal parts.
  // Tapered (taper = T): 1/T, 1/T, 2/T, ... 1/2 on the way down and the mirror image on
  // the way up, so the first upload and the last download are short and most of the
  // chain runs in large parts.
  std::vector<std::pair<uint32_t, uint32_t>> down, up;
  if (taper >= 4) {
    down.push_back({0, taper});
    for (uint32_t T = taper; T >= 2; T /= 2) down.push_back({1, T});
    for (uint32_t T = 2; T <= taper; T *= 2) up.push_back({T - 2, T});
    up.push_back({taper - 1, taper});
  } else {
    for (uint32_t c = 0; c < chunks; ++c) {
      down.push_back({c, chunks});
      up.push_back({c, chunks});
    }
  }
  const uint32_t nc = static_cast<uint32_t>(down.size());
  // ev[0]: fork; ev[1 .. nc]: inputs landed; ev[nc+1 .. 2 nc]: outputs ready; ev[2 nc+1]: join;
  // ev[2 nc+2 ..]: down halves finished on the second compute stream
  // With a second compute stream (aux) the down halves of odd parts run there, each on its own
  // slice of the workspace: a part's small launches fill the tails of its neighbour's (the up
  // halves stay in order on `run`: the large part must finish first so that its download
  // overlaps the rest).
  BF_CUDA(cudaEventRecord(ev[0], run));
  BF_CUDA(cudaStreamWaitEvent(cp, ev[0], 0));
  for (uint32_t c = 0; c < nc; ++c) {
    const uint64_t rows_c = pl.n / down[c].second;
    const uint64_t off = down[c].first * rows_c * k * es;
    BF_CUDA(cudaMemcpyAsync(static_cast<char*>(din) + off, static_cast<const char*>(in_host) + off, rows_c * k * es,
                            cudaMemcpyHostToDevice, cp));
    BF_CUDA(cudaEventRecord(ev[1 + c], cp));
  }
  uint64_t ws_off = 0;
  for (uint32_t c = 0; c < nc; ++c) {
    cudaStream_t sc = (aux && (c & 1)) ? aux : run;
    BF_CUDA(cudaStreamWaitEvent(sc, ev[1 + c], 0));
    const Plan v = part_view(pl, down[c].first, down[c].second);
    const uint64_t rows_c = pl.n / down[c].second, mid_c = mid_rows / down[c].second;
    // (with aux every part has its own workspace slice: 2 dim_max k / nparts elements)
    void* wsc = aux ? static_cast<char*>(ws) + ws_off : ws;
    if (aux) ws_off += 2 * (pl.dim_max / down[c].second) * k * es;
    int rc = plan_apply_half(v, 0, static_cast<char*>(din) + down[c].first * rows_c * k * es,
                             static_cast<char*>(mid) + down[c].first * mid_c * k * es, k, adjoint, wsc, sc);
    if (rc) return rc;
    if (sc == aux) {
      BF_CUDA(cudaEventRecord(ev[2 + 2 * nc + c], aux));
      BF_CUDA(cudaStreamWaitEvent(run, ev[2 + 2 * nc + c], 0));
    }
  }
  int rc = pl.dtype == BF_C128 ? launch_middle<double2>(pl, mid, mid2, k, adjoint, run)
                               : launch_middle<float2>(pl, mid, mid2, k, adjoint, run);
  if (rc) return rc;
  for (uint32_t e = 0; e < nc; ++e) {
    const Plan v = part_view(pl, up[e].first, up[e].second);
    const uint64_t rows_c = pl.n / up[e].second, mid_c = mid_rows / up[e].second;
    const uint64_t off = up[e].first * rows_c * k * es;
    rc = plan_apply_half(v, 1, static_cast<char*>(mid2) + up[e].first * mid_c * k * es, static_cast<char*>(dout) + off,
                         k, adjoint, ws, run);
    if (rc) return rc;
    BF_CUDA(cudaEventRecord(ev[1 + nc + e], run));
    BF_CUDA(cudaStreamWaitEvent(cp, ev[1 + nc + e], 0));
    BF_CUDA(cudaMemcpyAsync(static_cast<char*>(out_host) + off, static_cast<char*>(dout) + off, rows_c * k * es,
                            cudaMemcpyDeviceToHost, cp));
  }
  BF_CUDA(cudaEventRecord(ev[1 + 2 * nc], cp));
  BF_CUDA(cudaStreamWaitEvent(run, ev[1 + 2 * nc], 0));
  return 0;
}

}  // namespace bfly
