// plan.h — device-resident factor chain (the C++ side of bf_plan).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <vector>

#include "../../include/bfly.h"

namespace bfly {

// One transfer level ascending from half (construct.py:_level_geometry, 216-227).
struct LevelGeo {
  uint32_t level;
  bool splits;
  uint64_t G, P;       // nodes, pairs
  uint64_t nblocks;    // G * (splits ? 2 : 1) * P
};

struct Plan {
  int device = 0, dtype = BF_C128, sms = 148;
  uint64_t n = 0;
  uint32_t levels = 0, half = 0, rank = 0, max_rhs = 1;
  uint32_t m = 0;            // middle nodes per side, 2^half
  uint32_t branch = 2;       // tree branching: 2 (reference, 1-D), 4 (quadtree, BASELINE configs 3/4b)
  uint32_t part = 0, nparts = 1;  // sharded plans hold slice `part` of `nparts`
  uint64_t side = 0;         // n / m
  uint32_t nlev = 0;         // transfer levels per side
  std::vector<LevelGeo> lev;
  uint64_t leaf_nb = 0;      // leaf blocks
  uint32_t leaf_n0 = 0;      // rows per leaf block
  uint64_t dim_max = 0;      // largest intermediate vector length (2^L r)
  // device storage: one allocation, carved per factor
  void* base = nullptr;
  uint64_t base_bytes = 0;
  void* u_leaf = nullptr;
  void* v_leaf = nullptr;
  void* weights = nullptr;   // f64 (C128) or f32 (C64)
  std::vector<void*> g_lev, h_lev;
  // leaf factors folded into the outermost transfer level at upload (plan_fold_leaves):
  // blocks (G, nt, 1, n0, C) = leaf block (n0 x r) times level block (r x C); the chain then
  // runs that level with R = n0 and skips the two leaf launches
  void* g_fold = nullptr;    // U^L folded into G^{L-1}
  void* h_fold = nullptr;    // V^L folded into H^{L-1}
  void* fold_base = nullptr; // their allocation (owned by the full plan, not by part views)
  bool uploaded = false;

  size_t elem() const { return dtype == BF_C128 ? 16 : 8; }
  size_t real() const { return dtype == BF_C128 ? 8 : 4; }
};

// Optional per-launch event recorder (bf_timer): ev[2i], ev[2i+1] bracket launch i.
struct LaunchRecorder {
  cudaEvent_t* ev = nullptr;
  uint32_t cap = 0, used = 0;
  int before(cudaStream_t st) {
    if (!ev || used >= cap) return 0;
    return cudaEventRecord(ev[2 * used], st) == cudaSuccess ? 0 : BF_ECUDA;
  }
  int after(cudaStream_t st) {
    if (!ev || used >= cap) return 0;
    return cudaEventRecord(ev[2 * used++ + 1], st) == cudaSuccess ? 0 : BF_ECUDA;
  }
};

int plan_apply(const Plan& pl, const void* in, void* out, uint32_t k, int adjoint, void* ws, cudaStream_t st,
               LaunchRecorder* rec = nullptr);
int plan_apply_half(const Plan& pl, int up, const void* in, void* out, uint32_t k, int adjoint, void* ws,
                    cudaStream_t st);
int plan_apply_down_push(const Plan& pl, const void* in, void* const* peers, uint32_t k, int adjoint, void* ws,
                         cudaStream_t st);
int plan_middle_exchange(const Plan& pl, int unpack, const void* in, void* out, uint32_t k, int adjoint,
                         cudaStream_t st);
Plan part_view(const Plan& full, uint32_t part, uint32_t nparts);
int plan_fold_leaves(Plan& pl, cudaStream_t st);
Plan* plan_build_radix4(const Plan& p, cudaStream_t st);
void plan_free_radix4(Plan* q);
int plan_apply_host_pipelined(const Plan& pl, const void* in_host, void* out_host, void* din, void* dout, void* mid,
                              void* mid2, void* ws, uint32_t k, int adjoint, uint32_t chunks, cudaStream_t run,
                              cudaStream_t cp, cudaEvent_t* ev, uint32_t taper = 0, cudaStream_t aux = nullptr);
int plan_apply_factor(const Plan& pl, int which, int lvl_idx, int adjoint, const void* in, void* out, uint32_t k,
                      cudaStream_t st);
int entries(int kernel_id, uint64_t n, const int64_t* rows, uint32_t nr, const int64_t* cols, uint32_t nc, void* out,
            cudaStream_t st);
int sampled_rows(int kernel_id, uint64_t n, const void* dense, const int64_t* rows, uint32_t nr, const void* g,
                 uint32_t k, void* out, void* workspace, uint64_t ws_bytes, cudaStream_t st);
uint64_t sampled_rows_workspace(uint64_t n, uint32_t nr, uint32_t k);
int convert_c128_to_c64(const void* src, void* dst, uint64_t count, cudaStream_t st);
int convert_f64_to_f32(const void* src, void* dst, uint64_t count, cudaStream_t st);

}  // namespace bfly

struct bf_plan {
  bfly::Plan p;
  // bf_apply graph cache (the plan itself stays immutable; the cache is guarded)
  struct GraphEntry {
    const void* in;
    void* out;
    void* ws;
    uint32_t k;
    int adjoint;
    cudaStream_t stream;
    cudaGraphExec_t exec;
  };
  bool graphs_enabled = true;
  mutable std::mutex gmu;
  mutable std::vector<GraphEntry> graphs;
  mutable cudaStream_t own_stream = nullptr;
  // bf_apply_host device buffers
  mutable void* host_in = nullptr;
  mutable void* host_out = nullptr;
  mutable void* host_ws = nullptr;
  mutable uint64_t host_io_bytes = 0, host_ws_bytes = 0;
  mutable cudaStream_t copy_stream = nullptr;      // host pipeline transfers
  mutable cudaStream_t aux_stream = nullptr;       // host pipeline: odd parts of the down half
  // branching-4 twin of the chain for many right-hand sides (plan_build_radix4), built on first use
  mutable bfly::Plan* r4 = nullptr;
  mutable bool r4_tried = false;
  mutable std::mutex r4mu;
  mutable std::vector<cudaEvent_t> pipe_events;
};

struct bf_timer {
  uint32_t max_steps = 0, max_launches = 0, steps = 0, launches = 0;
  std::vector<cudaEvent_t> ev;  // [step][launch][2]
};
