// capi.cu — the extern "C" boundary declared in include/bfly.h.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "common.cuh"
#include "plan.h"

namespace bfly {

namespace {
thread_local std::string g_last_error;

using DeviceGuard = DeviceGuardScope;

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

// Copy `count` complex128 values (host or device) into plan storage of the plan dtype.
int upload_complex(const Plan& pl, const void* src, void* dst, uint64_t count, void* tmp, uint64_t tmp_elems,
                   cudaStream_t st) {
  if (!count) return 0;
  if (!src) return fail(BF_EINVAL, "null factor pointer");
  if (pl.dtype == BF_C128) {
    BF_CUDA(cudaMemcpyAsync(dst, src, count * 16, cudaMemcpyDefault, st));
    return 0;
  }
  for (uint64_t off = 0; off < count; off += tmp_elems) {
    const uint64_t c = count - off < tmp_elems ? count - off : tmp_elems;
    BF_CUDA(cudaMemcpyAsync(tmp, static_cast<const double2*>(src) + off, c * 16, cudaMemcpyDefault, st));
    int rc = convert_c128_to_c64(tmp, static_cast<float2*>(dst) + off, c, st);
    if (rc) return rc;
  }
  return 0;
}
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") in " + what;
  return e == cudaErrorMemoryAllocation ? BF_ENOMEM : BF_ECUDA;
}

}  // namespace bfly

using namespace bfly;

extern "C" {

int bf_version(void) { return 1; }

int bf_last_error(char* buf, size_t len) {
  if (!buf || !len) return BF_EINVAL;
  std::snprintf(buf, len, "%s", g_last_error.c_str());
  return BF_OK;
}

static int create_plan(bf_plan** out, uint64_t n, uint32_t levels, uint32_t rank, uint32_t max_rhs, int dtype,
                       int device, uint32_t part, uint32_t nparts, uint32_t branch) {
  if (!out) return fail(BF_EINVAL, "null plan output pointer");
  *out = nullptr;
  // DyadicPartition.__post_init__ (partition.py:25-34)
  if (n < 4 || !is_pow2(n)) return fail(BF_EINVAL, "matrix dimension must be a power of two >= 4");
  if (levels < 2 || levels % 2) return fail(BF_EINVAL, "tree depth must be even and >= 2");
  if (branch != 2 && branch != 4) return fail(BF_EINVAL, "branching must be 2 (binary tree) or 4 (quadtree)");
  const uint32_t lb = branch == 4 ? 2 : 1;  // log2(branching)
  if (branch == 4 && ((63 - __builtin_clzll(n)) % 2)) return fail(BF_EINVAL, "quadtree dimension must be a power of 4");
  if (levels > 40 || lb * (levels / 2) >= 63 || (1ull << (lb * (levels / 2))) > n)
    return fail(BF_EINVAL, "depth puts more nodes than n on the middle level");
  if (rank < 1) return fail(BF_EINVAL, "rank must be positive");
  if (dtype != BF_C128 && dtype != BF_C64) return fail(BF_EINVAL, "dtype must be BF_C128 or BF_C64");
  if (nparts < 1 || part >= nparts || ((1ull << (lb * (levels / 2))) % nparts) != 0)
    return fail(BF_EINVAL, "nparts must divide the middle node count and part < nparts");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(BF_EINVAL, "no such CUDA device");
  bf_plan* h = new (std::nothrow) bf_plan();
  if (!h) return fail(BF_ENOMEM, "host allocation failed");
  const char* ng = std::getenv("BF_NO_GRAPHS");
  h->graphs_enabled = !(ng && ng[0] && ng[0] != '0');
  Plan& p = h->p;
  p.device = device;
  p.dtype = dtype;
  p.n = n;
  p.levels = levels;
  p.half = levels / 2;
  p.rank = rank;
  p.max_rhs = max_rhs ? max_rhs : 1;
  p.branch = branch;
  p.m = 1u << (lb * p.half);
  p.part = part;
  p.nparts = nparts;
  p.side = n / p.m;
  // construct.py:_level_geometry (216-227)
  uint64_t nodes = p.m, rows = p.side;
  for (uint32_t lvl = p.half; lvl < levels; ++lvl) {
    LevelGeo g;
    g.level = lvl;
    g.P = 1ull << (lb * (levels - lvl - 1));
    g.G = nodes / nparts;  // this part's groups (the leading index carries the middle node)
    g.splits = rows >= branch;
    g.nblocks = g.G * (g.splits ? branch : 1) * g.P;
    if (g.splits) {
      nodes *= branch;
      rows /= branch;
    }
    p.lev.push_back(g);
  }
  p.nlev = static_cast<uint32_t>(p.lev.size());
  p.leaf_nb = nodes / nparts;
  p.leaf_n0 = static_cast<uint32_t>(rows);
  const uint64_t full = (1ull << (lb * levels)) * rank;
  p.dim_max = (full > n ? full : n) / nparts;
  {
    DeviceGuard dg(device);
    cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, device);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  *out = h;
  return BF_OK;
}

int bf_plan_create(bf_plan** out, uint64_t n, uint32_t levels, uint32_t rank, uint32_t max_rhs, int dtype,
                   int device) {
  return create_plan(out, n, levels, rank, max_rhs, dtype, device, 0, 1, 2);
}

int bf_plan_create_sharded(bf_plan** out, uint64_t n, uint32_t levels, uint32_t rank, int dtype, int device,
                           uint32_t part, uint32_t nparts) {
  return create_plan(out, n, levels, rank, 1, dtype, device, part, nparts, 2);
}

int bf_plan_create_tree(bf_plan** out, uint64_t n, uint32_t levels, uint32_t rank, uint32_t branching, int dtype,
                        int device, uint32_t part, uint32_t nparts) {
  return create_plan(out, n, levels, rank, 1, dtype, device, part, nparts, branching);
}

void bf_plan_destroy(bf_plan* plan) {
  if (!plan) return;
  DeviceGuard dg(plan->p.device);
  for (auto& gentry : plan->graphs) cudaGraphExecDestroy(gentry.exec);
  if (plan->host_in) cudaFree(plan->host_in);
  if (plan->host_out) cudaFree(plan->host_out);
  if (plan->host_ws) cudaFree(plan->host_ws);
  for (auto e : plan->pipe_events) cudaEventDestroy(e);
  if (plan->copy_stream) cudaStreamDestroy(plan->copy_stream);
  if (plan->aux_stream) cudaStreamDestroy(plan->aux_stream);
  if (plan->own_stream) cudaStreamDestroy(plan->own_stream);
  plan_free_radix4(plan->r4);
  if (plan->p.fold_base) cudaFree(plan->p.fold_base);
  if (plan->p.base) cudaFree(plan->p.base);
  delete plan;
}

int bf_plan_geometry(const bf_plan* plan, uint32_t* nlev, int8_t* splits, uint64_t* dims, uint64_t* leaf) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (nlev) *nlev = p.nlev;
  for (uint32_t i = 0; i < p.nlev; ++i) {
    const LevelGeo& g = p.lev[i];
    if (splits) splits[i] = g.splits ? 1 : 0;
    if (dims) {
      uint64_t* d = dims + 5ull * i;
      if (g.splits) {
        d[0] = g.G; d[1] = p.branch; d[2] = g.P; d[3] = p.rank; d[4] = static_cast<uint64_t>(p.branch) * p.rank;
      } else {
        d[0] = g.G; d[1] = g.P; d[2] = p.rank; d[3] = static_cast<uint64_t>(p.branch) * p.rank; d[4] = 0;
      }
    }
  }
  if (leaf) {
    leaf[0] = p.leaf_nb;
    leaf[1] = p.leaf_n0;
    leaf[2] = p.rank;
  }
  return BF_OK;
}

int bf_plan_upload(bf_plan* plan, const void* u_leaf, const void* const* g_levels, const double* weights,
                   const void* const* h_levels, const void* v_leaf) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  if (!g_levels || !h_levels) return fail(BF_EINVAL, "null level pointer array");
  Plan& p = plan->p;
  DeviceGuard dg(p.device);
  const uint64_t es = p.elem(), rs = p.real();
  const uint64_t leaf_elems = p.leaf_nb * p.leaf_n0 * p.rank;
  const uint64_t w_elems = static_cast<uint64_t>(p.m) * p.m * p.rank;
  uint64_t bytes = 2 * align_up(leaf_elems * es, 256) + align_up(w_elems * rs, 256);
  for (const LevelGeo& g : p.lev) bytes += 2 * align_up(g.nblocks * p.rank * p.branch * p.rank * es, 256);
  if (!p.base) {
    cudaError_t e = cudaMalloc(&p.base, bytes);
    if (e != cudaSuccess) {
      p.base = nullptr;
      return cuda_fail(e, "cudaMalloc(factor storage)");
    }
    p.base_bytes = bytes;
  }
  char* cur = static_cast<char*>(p.base);
  auto carve = [&](uint64_t b) {
    void* r = cur;
    cur += align_up(b, 256);
    return r;
  };
  p.u_leaf = carve(leaf_elems * es);
  p.v_leaf = carve(leaf_elems * es);
  p.weights = carve(w_elems * rs);
  p.g_lev.assign(p.nlev, nullptr);
  p.h_lev.assign(p.nlev, nullptr);
  for (uint32_t i = 0; i < p.nlev; ++i) p.g_lev[i] = carve(p.lev[i].nblocks * p.rank * p.branch * p.rank * es);
  for (uint32_t i = 0; i < p.nlev; ++i) p.h_lev[i] = carve(p.lev[i].nblocks * p.rank * p.branch * p.rank * es);

  cudaStream_t st = nullptr;
  void* tmp = nullptr;
  const uint64_t tmp_elems = 1ull << 25;  // 512 MiB of complex128 staging for the C64 conversion
  if (p.dtype == BF_C64) BF_CUDA(cudaMalloc(&tmp, tmp_elems * 16));
  int rc = upload_complex(p, u_leaf, p.u_leaf, leaf_elems, tmp, tmp_elems, st);
  if (!rc) rc = upload_complex(p, v_leaf, p.v_leaf, leaf_elems, tmp, tmp_elems, st);
  for (uint32_t i = 0; !rc && i < p.nlev; ++i) {
    const uint64_t c = p.lev[i].nblocks * p.rank * p.branch * p.rank;
    rc = upload_complex(p, g_levels[i], p.g_lev[i], c, tmp, tmp_elems, st);
    if (!rc) rc = upload_complex(p, h_levels[i], p.h_lev[i], c, tmp, tmp_elems, st);
  }
  if (!rc) {
    if (!weights) {
      rc = fail(BF_EINVAL, "null middle weights");
    } else if (p.dtype == BF_C128) {
      cudaError_t e = cudaMemcpyAsync(p.weights, weights, w_elems * 8, cudaMemcpyDefault, st);
      if (e != cudaSuccess) rc = cuda_fail(e, "upload weights");
    } else {
      cudaError_t e = cudaMemcpyAsync(tmp, weights, w_elems * 8, cudaMemcpyDefault, st);
      rc = e != cudaSuccess ? cuda_fail(e, "upload weights") : convert_f64_to_f32(tmp, p.weights, w_elems, st);
    }
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (tmp) cudaFree(tmp);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "bf_plan_upload");
  p.uploaded = true;
  return plan_fold_leaves(p, st);
}

uint64_t bf_apply_workspace_bytes(const bf_plan* plan, uint32_t k) {
  if (!plan) return 0;
  return 2ull * plan->p.dim_max * (k ? k : 1) * plan->p.elem();
}

// Destroys every cached graph of the plan (caller holds gmu and has synchronised the
// streams the graphs ran on).
static void drop_graphs_locked(const bf_plan* plan) {
  for (auto& gentry : plan->graphs) cudaGraphExecDestroy(gentry.exec);
  plan->graphs.clear();
}

// The plan a k-column apply runs on: the branching-4 twin (pairs of levels folded,
// plan_build_radix4) for many right-hand sides once it exists, else the plan itself.
// Built on first use (never inside a stream capture: callers resolve the plan first).
static const Plan& chain_plan(const bf_plan* plan, uint32_t k, cudaStream_t st = nullptr) {
  if (k < 8) return plan->p;
  std::lock_guard<std::mutex> lock(plan->r4mu);
  if (!plan->r4_tried && st) {   // a caller-side capture in progress: no allocation, no build
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return plan->p;
    }
  }
  if (!plan->r4_tried) {
    plan->r4_tried = true;
    plan->r4 = plan_build_radix4(plan->p, nullptr);
  }
  return plan->r4 ? *plan->r4 : plan->p;
}

// The chain is a fixed sequence of 2 + 2(L-h) launches: replay it as one CUDA
// graph per (buffers, k, direction, stream). A NULL stream is the legacy default
// stream, which cannot be captured; the graph then runs on a plan-owned blocking
// stream, which the legacy stream orders against implicitly. Caller holds gmu.
static int apply_graph_locked(const bf_plan* plan, const void* in, void* out, uint32_t k, int adjoint,
                              void* workspace, cudaStream_t st) {
  const Plan& p = chain_plan(plan, k, st);
  cudaStream_t run = st;
  if (!run) {
    if (!plan->own_stream) BF_CUDA(cudaStreamCreate(&plan->own_stream));
    run = plan->own_stream;
  }
  for (const auto& gentry : plan->graphs)
    if (gentry.in == in && gentry.out == out && gentry.ws == workspace && gentry.k == k && gentry.adjoint == adjoint &&
        gentry.stream == st) {
      BF_CUDA(cudaGraphLaunch(gentry.exec, run));
      return BF_OK;
    }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  BF_CUDA(cudaStreamIsCapturing(run, &cap));
  if (cap != cudaStreamCaptureStatusNone) return plan_apply(p, in, out, k, adjoint ? 1 : 0, workspace, st);
  BF_CUDA(cudaStreamBeginCapture(run, cudaStreamCaptureModeThreadLocal));
  const int rc = plan_apply(p, in, out, k, adjoint ? 1 : 0, workspace, run);
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(run, &graph);
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) return cuda_fail(ei, "cudaGraphInstantiate");
  if (plan->graphs.size() >= 16) {
    cudaGraphExecDestroy(plan->graphs.front().exec);
    plan->graphs.erase(plan->graphs.begin());
  }
  plan->graphs.push_back({in, out, workspace, k, adjoint, st, exec});
  BF_CUDA(cudaGraphLaunch(exec, run));
  return BF_OK;
}

int bf_apply(const bf_plan* plan, const void* in, void* out, uint32_t k, int adjoint, void* workspace,
             uint64_t workspace_bytes, void* stream) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors (call bf_plan_upload)");
  if (k < 1) return fail(BF_EINVAL, "need at least one right-hand side");
  if (!in || !out) return fail(BF_EINVAL, "null input/output pointer");
  if (!workspace || workspace_bytes < bf_apply_workspace_bytes(plan, k))
    return fail(BF_EINVAL, "workspace too small (see bf_apply_workspace_bytes)");
  if (p.nparts != 1) return fail(BF_EINVAL, "sharded plan: use bf_apply_down / bf_middle_pack / bf_apply_up");
  DeviceGuard dg(p.device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!plan->graphs_enabled) return plan_apply(chain_plan(plan, k, st), in, out, k, adjoint ? 1 : 0, workspace, st);
  std::lock_guard<std::mutex> lock(plan->gmu);
  return apply_graph_locked(plan, in, out, k, adjoint, workspace, st);
}

int bf_apply_down(const bf_plan* plan, const void* in, void* mid, uint32_t k, int adjoint, void* workspace,
                  uint64_t workspace_bytes, void* stream) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors (call bf_plan_upload)");
  if (k < 1 || !in || !mid) return fail(BF_EINVAL, "bad k or null pointer");
  if (!workspace || workspace_bytes < bf_apply_workspace_bytes(plan, k))
    return fail(BF_EINVAL, "workspace too small (see bf_apply_workspace_bytes)");
  DeviceGuard dg(p.device);
  return plan_apply_half(chain_plan(plan, k, static_cast<cudaStream_t>(stream)), 0, in, mid, k, adjoint ? 1 : 0, workspace, static_cast<cudaStream_t>(stream));
}

int bf_apply_up(const bf_plan* plan, const void* mid, void* out, uint32_t k, int adjoint, void* workspace,
                uint64_t workspace_bytes, void* stream) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors (call bf_plan_upload)");
  if (k < 1 || !mid || !out) return fail(BF_EINVAL, "bad k or null pointer");
  if (!workspace || workspace_bytes < bf_apply_workspace_bytes(plan, k))
    return fail(BF_EINVAL, "workspace too small (see bf_apply_workspace_bytes)");
  DeviceGuard dg(p.device);
  return plan_apply_half(chain_plan(plan, k, static_cast<cudaStream_t>(stream)), 1, mid, out, k, adjoint ? 1 : 0, workspace, static_cast<cudaStream_t>(stream));
}

int bf_apply_down_push(const bf_plan* plan, const void* in, void* const* peers, uint32_t k, int adjoint,
                       void* workspace, uint64_t workspace_bytes, void* stream) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors (call bf_plan_upload)");
  if (k < 1 || !in || !peers) return fail(BF_EINVAL, "bad k or null pointer");
  for (uint32_t d = 0; d < p.nparts; ++d)
    if (!peers[d]) return fail(BF_EINVAL, "null peer receive buffer");
  if (!workspace || workspace_bytes < bf_apply_workspace_bytes(plan, k))
    return fail(BF_EINVAL, "workspace too small (see bf_apply_workspace_bytes)");
  DeviceGuard dg(p.device);
  return plan_apply_down_push(p, in, peers, k, adjoint ? 1 : 0, workspace, static_cast<cudaStream_t>(stream));
}

int bf_middle_pack(const bf_plan* plan, const void* mid, void* send, uint32_t k, int adjoint, void* stream) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors (call bf_plan_upload)");
  if (k < 1 || !mid || !send) return fail(BF_EINVAL, "bad k or null pointer");
  DeviceGuard dg(p.device);
  return plan_middle_exchange(p, 0, mid, send, k, adjoint ? 1 : 0, static_cast<cudaStream_t>(stream));
}

int bf_middle_unpack(const bf_plan* plan, const void* recv, void* mid, uint32_t k, int adjoint, void* stream) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors (call bf_plan_upload)");
  if (k < 1 || !recv || !mid) return fail(BF_EINVAL, "bad k or null pointer");
  DeviceGuard dg(p.device);
  return plan_middle_exchange(p, 1, recv, mid, k, adjoint ? 1 : 0, static_cast<cudaStream_t>(stream));
}

int bf_timer_create(bf_timer** out, uint32_t max_steps, uint32_t max_launches) {
  if (!out || !max_steps || !max_launches) return fail(BF_EINVAL, "bad timer arguments");
  *out = nullptr;
  bf_timer* t = new (std::nothrow) bf_timer();
  if (!t) return fail(BF_ENOMEM, "host allocation failed");
  t->max_steps = max_steps;
  t->max_launches = max_launches;
  t->ev.assign(2ull * max_steps * max_launches, nullptr);
  for (auto& e : t->ev) {
    cudaError_t err = cudaEventCreate(&e);
    if (err != cudaSuccess) {
      e = nullptr;
      bf_timer_destroy(t);
      return cuda_fail(err, "cudaEventCreate");
    }
  }
  *out = t;
  return BF_OK;
}

void bf_timer_destroy(bf_timer* timer) {
  if (!timer) return;
  for (auto e : timer->ev)
    if (e) cudaEventDestroy(e);
  delete timer;
}

int bf_apply_timed(const bf_plan* plan, const void* in, void* out, uint32_t k, int adjoint, void* workspace,
                   uint64_t workspace_bytes, void* stream, bf_timer* timer) {
  if (!timer) return fail(BF_EINVAL, "null timer");
  if (timer->steps >= timer->max_steps) return fail(BF_EINVAL, "timer is full");
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors (call bf_plan_upload)");
  if (k < 1 || !in || !out) return fail(BF_EINVAL, "bad k or null pointer");
  if (!workspace || workspace_bytes < bf_apply_workspace_bytes(plan, k))
    return fail(BF_EINVAL, "workspace too small (see bf_apply_workspace_bytes)");
  if (p.nparts != 1) return fail(BF_EINVAL, "sharded plan: use bf_apply_down / bf_middle_pack / bf_apply_up");
  DeviceGuard dg(p.device);
  LaunchRecorder rec;
  rec.ev = timer->ev.data() + 2ull * timer->steps * timer->max_launches;
  rec.cap = timer->max_launches;
  int rc = plan_apply(chain_plan(plan, k), in, out, k, adjoint ? 1 : 0, workspace, static_cast<cudaStream_t>(stream), &rec);
  if (rc) return rc;
  if (timer->steps == 0) timer->launches = rec.used;
  if (rec.used != timer->launches) return fail(BF_EINVAL, "launch count changed between timed steps");
  ++timer->steps;
  return BF_OK;
}

int bf_timer_read(bf_timer* timer, float* launch_ms, uint32_t* steps, uint32_t* launches) {
  if (!timer) return fail(BF_EINVAL, "null timer");
  if (steps) *steps = timer->steps;
  if (launches) *launches = timer->launches;
  if (!launch_ms) return BF_OK;
  for (uint32_t s = 0; s < timer->steps; ++s)
    for (uint32_t i = 0; i < timer->launches; ++i) {
      cudaEvent_t* e = timer->ev.data() + 2ull * (static_cast<uint64_t>(s) * timer->max_launches + i);
      BF_CUDA(cudaEventSynchronize(e[1]));
      float ms = 0;
      BF_CUDA(cudaEventElapsedTime(&ms, e[0], e[1]));
      launch_ms[static_cast<uint64_t>(s) * timer->launches + i] = ms;
    }
  return BF_OK;
}

int bf_apply_host(const bf_plan* plan, const void* in_host, void* out_host, uint32_t k, int adjoint, void* stream) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors (call bf_plan_upload)");
  if (k < 1) return fail(BF_EINVAL, "need at least one right-hand side");
  if (!in_host || !out_host) return fail(BF_EINVAL, "null input/output pointer");
  if (p.nparts != 1) return fail(BF_EINVAL, "sharded plan: use bf_apply_down / bf_middle_pack / bf_apply_up");
  DeviceGuard dg(p.device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t io = p.n * k * p.elem();
  const uint64_t wsb = bf_apply_workspace_bytes(plan, k);
  // persistent device buffers (grown on demand) keep the pointers stable, so the chain
  // replays from the graph cache; the plan mutex serialises host applies on one plan
  std::lock_guard<std::mutex> lock(plan->gmu);
  cudaStream_t run = st;
  if (!run) {
    if (!plan->own_stream) BF_CUDA(cudaStreamCreate(&plan->own_stream));
    run = plan->own_stream;
  }
  // large transfers: pipeline H2D/D2H chunks (per middle-node range) against the chain
  uint32_t chunks = p.m >= 4 ? 4 : 1;  // measured best at cfg2 (tools/e2e_probe.py: 1 2.11 ms, 4 1.86, 8 1.98, 16 2.49)
  if (const char* env = getenv("BF_PIPE_CHUNKS")) {  // tuning knob: power of two <= m
    const long v = strtol(env, nullptr, 10);
    if (v >= 1 && v <= static_cast<long>(p.m) && (v & (v - 1)) == 0) chunks = static_cast<uint32_t>(v);
  }
  // tapered parts (1/T, 1/T, 2/T, ... 1/2 down, the mirror image up): the first upload and the
  // last download are 1/T of the vector and most of the chain runs in large parts.
  // BF_PIPE_TAPER=0 keeps `chunks` equal parts; setting BF_PIPE_CHUNKS does too.
  uint32_t taper = (p.m >= 8 && !getenv("BF_PIPE_CHUNKS")) ? 8 : 0;
  if (const char* env = getenv("BF_PIPE_TAPER")) {
    const long v = strtol(env, nullptr, 10);
    taper = (v >= 4 && v <= static_cast<long>(p.m) && (v & (v - 1)) == 0) ? static_cast<uint32_t>(v) : 0;
  }
  uint32_t nchunk = chunks, biggest = chunks;   // number of parts; the largest part is 1/biggest
  if (taper) {
    nchunk = 1;
    for (uint32_t T = taper; T >= 2; T /= 2) ++nchunk;
    biggest = 2;
  }
  // (graph capture of a memcpy needs page-locked host memory)
  auto pinned = [](const void* ptr) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool pipelined =
      plan->graphs_enabled && chunks > 1 && io >= (4ull << 20) && pinned(in_host) && pinned(out_host);
  const uint64_t mid_bytes = static_cast<uint64_t>(p.m) * p.m * p.rank * k * p.elem();
  // BF_PIPE_STREAMS=2: the down halves of odd parts on a second compute stream (own workspace slices)
  static const bool two_streams = [] {
    const char* e = getenv("BF_PIPE_STREAMS");
    return e && atoi(e) == 2;
  }();
  const uint64_t part_ws = two_streams ? 2 * p.dim_max * k * p.elem() * 2 : 2 * (p.dim_max / biggest) * k * p.elem();
  const uint64_t need_ws = pipelined ? 2 * mid_bytes + part_ws : wsb;
  if (plan->host_io_bytes < io || plan->host_ws_bytes < need_ws) {
    BF_CUDA(cudaStreamSynchronize(run));
    // every cached graph that captured the old device buffers would replay against freed
    // memory (a k=1 graph found again after a k=4 call grew them): drop them all
    drop_graphs_locked(plan);
    if (plan->host_in) cudaFree(plan->host_in);
    if (plan->host_out) cudaFree(plan->host_out);
    if (plan->host_ws) cudaFree(plan->host_ws);
    plan->host_in = plan->host_out = plan->host_ws = nullptr;
    plan->host_io_bytes = plan->host_ws_bytes = 0;
    BF_CUDA(cudaMalloc(&plan->host_in, io));
    BF_CUDA(cudaMalloc(&plan->host_out, io));
    BF_CUDA(cudaMalloc(&plan->host_ws, need_ws));
    plan->host_io_bytes = io;
    plan->host_ws_bytes = need_ws;
  }
  if (pipelined) {
    if (!plan->copy_stream) BF_CUDA(cudaStreamCreateWithFlags(&plan->copy_stream, cudaStreamNonBlocking));
    if (two_streams && !plan->aux_stream) BF_CUDA(cudaStreamCreateWithFlags(&plan->aux_stream, cudaStreamNonBlocking));
    if (plan->pipe_events.size() < 3 * nchunk + 3) {  // BF_PIPE_CHUNKS is re-read on every call
      BF_CUDA(cudaStreamSynchronize(run));
      drop_graphs_locked(plan);  // captured graphs reference the old events
      for (auto e : plan->pipe_events) cudaEventDestroy(e);
      plan->pipe_events.assign(3 * nchunk + 3, nullptr);
      for (auto& e : plan->pipe_events) BF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    void* const key_ws = reinterpret_cast<void*>(static_cast<uintptr_t>(1));  // marks the pipelined graph
    for (const auto& gentry : plan->graphs)
      if (gentry.in == in_host && gentry.out == out_host && gentry.ws == key_ws && gentry.k == k &&
          gentry.adjoint == adjoint && gentry.stream == run) {
        BF_CUDA(cudaGraphLaunch(gentry.exec, run));
        BF_CUDA(cudaStreamSynchronize(run));
        return BF_OK;
      }
    char* w = static_cast<char*>(plan->host_ws);
    (void)chain_plan(plan, k);   // build the many-RHS twin, if any, outside the capture
    BF_CUDA(cudaStreamBeginCapture(run, cudaStreamCaptureModeThreadLocal));
    const Plan& cp = chain_plan(plan, k);   // (resolved above, before the capture began)
    const int rc = plan_apply_host_pipelined(cp, in_host, out_host, plan->host_in, plan->host_out, w, w + mid_bytes,
                                             w + 2 * mid_bytes, k, adjoint ? 1 : 0, chunks, run, plan->copy_stream,
                                             plan->pipe_events.data(), taper, two_streams ? plan->aux_stream : nullptr);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(run, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture (host pipeline)");
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) return cuda_fail(ei, "cudaGraphInstantiate (host pipeline)");
    if (plan->graphs.size() >= 16) {
      cudaGraphExecDestroy(plan->graphs.front().exec);
      plan->graphs.erase(plan->graphs.begin());
    }
    plan->graphs.push_back({in_host, out_host, key_ws, k, adjoint ? 1 : 0, run, exec});
    BF_CUDA(cudaGraphLaunch(exec, run));
    BF_CUDA(cudaStreamSynchronize(run));
    return BF_OK;
  }
  BF_CUDA(cudaMemcpyAsync(plan->host_in, in_host, io, cudaMemcpyHostToDevice, run));
  int rc = plan->graphs_enabled
               ? apply_graph_locked(plan, plan->host_in, plan->host_out, k, adjoint ? 1 : 0, plan->host_ws, run)
               : plan_apply(chain_plan(plan, k), plan->host_in, plan->host_out, k, adjoint ? 1 : 0, plan->host_ws, run);
  if (rc) return rc;
  BF_CUDA(cudaMemcpyAsync(out_host, plan->host_out, io, cudaMemcpyDeviceToHost, run));
  BF_CUDA(cudaStreamSynchronize(run));
  return BF_OK;
}

int bf_apply_factor(const bf_plan* plan, int which, uint32_t level, int adjoint, const void* in, void* out,
                    uint32_t k, void* stream) {
  if (!plan) return fail(BF_EINVAL, "null plan");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors (call bf_plan_upload)");
  if (which < BF_FACTOR_V || which > BF_FACTOR_U) return fail(BF_EINVAL, "unknown factor selector");
  if (k < 1 || !in || !out) return fail(BF_EINVAL, "bad k or null pointer");
  int idx = 0;
  if (which == BF_FACTOR_G || which == BF_FACTOR_H) {
    if (level < p.half || level >= p.levels) return fail(BF_EINVAL, "transfer level outside [half, levels)");
    idx = static_cast<int>(level - p.half);
  }
  DeviceGuard dg(p.device);
  return plan_apply_factor(p, which, idx, adjoint ? 1 : 0, in, out, k, static_cast<cudaStream_t>(stream));
}

uint64_t bf_sampled_rows_workspace(uint64_t n, uint32_t nr, uint32_t k) { return sampled_rows_workspace(n, nr, k); }

int bf_sampled_rows(int kernel_id, uint64_t n, const void* dense, const int64_t* rows, uint32_t nr, const void* g,
                    uint32_t k, void* out, void* workspace, uint64_t ws_bytes, void* stream) {
  if (kernel_id < BF_KERNEL_FIO || kernel_id > BF_KERNEL_DFT) return fail(BF_EINVAL, "unknown entry kernel id");
  if (kernel_id == BF_KERNEL_DENSE && !dense) return fail(BF_EINVAL, "dense oracle needs a matrix pointer");
  if (n < 1 || k < 1) return fail(BF_EINVAL, "n and k must be positive");
  if (!nr) return BF_OK;
  if (!rows || !g || !out || !workspace) return fail(BF_EINVAL, "null pointer");
  return sampled_rows(kernel_id, n, dense, rows, nr, g, k, out, workspace, ws_bytes, static_cast<cudaStream_t>(stream));
}

int bf_entries(int kernel_id, uint64_t n, const int64_t* rows, uint32_t nr, const int64_t* cols, uint32_t nc,
               void* out, void* stream) {
  if (n < 1) return fail(BF_EINVAL, "n must be positive");
  if ((nr && !rows) || (nc && !cols) || (static_cast<uint64_t>(nr) * nc != 0 && !out))
    return fail(BF_EINVAL, "null pointer");
  return entries(kernel_id, n, rows, nr, cols, nc, out, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
