// common.cuh — sm_100a helpers shared by the libbfly kernels: complex
// arithmetic on interleaved (re, im) pairs, mbarrier + cp.async.bulk (TMA
// bulk-copy engine) wrappers, and error plumbing for the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace bfly {

// ---------------------------------------------------------------- complex
template <typename E> struct Cx;  // element traits: E = double2 | float2
template <> struct Cx<double2> {
  using R = double;
  static __host__ __device__ __forceinline__ double2 make(double a, double b) { return make_double2(a, b); }
};
template <> struct Cx<float2> {
  using R = float;
  static __host__ __device__ __forceinline__ float2 make(float a, float b) { return make_float2(a, b); }
};

// acc += a * b
template <typename E>
__device__ __forceinline__ void cmac(E& acc, const E a, const E b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
template <typename E>
__device__ __forceinline__ void cmac_conj(E& acc, const E a, const E b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}

template <typename E>
__device__ __forceinline__ E shfl_xor(E v, int mask) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, mask);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, mask);
  return v;
}

// ---------------------------------------------------------------- PTX: mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "BF_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra BF_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// L2 policy: streamed-once data (factor blocks) is evicted first so the
// chain's intermediate vectors stay L2-resident between levels.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// TMA bulk engine: global -> shared, completion signalled as tx bytes on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// -x by a sign-bit flip on the integer pipe (a DADD would queue behind DMMAs on the FP64 datapath)
__device__ __forceinline__ double neg(double x) {
  return __hiloint2double(__double2hiint(x) ^ static_cast<int>(0x80000000u), __double2loint(x));
}

// TMA bulk engine: shared -> global (bulk async-group completion, per issuing thread).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// all but the newest N committed groups of this thread have finished reading shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// every committed group of this thread has completed (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes become visible to the async proxy (TMA reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- launch limits
// Dynamic shared memory opt-in set once to the sm_100a maximum for every kernel
// (not per launch to the launch's own size): concurrent launches of one kernel
// with different sizes cannot race on the attribute, and a profiler replaying a
// captured graph node in isolation sees an attribute large enough for it.
constexpr int kMaxDynSmem = 227 * 1024;

// Opt a kernel in to the largest dynamic shared memory its static shared memory leaves.
template <typename Kernel>
inline cudaError_t allow_max_dyn_smem(Kernel* kern) {
  cudaFuncAttributes fa{};
  const cudaError_t e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kMaxDynSmem - static_cast<int>(fa.sharedSizeBytes));
}

// ---------------------------------------------------------------- device scope
// Makes `dev` current for the scope and restores the caller's device after.
struct DeviceGuardScope {
  int prev = -1;
  explicit DeviceGuardScope(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuardScope() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

}  // namespace bfly

#define BF_CUDA(call)                                        \
  do {                                                       \
    cudaError_t bf_e_ = (call);                              \
    if (bf_e_ != cudaSuccess) return ::bfly::cuda_fail(bf_e_, #call); \
  } while (0)
