// entries.cu — kernel-entry evaluator K(x, xi) = exp(2 pi i Phi(x, xi)) on
// index sets, plus dtype conversion kernels used by plan upload.
//
// FIO (kernels.py:23-38): x = i/N, xi = j - N/2, Phi = x xi + c(x)|xi|,
// c(x) = (2 + sin(2 pi x))/8, value exp(2 pi i Phi). The reference evaluates
// in NumPy with one rounding per operation and no fused multiply-add; every
// product/sum here uses the _rn intrinsics so nvcc cannot contract them
// (contraction changes ~22% of phases). Only the final
// sin/cos may differ from glibc by an ulp or two.
// DFTP (BASELINE config 1): exp(+2 pi i (j k mod N)/N), phase exact in int64.
#include "common.cuh"
#include "entry_eval.cuh"
#include "plan.h"

namespace bfly {

namespace {

__global__ void entries_kernel(int kind, uint64_t n, const int64_t* __restrict__ rows, uint32_t nr,
                               const int64_t* __restrict__ cols, uint32_t nc, double2* __restrict__ out) {
  const uint64_t total = static_cast<uint64_t>(nr) * nc;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = rows[x / nc], j = cols[x % nc];
    out[x] = kind == BF_KERNEL_FIO ? fio_entry(n, i, j) : kind == BF_KERNEL_DFTP ? dftp_entry(n, i, j) : radon2d_entry(n, i, j);
  }
}

__global__ void c128_to_c64(const double2* __restrict__ src, float2* __restrict__ dst, uint64_t count) {
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < count;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double2 v = src[x];
    dst[x] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
  }
}

__global__ void f64_to_f32(const double* __restrict__ src, float* __restrict__ dst, uint64_t count) {
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < count;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[x] = static_cast<float>(src[x]);
}

unsigned grid_for(uint64_t total) {
  uint64_t g = (total + 255) / 256;
  return static_cast<unsigned>(g > 148 * 16 ? 148 * 16 : (g ? g : 1));
}

}  // namespace

int entries(int kernel_id, uint64_t n, const int64_t* rows, uint32_t nr, const int64_t* cols, uint32_t nc, void* out,
            cudaStream_t st) {
  if (kernel_id != BF_KERNEL_FIO && kernel_id != BF_KERNEL_DFTP && kernel_id != BF_KERNEL_RADON2D)
    return fail(BF_EINVAL, "unknown entry kernel id");
  if (static_cast<uint64_t>(nr) * nc == 0) return 0;
  entries_kernel<<<grid_for(static_cast<uint64_t>(nr) * nc), 256, 0, st>>>(kernel_id, n, rows, nr, cols, nc,
                                                                          static_cast<double2*>(out));
  BF_CUDA(cudaGetLastError());
  return 0;
}

int convert_c128_to_c64(const void* src, void* dst, uint64_t count, cudaStream_t st) {
  if (!count) return 0;
  c128_to_c64<<<grid_for(count), 256, 0, st>>>(static_cast<const double2*>(src), static_cast<float2*>(dst), count);
  BF_CUDA(cudaGetLastError());
  return 0;
}

int convert_f64_to_f32(const void* src, void* dst, uint64_t count, cudaStream_t st) {
  if (!count) return 0;
  f64_to_f32<<<grid_for(count), 256, 0, st>>>(static_cast<const double*>(src), static_cast<float*>(dst), count);
  BF_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace bfly
