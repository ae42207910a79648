// tcgen05 probe: one D (128 x N, fp32 in TMEM) = A (128 x K, tf32) * B (N x K, tf32)^T with
// both operands K-major in the canonical no-swizzle ("interleave") shared-memory layout,
// issued by one thread, read back with tcgen05.ld, compared with a CPU product. Checks the
// descriptor encoding (LBO / SBO / version) and the TMEM lane/column mapping used by
// csrc/tc_kernel.cuh. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tcgen05_probe tools/tcgen05_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, N = 32, K = 32;

// canonical K-major no-swizzle: element (row, k) of a rows x K operand
__host__ __device__ inline uint32_t canon(uint32_t row, uint32_t k, uint32_t Kdim) {
  return (k / 4) * 128 + (row / 8) * (Kdim / 4) * 128 + (row % 8) * 16 + (k % 4) * 4;  // bytes
}

__device__ inline uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // version 1 (Blackwell)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

__device__ inline uint32_t idesc_tf32(int m, int n, int a_neg) {
  uint32_t d = 0;
  d |= 1u << 4;              // c_format F32
  d |= 2u << 7;              // a_format TF32
  d |= 2u << 10;             // b_format TF32
  d |= static_cast<uint32_t>(a_neg) << 13;
  // a_major = b_major = 0 (K-major)
  d |= static_cast<uint32_t>(n >> 3) << 17;
  d |= static_cast<uint32_t>(m >> 4) << 24;
  return d;
}

__global__ void probe(const float* A, const float* B, float* D, int neg) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  unsigned char* sa = sm;
  unsigned char* sb = sm + M * K * 4;
  for (int x = threadIdx.x; x < M * K; x += blockDim.x) {
    const int row = x / K, k = x % K;
    *reinterpret_cast<float*>(sa + canon(row, k, K)) = A[row * K + k];
  }
  for (int x = threadIdx.x; x < N * K; x += blockDim.x) {
    const int row = x / K, k = x % K;
    *reinterpret_cast<float*>(sb + canon(row, k, K)) = B[row * K + k];
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base))), "n"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&mbar))));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(sa));
    const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(sb));
    const uint32_t id = idesc_tf32(M, N, neg);
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t ad = smem_desc(a0 + ks * 256, 128, (K / 4) * 128);
      const uint64_t bd = smem_desc(b0 + ks * 256, 128, (K / 4) * 128);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
          "l"(ad), "l"(bd), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&mbar)))
                 : "memory");
  }
  // wait for the MMAs
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(&mbar)))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t v[32];
  const uint32_t taddr = tbase + (static_cast<uint32_t>(w * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  const int row = w * 32 + lane;
#pragma unroll
  for (int n = 0; n < 32; ++n) D[row * N + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(64));
}

int main() {
  float *A, *B, *D;
  cudaMallocManaged(&A, M * K * 4);
  cudaMallocManaged(&B, N * K * 4);
  cudaMallocManaged(&D, M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) A[i] = (rand() % 17 - 8) / 8.0f;  // exact in tf32
  for (int i = 0; i < N * K; ++i) B[i] = (rand() % 13 - 6) / 4.0f;
  const size_t smem = (M + N) * K * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int neg = 0; neg < 2; ++neg) {
    probe<<<1, 128, smem>>>(A, B, D, neg);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
      return 1;
    }
    double maxerr = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[i * K + k] * B[j * K + k];
        if (neg) ref = -ref;
        maxerr = fmax(maxerr, fabs(ref - D[i * N + j]));
      }
    printf("neg=%d max abs err %.3e  D[0][0]=%f D[5][7]=%f\n", neg, maxerr, D[0], D[5 * N + 7]);
  }
  return 0;
}
