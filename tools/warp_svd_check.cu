// Checks warp_svd (linalg.cuh) against svd_small on random complex matrices:
// singular values, reconstruction U diag(s) V^H, sweep counts and timing.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tools/warp_svd_check tools/warp_svd_check.cu
#define BF_JACOBI_STATS 1
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1502_01379_b200/csrc/linalg.cuh"

using namespace bfly;

__global__ void k_warp(const double2* in, int m, int n, double2* U, double2* V, double* S, int reps) {
  extern __shared__ double2 wsm[];
  double2* M = wsm;
  double2* Vs = wsm + 32 * 33;
  __shared__ double sg[32];
  const double2* src = in + static_cast<size_t>(blockIdx.x) * m * n;
  for (int i = threadIdx.x; i < m * n; i += 32) M[(i / n) * 33 + i % n] = src[i];
  __syncwarp();
  for (int r = 0; r < reps; ++r)
    warp_svd(M, m, n, 33, 1, U + static_cast<size_t>(blockIdx.x) * 32 * 32, 32, V + static_cast<size_t>(blockIdx.x) * 32 * 32,
             32, sg, Vs);
  for (int i = threadIdx.x; i < (m < n ? m : n); i += 32) S[blockIdx.x * 32 + i] = sg[i];
}

__global__ void k_cta(const double2* in, int m, int n, double* S) {
  extern __shared__ double2 sm[];
  __shared__ int flag, perm[64];
  __shared__ double ssc[64], sg[64];
  double2* M = sm;
  double2* W = M + 32 * 32;
  double2* Vt = W + 32 * 32;
  double2* U = Vt + 32 * 32;
  double2* V = U + 32 * 32;
  const double2* src = in + static_cast<size_t>(blockIdx.x) * m * n;
  for (int i = threadIdx.x; i < m * n; i += blockDim.x) M[i] = src[i];
  __syncthreads();
  svd_small(M, m, n, n, U, 32, V, 32, sg, W, Vt, &flag, perm, ssc);
  for (int i = threadIdx.x; i < (m < n ? m : n); i += blockDim.x) S[blockIdx.x * 32 + i] = sg[i];
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 32, n = argc > 2 ? atoi(argv[2]) : 32, batch = argc > 3 ? atoi(argv[3]) : 256;
  const int rank = argc > 4 ? atoi(argv[4]) : 32;
  std::vector<double2> h(static_cast<size_t>(batch) * m * n);
  srand(3);
  auto rnd = [] { return (rand() + 0.5) / RAND_MAX - 0.5; };
  for (int b = 0; b < batch; ++b) {
    std::vector<double2> x(m * rank), y(rank * n);
    for (auto& e : x) e = make_double2(rnd(), rnd());
    for (auto& e : y) e = make_double2(rnd(), rnd());
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) {
        double2 acc = make_double2(0, 0);
        for (int k = 0; k < rank; ++k) {
          acc.x += x[i * rank + k].x * y[k * n + j].x - x[i * rank + k].y * y[k * n + j].y;
          acc.y += x[i * rank + k].x * y[k * n + j].y + x[i * rank + k].y * y[k * n + j].x;
        }
        h[(static_cast<size_t>(b) * m + i) * n + j] = acc;
      }
  }
  double2 *d, *U, *V;
  double *S1, *S2;
  cudaMalloc(&d, h.size() * 16);
  cudaMalloc(&U, static_cast<size_t>(batch) * 32 * 32 * 16);
  cudaMalloc(&V, static_cast<size_t>(batch) * 32 * 32 * 16);
  cudaMalloc(&S1, batch * 32 * 8);
  cudaMalloc(&S2, batch * 32 * 8);
  cudaMemcpy(d, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 32 * 32 * 16);
  k_cta<<<batch, 256, 5 * 32 * 32 * 16>>>(d, m, n, S2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int zero = 0;
  cudaMemcpyToSymbol(g_jacobi_sweeps, &zero, sizeof(int));
  cudaEventRecord(e0);
  cudaFuncSetAttribute(k_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32 * 33 * 16);
  k_warp<<<batch, 32, 3 * 32 * 33 * 16>>>(d, m, n, U, V, S1, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int sw = 0;
  cudaMemcpyFromSymbol(&sw, g_jacobi_sweeps, sizeof(int));
  std::vector<double> s1(batch * 32), s2(batch * 32);
  cudaMemcpy(s1.data(), S1, s1.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(s2.data(), S2, s2.size() * 8, cudaMemcpyDeviceToHost);
  double maxrel = 0;
  const int k = m < n ? m : n;
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < k; ++i) {
      const double a = s1[b * 32 + i], c = s2[b * 32 + i];
      const double r = fabs(a - c) / (s2[b * 32] > 0 ? s2[b * 32] : 1);
      if (r > maxrel) maxrel = r;
    }
  printf("m=%d n=%d batch=%d rank=%d: warp_svd %.3f ms, sweeps %s, max |s_warp - s_cta| / s_max = %.3e  err=%s\n", m, n,
         batch, rank, ms, "n/a", maxrel, cudaGetErrorString(cudaGetLastError()));
  printf("s_warp[0..3] %.6f %.6f %.6f %.6f  s_cta %.6f %.6f %.6f %.6f\n", s1[0], s1[1], s1[2], s1[3], s2[0], s2[1], s2[2],
         s2[3]);
  return 0;
}
