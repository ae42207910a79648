// Standalone timing of the construction's shared-memory SVD (svd_small /
// jacobi_cols in linalg.cuh) on batches of random complex matrices; reports
// time per batch and the mean Jacobi sweep count. Build: make -C tools jacobi_bench
#define BF_JACOBI_STATS 1
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1502_01379_b200/csrc/linalg.cuh"

using namespace bfly;

__global__ void k_svd(const double2* in, int m, int n, double2* U, double2* V, double* S) {
  extern __shared__ double2 sm[];
  __shared__ int flag, perm[64];
  __shared__ double ssc[64];
  const int ld = n;
  double2* M = sm;
  double2* W = M + m * n;
  double2* Vt = W + (m > n ? m : n) * (m < n ? m : n);
  const double2* src = in + static_cast<size_t>(blockIdx.x) * m * n;
  for (int i = threadIdx.x; i < m * n; i += blockDim.x) M[i] = src[i];
  __syncthreads();
  svd_small(M, m, n, ld, U + static_cast<size_t>(blockIdx.x) * m * 64, 64, V + static_cast<size_t>(blockIdx.x) * 64 * 64,
            64, S + blockIdx.x * 64, W, Vt, &flag, perm, ssc);
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 32, n = argc > 2 ? atoi(argv[2]) : 32;
  const int batch = argc > 3 ? atoi(argv[3]) : 256, threads = argc > 4 ? atoi(argv[4]) : 256;
  const int rank = argc > 5 ? atoi(argv[5]) : n;  // rank of the random matrices
  std::vector<double2> h(static_cast<size_t>(batch) * m * n);
  srand(1);
  auto rnd = [] { return (rand() + 0.5) / RAND_MAX - 0.5; };
  for (int b = 0; b < batch; ++b) {
    std::vector<double2> a(m * rank), c(rank * n);
    for (auto& x : a) x = make_double2(rnd(), rnd());
    for (auto& x : c) x = make_double2(rnd(), rnd());
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) {
        double2 acc = make_double2(0, 0);
        for (int k = 0; k < rank; ++k) {
          acc.x += a[i * rank + k].x * c[k * n + j].x - a[i * rank + k].y * c[k * n + j].y;
          acc.y += a[i * rank + k].x * c[k * n + j].y + a[i * rank + k].y * c[k * n + j].x;
        }
        h[(static_cast<size_t>(b) * m + i) * n + j] = acc;
      }
  }
  double2 *d, *U, *V;
  double* S;
  cudaMalloc(&d, h.size() * 16);
  cudaMalloc(&U, static_cast<size_t>(batch) * 64 * 64 * 16 * 2);
  cudaMalloc(&V, static_cast<size_t>(batch) * 64 * 64 * 16);
  cudaMalloc(&S, static_cast<size_t>(batch) * 64 * 8);
  cudaMemcpy(d, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  const int smem = (m * n + 2 * (m > n ? m : n) * (m < n ? m : n)) * 16;
  cudaFuncSetAttribute(k_svd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    int zero = 0;
    cudaMemcpyToSymbol(g_jacobi_sweeps, &zero, sizeof(int));
    cudaEventRecord(e0);
    k_svd<<<batch, threads, smem>>>(d, m, n, U, V, S);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int sw = 0;
    cudaMemcpyFromSymbol(&sw, g_jacobi_sweeps, sizeof(int));
    printf("m=%d n=%d batch=%d threads=%d rank=%d smem=%d: %.3f ms, sweeps/problem %.2f  err=%s\n", m, n, batch,
           threads, rank, smem, ms, double(sw) / batch, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
