// Dependent-chain latency of DFMA, DADD, DMMA (m8n8k4 f64) and LDS.128 on one warp (clock64),
// to size ILP in latency-bound kernels. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double a, double b) {
  __shared__ double2 sm[64];
  double x = a, y = b;
  if (threadIdx.x < 64) sm[threadIdx.x] = make_double2(a, b);
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, y, a);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = x + y;
  long long t2 = clock64();
  double d0 = x, d1 = y;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  long long t3 = clock64();
  int idx = threadIdx.x & 63;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    double2 v = sm[idx];
    idx = (static_cast<int>(v.x) + idx) & 63;
  }
  long long t4 = clock64();
  out[threadIdx.x] = x + d0 + d1 + idx;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 1024;
    cyc[1] = (t2 - t1) / 1024;
    cyc[2] = (t3 - t2) / 1024;
    cyc[3] = (t4 - t3) / 1024;
  }
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 1024 * 8);
  cudaMallocManaged(&c, 64);
  lat<<<1, 32>>>(o, c, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  printf("dependent latency (cycles): DFMA %lld  DADD %lld  DMMA.8x8x4 %lld  LDS.128+IADD %lld\n", c[0], c[1], c[2], c[3]);
  return 0;
}
