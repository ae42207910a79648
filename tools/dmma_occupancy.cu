// DMMA (mma.sync m8n8k4 f64) throughput vs resident warps per SM and independent
// accumulators per warp: how many warps the many-RHS consumer needs to fill the
// FP64 tensor pipe. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_occupancy tools/dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int ACC>
__global__ void loop(double* out, int iters) {
  double d[ACC][2];
  double a = threadIdx.x * 1e-3, b = 0.5;
#pragma unroll
  for (int j = 0; j < ACC; ++j) d[j][0] = d[j][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < ACC; ++j) dmma(d[j][0], d[j][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < ACC; ++j) s += d[j][0] + d[j][1];
  if (s == 12345.0) out[0] = s;
}

template <int ACC>
void run(int sms, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w : {1, 2, 3, 4, 6, 8, 12, 16}) {
    const int iters = 4096 * 8 / ACC;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      loop<ACC><<<sms, w * 32>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double fl = 2.0 * 8 * 8 * 4 * (double)ACC * iters * w * sms;
    printf("acc %2d warps/SM %2d: %.2f TF/s\n", ACC, w, fl / (best * 1e-3) / 1e12);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  run<4>(sms, out);
  run<8>(sms, out);
  run<16>(sms, out);
  run<24>(sms, out);
  return 0;
}
