// Microbenchmark: FP64 peaks on B200 (DFMA pipe vs DMMA tensor path) and a
// streaming-read kernel. Used to fix the roofline denominators the apply
// chain is judged against. Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_m8n8k4_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double d[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_m16n8k16_loop(double* out, int iters) {
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 0.5 + j;
  double d[2][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(d[j][0]), "+d"(d[j][1]), "+d"(d[j][2]), "+d"(d[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int j = 0; j < 2; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void read_stream(const double2* __restrict__ in, size_t n, double* out) {
  double sx = 0, sy = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = __ldcs(in + i);
    sx += v.x; sy += v.y;
  }
  if (sx == 12345.678) out[0] = sy;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int blocks = sms * 4, threads = 256, iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  double fl = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  printf("{\"dfma_tflops\": %.2f, ", fl / ms / 1e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); dmma_m8n8k4_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  fl = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * threads / 32;
  printf("\"dmma_m8n8k4_tflops\": %.2f, ", fl / ms / 1e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); dmma_m16n8k16_loop<<<blocks, threads>>>(out, iters / 4); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  fl = 2.0 * 16 * 8 * 16 * 2 * (double)(iters / 4) * blocks * threads / 32;
  printf("\"dmma_m16n8k16_tflops\": %.2f, ", fl / ms / 1e9);
  size_t n = (size_t)1 << 29;  // 8 GiB of double2
  double2* buf; CK(cudaMalloc(&buf, n * sizeof(double2)));
  CK(cudaMemset(buf, 0, n * sizeof(double2)));
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0); read_stream<<<sms * 8, 512>>>(buf, n, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("\"read_gbs\": %.1f, ", n * sizeof(double2) / best / 1e6);
  best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0); CK(cudaMemcpyAsync(buf + n / 2, buf, n / 2 * sizeof(double2), cudaMemcpyDeviceToDevice)); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("\"copy_gbs\": %.1f, \"sms\": %d}\n", n * sizeof(double2) / best / 1e6, sms);
  return 0;
}
