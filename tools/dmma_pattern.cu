// DMMA issue rate of the many-RHS consumer's exact instruction pattern with operands from
// shared memory but no global traffic: the Gauss (2 x 4 tiles: 24 DMMAs per k-step, 6
// fragment loads) and 4-product forms, 8 warps per SM. Separates the tensor-pipe ceiling
// of the inner loop from the pipeline/memory effects of the real kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_pattern tools/dmma_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MT, int NT, bool GAUSS, bool SMEM>
__global__ void loop(double* out, int iters) {
  __shared__ double2 sA[16 * 36], sB[32 * 66];
  for (int i = threadIdx.x; i < 16 * 36; i += blockDim.x) sA[i] = make_double2(i * 1e-3, 1 - i * 1e-3);
  for (int i = threadIdx.x; i < 32 * 66; i += blockDim.x) sB[i] = make_double2(i * 2e-3, 0.5 - i * 1e-3);
  __syncthreads();
  const int lane = threadIdx.x & 31, lr = lane >> 2, lk = lane & 3;
  double cr[MT][NT][2] = {}, ci[MT][NT][2] = {}, cs[MT][NT][2] = {};
  for (int it = 0; it < iters; ++it) {
    const int k0 = (it & 7) * 4;
    double ar[MT], ai[MT], br[NT], bi[NT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      double2 v = SMEM ? sA[(8 * i + lr) * 36 + k0 + lk] : make_double2(it * 1e-9 + i, lk);
      ar[i] = v.x;
      ai[i] = v.y;
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      double2 v = SMEM ? sB[(k0 + lk) * 66 + 8 * j + lr] : make_double2(it * 1e-9 + j, lr);
      br[j] = v.x;
      bi[j] = v.y;
    }
    if (GAUSS) {
      double as[MT], bs[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) as[i] = ar[i] + ai[i];
#pragma unroll
      for (int j = 0; j < NT; ++j) bs[j] = br[j] + bi[j];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], ar[i], br[j]);
          dmma(ci[i][j][0], ci[i][j][1], ai[i], bi[j]);
        }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(cs[i][j][0], cs[i][j][1], as[i], bs[j]);
    } else {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], ar[i], br[j]);
          dmma(ci[i][j][0], ci[i][j][1], ar[i], bi[j]);
        }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], -ai[i], bi[j]);
          dmma(ci[i][j][0], ci[i][j][1], ai[i], br[j]);
        }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) s += cr[i][j][0] + cr[i][j][1] + ci[i][j][0] + ci[i][j][1] + cs[i][j][0];
  if (s == 12345.0) out[0] = s;
}

template <int MT, int NT, bool GAUSS, bool SMEM>
void run(const char* name, int sms, double* out, int warps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8192;
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    loop<MT, NT, GAUSS, SMEM><<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double dmmas = (GAUSS ? 3.0 : 4.0) * MT * NT * iters * warps * sms;
  const double tensor = 2.0 * 8 * 8 * 4 * dmmas;  // tensor-pipe flops
  const double alg = 8.0 * 8 * 8 * 4 * MT * NT * iters * warps * sms;  // complex-algorithmic flops
  printf("%-28s warps %2d: tensor %.2f TF/s, algorithmic %.2f TF/s\n", name, warps, tensor / (best * 1e-3) / 1e12,
         alg / (best * 1e-3) / 1e12);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int w : {4, 8}) {
    run<2, 4, true, true>("gauss 2x4 smem", sms, out, w);
    run<2, 4, true, false>("gauss 2x4 regs", sms, out, w);
    run<2, 4, false, true>("4-product 2x4 smem", sms, out, w);
    run<2, 2, true, true>("gauss 2x2 smem", sms, out, w);
    run<1, 2, true, true>("gauss 1x2 smem", sms, out, w);
  }
  return 0;
}
