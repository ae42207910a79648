// Launch-to-launch floor of dependent kernels on one stream, replayed as a CUDA graph:
// empty kernels, kernels with large dynamic shared memory, with and without programmatic
// dependent launch (PDL), 8 CTAs each (the node kernels' cfg0 grid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_latency tools/launch_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && p) p[blockIdx.x] += 1;
}

__global__ void k_smem(int* p) {
  extern __shared__ int s[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && p) p[blockIdx.x] += s[5];
}

static float run(void (*kern)(int*), size_t smem, bool pdl, int grid, int block, int* buf) {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 200;
  cudaGraph_t g;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < reps; ++i) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, buf);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphExec_t ex;
  cudaGraphInstantiate(&ex, g, 0);
  cudaGraphLaunch(ex, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  for (int i = 0; i < 5; ++i) cudaGraphLaunch(ex, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / (5 * reps);
}

int main() {
  int* buf;
  cudaMalloc(&buf, 1 << 20);
  for (int pdl = 0; pdl < 2; ++pdl) {
    printf("pdl=%d empty 8x96: %.2f us per kernel\n", pdl, run(k_empty, 0, pdl, 8, 96, buf));
    printf("pdl=%d smem 48KB 8x96: %.2f us\n", pdl, run(k_smem, 48 << 10, pdl, 8, 96, buf));
    printf("pdl=%d smem 140KB 8x96: %.2f us\n", pdl, run(k_smem, 140 << 10, pdl, 8, 96, buf));
    printf("pdl=%d smem 140KB 256x512: %.2f us\n", pdl, run(k_smem, 140 << 10, pdl, 256, 512, buf));
    printf("pdl=%d empty 148x128: %.2f us\n", pdl, run(k_empty, 0, pdl, 148, 128, buf));
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
