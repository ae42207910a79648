// Confirms the m8n8k4 f64 mma.sync fragment layouts used by the many-RHS DMMA consumer.
#include <cstdio>
__global__ void k(double* out) {
  int lane = threadIdx.x;
  // A[i][kk] = i*10 + kk ; B[kk][j] = (kk+1)*100 + j
  double a = (lane >> 2) * 10 + (lane & 3);          // assumed: row lane>>2, col lane&3
  double b = ((lane & 3) + 1) * 100 + (lane >> 2);    // assumed: row lane&3, col lane>>2
  double d0 = 0, d1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  out[lane * 2] = d0;
  out[lane * 2 + 1] = d1;
}
int main() {
  double* d; cudaMalloc(&d, 64 * 8);
  k<<<1, 32>>>(d);
  double h[64]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int lane = 0; lane < 32; ++lane)
    for (int q = 0; q < 2; ++q) {
      int i = lane >> 2, j = (lane & 3) * 2 + q;   // assumed C layout
      double want = 0;
      for (int kk = 0; kk < 4; ++kk) want += (i * 10 + kk) * ((kk + 1) * 100 + j);
      if (h[lane * 2 + q] != want) ++bad;
    }
  printf("dmma layout mismatches: %d\n", bad);
  return 0;
}
