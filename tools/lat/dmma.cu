// Dev microbenchmark: FP64 mma.sync m8n8k4 throughput vs DFMA on sm_100a.
#include <cstdio>
__global__ void k(double* x, long long* out, int n) {
  double a = x[threadIdx.x], b = x[threadIdx.x + 256];
  double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  double g[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) g[q] = fma(a, g[q], b);
  }
  __syncthreads();
  long long t2 = clock64();
  x[threadIdx.x] = c0 + c1 + d0 + d1 + e0 + e1 + f0 + f1 + g[0] + g[1] + g[2] + g[3] + g[4] + g[5] + g[6] + g[7];
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; }
}
int main() {
  double* x; long long* o; cudaMalloc(&x, 1024 * 8); cudaMalloc(&o, 16);
  cudaMemset(x, 0, 1024 * 8);
  int n = 1000;
  for (int w = 1; w <= 8; w *= 2) {
    k<<<1, 32 * w>>>(x, o, n); cudaDeviceSynchronize();
    k<<<1, 32 * w>>>(x, o, n);
    long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    double fma_mma = 4.0 * n * 256 * w, fma_d = 8.0 * n * 32 * w;
    printf("warps %d: DMMA %.1f FMA/clk/SM  DFMA %.1f FMA/clk/SM\n", w, fma_mma / h[0], fma_d / h[1]);
  }
}
