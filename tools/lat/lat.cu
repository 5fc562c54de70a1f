// Dev microbenchmark: dependent-chain latencies on sm_100a (cycles per op).
#include <cstdio>
__global__ void k(double* x, long long* out, int n) {
  double a = x[threadIdx.x], b = x[threadIdx.x + 32];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, 0.5);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) a = rsqrt(a + 2.0);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31);
  long long t3 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = __shfl_sync(0xffffffffu, f, (threadIdx.x + 1) & 31);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) a = a * b;
  long long t5 = clock64();
  x[threadIdx.x] = a + f;
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; }
}
int main() {
  double* x; long long* o; cudaMalloc(&x, 64 * 8); cudaMalloc(&o, 5 * 8);
  cudaMemset(x, 0, 64 * 8);
  int n = 1000;
  k<<<1, 32>>>(x, o, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(x, o, n);
  long long h[5]; cudaMemcpy(h, o, 40, cudaMemcpyDeviceToHost);
  printf("dfma %.1f rsqrt(+dadd) %.1f shfl64 %.1f shfl32 %.1f dmul %.1f cycles\n", h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
}
