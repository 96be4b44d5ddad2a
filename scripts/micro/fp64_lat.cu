// Latency of dependent FP64 sqrt / div / fma / shfl chains on one warp (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0) {
  double x = x0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) x = sqrt(x) + 1.5;
  long long t1 = clock64();
  for (int i = 0; i < 256; ++i) x = 3.0 / x + 1.0;
  long long t2 = clock64();
  for (int i = 0; i < 256; ++i) x = fma(x, 0.999, 0.5);
  long long t3 = clock64();
  for (int i = 0; i < 256; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * 1.0000001;
  long long t4 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 4 * 8);
  k<<<1, 32>>>(o, c, 2.0); k<<<1, 32>>>(o, c, 2.0);
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("per op cycles: sqrt+add %.1f  div+add %.1f  fma %.1f  shfl64+mul %.1f\n", h[0] / 256.0, h[1] / 256.0, h[2] / 256.0, h[3] / 256.0);
  return 0;
}
