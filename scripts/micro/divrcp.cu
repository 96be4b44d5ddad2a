// Is q' = fma(fma(-q, d, a), y, q), q = a * y, y = 1 / d (IEEE), equal to the
// IEEE quotient a / d for every (a, d)?  (Markstein's correction with a
// correctly rounded reciprocal.)  Counts mismatches over random operands with
// mixed exponents; prints the first few.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
__device__ __forceinline__ double rnd(unsigned long long s, int emin, int emax) {
  const unsigned long long h = mix(s);
  const double m = 1.0 + (double)(h >> 12) * (1.0 / 4503599627370496.0);  // [1, 2)
  const int e = emin + (int)((h & 0xfff) % (unsigned)(emax - emin + 1));
  return ((h >> 11) & 1 ? -1.0 : 1.0) * ldexp(m, e);
}
__global__ void k(unsigned long long base, long per, int mode, unsigned long long* bad, double* ex) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long nb = 0;
  for (long i = 0; i < per; ++i) {
    const unsigned long long s = base + (unsigned long long)(t * per + i) * 2;
    double a = rnd(s, -60, 60);
    double d = rnd(s + 1, -60, 60);
    if (mode == 1) d = sqrt(fabs(d));   // Cholesky pivots
    if (mode == 2) { a = rnd(s, -1000, 1000); d = fabs(rnd(s + 1, -1000, 1000)); }
    const double y = 1.0 / d;
    const double q = a * y;
    const double r = fma(-q, d, a);
    const double q2 = fma(r, y, q);
    const double ref = a / d;
    if (q2 != ref && !(isnan(q2) && isnan(ref))) {
      ++nb;
      if (nb == 1 && ex) { ex[2 * (t % 8)] = a; ex[2 * (t % 8) + 1] = d; }
    }
  }
  if (nb) atomicAdd(bad, nb);
}
int main() {
  unsigned long long* bad; double* ex;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&ex, 16 * 8);
  for (int mode = 0; mode < 3; ++mode) {
    *bad = 0;
    for (int k8 = 0; k8 < 16; ++k8) ex[k8] = 0;
    const int grid = 148 * 16, tpb = 256;
    const long per = 4096;
    for (int rep = 0; rep < 4; ++rep)
      k<<<grid, tpb>>>(0x1234567ULL + rep * 0x9E3779B97F4A7C15ULL + mode, per, mode, bad, ex);
    cudaDeviceSynchronize();
    printf("mode %d: %.3e samples, mismatches %llu (example a=%.17g d=%.17g)\n", mode,
           4.0 * grid * tpb * per, *bad, ex[0], ex[1]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
