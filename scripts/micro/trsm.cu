// Isolated timing of the residual kernel's TRSM step (rows below a 32x32
// diagonal block, one thread per row, row in registers) and of the warp-0
// diagonal factorisation, on one CTA of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int CB = 32, CS = 33, NT = 256;
__global__ void k_trsm(double* A, int U, long long* cyc, int reps) {
  __shared__ double Lj[CB * CS];
  for (int t = threadIdx.x; t < CB * CS; t += NT) Lj[t] = 1.0 + (t % 7) * 0.01;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    const int j0 = 0, bw = 32, j1 = 32;
    for (int i = j1 + threadIdx.x; i < U; i += NT) {
      double a[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) a[c] = c < bw ? A[i + (long)U * (j0 + c)] : 0.0;
#pragma unroll
      for (int k = 0; k < CB; ++k) {
        if (k < bw) {
          a[k] = a[k] / Lj[k * CS + k];
#pragma unroll
          for (int j = k + 1; j < CB; ++j)
            if (j < bw) a[j] = fma(-a[k], Lj[j * CS + k], a[j]);
        }
      }
#pragma unroll
      for (int c = 0; c < CB; ++c)
        if (c < bw) A[i + (long)U * (j0 + c)] = a[c];
    }
    __syncthreads();
  }
  long long t1 = clock64();
  // warp-0 diagonal factorisation in shared memory
  __shared__ double D[CB * CS];
  long long t2 = 0, t3 = 0;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    t2 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
      for (int c = 0; c <= lane; ++c) D[lane * CS + c] = (c == lane) ? 40.0 : 0.3 + 0.001 * c;
      __syncwarp();
      for (int k = 0; k < CB; ++k) {
        const double akk = D[k * CS + k];
        if (akk <= 0.0) break;
        const double d = sqrt(akk);
        if (lane > k) D[lane * CS + k] = D[lane * CS + k] / d;
        __syncwarp();
        if (lane == k) D[k * CS + k] = d;
        if (lane > k) {
          const double lik = D[lane * CS + k];
          for (int j = k + 1; j <= lane; ++j) D[lane * CS + j] = fma(-lik, D[j * CS + k], D[lane * CS + j]);
        }
        __syncwarp();
      }
    }
    t3 = clock64();
  }
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; cyc[1] = (t3 - t2) / reps; A[0] += D[5]; }
}
int main() {
  const int U = 300;
  double* A; long long* c;
  cudaMalloc(&A, sizeof(double) * U * U); cudaMalloc(&c, 16);
  cudaMemset(A, 0, sizeof(double) * U * U);
  k_trsm<<<1, NT>>>(A, U, c, 4);
  k_trsm<<<1, NT>>>(A, U, c, 20);
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("TRSM step (268 rows, 256 threads): %lld cycles; warp diag factor 32x32: %lld cycles\n", h[0], h[1]);
  k_trsm<<<148, NT>>>(A, U, c, 20);
  cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("(148 CTAs concurrently) TRSM %lld, diag %lld\n", h[0], h[1]);
  return 0;
}
