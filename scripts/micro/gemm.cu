// Standalone timing of the residual kernel's 2 J^T J (lower triangle) GEMM
// variants on one CTA of 256 threads (and 148 CTAs), U = 300.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NT = 256, GB = 64, GK = 32, GP = GB + 1;
__device__ __forceinline__ void gn_load(const double* J, int U, int a0, int b0, int k0, double (&pa)[8], double (&pb)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int t = threadIdx.x + NT * q;
    const int col = t / GK, kk = t - col * GK;
    const int k = k0 + kk, a = a0 + col, b = b0 + col;
    pa[q] = (k < U && a < U) ? 2.0 * J[k + (long)U * a] : 0.0;
    pb[q] = (k < U && b < U) ? J[k + (long)U * b] : 0.0;
  }
}
template <int VAR>
__global__ void k_gn(const double* Jall, double* GNall, int U, long long* cyc, int reps) {
  extern __shared__ double sm[];
  const double* J = Jall + (long)blockIdx.x * U * U;
  double* GN = GNall + (long)blockIdx.x * U * U;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int nb = (U + GB - 1) / GB, nk = (U + GK - 1) / GK;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep)
    for (int bi = 0; bi < nb; ++bi)
      for (int bj = 0; bj <= bi; ++bj) {
        const int a0 = bi * GB, b0 = bj * GB;
        double acc[4][4];
        double pa[8], pb[8];
        gn_load(J, U, a0, b0, 0, pa, pb);
        for (int c = 0; c < nk; ++c) {
          double* As = sm + (c & 1) * 2 * GK * GP;
          double* Bs = As + GK * GP;
          if (VAR != 2 || c < 2) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int t = tid + NT * q;
              const int col = t / GK, kk = t - col * GK;
              As[kk * GP + col] = pa[q];
              Bs[kk * GP + col] = pb[q];
            }
          }
          __syncthreads();
          if (c + 1 < nk && VAR != 2) gn_load(J, U, a0, b0, (c + 1) * GK, pa, pb);
          const int kc = min(GK, U - c * GK);
          int kk = 0;
          if (c == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[i][j] = As[ty + 16 * i] * Bs[tx + 16 * j];
            kk = 1;
          }
          if (kc == GK) {
#pragma unroll 8
            for (; kk < GK; ++kk) {
              double av[4], bv[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) av[i] = As[kk * GP + ty + 16 * i];
#pragma unroll
              for (int j = 0; j < 4; ++j) bv[j] = Bs[kk * GP + tx + 16 * j];
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
            }
          } else {
            for (; kk < kc; ++kk) {
              double av[4], bv[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) av[i] = As[kk * GP + ty + 16 * i];
#pragma unroll
              for (int j = 0; j < 4; ++j) bv[j] = Bs[kk * GP + tx + 16 * j];
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int a = a0 + ty + 16 * i, b = b0 + tx + 16 * j;
            if (a < U && b <= a) GN[a + (long)U * b] = 0.5 * (acc[i][j] + acc[i][j]);
          }
        __syncthreads();
      }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

__device__ __forceinline__ void cpa8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__global__ void k_gn1(const double* Jall, double* GNall, int U, long long* cyc, int reps) {
  extern __shared__ double sm[];
  const double* J = Jall + (long)blockIdx.x * U * U;
  double* GN = GNall + (long)blockIdx.x * U * U;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int nb = (U + GB - 1) / GB, nk = (U + GK - 1) / GK;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep)
    for (int bi = 0; bi < nb; ++bi)
      for (int bj = 0; bj <= bi; ++bj) {
        const int a0 = bi * GB, b0 = bj * GB;
        double acc[4][4];
        auto issue = [&](int c) {
          double* As = sm + (c & 1) * 2 * GK * GP;
          double* Bs = As + GK * GP;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int t = tid + NT * q;
            const int col = t / GK, kk = t - col * GK;
            const int k = c * GK + kk, a = a0 + col, b = b0 + col;
            if (k < U && a < U) cpa8(As + kk * GP + col, J + k + (long)U * a); else As[kk * GP + col] = 0.0;
            if (k < U && b < U) cpa8(Bs + kk * GP + col, J + k + (long)U * b); else Bs[kk * GP + col] = 0.0;
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        };
        issue(0);
        for (int c = 0; c < nk; ++c) {
          double* As = sm + (c & 1) * 2 * GK * GP;
          double* Bs = As + GK * GP;
          __syncthreads();
          if (c + 1 < nk) {
            issue(c + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int t = tid + NT * q;
            const int col = t / GK, kk = t - col * GK;
            As[kk * GP + col] = 2.0 * As[kk * GP + col];
          }
          __syncthreads();
          const int kc = min(GK, U - c * GK);
          int kk = 0;
          if (c == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[i][j] = As[ty + 16 * i] * Bs[tx + 16 * j];
            kk = 1;
          }
          if (kc == GK) {
#pragma unroll 8
            for (; kk < GK; ++kk) {
              double av[4], bv[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) av[i] = As[kk * GP + ty + 16 * i];
#pragma unroll
              for (int j = 0; j < 4; ++j) bv[j] = Bs[kk * GP + tx + 16 * j];
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
            }
          } else {
            for (; kk < kc; ++kk) {
              double av[4], bv[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) av[i] = As[kk * GP + ty + 16 * i];
#pragma unroll
              for (int j = 0; j < 4; ++j) bv[j] = Bs[kk * GP + tx + 16 * j];
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int a = a0 + ty + 16 * i, b = b0 + tx + 16 * j;
            if (a < U && b <= a) GN[a + (long)U * b] = 0.5 * (acc[i][j] + acc[i][j]);
          }
      }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

constexpr int GP2 = 2 * GB + 1;
// tiles in pairs (bi, bj) + (bi, bj+1): 4 x 8 per thread, A shared
__global__ void k_gn3(const double* Jall, double* GNall, int U, long long* cyc, int reps) {
  extern __shared__ double sm[];
  const double* J = Jall + (long)blockIdx.x * U * U;
  double* GN = GNall + (long)blockIdx.x * U * U;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int nb = (U + GB - 1) / GB, nk = (U + GK - 1) / GK;
  constexpr int BUF = GK * GP + GK * GP2;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep)
    for (int bi = 0; bi < nb; ++bi)
      for (int bj = 0; bj <= bi; bj += 2) {
        const int a0 = bi * GB, b0 = bj * GB;
        const int nbw = (bj + 1 <= bi) ? 2 * GB : GB;  // columns staged
        double acc[4][8];
        auto issue = [&](int c) {
          double* As = sm + (c & 1) * BUF;
          double* Bs = As + GK * GP;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int t = tid + NT * q;
            const int col = t / GK, kk = t - col * GK;
            const int k = c * GK + kk, a = a0 + col;
            if (k < U && a < U) cpa8(As + kk * GP + col, J + k + (long)U * a); else As[kk * GP + col] = 0.0;
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int t = tid + NT * q;
            const int col = t / GK, kk = t - col * GK;
            const int k = c * GK + kk, b = b0 + col;
            if (col < nbw) {
              if (k < U && b < U) cpa8(Bs + kk * GP2 + col, J + k + (long)U * b); else Bs[kk * GP2 + col] = 0.0;
            }
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        };
        issue(0);
        for (int c = 0; c < nk; ++c) {
          double* As = sm + (c & 1) * BUF;
          double* Bs = As + GK * GP;
          __syncthreads();
          if (c + 1 < nk) {
            issue(c + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int t = tid + NT * q;
            const int col = t / GK, kk = t - col * GK;
            As[kk * GP + col] = 2.0 * As[kk * GP + col];
          }
          __syncthreads();
          const int kc = min(GK, U - c * GK);
          int kk = 0;
          if (c == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[i][j] = As[ty + 16 * i] * Bs[tx + 16 * j];
            kk = 1;
          }
#pragma unroll 4
          for (; kk < kc; ++kk) {
            double av[4], bv[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk * GP + ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 8; ++j) bv[j] = Bs[kk * GP2 + tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int a = a0 + ty + 16 * i, b = b0 + tx + 16 * j;
            if (a < U && b <= a && (j < 4 || nbw == 2 * GB)) GN[a + (long)U * b] = 0.5 * (acc[i][j] + acc[i][j]);
          }
      }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}
int main() {
  const int U = 300, B = 148;
  double *J, *G; long long* c;
  cudaMalloc(&J, sizeof(double) * U * U * B); cudaMalloc(&G, sizeof(double) * U * U * B); cudaMalloc(&c, 8 * B);
  cudaMemset(J, 0, sizeof(double) * U * U * B);
  const int smem = 4 * GK * GP * 8;
  cudaFuncSetAttribute(k_gn<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_gn<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[B];
  cudaFuncSetAttribute(k_gn1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int nb : {1, 148}) {
    k_gn1<<<nb, NT, smem>>>(J, G, U, c, 3);
    cudaDeviceSynchronize();
    cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("var 1 (cp.async) blocks %d: %lld cycles per GN (%.1f FMA/clk/SM)\n", nb, h[0], 18.4e6 / h[0]);
  }
  const int smem3 = 2 * (GK * GP + GK * GP2) * 8;
  cudaFuncSetAttribute(k_gn3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
  for (int nb : {1, 148}) {
    k_gn3<<<nb, NT, smem3>>>(J, G, U, c, 3);
    cudaDeviceSynchronize();
    cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("var 3 (pairs, cp.async) blocks %d: %lld cycles per GN\n", nb, h[0]);
  }
  for (int var = 0; var < 3; var += 2) {
    for (int nb : {1, 148}) {
      if (var == 0) k_gn<0><<<nb, NT, smem>>>(J, G, U, c, 3); else k_gn<2><<<nb, NT, smem>>>(J, G, U, c, 3);
      cudaDeviceSynchronize();
      cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
      printf("var %d (%s) blocks %d: %lld cycles per GN (18.4M FMA -> %.1f FMA/clk/SM)\n", var,
             var == 0 ? "current" : "no global staging", nb, h[0], 18.4e6 / h[0]);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
