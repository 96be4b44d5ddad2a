// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) probe: (1) dump D = A B + C
// for random tiles so the host can compare it bit for bit with the k-ascending
// fma chain the PBAD numeric contract needs; (2) DMMA vs DFMA throughput.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// tiles: A [T][8][4] row-major, B [T][4][8] row-major, C/D [T][8][8]
__global__ void k_tiles(const double* A, const double* B, const double* C, double* D, int T) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= T) return;
  const int g = lane >> 2, t = lane & 3;
  const double a = A[warp * 32 + g * 4 + t];
  const double b = B[warp * 32 + t * 8 + g];
  const double c0 = C[warp * 64 + g * 8 + 2 * t], c1 = C[warp * 64 + g * 8 + 2 * t + 1];
  double d0, d1;
  dmma(d0, d1, a, b, c0, c1);
  D[warp * 64 + g * 8 + 2 * t] = d0;
  D[warp * 64 + g * 8 + 2 * t + 1] = d1;
}

template <int CH>
__global__ void k_dmma_rate(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = c * 1e-3;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b, d[c][0], d[c][1]);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void k_dfma_rate(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double d[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c] = c * 1e-3;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c] = fma(a, d[c], b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c];
  if (s == 12345.678) out[0] = s;
}

static double rnd(unsigned long long& s) {
  s = s * 6364136223846793005ULL + 1442695040888963407ULL;
  const double u = ((s >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
  s = s * 6364136223846793005ULL + 1442695040888963407ULL;
  const int e = (int)((s >> 33) % 41) - 20;  // 2^-20 .. 2^20 magnitudes: cancellation + alignment
  return ldexp(u, e);
}

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 20000;
  const char* path = argc > 2 ? argv[2] : "gpurun_out/dmma_tiles.bin";
  size_t nA = (size_t)T * 32, nC = (size_t)T * 64;
  double *hA = (double*)malloc(nA * 8), *hB = (double*)malloc(nA * 8), *hC = (double*)malloc(nC * 8),
         *hD = (double*)malloc(nC * 8);
  unsigned long long s = 12345;
  for (size_t i = 0; i < nA; ++i) hA[i] = rnd(s);
  for (size_t i = 0; i < nA; ++i) hB[i] = rnd(s);
  for (size_t i = 0; i < nC; ++i) hC[i] = rnd(s);
  double *A, *B, *C, *D;
  cudaMalloc(&A, nA * 8); cudaMalloc(&B, nA * 8); cudaMalloc(&C, nC * 8); cudaMalloc(&D, nC * 8);
  cudaMemcpy(A, hA, nA * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, nA * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(C, hC, nC * 8, cudaMemcpyHostToDevice);
  k_tiles<<<(T * 32 + 127) / 128, 128>>>(A, B, C, D, T);
  cudaMemcpy(hD, D, nC * 8, cudaMemcpyDeviceToHost);
  FILE* f = fopen(path, "wb");
  fwrite(&T, 4, 1, f);
  fwrite(hA, 8, nA, f); fwrite(hB, 8, nA, f); fwrite(hC, 8, nC, f); fwrite(hD, 8, nC, f);
  fclose(f);
  // throughput
  double* o;
  cudaMalloc(&o, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int blocks_per_sm = 1; blocks_per_sm <= 4; blocks_per_sm *= 2) {
    const int grid = 148 * blocks_per_sm, tpb = 256;
    k_dmma_rate<4><<<grid, tpb>>>(o, 100);
    cudaEventRecord(e0);
    k_dmma_rate<4><<<grid, tpb>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 256 * 4 * (double)iters * (grid * tpb / 32);
    printf("DMMA m8n8k4 grid %d x %d: %.2f TFLOP/s\n", grid, tpb, flops / ms / 1e9);
    k_dfma_rate<8><<<grid, tpb>>>(o, 100);
    cudaEventRecord(e0);
    k_dfma_rate<8><<<grid, tpb>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops2 = 2.0 * 8 * (double)iters * grid * tpb;
    printf("DFMA         grid %d x %d: %.2f TFLOP/s\n", grid, tpb, flops2 / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
