// pbad_peak.cu -- FP64 microbenchmarks for the roofline denominator.
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the PBAD kernels are
// FP64 (DFMA/DMUL/DADD), so bench.py measures the sustained DFMA rate and the
// dependent-DFMA latency on the same box, with the same launch style.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace {

// 8 independent FMA chains per thread; FLOPs = 2 * 8 * iters * threads
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 123.456) out[blockIdx.x] = s;  // keep the chains alive
}

// one dependent chain, one thread: cycles per DFMA
__global__ void k_dfma_latency(double* out, long long* cycles, int iters, double a, double b) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  const long long t1 = clock64();
  out[0] = x;
  cycles[0] = t1 - t0;
}

// FP64 tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), 256 FMA per warp
// instruction; 8 independent accumulator tiles per warp
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma884(c[k][0], c[k][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 123.456) out[blockIdx.x] = s;
}

}  // namespace

// DMMA (FP64 tensor core) rate in TFLOP/s, FMA = 2 FLOPs
extern "C" int pbad_peak_dmma(int device, double* tflops, double* ms) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, device);
  double* d = nullptr;
  cudaMalloc(&d, sizeof(double) * 65536);
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 8192;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dmma_peak<<<blocks, threads>>>(d, 64, 0.999999, 1e-7);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_dmma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    if (t < best) best = t;
  }
  const double warps = (double)blocks * threads / 32.0;
  const double flops = 2.0 * 256.0 * 8.0 * (double)iters * warps;
  *tflops = flops / (best * 1e-3) / 1e12;
  *ms = best;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int pbad_peak_fp64(int device, double* tflops, double* ms, double* latency_cycles) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, device);
  double* d = nullptr;
  long long* dc = nullptr;
  cudaMalloc(&d, sizeof(double) * 65536);
  cudaMalloc(&dc, sizeof(long long));
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma_peak<<<blocks, threads>>>(d, 64, 0.999999, 1e-7);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    if (t < best) best = t;
  }
  const double flops = 2.0 * 8.0 * 16.0 * (double)iters * (double)blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  *ms = best;
  k_dfma_latency<<<1, 1>>>(d, dc, 4096, 0.999999, 1e-7);
  long long cyc = 0;
  cudaMemcpy(&cyc, dc, sizeof cyc, cudaMemcpyDeviceToHost);
  *latency_cycles = (double)cyc / (4096.0 * 16.0);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  cudaFree(dc);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
