// pbad_chain_ops.cuh -- per-row link algebra of serial chains of
// axis-aligned hinges (identity offset rotation), shared by the chain
// kernels pbad_chain4.cu (quad per environment) and pbad_chain5.cu (warp per
// environment), plus the TMA bulk-copy / mbarrier helpers they stream link
// records with.  Every function is the reference's operation sequence for
// one row of a 4x4 transform (kinematics.cpp:20-181, adjoint.cpp:9-64);
// the dropped terms of the axis-aligned products are fma(x, +-0, acc) with
// finite x (pbad_chain.cu), so results are bit-identical to oracle/.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pbad_math.cuh"

namespace pbad_gpu {
namespace chain_ops {

// ---- TMA bulk copy + mbarrier (sm_90+ PTX; SASS UBLKCP / SYNCS) -----------
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(double* dst, const double* src, unsigned bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
// the same with an L2 evict-first policy (the copy is the data's last read)
__device__ __forceinline__ void bulk_load_ef(double* dst, const double* src, unsigned bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  long spins = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
    if (!ok && ++spins > (1L << 28)) __trap();  // a lost transfer fails the launch instead of hanging
  } while (!ok);
}

// ---- per-link joint algebra (axis-aligned hinge, identity offset rotation) --
// rotation_coeffs (kinematics.cpp:20-45) for a unit-axis angle q: s = A q, c = 1 - B q^2
__device__ __forceinline__ void hinge_cs(double q, double* c, double* s) {
  const double k2 = q * q;
  // sqrt(fl(q*q)) == |q| in binary64 round-to-nearest barring underflow of
  // q*q; an underflowed q lands in the Taylor branch where A = 1, B = 1/2
  // exactly either way, so fabs is bit-identical and saves the DP sqrt.
  const double n = isinf(k2) ? k2 : fabs(q);
  const double n2 = n * n;
  double A, B;
  if (n < 1e-4) {
    const double n4 = n2 * n2;
    A = 1.0 - n2 / 6.0 + n4 / 120.0;
    B = 0.5 - n2 / 24.0 + n4 / 720.0;
  } else {
    double sn, co;
    pbad_sincos(n, &sn, &co);
    A = sn / n;
    B = (1.0 - co) / n2;
  }
  *s = A * q;
  *c = 1.0 - B * k2;
}

// T <- T * L (row of the world transform; kinematics.cpp:171-181)
template <int JK>
__device__ __forceinline__ void fk(double c, double s, const double* t, double* T) {
  double tc = T[0] * t[0];
  tc = fma(T[1], t[1], tc);
  tc = fma(T[2], t[2], tc);
  tc = tc + T[3];
  double n0, n1, n2;
  if (JK == 1) {
    n0 = T[0];
    n1 = fma(T[2], s, T[1] * c);
    n2 = fma(T[2], c, T[1] * (-s));
  } else if (JK == 2) {
    n0 = fma(T[2], -s, T[0] * c);
    n1 = T[1];
    n2 = fma(T[2], c, T[0] * s);
  } else {
    n0 = fma(T[1], s, T[0] * c);
    n1 = fma(T[1], c, T[0] * (-s));
    n2 = T[2];
  }
  T[0] = n0;
  T[1] = n1;
  T[2] = n2;
  T[3] = tc;
}
// lever row T_parent * dL/dq: its two non-zero columns (adjoint.cpp:22-25)
template <int JK>
__device__ __forceinline__ void lever(double c, double s, const double* T, double& l0, double& l1) {
  if (JK == 1) {
    l0 = fma(T[2], c, T[1] * (-s));
    l1 = fma(T[2], -s, T[1] * (-c));
  } else if (JK == 2) {
    l0 = fma(T[2], -c, T[0] * (-s));
    l1 = fma(T[2], -s, T[0] * c);
  } else {
    l0 = fma(T[1], c, T[0] * (-s));
    l1 = fma(T[1], -s, T[0] * (-c));
  }
}
template <int JK>
__device__ __forceinline__ double lever_dot(double l0, double l1, const double* a) {
  if (JK == 1) return fma(l1, a[2], l0 * a[1]);
  if (JK == 2) return fma(l1, a[2], l0 * a[0]);
  return fma(l1, a[1], l0 * a[0]);
}
// o = a * L^T (adjoint transport to the parent, adjoint.cpp:49-64)
template <int JK>
__device__ __forceinline__ void transport(double c, double s, const double* t, const double* a, double* o) {
  if (JK == 1) {
    o[0] = fma(a[3], t[0], a[0]);
    o[1] = fma(a[3], t[1], fma(a[2], -s, a[1] * c));
    o[2] = fma(a[3], t[2], fma(a[2], c, a[1] * s));
  } else if (JK == 2) {
    o[0] = fma(a[3], t[0], fma(a[2], s, a[0] * c));
    o[1] = fma(a[3], t[1], a[1]);
    o[2] = fma(a[3], t[2], fma(a[2], c, a[0] * (-s)));
  } else {
    o[0] = fma(a[3], t[0], fma(a[1], -s, a[0] * c));
    o[1] = fma(a[3], t[1], fma(a[1], c, a[0] * s));
    o[2] = fma(a[3], t[2], a[2]);
  }
  o[3] = a[3];
}
// row of (a * S), S packed column-major
__device__ __forceinline__ void row_s(const double* a, const double* S, double* out) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double acc = a[0] * S[4 * c];
    acc = fma(a[1], S[1 + 4 * c], acc);
    acc = fma(a[2], S[2 + 4 * c], acc);
    acc = fma(a[3], S[3 + 4 * c], acc);
    out[c] = acc;
  }
}
__device__ __forceinline__ void lds16(const double* p, double* S) {
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    const double2 v = *reinterpret_cast<const double2*>(p + k);
    S[k] = v.x;
    S[k + 1] = v.y;
  }
}

}  // namespace chain_ops
}  // namespace pbad_gpu
