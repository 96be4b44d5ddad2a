// pbad_chain5.cu -- warp-per-environment chain kernel ("v5") for serial
// chains of axis-aligned hinges (energy form, L-BFGS): the C1/C2/C3
// workloads, one PBAD step (stepper.cpp:83-147) per launch.
//
// One warp owns one environment for the whole step, so the L-BFGS solver
// (optim.cpp:141-232) runs with warp-uniform control flow and its entire
// state is resident in shared memory: the s/y history ring (2 m n doubles,
// 25.6 KB at C3), the iterate, gradient, direction, candidate and candidate
// gradient.  Only the per-link records of the reverse sweep (joint rotation,
// lever rows, inertial seed rows) leave the SM: the forward sweep writes
// them to global memory (L2-resident: a wave of ~600 environments holds
// ~13 MB) and the reverse sweep streams them back in descending 16-link
// chunks with TMA bulk copies into a 3-slot ring.
//
// Lanes inside a forward sweep (per link, l = 4 g + r, row r of a 4x4):
//   g = 0      world transform T row r (current iterate), lever row
//   g = 1, 2   history transforms A = FK(hist1), H = FK(hist0) row r
//   g = 3      gravity term cg . T
//   g = 4..6   inertial seed row g - 4: S (T - 2 A + H) / dt^2
// All lanes execute one instruction stream with lane-selected operands
// (no divergence); the rows are exchanged through a double-buffered
// shared-memory slot per link.  The reverse sweep runs the inertial and
// gravity adjoint recursions in lanes 0-3 and 4-7 (adjoint.cpp:49-64).
// Vectors are element-interleaved over the 32 lanes (element k in lane
// k % 32), which is exactly the reference's 32-partial dot order; the
// partial-sum tree is a xor butterfly (numeric contract).
//
// Every scalar keeps the reference's operation sequence (pbad_chain_ops.cuh,
// the same per-row functions as the v4 kernel), so results are
// bit-identical to oracle/ and to the reference build.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "pbad_chain_ops.cuh"
#include "pbad_kernels.cuh"
#include "pbad_launch.h"
#include "pbad_math.cuh"

namespace pbad_gpu {
namespace c5 {

using namespace chain_ops;

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_FAILED = 2 };
enum { TR_OK = 0, TR_FAIL_LIMIT = 1, TR_NONFINITE_INIT = 2, TR_NONFINITE_CFG = 3, TR_RUNNING = 4 };

constexpr int CH = 32;    // links per forward chunk (one per lane)
constexpr int RCH = 16;   // links per reverse chunk (one TMA bulk copy)
constexpr int kRing = 3;  // reverse ring slots
constexpr int kRecMass = 20;  // per-link record doubles: cs | lev[3][2] | seed[3][4] (massless links: 8)
constexpr int kMaxMem = 32;
constexpr int kHistW = 6;  // hist record per link: c0 s0 | c1 s1 | cx sx
#ifndef PBAD_C5_UNROLL
#define PBAD_C5_UNROLL 4
#endif
constexpr int kUnroll = PBAD_C5_UNROLL;  // forward links unrolled per loop trip (single-kind chains)

// per-warp shared-memory layout (doubles); n2 = n rounded up to even
struct WarpLayout {
  int x, g, d, c, e, tau, hs, hy, hsy, alpha, buf, rows, ring, scr, bar, total;
};
__host__ __device__ inline WarpLayout warp_layout(int n, int mem) {
  WarpLayout w;
  const int n2 = (n + 1) & ~1, m = mem > 0 ? mem : 1;
  int o = 0;
  auto take = [&](int cnt) {
    const int at = o;
    o += (cnt + 1) & ~1;  // 16-byte alignment
    return at;
  };
  w.x = take(n2);
  w.g = take(n2);
  w.d = take(n2);
  w.c = take(n2);
  w.e = take(n2);
  w.tau = take(n2);
  w.hs = take(m * n2);
  w.hy = take(m * n2);
  w.hsy = take(m);
  w.alpha = take(m);
  w.buf = take(CH * 6);
  w.rows = take(2 * 12 * 4);
  w.ring = take(kRing * RCH * kRecMass);
  w.scr = take(16);
  w.bar = take(kRing);
  w.total = o;
  return w;
}
__host__ __device__ inline size_t block_smem_bytes(int N, int n, int mem, int warps) {
  return (size_t)(20L * N + (long)warps * warp_layout(n, mem).total) * sizeof(double) +
         (size_t)(2 * N + 1) * sizeof(int);
}

// ---- warp context -------------------------------------------------------------
struct W {
  int N, n, mem, lane, g, r;
  long e, B;
  const double* mrec;  // shared model records [N][20]: S (16), offset translation (3)
  const int* kind;     // shared link classes (jk | sk << 2)
  const int* roff;     // shared per-env record offsets [N+1]
  double* s;           // this warp's shared area
  WarpLayout L;
  uint64_t* bar;
  double* rec;         // this env's link records (global)
  double* hist;        // this env's history rotations [N][6] (global)
  double *gh0, *gh1;   // hist0 / hist1 in the chain layout (quad-interleaved, global)
  double* histc;
  int* ci;
  long n4;
  double dt, inv_dt2, wm, gr;
  double gz[3];
  DOpt o;
  unsigned nload;      // reverse chunks consumed (ring slot and phase)
};

__device__ __forceinline__ int& ival(const W& w, int slot) { return w.ci[(long)slot * w.B + w.e]; }
// element k of this env in a quad-interleaved chain-layout vector (pbad_chain.cu)
__device__ __forceinline__ double& qv(const W& w, double* base, int k) {
  return base[((w.e >> 3) * w.n4 + (k >> 2)) * 32 + (w.e & 7) * 4 + (k & 3)];
}

// ---- 32-lane vector ops (canonical 32-partial order) --------------------------
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}
__device__ __forceinline__ double vdot(const W& w, const double* a, const double* b) {
  double acc = 0.0;
  for (int k = w.lane; k < w.n; k += 32) acc = fma(a[k], b[k], acc);
  return wsum(acc);
}
__device__ __forceinline__ double vinf(const W& w, const double* a) {
  double m = 0.0;
  for (int k = w.lane; k < w.n; k += 32) m = fmax(m, fabs(a[k]));
  return wmax(m);
}
__device__ __forceinline__ bool vfinite(const W& w, const double* a) {
  bool ok = true;
  for (int k = w.lane; k < w.n; k += 32) ok = ok && isfinite(a[k]);
  return __all_sync(0xffffffffu, ok);
}
__device__ __forceinline__ bool qfinite(const W& w, double* base) {
  bool ok = true;
  for (int k = w.lane; k < w.n; k += 32) ok = ok && isfinite(qv(w, base, k));
  return __all_sync(0xffffffffu, ok);
}

// ---- forward sweep ---------------------------------------------------------------
// StepObjective::value at X (objective.cpp:215-239), writing the reverse
// sweep's per-link records.
template <int CK>
__device__ __forceinline__ void fwd_link(const W& w, int j, int i, double* R, double& sum, int par) {
  constexpr int JK = CK & 3;
  constexpr bool SK = (CK >> 2) != 0;
  const int l = w.lane;
  // this lane's chain: T (current), A (hist1), H (hist0); other lanes follow T
  const int co = (w.g == 1) ? 4 : (w.g == 2) ? 2 : 0;
  const double2 cs = *reinterpret_cast<const double2*>(w.s + w.L.buf + j * 6 + co);
  const double* mr = w.mrec + 20 * i;
  const double2 t01 = *reinterpret_cast<const double2*>(mr + 16);
  const double t[3] = {t01.x, t01.y, mr[18]};
  double* rp = w.rec + w.roff[i];
  double l0, l1;
  lever<JK>(cs.x, cs.y, R, l0, l1);  // T_parent row times dL/dq (adjoint.cpp:22-25)
  if (l < 3) *reinterpret_cast<double2*>(rp + 2 + 2 * l) = make_double2(l0, l1);
  fk<JK>(cs.x, cs.y, t, R);
  if (SK) {
    double* rows = w.s + w.L.rows + par * 48;
    if (l < 12) {
      *reinterpret_cast<double2*>(rows + 4 * l) = make_double2(R[0], R[1]);
      *reinterpret_cast<double2*>(rows + 4 * l + 2) = make_double2(R[2], R[3]);
    }
    __syncwarp();
    const int sel = (l < 16) ? w.r : (l < 28 ? w.g - 4 : 3);
    double Tr[4], Ar[4], Hr[4];
    {
      const double2 a = *reinterpret_cast<const double2*>(rows + 4 * sel);
      const double2 b = *reinterpret_cast<const double2*>(rows + 4 * sel + 2);
      const double2 c = *reinterpret_cast<const double2*>(rows + 16 + 4 * sel);
      const double2 d = *reinterpret_cast<const double2*>(rows + 16 + 4 * sel + 2);
      const double2 e = *reinterpret_cast<const double2*>(rows + 32 + 4 * sel);
      const double2 f = *reinterpret_cast<const double2*>(rows + 32 + 4 * sel + 2);
      Tr[0] = a.x; Tr[1] = a.y; Tr[2] = b.x; Tr[3] = b.y;
      Ar[0] = c.x; Ar[1] = c.y; Ar[2] = d.x; Ar[3] = d.y;
      Hr[0] = e.x; Hr[1] = e.y; Hr[2] = f.x; Hr[3] = f.y;
    }
    double S[16];
    lds16(mr, S);
    // seed lanes: dd = (T - 2A + H) / dt^2 of row sel
    double in[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double dd = Tr[k] - 2.0 * Ar[k];
      dd = dd + Hr[k];
      dd = w.inv_dt2 * dd;
      in[k] = (l < 12) ? R[k] : dd;
    }
    double P[4];
    row_s(in, S, P);
    if (w.g == 3) {
#pragma unroll
      for (int k = 0; k < 4; ++k) P[k] = (-w.gr) * S[12 + k];
    }
    const double ev = ddot_row(P, Tr);
    // term g of this link: ((row0 + row1) + row2) + row3, added in link order
    const double e1 = __shfl_down_sync(0xffffffffu, ev, 1);
    const double e2 = __shfl_down_sync(0xffffffffu, ev, 2);
    const double e3 = __shfl_down_sync(0xffffffffu, ev, 3);
    sum += ((ev + e1) + e2) + e3;  // meaningful in lanes 0, 4, 8, 12
    if (l >= 16 && l < 28 && w.r == 0) {
      double* sp = rp + 8 + 4 * (w.g - 4);
      *reinterpret_cast<double2*>(sp) = make_double2(P[0], P[1]);
      *reinterpret_cast<double2*>(sp + 2) = make_double2(P[2], P[3]);
    }
  }
}

__device__ __forceinline__ void fwd_link_dyn(const W& w, int j, int i, double* R, double& sum, int par) {
  switch (w.kind[i]) {
    case 1: fwd_link<1>(w, j, i, R, sum, par); break;
    case 2: fwd_link<2>(w, j, i, R, sum, par); break;
    case 3: fwd_link<3>(w, j, i, R, sum, par); break;
    case 5: fwd_link<5>(w, j, i, R, sum, par); break;
    case 6: fwd_link<6>(w, j, i, R, sum, par); break;
    default: fwd_link<7>(w, j, i, R, sum, par); break;
  }
}

// link-pattern code: P | K0 << 2 | K1 << 5 (P = period 1 or 2; 0 = per-link dispatch)
template <int PAT>
__device__ __forceinline__ void fwd_any(const W& w, int j, int i, double* R, double& sum, int par) {
  constexpr int P = PAT & 3, K0 = (PAT >> 2) & 7, K1 = (PAT >> 5) & 7;
  if constexpr (P == 1) {
    fwd_link<K0>(w, j, i, R, sum, par);
  } else if constexpr (P == 2) {
    if (i & 1) fwd_link<K1>(w, j, i, R, sum, par);
    else fwd_link<K0>(w, j, i, R, sum, par);
  } else {
    fwd_link_dyn(w, j, i, R, sum, par);
  }
}

template <int PAT>
__device__ double forward(W& w, const double* X, double tdx) {
  const int N = w.N, l = w.lane;
  double R[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) R[k] = (w.r == k) ? 1.0 : 0.0;
  double sum = 0.0;
  double4 hn = make_double4(0.0, 0.0, 0.0, 0.0);
  if (l < N) {
    const double* hp = w.hist + (long)l * kHistW;
    const double2 a = *reinterpret_cast<const double2*>(hp);
    const double2 b = *reinterpret_cast<const double2*>(hp + 2);
    hn = make_double4(a.x, a.y, b.x, b.y);
  }
  int par = 0;
  for (int lo = 0; lo < N; lo += CH) {
    const int cnt = min(CH, N - lo), i = lo + l;
    const double4 hc = hn;
    double c = 1.0, s = 0.0;
    if (i < N) hinge_cs(X[i], &c, &s);
    if (lo + CH + l < N) {  // next chunk's history rotations
      const double* hp = w.hist + (long)(lo + CH + l) * kHistW;
      const double2 a = *reinterpret_cast<const double2*>(hp);
      const double2 b = *reinterpret_cast<const double2*>(hp + 2);
      hn = make_double4(a.x, a.y, b.x, b.y);
    }
    __syncwarp();  // the previous chunk's readers are done with the buffer
    if (i < N) {
      double* b = w.s + w.L.buf + l * 6;
      *reinterpret_cast<double2*>(b) = make_double2(c, s);
      *reinterpret_cast<double2*>(b + 2) = make_double2(hc.x, hc.y);
      *reinterpret_cast<double2*>(b + 4) = make_double2(hc.z, hc.w);
      *reinterpret_cast<double2*>(w.rec + w.roff[i]) = make_double2(c, s);
    }
    __syncwarp();
    if constexpr ((PAT & 3) == 1) {
      // one link kind: the massive flag is a compile-time constant; unrolled so
      // consecutive links' independent work can overlap
      constexpr int PK = ((PAT >> 2) & 7) >> 2;
#pragma unroll kUnroll
      for (int j = 0; j < cnt; ++j) {
        fwd_any<PAT>(w, j, lo + j, R, sum, par);
        par ^= PK;
      }
    } else {
      for (int j = 0; j < cnt; ++j) {
        fwd_any<PAT>(w, j, lo + j, R, sum, par);
        par ^= (w.kind[lo + j] >> 2);
      }
    }
  }
  const double sa = __shfl_sync(0xffffffffu, sum, 0), sb = __shfl_sync(0xffffffffu, sum, 4);
  const double sc = __shfl_sync(0xffffffffu, sum, 8), sg = __shfl_sync(0xffffffffu, sum, 12);
  const double wm = w.wm;
  const double cpp = sa - wm, c1p = sb - wm, c2p = sc - wm;
  const double inertial = 0.5 * w.inv_dt2 * (cpp - 4.0 * c1p + 2.0 * c2p + *w.histc);
  return inertial + sg - tdx;
}

// ---- reverse sweep ---------------------------------------------------------------
// functional_grad twice (adjoint.cpp:49-64): gradient = inertial adjoint +
// gravity adjoint - tau (objective.cpp:241-250) into G.
template <int CK>
__device__ __forceinline__ void rev_link(const W& w, const double* rp, int i, double* c, double* G) {
  constexpr int JK = CK & 3;
  constexpr bool SK = (CK >> 2) != 0;
  const double2 cs = *reinterpret_cast<const double2*>(rp);
  const bool own = w.r < 3;  // row 3 of the lever and of the seed is exactly zero
  double l0 = 0.0, l1 = 0.0;
  if (own) {
    const double2 lv = *reinterpret_cast<const double2*>(rp + 2 + 2 * w.r);
    l0 = lv.x;
    l1 = lv.y;
  }
  const double* mr = w.mrec + 20 * i;
  double a[4];
  if (SK) {
    // inertial lanes: the seed row from the record; gravity lanes: the
    // gravity cotangent row (0 + (-g_r) S[12..15])
    double sd[4] = {0.0, 0.0, 0.0, 0.0};
    if (own && w.g == 0) {
      const double2 s01 = *reinterpret_cast<const double2*>(rp + 8 + 4 * w.r);
      const double2 s23 = *reinterpret_cast<const double2*>(rp + 8 + 4 * w.r + 2);
      sd[0] = s01.x;
      sd[1] = s01.y;
      sd[2] = s23.x;
      sd[3] = s23.y;
    }
    const double2 u01 = *reinterpret_cast<const double2*>(mr + 12);
    const double2 u23 = *reinterpret_cast<const double2*>(mr + 14);
    const double u[4] = {u01.x, u01.y, u23.x, u23.y};
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = c[k] + ((w.g == 0) ? sd[k] : (0.0 + (-w.gr) * u[k]));
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = c[k];
  }
  const double p = lever_dot<JK>(l0, l1, a);
  const double p1 = __shfl_down_sync(0xffffffffu, p, 1);
  const double p2 = __shfl_down_sync(0xffffffffu, p, 2);
  const double p3 = __shfl_down_sync(0xffffffffu, p, 3);
  const double gsum = 0.0 + (((p + p1) + p2) + p3);  // lane 0: inertial, lane 4: gravity
  const double gp = __shfl_sync(0xffffffffu, gsum, 4);
  if (w.lane == 0) G[i] = (gsum + gp) - w.s[w.L.tau + i];
  if (i > 0) {
    const double2 t01 = *reinterpret_cast<const double2*>(mr + 16);
    const double t[3] = {t01.x, t01.y, mr[18]};
    double o[4];
    transport<JK>(cs.x, cs.y, t, a, o);
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = 0.0 + o[k];
  }
}

__device__ __forceinline__ void rev_link_dyn(const W& w, const double* rp, int i, double* c, double* G) {
  switch (w.kind[i]) {
    case 1: rev_link<1>(w, rp, i, c, G); break;
    case 2: rev_link<2>(w, rp, i, c, G); break;
    case 3: rev_link<3>(w, rp, i, c, G); break;
    case 5: rev_link<5>(w, rp, i, c, G); break;
    case 6: rev_link<6>(w, rp, i, c, G); break;
    default: rev_link<7>(w, rp, i, c, G); break;
  }
}

template <int PAT>
__device__ __forceinline__ void rev_any(const W& w, const double* rp, int i, double* c, double* G) {
  constexpr int P = PAT & 3, K0 = (PAT >> 2) & 7, K1 = (PAT >> 5) & 7;
  if constexpr (P == 1) {
    rev_link<K0>(w, rp, i, c, G);
  } else if constexpr (P == 2) {
    if (i & 1) rev_link<K1>(w, rp, i, c, G);
    else rev_link<K0>(w, rp, i, c, G);
  } else {
    rev_link_dyn(w, rp, i, c, G);
  }
}

__device__ __forceinline__ void issue_chunk(W& w, int ch, unsigned k) {
  const int lo = RCH * ch, hi = min(w.N, lo + RCH);
  const int slot = (int)(k % kRing);
  const unsigned bytes = (unsigned)(w.roff[hi] - w.roff[lo]) * 8u;
  bulk_load(w.s + w.L.ring + slot * RCH * kRecMass, w.rec + w.roff[lo], bytes, w.bar + slot);
}

template <int PAT>
__device__ void reverse(W& w, double* G) {
  const int N = w.N, nch = (N + RCH - 1) / RCH;
  fence_async_global();  // this lane's record stores -> the bulk copies below
  __syncwarp();
  const unsigned k0 = w.nload;
  if (w.lane == 0) {
    fence_async_smem();  // previous readers of the ring before the async writes
    for (int p = 0; p < kRing && p < nch; ++p) issue_chunk(w, nch - 1 - p, k0 + p);
  }
  double c[4] = {0.0, 0.0, 0.0, 0.0};
  for (int idx = 0; idx < nch; ++idx) {
    const int ch = nch - 1 - idx;
    const int lo = RCH * ch, cnt = min(RCH, N - lo);
    const unsigned k = k0 + idx;
    const int slot = (int)(k % kRing);
    mbar_wait(w.bar + slot, (k / kRing) & 1u);
    const double* base = w.s + w.L.ring + slot * RCH * kRecMass - w.roff[lo];
    for (int j = cnt - 1; j >= 0; --j) rev_any<PAT>(w, base + w.roff[lo + j], lo + j, c, G);
    __syncwarp();
    if (idx + kRing < nch && w.lane == 0) {
      fence_async_smem();
      issue_chunk(w, ch - kRing, k + kRing);
    }
  }
  w.nload = k0 + nch;
  __syncwarp();
}

// ---- per-step passes (once per PBAD step) ----------------------------------------
// joint rotations of V into hist slot `slot` (0: hist0, 1: hist1, 2: x)
__device__ __forceinline__ void hist_rotations_q(const W& w, double* base, int slot) {
  for (int i = w.lane; i < w.N; i += 32) {
    double c, s;
    hinge_cs(qv(w, base, i), &c, &s);
    *reinterpret_cast<double2*>(w.hist + (long)i * kHistW + 2 * slot) = make_double2(c, s);
  }
  __syncwarp();
}
__device__ __forceinline__ void hist_rotations_s(const W& w, const double* V, int slot) {
  for (int i = w.lane; i < w.N; i += 32) {
    double c, s;
    hinge_cs(V[i], &c, &s);
    *reinterpret_cast<double2*>(w.hist + (long)i * kHistW + 2 * slot) = make_double2(c, s);
  }
  __syncwarp();
}

__device__ __forceinline__ void fk_dyn(int jk, double c, double s, const double* t, double* T) {
  if (jk == 1) fk<1>(c, s, t, T);
  else if (jk == 2) fk<2>(c, s, t, T);
  else fk<3>(c, s, t, T);
}
// ((v_0 + v_1) + v_2) + v_3 over the quad (every quad computes the same rows)
__device__ __forceinline__ double quad_rows(double v) {
  const double v0 = __shfl_sync(0xffffffffu, v, 0, 4), v1 = __shfl_sync(0xffffffffu, v, 1, 4);
  const double v2 = __shfl_sync(0xffffffffu, v, 2, 4), v3 = __shfl_sync(0xffffffffu, v, 3, 4);
  return ((v0 + v1) + v2) + v3;
}

// hist_const = 4 cv(tk, tk) + cv(tk1, tk1) - 4 cv(tk, tk1) (objective.cpp:162-185),
// tk = FK(hist1), tk1 = FK(hist0); massless links add exact zeros and are skipped
__device__ double hist_const(const W& w) {
  double A[4], H[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) A[k] = H[k] = (w.r == k) ? 1.0 : 0.0;
  double vAA = 0.0, vHH = 0.0, vAH = 0.0;
  for (int i = 0; i < w.N; ++i) {
    const int ck = w.kind[i];
    const double* hp = w.hist + (long)i * kHistW;
    const double* mr = w.mrec + 20 * i;
    const double t[3] = {mr[16], mr[17], mr[18]};
    fk_dyn(ck & 3, hp[2], hp[3], t, A);
    fk_dyn(ck & 3, hp[0], hp[1], t, H);
    if (ck >> 2) {
      double S[16], as[4], hs[4];
      lds16(mr, S);
      row_s(A, S, as);
      row_s(H, S, hs);
      vAA += quad_rows(ddot_row(as, A));
      vHH += quad_rows(ddot_row(hs, H));
      vAH += quad_rows(ddot_row(as, H));
    }
  }
  return 4.0 * (vAA - w.wm) + (vHH - w.wm) - 4.0 * (vAH - w.wm);
}

// fd_kinetic (stepper.cpp:14-22) + gravity_potential (baseline.cpp:219-229)
// between FK(hist slot 1) and FK(hist slot 2)
__device__ void step_energy(const W& w, double* ke, double* pe) {
  double P[4], Q[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) P[k] = Q[k] = (w.r == k) ? 1.0 : 0.0;
  double kk = 0.0, pp = 0.0;
  const double ghat[4] = {w.gz[0], w.gz[1], w.gz[2], 0.0};
  for (int i = 0; i < w.N; ++i) {
    const int ck = w.kind[i];
    const double* hp = w.hist + (long)i * kHistW;
    const double* mr = w.mrec + 20 * i;
    const double t[3] = {mr[16], mr[17], mr[18]};
    fk_dyn(ck & 3, hp[2], hp[3], t, P);
    fk_dyn(ck & 3, hp[4], hp[5], t, Q);
    if (ck >> 2) {
      double S[16], td[4], tds[4];
      lds16(mr, S);
#pragma unroll
      for (int c = 0; c < 4; ++c) td[c] = (Q[c] - P[c]) / w.dt;
      row_s(td, S, tds);
      double wu = Q[0] * S[12];
      wu = fma(Q[1], S[13], wu);
      wu = fma(Q[2], S[14], wu);
      wu = fma(Q[3], S[15], wu);
      const double term = quad_rows(ddot_row(tds, td));
      const double u0 = __shfl_sync(0xffffffffu, wu, 0, 4), u1 = __shfl_sync(0xffffffffu, wu, 1, 4);
      const double u2 = __shfl_sync(0xffffffffu, wu, 2, 4), u3 = __shfl_sync(0xffffffffu, wu, 3, 4);
      double d = ghat[0] * u0;
      d = fma(ghat[1], u1, d);
      d = fma(ghat[2], u2, d);
      d = fma(ghat[3], u3, d);
      kk += 0.5 * term;
      pp -= d;
    }
  }
  *ke = kk;
  *pe = pp;
}

// ForceModel::tau_at (objective.hpp:28-58) into the shared tau vector
__device__ void tau_at(const W& w, const DForces& f, double t) {
  const int n = w.n;
  double* tau = w.s + w.L.tau;
  for (int i = w.lane; i < n; i += 32) {
    double v;
    if (f.has_act && f.act_len == n) {
      if (f.act_kind == 0) {
        v = f.act_amp[i];
      } else {
        const double ph = i < f.act_phase_len ? f.act_phase[i] : 0.0;
        double s, c;
        pbad_sincos(2.0 * 3.141592653589793 * f.act_freq * t + ph, &s, &c);
        v = f.act_amp[i] * s;
      }
    } else if (f.tau_len == n) {
      v = f.tau[i];
    } else {
      v = 0.0;
    }
    tau[i] = v;
  }
  __syncwarp();
}

// ---- L-BFGS (LbfgsSolver, optim.cpp:141-232) --------------------------------------
struct Solver {
  double value, grad0, ginf, xinf;
  int status, iters, stag, acc, h0, hc;
};

__device__ __forceinline__ double* hist_s(const W& w, const Solver& s, int i) {
  return w.s + w.L.hs + ((s.h0 + i) % w.mem) * ((w.n + 1) & ~1);
}
__device__ __forceinline__ double* hist_y(const W& w, const Solver& s, int i) {
  return w.s + w.L.hy + ((s.h0 + i) % w.mem) * ((w.n + 1) & ~1);
}
__device__ __forceinline__ double hist_sy(const W& w, const Solver& s, int i) {
  return w.s[w.L.hsy + (s.h0 + i) % w.mem];
}

// dir = -two_loop(g) (optim.cpp:213-229); returns dir . g
__device__ double direction(const W& w, const Solver& s) {
  double* q = w.s + w.L.d;
  const double* g = w.s + w.L.g;
  double* alpha = w.s + w.L.alpha;
  const int n = w.n, hc = s.hc;
  for (int k = w.lane; k < n; k += 32) q[k] = g[k];
  __syncwarp();
  for (int i = hc - 1; i >= 0; --i) {
    const double* sv = hist_s(w, s, i);
    const double* yv = hist_y(w, s, i);
    const double a = vdot(w, sv, q) / hist_sy(w, s, i);
    if (w.lane == 0) alpha[i] = a;
    for (int k = w.lane; k < n; k += 32) q[k] = q[k] - a * yv[k];
    __syncwarp();
  }
  if (hc > 0) {
    const double* yl = hist_y(w, s, hc - 1);
    const double scl = hist_sy(w, s, hc - 1) / vdot(w, yl, yl);
    for (int k = w.lane; k < n; k += 32) q[k] = q[k] * scl;
    __syncwarp();
  }
  for (int i = 0; i < hc; ++i) {
    const double* sv = hist_s(w, s, i);
    const double* yv = hist_y(w, s, i);
    const double beta = vdot(w, yv, q) / hist_sy(w, s, i);
    const double cc = alpha[i] - beta;
    for (int k = w.lane; k < n; k += 32) q[k] = q[k] + cc * sv[k];
    __syncwarp();
  }
  double acc = 0.0;
  for (int k = w.lane; k < n; k += 32) {
    const double d = -q[k];
    q[k] = d;
    acc = fma(d, g[k], acc);
  }
  __syncwarp();
  return wsum(acc);
}

__device__ __forceinline__ double steepest(const W& w) {
  double* d = w.s + w.L.d;
  const double* g = w.s + w.L.g;
  double acc = 0.0;
  for (int k = w.lane; k < w.n; k += 32) {
    const double v = -g[k];
    d[k] = v;
    acc = fma(v, g[k], acc);
  }
  __syncwarp();
  return wsum(acc);
}

// candidate x + t dir; returns all-finite, tau . cand in *tdx
__device__ __forceinline__ bool candidate(const W& w, double t, double* tdx) {
  const double *x = w.s + w.L.x, *d = w.s + w.L.d, *tau = w.s + w.L.tau;
  double* c = w.s + w.L.c;
  double acc = 0.0;
  bool fin = true;
  for (int k = w.lane; k < w.n; k += 32) {
    const double cv = x[k] + t * d[k];
    c[k] = cv;
    fin = fin && isfinite(cv);
    acc = fma(tau[k], cv, acc);
  }
  __syncwarp();
  *tdx = wsum(acc);
  return __all_sync(0xffffffffu, fin);
}

// accepted step (optim.cpp:176-205): s = t dir, y = evg - g, push if
// s.y > 1e-12 (dropping the oldest pair beyond m), x = cand, g = evg
__device__ void accept_step(const W& w, Solver& s, double t, double v, double fval) {
  const int n = w.n, n2 = (n + 1) & ~1;
  double *x = w.s + w.L.x, *g = w.s + w.L.g;
  const double *d = w.s + w.L.d, *c = w.s + w.L.c, *e = w.s + w.L.e;
  double acc = 0.0;
  for (int k = w.lane; k < n; k += 32) acc = fma(t * d[k], e[k] - g[k], acc);
  const double sy = wsum(acc);
  const bool push = sy > 1e-12 && w.mem > 0;
  int slot = 0;
  if (push) {
    if (s.hc < w.mem) {
      slot = (s.h0 + s.hc) % w.mem;
      ++s.hc;
    } else {  // the deque pops its front: the new pair takes the oldest slot
      slot = s.h0;
      s.h0 = (s.h0 + 1) % w.mem;
    }
  }
  double* sv = w.s + w.L.hs + slot * n2;
  double* yv = w.s + w.L.hy + slot * n2;
  double gm = 0.0, xm = 0.0;
  for (int k = w.lane; k < n; k += 32) {
    const double ek = e[k], ck = c[k];
    if (push) {
      sv[k] = t * d[k];
      yv[k] = ek - g[k];
    }
    x[k] = ck;
    g[k] = ek;
    gm = fmax(gm, fabs(ek));
    xm = fmax(xm, fabs(ck));
  }
  if (push && w.lane == 0) w.s[w.L.hsy + slot] = sy;
  __syncwarp();
  s.ginf = wmax(gm);
  s.xinf = wmax(xm);
  s.value = v;
  ++s.acc;
  if (fval - v <= w.o.ftol * fmax(1.0, fabs(fval))) ++s.stag;
  else s.stag = 0;
  if (s.stag >= 2) s.status = ST_CONVERGED;
}

__device__ __forceinline__ void stage(const DModel& m, double* smem) {
  double* rec = smem;
  int* kind = reinterpret_cast<int*>(rec + 20L * m.N);
  int* roff = kind + m.N;
  const double2* src = reinterpret_cast<const double2*>(m.crec);
  double2* dst = reinterpret_cast<double2*>(rec);
  for (int k = threadIdx.x; k < 10 * m.N; k += blockDim.x) dst[k] = __ldg(src + k);
  for (int k = threadIdx.x; k < m.N; k += blockDim.x) kind[k] = __ldg(m.ckind + k);
  // per-environment record offsets (the v4 offsets are per 8-environment warp)
  for (int k = threadIdx.x; k <= m.N; k += blockDim.x) roff[k] = __ldg(m.croff + k) / 8;
  __syncthreads();
}

// One PBAD step for this warp's environment: begin_step, L-BFGS to
// completion, finish_step (stepper.cpp:83-147).
template <int PAT>
__global__ void __launch_bounds__(256, 1) k_chain5_step(DModel m, DForces f, DSchedule sc, ChainLayout CL, double* cw,
                                                     int* ci, long B, long recw, Outputs out) {
  extern __shared__ __align__(16) double smem[];
  stage(m, smem);
  W w;
  w.N = m.N;
  w.n = m.n;
  w.mem = sc.opt.mem;
  w.lane = threadIdx.x & 31;
  w.g = w.lane >> 2;
  w.r = w.lane & 3;
  w.e = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  w.B = B;
  if (w.e >= B) return;
  w.mrec = smem;
  w.kind = reinterpret_cast<const int*>(smem + 20L * m.N);
  w.roff = w.kind + m.N;
  w.L = warp_layout(m.n, sc.opt.mem);
  const size_t mbytes = (20L * m.N) * sizeof(double) + (2 * m.N + 1) * sizeof(int);
  w.s = smem + (mbytes + 15) / 16 * 2 + (long)(threadIdx.x >> 5) * w.L.total;
  w.bar = reinterpret_cast<uint64_t*>(w.s + w.L.bar);
  w.rec = cw + CL.rec + w.e * recw;
  w.hist = cw + CL.hist + w.e * (long)m.N * kHistW;
  w.n4 = (m.n + 3) >> 2;
  w.gh0 = cw + CL.h0;
  w.gh1 = cw + CL.h1;
  w.histc = cw + CL.histc + w.e;
  w.ci = ci;
  w.dt = sc.dt;
  w.inv_dt2 = 1.0 / (sc.dt * sc.dt);
  w.wm = m.weighted_mass;
  w.gz[0] = f.gravity[0];
  w.gz[1] = f.gravity[1];
  w.gz[2] = f.gravity[2];
  w.gr = (w.r == 0) ? f.gravity[0] : (w.r == 1) ? f.gravity[1] : (w.r == 2) ? f.gravity[2] : 0.0;
  w.o = sc.opt;
  w.nload = 0;
  if (w.lane == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(w.bar + s);
    fence_mbar_init();
  }
  __syncwarp();
  if (ival(w, IS_RUN) != TR_RUNNING) return;
  const int n = m.n;
  const int step = ival(w, IS_STEP);
  // StepObjective ctor validates the history (objective.cpp:176-177)
  if (!qfinite(w, w.gh0) || !qfinite(w, w.gh1)) {
    if (w.lane == 0) ival(w, IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  double* x = w.s + w.L.x;
  double* g = w.s + w.L.g;
  // begin_step: actuation at the step end, warm start (stepper.cpp:83-115)
  tau_at(w, f, step * sc.dt + sc.times[2] * sc.dt);
  {
    const double span = -sc.times[0];
    const double tau_m = sc.times[2];
    const bool ws = sc.warm_start != 0;
    for (int k = w.lane; k < n; k += 32) {
      const double h1 = qv(w, w.gh1, k), h0 = qv(w, w.gh0, k);
      x[k] = ws ? h1 + (tau_m / span) * (h1 - h0) : h1;
    }
  }
  hist_rotations_q(w, w.gh0, 0);
  hist_rotations_q(w, w.gh1, 1);
  const double hc = hist_const(w);
  if (w.lane == 0) *w.histc = hc;
  __syncwarp();
  if (!vfinite(w, x)) {
    if (w.lane == 0) ival(w, IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  // LbfgsSolver ctor: first evaluation (optim.cpp:143-150)
  Solver s{};
  s.status = ST_RUNNING;
  double* itv = out.itv ? out.itv + out.rrow(w.e, step) * out.itv_n : nullptr;
  {
    const double tdx0 = vdot(w, w.s + w.L.tau, x);
    s.xinf = vinf(w, x);
    const double v0 = forward<PAT>(w, x, tdx0);
    reverse<PAT>(w, g);
    if (!isfinite(v0)) {
      if (w.lane == 0) ival(w, IS_RUN) = TR_NONFINITE_INIT;
      return;
    }
    s.value = v0;
    s.grad0 = vinf(w, g);
    s.ginf = s.grad0;
  }
  for (;;) {
    // LbfgsSolver::iterate (optim.cpp:152-205)
    if (s.iters >= w.o.max_iters) {
      s.status = ST_FAILED;
      break;
    }
    if (s.ginf <= w.o.grad_tol * fmax(1.0, s.xinf) || (w.o.grad_rtol > 0.0 && s.ginf <= w.o.grad_rtol * s.grad0)) {
      s.status = ST_CONVERGED;
      break;
    }
    double slope = direction(w, s);
    if (!(slope < 0.0)) {
      s.hc = 0;
      s.h0 = 0;
      slope = steepest(w);
    }
    const double fval = s.value;
    double t = 1.0;
    bool accepted = false;
    for (int trial = 0; trial < w.o.max_line_search; ++trial) {
      double tdx;
      if (candidate(w, t, &tdx)) {
        const double v = forward<PAT>(w, w.s + w.L.c, tdx);
        if (isfinite(v) && v <= fval + w.o.armijo_c1 * t * slope && v < fval) {
          reverse<PAT>(w, w.s + w.L.e);
          accept_step(w, s, t, v, fval);
          accepted = true;
          break;
        }
      }
      t *= w.o.backtrack_factor;
    }
    if (!accepted) s.status = ST_FAILED;  // best-so-far state retained
    if (itv && w.lane == 0) itv[s.iters] = s.value;
    ++s.iters;
    if (s.status == ST_RUNNING && s.iters >= w.o.max_iters) s.status = ST_FAILED;
    if (s.status != ST_RUNNING) break;
  }
  // finish_step (stepper.cpp:117-147)
  const bool converged = s.status == ST_CONVERGED;
  const double gnorm = vinf(w, g);
  if (w.lane == 0) {
    if (out.iterations) out.iterations[out.rrow(w.e, step)] = s.iters;
    if (out.converged) out.converged[out.rrow(w.e, step)] = converged;
    if (out.accepted) out.accepted[out.rrow(w.e, step)] = s.acc;
    if (out.final_value) out.final_value[out.rrow(w.e, step)] = s.value;
    if (out.final_grad_norm) out.final_grad_norm[out.rrow(w.e, step)] = gnorm;
    ival(w, IS_NREP) = step + 1;
  }
  const int fs = converged ? 0 : ival(w, IS_FAIL) + 1;
  __syncwarp();
  if (w.lane == 0) ival(w, IS_FAIL) = fs;
  if (fs > sc.fail_limit) {
    if (w.lane == 0) ival(w, IS_RUN) = TR_FAIL_LIMIT;
    return;
  }
  hist_rotations_s(w, x, 2);
  double ke, pe;
  step_energy(w, &ke, &pe);
  for (int k = w.lane; k < n; k += 32) {
    qv(w, w.gh0, k) = qv(w, w.gh1, k);
    qv(w, w.gh1, k) = x[k];
    if (out.q) out.q[out.qrow(w.e, step + 1) * n + k] = x[k];
  }
  if (w.lane == 0) {
    if (out.energy) {
      out.energy[out.qrow(w.e, step + 1) * 2] = ke;
      out.energy[out.qrow(w.e, step + 1) * 2 + 1] = pe;
    }
    ival(w, IS_STEP) = step + 1;
    ival(w, IS_NSAMP) = step + 2;
    if (step + 1 >= sc.total_steps) ival(w, IS_RUN) = TR_OK;
  }
}

inline int warps_per_block(int N, int n, int mem) {
  // 4 warps (one per SM sub-partition) unless the shared memory of four
  // environments does not fit, then fewer
  for (int wpb = 4; wpb >= 1; --wpb)
    if (block_smem_bytes(N, n, mem, wpb) + 64 <= 227 * 1024) return wpb;
  return 0;
}
// Warps per block for a batch of B environments on `sms` SMs: the batch spread
// evenly, one block per SM (up to 8 warps, as shared memory allows), so no SM
// runs more warps than the mean (C2: 7 warps per SM instead of 8 on 108 SMs
// and 4 on 40), at least the 4 of warps_per_block
inline int launch_wpb(int N, int n, int mem, long B, int sms) {
  const int base = warps_per_block(N, n, mem);
  if (base < 4) return base;
  int w = (int)std::min<long>(8, std::max<long>(4, (B + sms - 1) / sms));
  while (w > 4 && block_smem_bytes(N, n, mem, w) + 64 > 227 * 1024) --w;
  return w;
}
inline int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

template <int PAT>
cudaError_t launch(const ChainArgs& a, long recw, const Outputs& out, cudaStream_t s) {
  const int wpb = launch_wpb(a.m.N, a.m.n, a.sc.opt.mem, a.B, sm_count());
  const size_t sm = block_smem_bytes(a.m.N, a.m.n, a.sc.opt.mem, wpb) + 64;
  static SmemAttr attr_;
  size_t& configured = attr_.here();
  if (sm > configured) {
    const cudaError_t e = cudaFuncSetAttribute(k_chain5_step<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    configured = sm;
  }
  const unsigned grid = (unsigned)((a.B + wpb - 1) / wpb);
  k_chain5_step<PAT><<<grid, 32 * wpb, sm, s>>>(a.m, a.f, a.sc, a.L, a.cw, a.ci, a.B, recw, out);
  return cudaGetLastError();
}

}  // namespace c5

bool chain5_fits(int N, int n, int mem) { return mem <= c5::kMaxMem && c5::warps_per_block(N, n, mem) > 0; }

namespace {
constexpr int p16 = 1 | (6 << 2), p2 = 2 | (3 << 2) | (6 << 5);
template <int PAT>
int c5_blocks_per_sm(size_t sm, int threads) {
  if (cudaFuncSetAttribute(c5::k_chain5_step<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
    return 0;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, c5::k_chain5_step<PAT>, threads, sm) != cudaSuccess) return 0;
  return nb;
}
}  // namespace

// Waves of resident blocks a batch of B environments needs on `device`
// (0 if the kernel does not fit).  One warp per environment is the faster
// mapping while the whole batch is resident at once; beyond one wave the
// quad-per-environment v4 kernel, eight environments per warp, does more
// useful work per instruction.
int chain5_waves(int N, int n, int mem, long B, int pattern, int device) {
  if (c5::warps_per_block(N, n, mem) != 4 || mem > c5::kMaxMem) return 0;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  const int wpb = c5::launch_wpb(N, n, mem, B, sms);  // what launch() will use
  const size_t sm = c5::block_smem_bytes(N, n, mem, wpb) + 64;
  const int th = 32 * wpb;
  const int nb = pattern == p16 ? c5_blocks_per_sm<p16>(sm, th) : pattern == p2 ? c5_blocks_per_sm<p2>(sm, th)
                                                                                  : c5_blocks_per_sm<0>(sm, th);
  if (nb < 1) return 0;
  const long blocks = (B + wpb - 1) / wpb;
  return (int)((blocks + (long)nb * sms - 1) / ((long)nb * sms));
}

cudaError_t launch_chain5_step(const ChainArgs& a, int pattern, long recw, const Outputs& out, cudaStream_t s) {
  switch (pattern) {
    case p16: return c5::launch<p16>(a, recw, out, s);
    case p2: return c5::launch<p2>(a, recw, out, s);
    default: return c5::launch<0>(a, recw, out, s);
  }
}

}  // namespace pbad_gpu
