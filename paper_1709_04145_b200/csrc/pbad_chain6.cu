// pbad_chain6.cu -- chain kernel "v6": the v4 warp-synchronous chain kernel
// (pbad_chain4.cu) with two lanes per transform row, for serial chains of
// axis-aligned hinges (energy form, L-BFGS) in batches larger than one wave
// of the v5 kernel (C3: 4096 x 200 DOF).
//
// v4 maps a quad (4 lanes, one per row) to an environment and runs 8
// environments per warp: the C3 batch is 512 warps, fewer than the 592 SM
// sub-partitions, so every FP64 dependency and memory latency is exposed
// (ncu: issue 17 %).  v6 runs 4 environments per warp with 8 lanes each,
// l = 8 e + 4 h + r, doubling the warps and halving each lane's work:
//  * forward sweep: half h = 0 carries the world transform T (plus the lever
//    rows, T S, the gravity term and the inertial seed S (T - 2A + H)/dt^2),
//    half h = 1 the history transforms A = FK(hist1) and H = FK(hist0) (and
//    A S, H S); one shuffle per row exchanges T and A between the halves,
//    every other operand is lane-local; both halves execute one
//    instruction stream with half-selected operands;
//  * reverse sweep: the inertial adjoint in h = 0, the gravity adjoint in
//    h = 1 (adjoint.cpp:49-64);
//  * vectors: element k of an environment in lane k % 8 (groups of 8 per
//    32-double line), the reference's 32-partial dot order with 4 partials
//    per lane and a xor-4/2/1 butterfly (numeric contract);
//    every L-BFGS pass touches half as many elements per lane.
// Per-link records (rotation, lever rows, seed rows) go through global
// memory and come back by TMA bulk copies into a shared-memory ring exactly
// as in v4; the s/y history stays in HBM / L2 with L2 prefetches.
//
// Every value is produced by the reference's operation sequence (the
// per-row functions of pbad_chain_ops.cuh), so results are bit-identical to
// v4, v5, oracle/ and the reference build.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>

#include "pbad_chain_ops.cuh"
#include "pbad_kernels.cuh"
#include "pbad_launch.h"
#include "pbad_math.cuh"

namespace pbad_gpu {
namespace c6 {

using namespace chain_ops;

enum { PH_DIR = 0, PH_GEN = 1, PH_EVAL = 2, PH_DONE = 3 };
enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_FAILED = 2 };
enum { TR_OK = 0, TR_FAIL_LIMIT = 1, TR_NONFINITE_INIT = 2, TR_NONFINITE_CFG = 3, TR_RUNNING = 4 };

constexpr int kE = 4;   // environments per warp
constexpr int kL = 8;   // lanes per environment
// warps per block: a launch-time choice among 4, 7 and 8 (launch()): one
// block per SM of up to 8 warps shares the per-block model records and leaves
// the most L1 beside the warps' shared areas (C3: 4 -> 7 warps, 118 -> 106 ms)
constexpr int CL = 8;   // links per chunk (one per lane of an environment)
#ifndef PBAD_C6_RING
#define PBAD_C6_RING 3
#endif
constexpr int kRing = PBAD_C6_RING;
constexpr int kMaxMem = 16;
constexpr long kGS = 32;  // vector group stride (doubles): 8 elements x 4 environments
// per-link record (doubles, per warp): cs [env][2] | lev [3*env+row][2] | seed [3*env+row][4]
constexpr int kRecCS = 0, kRecLev = 8, kRecSd = 32;
constexpr int kRecLight = 32, kRecMass = 80;
constexpr int kSlot = CL * kRecMass;  // ring slot (doubles)
static_assert(kRecLight == kRecSd && kRecMass == kRecSd + 12 * kE, "record layout");
// per-warp shared memory (doubles)
// Shared-memory strides padded against bank conflicts (ncu round 2: 5.7 G
// excess wavefronts per C3 launch at strides 8 / 16 / 32):
constexpr int kRotS = 10;   // rotation record (c s | c0 s0 | c1 s1 | pad): 80 B apart
constexpr int kTermS = 20;  // energy-term row partials: 4 rows x 4 envs + 4 pad (term readers in distinct banks)
constexpr int kRedH = 18;   // gravity-chain offset inside a link's gradient partials (16 + 2 pad)
constexpr int kRedS = 34;   // gradient row partials of one link: 2 chains x 4 rows x 4 envs + 2 pad
constexpr int kFwdC = 0;                            // rotations of the chunk [CL][env]
constexpr int kFwdR = kFwdC + CL * kE * kRotS;      // energy row partials [CL][term][row][env]
constexpr int kFwdEnd = kFwdR + CL * 4 * kTermS;    // (the forward buffers overlay the ring)
constexpr int kRRed = kRing * kSlot;                // gradient row partials [CL][chain][row][env]
constexpr int kQScr = kRRed + CL * kRedS;           // per-environment scratch [env][16]
constexpr int kHsy = kQScr + kE * 16;          // per-environment s.y ring and alpha [env][kHsyW]
constexpr int kHsyW = 40;
constexpr int kBar = kHsy + kE * kHsyW;        // mbarriers
constexpr int kWarpD = kBar + 4;
static_assert(kFwdEnd <= kRing * kSlot, "forward buffers must fit in the ring");
static_assert(kHsyW >= 2 * kMaxMem + 1, "s.y ring + alpha");
static_assert(kWarpD % 2 == 0, "16-byte aligned warp areas");
constexpr int kHistW = 6;  // hist record per (link, env): c0 s0 | c1 s1 | cx sx

__host__ __device__ inline size_t smem_bytes(int N, int kw) {
  return (size_t)(kw * kWarpD + 20L * N) * sizeof(double) + (size_t)(2 * N + 1) * sizeof(int);
}

// ---- context ----------------------------------------------------------------
struct Ctx {
  int N, n, n8, nf, r, h, j, e;  // nf: groups whose 8 elements all exist (8 g + 7 < n)
  long ge, B, n4q;
  bool valid;
  unsigned em;         // this environment's 8 lanes
  double* ws;          // this warp's shared area
  uint64_t* bar;       // kRing mbarriers
  const double* mrec;  // shared model records [N][20]
  const int* kind;     // shared link classes
  const int* roff;     // shared per-warp record offsets [N+1]
  double* rec;         // this warp's link records (global)
  double* hist;        // this warp's history rotations [N][env][6] (global)
  double *gh0, *gh1;   // hist0 / hist1 in the quad chain layout (pbad_chain.cu)
  double *x, *g, *cand, *dir, *q, *evg, *tau, *hs, *hy;
  long VS;
  double* hsy;    // shared: this env's s.y ring [mem+1] then alpha [mem]
  double* histc;
  int* ci;
  double dt, inv_dt2, wm, gr;
  double gz[3];
  DOpt o;
  unsigned nload;  // ring chunks consumed (warp-uniform; sets slot and phase)
};

// shuffles inside an environment's 8 lanes; the solver steps of the four
// environments diverge, so the environment's own mask ...
__device__ __forceinline__ double eshfl(const Ctx& C, double v, int src) { return __shfl_sync(C.em, v, src, kL); }
__device__ __forceinline__ double eshfl_xor(const Ctx& C, double v, int m) {
  return __shfl_xor_sync(C.em, v, m, kL);
}
// ... except in the sweeps, which every lane of the warp executes together
__device__ __forceinline__ double wshfl_xor(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m, kL); }
__device__ __forceinline__ double wshfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src, kL); }
__device__ __forceinline__ void esync(const Ctx& C) { __syncwarp(C.em); }
__device__ __forceinline__ int& ival(const Ctx& C, int slot) { return C.ci[(long)slot * C.B + C.ge]; }
// element k of this environment: this lane's elements are k = 8 g + j
__device__ __forceinline__ double& vat(const Ctx& C, double* V, int k) {
  return V[(long)(k >> 3) * kGS + ((k & 7) - C.j)];
}
// element k of this environment in a quad-interleaved chain-layout vector
__device__ __forceinline__ double& qv(const Ctx& C, double* base, int k) {
  return base[((C.ge >> 3) * C.n4q + (k >> 2)) * 32 + (C.ge & 7) * 4 + (k & 3)];
}
__device__ __forceinline__ bool elem_ok(const Ctx& C, int g) { return g < C.n8 && 8 * g + C.j < C.n; }

// ---- 8-lane vector ops (32-partial canonical dot, optim.cpp) -----------------
// acc[a] holds partial 8 a + j of the reference's 32 interleaved partials
__device__ __forceinline__ double dot_finish(const Ctx& C, const double* acc) {
  double v = (acc[0] + acc[2]) + (acc[1] + acc[3]);  // partial tree levels xor 16, xor 8
  v = v + eshfl_xor(C, v, 4);
  v = v + eshfl_xor(C, v, 2);
  v = v + eshfl_xor(C, v, 1);
  return v;
}
__device__ __forceinline__ double emax(const Ctx& C, double mx) {
  mx = fmax(mx, eshfl_xor(C, mx, 4));
  mx = fmax(mx, eshfl_xor(C, mx, 2));
  mx = fmax(mx, eshfl_xor(C, mx, 1));
  return mx;
}
__device__ __forceinline__ double edot(const Ctx& C, const double* A, const double* Bv) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int g = 0; g < C.n8; ++g)
    if (elem_ok(C, g)) acc[g & 3] = fma(A[(long)g * kGS], Bv[(long)g * kGS], acc[g & 3]);
  return dot_finish(C, acc);
}
__device__ __forceinline__ double einfnorm(const Ctx& C, const double* A) {
  double mx = 0.0;
  for (int g = 0; g < C.n8; ++g)
    if (elem_ok(C, g)) mx = fmax(mx, fabs(A[(long)g * kGS]));
  return emax(C, mx);
}
__device__ __forceinline__ bool eallfinite(const Ctx& C, const double* A) {
  bool ok = true;
  for (int g = 0; g < C.n8; ++g)
    if (elem_ok(C, g)) ok = ok && isfinite(A[(long)g * kGS]);
  return __all_sync(C.em, ok);
}
__device__ __forceinline__ bool qallfinite(const Ctx& C, double* base) {
  bool ok = true;
  for (int k = C.j; k < C.n; k += kL) ok = ok && isfinite(qv(C, base, k));
  return __all_sync(C.em, ok);
}

// ---- forward sweep ------------------------------------------------------------
// StepObjective::value at X (objective.cpp:215-239), storing the reverse
// sweep's per-link records.  X1: T (h = 0) or A = FK(hist1) (h = 1);
// X2: H = FK(hist0) in both halves.
struct Rows {
  double X1[4], X2[4];
};

// predicated 16-byte global store without a branch around it
__device__ __forceinline__ void stg2_if(bool p, double* a, double x, double y) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.global.v2.f64 [%1], {%2, %3};\n}" ::"r"((int)p),
               "l"(a), "d"(x), "d"(y)
               : "memory");
}

template <int CK>
__device__ __forceinline__ void fwd_link(const Ctx& C, int jl, int i, Rows& R, double* rp) {
  constexpr int JK = CK & 3;
  constexpr bool SK = (CK >> 2) != 0;
  const double* rb = C.ws + kFwdC + (jl * kE + C.e) * kRotS;
  // X1's rotation: the iterate's (h = 0) or hist1's (h = 1); X2's: hist0's
  const double2 cs1 = *reinterpret_cast<const double2*>(rb + 4 * C.h);
  const double2 hc0 = *reinterpret_cast<const double2*>(rb + 2);
  const double c1 = cs1.x, s1 = cs1.y;
  const double* mr = C.mrec + 20 * i;
  const double2 t01 = *reinterpret_cast<const double2*>(mr + 16);
  const double t[3] = {t01.x, t01.y, mr[18]};
  const int row = 3 * C.e + C.r;
  const bool rec_lane = C.h == 0 && C.r < 3;
  double l0, l1;
  lever<JK>(c1, s1, R.X1, l0, l1);  // h = 0: T_parent row times dL/dq (adjoint.cpp:22-25)
  stg2_if(rec_lane, rp + kRecLev + 2 * row, l0, l1);
  fk<JK>(c1, s1, t, R.X1);
  fk<JK>(hc0.x, hc0.y, t, R.X2);
  if (SK) {
    double S[16];
    lds16(mr, S);
    double p[4];  // the other half's X1: A in h = 0, T in h = 1
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = wshfl_xor(R.X1[k], 4);
    double tr[4], y[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double dd = R.X1[k] - 2.0 * p[k];  // h = 0: (T - 2A + H) / dt^2
      dd = dd + R.X2[k];
      dd = C.inv_dt2 * dd;
      y[k] = C.h ? R.X2[k] : dd;
      tr[k] = C.h ? p[k] : R.X1[k];
    }
    double p1[4], p2[4], cg[4];
    row_s(R.X1, S, p1);  // h = 0: T S, h = 1: A S
    row_s(y, S, p2);     // h = 0: seed row, h = 1: H S
#pragma unroll
    for (int k = 0; k < 4; ++k) cg[k] = C.h ? p2[k] : (-C.gr) * S[12 + k];
    double* fr = C.ws + kFwdR + jl * 4 * kTermS + C.r * 4 + C.e;
    fr[C.h ? kTermS : 0] = ddot_row(p1, tr);           // term 0 (T S . T) / term 1 (A S . T)
    fr[C.h ? 2 * kTermS : 3 * kTermS] = ddot_row(cg, tr);  // term 3 (gravity) / term 2 (H S . T)
    double* sp = rp + kRecSd + 4 * row;
    stg2_if(rec_lane, sp, p2[0], p2[1]);
    stg2_if(rec_lane, sp + 2, p2[2], p2[3]);
  }
}

__device__ __forceinline__ void fwd_link_dyn(const Ctx& C, int jl, int i, Rows& R) {
  switch (C.kind[i]) {
    case 1: fwd_link<1>(C, jl, i, R, C.rec + C.roff[i]); break;
    case 2: fwd_link<2>(C, jl, i, R, C.rec + C.roff[i]); break;
    case 3: fwd_link<3>(C, jl, i, R, C.rec + C.roff[i]); break;
    case 5: fwd_link<5>(C, jl, i, R, C.rec + C.roff[i]); break;
    case 6: fwd_link<6>(C, jl, i, R, C.rec + C.roff[i]); break;
    default: fwd_link<7>(C, jl, i, R, C.rec + C.roff[i]); break;
  }
}

// link-pattern code: P | K0 << 2 | K1 << 5 (P = period 1 or 2; 0 = per-link dispatch)
template <int PAT, int J>
struct PatKind {
  static constexpr int P = PAT & 3;
  static constexpr int value = (P == 2 && (J & 1)) ? ((PAT >> 5) & 7) : ((PAT >> 2) & 7);
};
// record offset of chunk link J from the chunk's first record (compile-time
// for a link pattern: the chunk starts at a multiple of the period)
template <int PAT, int J>
struct RecOff {
  static constexpr int value =
      RecOff<PAT, J - 1>::value + (((PatKind<PAT, J - 1>::value >> 2) != 0) ? kRecMass : kRecLight);
};
template <int PAT>
struct RecOff<PAT, 0> {
  static constexpr int value = 0;
};
template <int PAT, int J>
struct FwdUnroll {
  static __device__ __forceinline__ void run(const Ctx& C, int lo, Rows& R, double* rc) {
    fwd_link<PatKind<PAT, J>::value>(C, J, lo + J, R, rc + RecOff<PAT, J>::value);
    FwdUnroll<PAT, J + 1>::run(C, lo, R, rc);
  }
};
template <int PAT>
struct FwdUnroll<PAT, CL> {
  static __device__ __forceinline__ void run(const Ctx&, int, Rows&, double*) {}
};

template <int PAT>
__device__ __forceinline__ void fwd_chunk(const Ctx& C, int lo, int cnt, Rows& R) {
  if constexpr ((PAT & 3) != 0) {
    if (cnt == CL) {
      FwdUnroll<PAT, 0>::run(C, lo, R, C.rec + C.roff[lo]);
      return;
    }
  }
  for (int jl = 0; jl < cnt; ++jl) fwd_link_dyn(C, jl, lo + jl, R);
}

template <int PAT>
__device__ __forceinline__ double forward(const Ctx& C, const double* X, double tdx) {
  const int N = C.N;
  const int nch = (N + CL - 1) / CL;
  Rows R;
#pragma unroll
  for (int k = 0; k < 4; ++k) R.X1[k] = R.X2[k] = (C.r == k) ? 1.0 : 0.0;
  double sum = 0.0;  // lane j < 4: running sum of energy term j
  // this lane's link of chunk c: 8 c + j (its own element of X)
  double xa = 0.0;
  double2 ha0 = make_double2(0.0, 0.0), ha1 = ha0;
  auto fetch = [&](int c) {
    const int la = CL * c + C.j;
    if (la < N) {
      xa = X[(long)c * kGS];
      const double* hp = C.hist + ((long)la * kE + C.e) * kHistW;
      ha0 = *reinterpret_cast<const double2*>(hp);
      ha1 = *reinterpret_cast<const double2*>(hp + 2);
    }
  };
  fetch(0);
  for (int c = 0; c < nch; ++c) {
    const int lo = CL * c, cnt = min(CL, N - lo);
    const int la = lo + C.j;
    // phase A: the joint rotation of this lane's link
    double ca, sa;
    hinge_cs(xa, &ca, &sa);
    const double2 h_a0 = ha0, h_a1 = ha1;
    if (c + 1 < nch) fetch(c + 1);
    __syncwarp();  // previous chunk's readers are done with the buffers
    if (la < N) {
      double* rb = C.ws + kFwdC + (C.j * kE + C.e) * kRotS;
      *reinterpret_cast<double2*>(rb) = make_double2(ca, sa);
      *reinterpret_cast<double2*>(rb + 2) = h_a0;
      *reinterpret_cast<double2*>(rb + 4) = h_a1;
      *reinterpret_cast<double2*>(C.rec + C.roff[la] + kRecCS + 2 * C.e) = make_double2(ca, sa);
    }
    __syncwarp();
    // phase B: the serial recursions over the chunk
    fwd_chunk<PAT>(C, lo, cnt, R);
    __syncwarp();
    // lane t < 4 adds term t of each massive link, link by link (serial order)
    if (C.j < 4) {
      const double* b0 = C.ws + kFwdR + C.j * kTermS + C.e;
      if ((PAT & 3) != 0 && cnt == CL) {
#pragma unroll
        for (int jl = 0; jl < CL; ++jl) {
          const int ck = ((PAT & 3) == 2 && (jl & 1)) ? ((PAT >> 5) & 7) : ((PAT >> 2) & 7);
          if (ck >> 2) {
            const double* b = b0 + jl * 4 * kTermS;
            sum += ((b[0] + b[4]) + b[8]) + b[12];
          }
        }
      } else {
        for (int jl = 0; jl < cnt; ++jl) {
          if (C.kind[lo + jl] >> 2) {
            const double* b = b0 + jl * 4 * kTermS;
            sum += ((b[0] + b[4]) + b[8]) + b[12];
          }
        }
      }
    }
  }
  const double sa = wshfl(sum, 0), sb = wshfl(sum, 1), sc = wshfl(sum, 2), sg = wshfl(sum, 3);
  const double wm = C.wm;
  const double cpp = sa - wm, c1p = sb - wm, c2p = sc - wm;
  const double inertial = 0.5 * C.inv_dt2 * (cpp - 4.0 * c1p + 2.0 * c2p + *C.histc);
  return inertial + sg - tdx;
}

// ---- reverse sweep ------------------------------------------------------------
// functional_grad twice (adjoint.cpp:49-64): gradient = inertial adjoint
// (h = 0) + gravity adjoint (h = 1) - tau (objective.cpp:241-250) into Gv.
template <int CK>
__device__ __forceinline__ void rev_link(const Ctx& C, const double* rp, int i, int jl, double* cc) {
  constexpr int JK = CK & 3;
  constexpr bool SK = (CK >> 2) != 0;
  const double2 cs = *reinterpret_cast<const double2*>(rp + kRecCS + 2 * C.e);
  const int row = 3 * C.e + C.r;
  const bool own = C.r < 3;  // row 3 of the lever and of the seed is exactly zero
  double l0 = 0.0, l1 = 0.0;
  if (own) {
    const double2 lv = *reinterpret_cast<const double2*>(rp + kRecLev + 2 * row);
    l0 = lv.x;
    l1 = lv.y;
  }
  const double* mr = C.mrec + 20 * i;
  double a[4];
  if (SK) {
    // inertial chain (h = 0, rows 0..2): a = cc + seed; gravity chain: a = cc +
    // (0.0 + (-g_r) u) with u = S column 3.  Both as cc + fma(m, v, 0.0): the
    // product m v is exact for m = 1, and fma(x, y, 0.0) == 0.0 + x * y.  The
    // only difference, the sign of a zero addend, cannot reach a: cc is never
    // -0 (it starts at +0 and is 0.0 + o afterwards), and row 3 (no seed)
    // takes m = 0.
    const bool sd_lane = own && C.h == 0;
    const double* vp = sd_lane ? rp + kRecSd + 4 * row : mr + 12;
    const double mlt = sd_lane ? 1.0 : (C.h ? -C.gr : 0.0);
    const double2 v01 = *reinterpret_cast<const double2*>(vp);
    const double2 v23 = *reinterpret_cast<const double2*>(vp + 2);
    const double v[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = cc[k] + fma(mlt, v[k], 0.0);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = cc[k];
  }
  C.ws[kRRed + jl * kRedS + C.h * kRedH + C.r * 4 + C.e] = lever_dot<JK>(l0, l1, a);
  if (i > 0) {
    const double2 t01 = *reinterpret_cast<const double2*>(mr + 16);
    const double t[3] = {t01.x, t01.y, mr[18]};
    double o[4];
    transport<JK>(cs.x, cs.y, t, a, o);
#pragma unroll
    for (int k = 0; k < 4; ++k) cc[k] = 0.0 + o[k];
  }
}

__device__ __forceinline__ void rev_link_dyn(const Ctx& C, const double* rp, int i, int jl, double* cc) {
  switch (C.kind[i]) {
    case 1: rev_link<1>(C, rp, i, jl, cc); break;
    case 2: rev_link<2>(C, rp, i, jl, cc); break;
    case 3: rev_link<3>(C, rp, i, jl, cc); break;
    case 5: rev_link<5>(C, rp, i, jl, cc); break;
    case 6: rev_link<6>(C, rp, i, jl, cc); break;
    default: rev_link<7>(C, rp, i, jl, cc); break;
  }
}

template <int PAT, int J>
struct RevUnroll {  // links J, J-1, ..., 0 of a full chunk
  static __device__ __forceinline__ void run(const Ctx& C, const double* sbase, int lo, double* cc) {
    rev_link<PatKind<PAT, J>::value>(C, sbase + RecOff<PAT, J>::value, lo + J, J, cc);
    RevUnroll<PAT, J - 1>::run(C, sbase, lo, cc);
  }
};
template <int PAT>
struct RevUnroll<PAT, -1> {
  static __device__ __forceinline__ void run(const Ctx&, const double*, int, double*) {}
};

template <int PAT>
__device__ __forceinline__ void rev_chunk(const Ctx& C, const double* sbase, int lo, int cnt, double* cc) {
  if constexpr ((PAT & 3) != 0) {
    if (cnt == CL) {
      RevUnroll<PAT, CL - 1>::run(C, sbase + C.roff[lo], lo, cc);
      return;
    }
  }
  for (int jl = cnt - 1; jl >= 0; --jl) rev_link_dyn(C, sbase + C.roff[lo + jl], lo + jl, jl, cc);
}

__device__ __forceinline__ void issue_chunk(Ctx& C, int c, unsigned k) {
  const int lo = CL * c, hi = min(C.N, lo + CL);
  const int slot = (int)(k % kRing);
  const unsigned bytes = (unsigned)(C.roff[hi] - C.roff[lo]) * 8u;
#if PBAD_C6_HINT & 2
  bulk_load_ef(C.ws + slot * kSlot, C.rec + C.roff[lo], bytes, C.bar + slot);
#else
  bulk_load(C.ws + slot * kSlot, C.rec + C.roff[lo], bytes, C.bar + slot);
#endif
}

template <int PAT>
__device__ __forceinline__ void reverse(Ctx& C, double* Gv) {
  const int N = C.N;
  const int nch = (N + CL - 1) / CL;
  fence_async_global();  // this lane's record stores -> the bulk copies below
  __syncwarp();
  const unsigned k0 = C.nload;
  if ((threadIdx.x & 31) == 0) {
    fence_async_smem();  // forward-buffer accesses in the ring area before the async writes
    for (int p = 0; p < kRing && p < nch; ++p) issue_chunk(C, nch - 1 - p, k0 + p);
  }
  double cc[4] = {0.0, 0.0, 0.0, 0.0};
  // tau of this lane's link of the next chunk (loaded a chunk ahead)
  double tau_n = (CL * (nch - 1) + C.j < N) ? C.tau[(long)(nch - 1) * kGS] : 0.0;
  for (int idx = 0; idx < nch; ++idx) {
    const int c = nch - 1 - idx;
    const int lo = CL * c, cnt = min(CL, N - lo);
    const unsigned k = k0 + idx;
    const int slot = (int)(k % kRing);
    mbar_wait(C.bar + slot, (k / kRing) & 1u);
    const double* sbase = C.ws + slot * kSlot - C.roff[lo];
    const double tau_c = tau_n;
    if (c > 0) tau_n = C.tau[(long)(c - 1) * kGS];
    rev_chunk<PAT>(C, sbase, lo, cnt, cc);
    __syncwarp();
    // the gradient entry of this lane's link of the chunk
    if (C.j < cnt) {
      const double* b = C.ws + kRRed + C.j * kRedS + C.e;
      const double gi = 0.0 + (((b[0] + b[4]) + b[8]) + b[12]);
      const double gp = 0.0 + (((b[kRedH] + b[kRedH + 4]) + b[kRedH + 8]) + b[kRedH + 12]);
      Gv[(long)c * kGS] = (gi + gp) - tau_c;
    }
    __syncwarp();
    if (idx + kRing < nch && (threadIdx.x & 31) == 0) {
      fence_async_smem();
      issue_chunk(C, c - kRing, k + kRing);
    }
  }
  C.nload = k0 + nch;
}

// ---- per-step history passes (once per PBAD step) ---------------------------
// joint rotations into hist slot `slot` (0: hist0, 1: hist1, 2: x)
__device__ __forceinline__ void hist_rotations_q(const Ctx& C, double* base, int slot) {
  for (int i = C.j; i < C.N; i += kL) {
    double c, s;
    hinge_cs(qv(C, base, i), &c, &s);
    *reinterpret_cast<double2*>(C.hist + ((long)i * kE + C.e) * kHistW + 2 * slot) = make_double2(c, s);
  }
  esync(C);
}
__device__ __forceinline__ void hist_rotations(const Ctx& C, const double* V, int slot) {
  for (int i = C.j; i < C.N; i += kL) {
    double c, s;
    hinge_cs(V[(long)(i >> 3) * kGS], &c, &s);
    *reinterpret_cast<double2*>(C.hist + ((long)i * kE + C.e) * kHistW + 2 * slot) = make_double2(c, s);
  }
  esync(C);
}

__device__ __forceinline__ void fk_dyn(int jk, double c, double s, const double* t, double* T) {
  if (jk == 1) fk<1>(c, s, t, T);
  else if (jk == 2) fk<2>(c, s, t, T);
  else fk<3>(c, s, t, T);
}
// ((v_0 + v_1) + v_2) + v_3 over the 4 rows (both halves compute the same rows)
__device__ __forceinline__ double rows4(const Ctx& C, double v) {
  const double v0 = __shfl_sync(C.em, v, 0, 4), v1 = __shfl_sync(C.em, v, 1, 4);
  const double v2 = __shfl_sync(C.em, v, 2, 4), v3 = __shfl_sync(C.em, v, 3, 4);
  return ((v0 + v1) + v2) + v3;
}

// hist_const = 4 cv(tk, tk) + cv(tk1, tk1) - 4 cv(tk, tk1) (objective.cpp:162-185),
// tk = FK(hist1), tk1 = FK(hist0); massless links add exact zeros and are skipped
__device__ __forceinline__ double hist_const(const Ctx& C) {
  double A[4], H[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) A[k] = H[k] = (C.r == k) ? 1.0 : 0.0;
  double vAA = 0.0, vHH = 0.0, vAH = 0.0;
  for (int i = 0; i < C.N; ++i) {
    const int ck = C.kind[i];
    const double* hp = C.hist + ((long)i * kE + C.e) * kHistW;
    const double* mr = C.mrec + 20 * i;
    const double t[3] = {mr[16], mr[17], mr[18]};
    fk_dyn(ck & 3, hp[2], hp[3], t, A);
    fk_dyn(ck & 3, hp[0], hp[1], t, H);
    if (ck >> 2) {
      double S[16], as[4], hs[4];
      lds16(mr, S);
      row_s(A, S, as);
      row_s(H, S, hs);
      vAA += rows4(C, ddot_row(as, A));
      vHH += rows4(C, ddot_row(hs, H));
      vAH += rows4(C, ddot_row(as, H));
    }
  }
  return 4.0 * (vAA - C.wm) + (vHH - C.wm) - 4.0 * (vAH - C.wm);
}

// fd_kinetic (stepper.cpp:14-22) + gravity_potential (baseline.cpp:219-229)
// between FK(hist slot 1) and FK(hist slot 2)
__device__ __forceinline__ void step_energy(const Ctx& C, double* ke, double* pe) {
  double P[4], W[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) P[k] = W[k] = (C.r == k) ? 1.0 : 0.0;
  double kk = 0.0, pp = 0.0;
  const double ghat[4] = {C.gz[0], C.gz[1], C.gz[2], 0.0};
  for (int i = 0; i < C.N; ++i) {
    const int ck = C.kind[i];
    const double* hp = C.hist + ((long)i * kE + C.e) * kHistW;
    const double* mr = C.mrec + 20 * i;
    const double t[3] = {mr[16], mr[17], mr[18]};
    fk_dyn(ck & 3, hp[2], hp[3], t, P);
    fk_dyn(ck & 3, hp[4], hp[5], t, W);
    if (ck >> 2) {
      double S[16], td[4], tds[4];
      lds16(mr, S);
#pragma unroll
      for (int c = 0; c < 4; ++c) td[c] = (W[c] - P[c]) / C.dt;
      row_s(td, S, tds);
      double wu = W[0] * S[12];
      wu = fma(W[1], S[13], wu);
      wu = fma(W[2], S[14], wu);
      wu = fma(W[3], S[15], wu);
      const double term = rows4(C, ddot_row(tds, td));
      const double u0 = __shfl_sync(C.em, wu, 0, 4), u1 = __shfl_sync(C.em, wu, 1, 4);
      const double u2 = __shfl_sync(C.em, wu, 2, 4), u3 = __shfl_sync(C.em, wu, 3, 4);
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

// ForceModel::tau_at (objective.hpp:28-58)
__device__ __forceinline__ void tau_at(const Ctx& C, const DForces& f, double t) {
  const int n = C.n;
  for (int i = C.j; i < n; i += kL) {
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
    vat(C, C.tau, i) = v;
  }
}

// ---- L-BFGS (LbfgsSolver, optim.cpp:141-232) ------------------------------
// The v4 kernel's fused vector passes (one per reduction of the two-loop
// recursion, one for the candidate, one for the accepted step) over this
// lane's elements 8 g + j; every dot keeps its 32-partial order.
struct Solver {
  double value, grad0, t, slope, fval;
  double ginf, xinf;  // |g|_inf, |x|_inf of the current iterate
  double tdx;         // tau . cand of the pending candidate
  int status, iters, stag, acc, h0, hc, trial, phase;
  double* itv;        // per_iteration_values row of this step (lane j = 0 writes), or null
  // s . g and y . y of the pair the last accepted step pushed (PBAD_C6_FUSE):
  // the two-loop's first dot and its y_{hc-1} . y_{hc-1}, computed in the
  // accepted-step pass with the same operands and partial order
  double pre_sg, pre_yy;
  bool pre;
};

#ifndef PBAD_C6_KB
#define PBAD_C6_KB 8
#endif
constexpr int kB = PBAD_C6_KB;  // groups per batch of loads (multiple of 4: dot partial index)
static_assert(kB % 4 == 0, "batch must keep the 32-partial dot order");

// Vector passes run in batches of kB groups.  Batches of groups below nf
// hold an element in every lane and run unpredicated from one base address
// (F = true); the tail batch checks every group (F = false).
// PBAD_C6_HINT (L2 eviction priority, bit mask): 1 (default): the two-loop
// passes that are a history vector's last read of the iteration (loop 2 and
// the scale pass) load it evict-first (ld.global.cs), leaving L2 to the link
// records and the hot vectors (C3 93.7 -> 91.7 ms); 2 (A/B only, slower):
// the reverse sweep's record bulk copies carry an L2 evict-first policy.
// Measured and dropped: evict-last record stores, evict-last
// loop-1 history loads, evict-first s / y stores.
#ifndef PBAD_C6_HINT
#define PBAD_C6_HINT 1
#endif
template <bool F, bool CS = false>
__device__ __forceinline__ void ldb(const Ctx& C, const double* V, int g0, double* out) {
  const double* p = V + (long)g0 * kGS;
#pragma unroll
  for (int jj = 0; jj < kB; ++jj) {
    if (CS) out[jj] = (F || g0 + jj < C.n8) ? __ldcs(p + jj * kGS) : 0.0;
    else out[jj] = (F || g0 + jj < C.n8) ? p[jj * kGS] : 0.0;
  }
}
template <bool F>
__device__ __forceinline__ bool gok(const Ctx& C, int g) { return F || elem_ok(C, g); }
__device__ __forceinline__ void l2_prefetch(const Ctx& C, const double* V) {
  if ((threadIdx.x & 31) == 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(V - (threadIdx.x & 31)),
                 "r"((unsigned)(C.n8 * kGS * sizeof(double)))
                 : "memory");
}

// two-loop passes: q' = op(q, w); then DOT 0: z . q'; 1: z . z; 2: dir = -q', dir . g
enum { M_COPY = 0, M_SUB = 1, M_SCALE = 2, M_ADD = 3, M_SUBSCALE = 4 };
// PBAD_C6_FUSE (default 1): with the pushed pair's s . g and y . y from the
// accepted-step pass, the two-loop skips its copy pass (q = g; the first
// M_SUB pass reads g as q) and merges the scale pass into loop 1's last pass
// (M_SUBSCALE: q = (q - a y_0) scl; y_0 . q): two of the iteration's vector
// passes fewer, every value unchanged.
#ifndef PBAD_C6_FUSE
#define PBAD_C6_FUSE 1
#endif
template <bool F, int MODE, int DOT>
__device__ __forceinline__ void tl_batch(const Ctx& C, const double* qs, const double* w, double a, double a2,
                                         const double* z, bool store_q, int g0, double* acc) {
  double qv_[kB], wv[kB], zv[kB];
  // loop 2 and the scale pass are a history vector's last read of the iteration
  constexpr bool LAST = (PBAD_C6_HINT & 1) && (MODE == M_ADD || MODE == M_SCALE || MODE == M_SUBSCALE);
  if (MODE != M_COPY) ldb<F>(C, qs, g0, qv_);
  if (MODE != M_SCALE) ldb<F, LAST>(C, w, g0, wv);
  if (DOT == 2) ldb<F>(C, C.g, g0, zv);
  else if (MODE != M_SUBSCALE) ldb<F, LAST>(C, z, g0, zv);  // M_SUBSCALE: z = w
  double* qo = C.q + (long)g0 * kGS;
  double* dout = C.dir + (long)g0 * kGS;
#pragma unroll
  for (int jj = 0; jj < kB; ++jj) {
    if (!gok<F>(C, g0 + jj)) continue;
    double qn;
    if (MODE == M_COPY) qn = wv[jj];
    else if (MODE == M_SUB) qn = qv_[jj] - a * wv[jj];
    else if (MODE == M_SCALE) qn = qv_[jj] * a;
    else if (MODE == M_SUBSCALE) qn = (qv_[jj] - a * wv[jj]) * a2;
    else qn = qv_[jj] + a * wv[jj];
    if (DOT == 2) {
      const double d = -qn;
      dout[jj * kGS] = d;
      acc[jj & 3] = fma(d, zv[jj], acc[jj & 3]);
    } else {
      if (store_q) qo[jj * kGS] = qn;
      if (DOT == 0 && MODE == M_SUBSCALE) acc[jj & 3] = fma(wv[jj], qn, acc[jj & 3]);
      else if (DOT == 0) acc[jj & 3] = fma(zv[jj], qn, acc[jj & 3]);
      else acc[jj & 3] = fma(zv[jj], zv[jj], acc[jj & 3]);
    }
  }
}
template <int MODE, int DOT>
__device__ __forceinline__ double tl_pass(const Ctx& C, const double* w, double a, const double* z, bool store_q,
                                         const double* qs = nullptr, double a2 = 0.0) {
  if (!qs) qs = C.q;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int g0 = 0;
  for (; g0 + kB <= C.nf; g0 += kB) tl_batch<true, MODE, DOT>(C, qs, w, a, a2, z, store_q, g0, acc);
  for (; g0 < C.n8; g0 += kB) tl_batch<false, MODE, DOT>(C, qs, w, a, a2, z, store_q, g0, acc);
  return dot_finish(C, acc);
}

// ring slot of deque entry i: (h0 + i) mod (mem + 1) with h0, i <= mem
__device__ __forceinline__ int hslot(const Ctx& C, const Solver& s, int i) {
  const int k = s.h0 + i;
  return k > C.o.mem ? k - (C.o.mem + 1) : k;
}
__device__ __forceinline__ const double* hist_s(const Ctx& C, const Solver& s, int i) {
  return C.hs + hslot(C, s, i) * C.VS;
}
__device__ __forceinline__ const double* hist_y(const Ctx& C, const Solver& s, int i) {
  return C.hy + hslot(C, s, i) * C.VS;
}
__device__ __forceinline__ double hist_sy(const Ctx& C, const Solver& s, int i) { return C.hsy[hslot(C, s, i)]; }

// loop 2 of the two-loop from q and y_0 . q (shared by both variants)
__device__ __forceinline__ double two_loop_2(const Ctx& C, const Solver& s, const double* alpha, double d) {
  const int hc = s.hc;
  double slope = 0.0;
  for (int i = 0; i < hc; ++i) {
    const double beta = d / hist_sy(C, s, i);
    const double c = alpha[i] - beta;
    if (i + 2 < hc) {
      l2_prefetch(C, hist_s(C, s, i + 1));
      l2_prefetch(C, hist_y(C, s, i + 2));
    } else if (i + 1 < hc) {
      l2_prefetch(C, hist_s(C, s, i + 1));
    }
    if (i + 1 < hc) d = tl_pass<M_ADD, 0>(C, hist_s(C, s, i), c, hist_y(C, s, i + 1), true);
    else slope = tl_pass<M_ADD, 2>(C, hist_s(C, s, i), c, nullptr, false);  // dir = -q; dir . g
  }
  return slope;
}

// the two-loop with the pushed pair's s . g and y . y known (PBAD_C6_FUSE):
// no copy pass (loop 1's first pass reads g as q) and loop 1's last pass
// applies the scale (M_SUBSCALE)
__device__ __forceinline__ double direction_fused(const Ctx& C, const Solver& s, double* alpha) {
  const int hc = s.hc;
  double d = s.pre_sg;  // s_{hc-1} . g
  const double scl = hist_sy(C, s, hc - 1) / s.pre_yy;
  for (int i = hc - 1; i >= 0; --i) {
    const double a = d / hist_sy(C, s, i);
    alpha[i] = a;
    if (i >= 2) {
      l2_prefetch(C, hist_y(C, s, i - 1));
      l2_prefetch(C, hist_s(C, s, i - 2));
    } else if (i == 1) {
      l2_prefetch(C, hist_y(C, s, 0));
    }
    const double* qs = (i == hc - 1) ? C.g : C.q;  // q = g before the first pass
    if (i > 0) d = tl_pass<M_SUB, 0>(C, hist_y(C, s, i), a, hist_s(C, s, i - 1), true, qs);
    else d = tl_pass<M_SUBSCALE, 0>(C, hist_y(C, s, 0), a, nullptr, true, qs, scl);  // q = (q - a y_0) scl; y_0 . q
  }
  l2_prefetch(C, hist_s(C, s, 0));
  if (hc > 1) l2_prefetch(C, hist_y(C, s, 1));
  return two_loop_2(C, s, alpha, d);
}

// two_loop (optim.cpp:213-229) fused with dir = -q and slope = dir . g
// (optim.cpp:162-170); returns the slope
__device__ __forceinline__ double direction(const Ctx& C, const Solver& s) {
  const int hc = s.hc;
  if (hc == 0) return tl_pass<M_COPY, 2>(C, C.g, 0.0, nullptr, false);
  l2_prefetch(C, hist_s(C, s, hc - 1));
  l2_prefetch(C, hist_y(C, s, hc - 1));
  if (hc > 1) l2_prefetch(C, hist_s(C, s, hc - 2));
  double* alpha = C.hsy + kMaxMem + 1;
  if (PBAD_C6_FUSE && s.pre) return direction_fused(C, s, alpha);
  double d = tl_pass<M_COPY, 0>(C, C.g, 0.0, hist_s(C, s, hc - 1), true);  // q = g; s . q
  double yy = 0.0;
  for (int i = hc - 1; i >= 0; --i) {
    const double a = d / hist_sy(C, s, i);
    alpha[i] = a;
    if (i >= 2) {
      l2_prefetch(C, hist_y(C, s, i - 1));
      l2_prefetch(C, hist_s(C, s, i - 2));
    } else if (i == 1) {
      l2_prefetch(C, hist_y(C, s, 0));
    }
    if (i > 0) d = tl_pass<M_SUB, 0>(C, hist_y(C, s, i), a, hist_s(C, s, i - 1), true);
    else yy = tl_pass<M_SUB, 1>(C, hist_y(C, s, 0), a, hist_y(C, s, hc - 1), true);
  }
  l2_prefetch(C, hist_s(C, s, 0));
  if (hc > 1) l2_prefetch(C, hist_y(C, s, 1));
  const double scl = hist_sy(C, s, hc - 1) / yy;
  d = tl_pass<M_SCALE, 0>(C, nullptr, scl, hist_y(C, s, 0), true);  // q *= scl; y_0 . q
  return two_loop_2(C, s, alpha, d);
}

// start of LbfgsSolver::iterate: termination tests, direction, slope
__device__ __forceinline__ void begin_iteration(const Ctx& C, Solver& s) {
  if (s.iters >= C.o.max_iters) {
    s.status = ST_FAILED;
    s.phase = PH_DONE;
    return;
  }
  // grad_converged (optim.cpp:35-41) on the norms of the current iterate
  if (s.ginf <= C.o.grad_tol * fmax(1.0, s.xinf) || (C.o.grad_rtol > 0.0 && s.ginf <= C.o.grad_rtol * s.grad0)) {
    s.status = ST_CONVERGED;
    s.phase = PH_DONE;
    return;
  }
  double slope = direction(C, s);
  s.pre = false;
  if (!(slope < 0.0)) {
    s.hc = 0;
    s.h0 = 0;
    slope = tl_pass<M_COPY, 2>(C, C.g, 0.0, nullptr, false);  // dir = -g
  }
  s.slope = slope;
  s.t = 1.0;
  s.trial = 0;
  s.fval = s.value;
  s.phase = PH_GEN;
}

template <bool F>
__device__ __forceinline__ void cand_batch(const Ctx& C, double t, int g0, double* acc, bool& fin) {
  double xv[kB], dv[kB], tv[kB];
  ldb<F>(C, C.x, g0, xv);
  ldb<F>(C, C.dir, g0, dv);
  ldb<F>(C, C.tau, g0, tv);
  double* co = C.cand + (long)g0 * kGS;
#pragma unroll
  for (int jj = 0; jj < kB; ++jj) {
    if (!gok<F>(C, g0 + jj)) continue;
    const double cv = xv[jj] + t * dv[jj];
    co[jj * kGS] = cv;
    fin = fin && isfinite(cv);
    acc[jj & 3] = fma(tv[jj], cv, acc[jj & 3]);
  }
}

// next finite candidate x + t dir of the backtracking line search, with
// tau . cand for its objective value
__device__ __forceinline__ void next_candidate(const Ctx& C, Solver& s) {
  while (s.trial < C.o.max_line_search) {
    const double t = s.t;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    bool fin = true;
    int g0 = 0;
    for (; g0 + kB <= C.nf; g0 += kB) cand_batch<true>(C, t, g0, acc, fin);
    for (; g0 < C.n8; g0 += kB) cand_batch<false>(C, t, g0, acc, fin);
    const double tdx = dot_finish(C, acc);
    if (__all_sync(C.em, fin)) {
      s.tdx = tdx;
      s.phase = PH_EVAL;
      return;
    }
    s.t *= C.o.backtrack_factor;
    ++s.trial;
  }
  s.status = ST_FAILED;  // no acceptable step
  if (s.itv && C.j == 0) s.itv[s.iters] = s.value;
  ++s.iters;
  s.phase = PH_DONE;
}

template <bool F>
__device__ __forceinline__ void acc_batch(const Ctx& C, double t, double* sv, double* yv, int g0, double* acc, double* asg,
                                          double* ayy, double& gm, double& xm) {
  double dv[kB], ev[kB], gv[kB], cv[kB];
  ldb<F>(C, C.dir, g0, dv);
  ldb<F>(C, C.evg, g0, ev);
  ldb<F>(C, C.g, g0, gv);
  ldb<F>(C, C.cand, g0, cv);
  const long o0 = (long)g0 * kGS;
#pragma unroll
  for (int jj = 0; jj < kB; ++jj) {
    if (!gok<F>(C, g0 + jj)) continue;
    const long o = o0 + jj * kGS;
    const double sj = t * dv[jj];
    const double yj = ev[jj] - gv[jj];
    sv[o] = sj;
    yv[o] = yj;
    C.x[o] = cv[jj];
    C.g[o] = ev[jj];
    acc[jj & 3] = fma(sj, yj, acc[jj & 3]);
    if (PBAD_C6_FUSE) {
      asg[jj & 3] = fma(sj, ev[jj], asg[jj & 3]);  // s . g(new): the copy pass's z . q
      ayy[jj & 3] = fma(yj, yj, ayy[jj & 3]);      // y . y: loop 1's DOT 1
    }
    gm = fmax(gm, fabs(ev[jj]));
    xm = fmax(xm, fabs(cv[jj]));
  }
}

// accepted step (optim.cpp:176-205) in one pass: s = t dir, y = evg - g,
// s . y, x = cand, g = evg, and the norms of the new iterate
__device__ __forceinline__ void accept_step(const Ctx& C, Solver& s, double v) {
  const int cap = C.o.mem + 1;
  const int slot = (s.h0 + s.hc) % cap;
  double* sv = C.hs + slot * C.VS;
  double* yv = C.hy + slot * C.VS;
  const double t = s.t;
  double acc[4] = {0.0, 0.0, 0.0, 0.0}, asg[4] = {0.0, 0.0, 0.0, 0.0}, ayy[4] = {0.0, 0.0, 0.0, 0.0};
  double gm = 0.0, xm = 0.0;
  int g0 = 0;
  for (; g0 + kB <= C.nf; g0 += kB) acc_batch<true>(C, t, sv, yv, g0, acc, asg, ayy, gm, xm);
  for (; g0 < C.n8; g0 += kB) acc_batch<false>(C, t, sv, yv, g0, acc, asg, ayy, gm, xm);
  const double sy = dot_finish(C, acc);
  s.pre = false;
  s.ginf = emax(C, gm);
  s.xinf = emax(C, xm);
  if (sy > 1e-12) {
    if (PBAD_C6_FUSE) {
      s.pre = true;
      s.pre_sg = dot_finish(C, asg);
      s.pre_yy = dot_finish(C, ayy);
    }
    if (C.j == 0) C.hsy[slot] = sy;
    ++s.hc;
    if (s.hc > C.o.mem) {
      s.h0 = (s.h0 + 1) % cap;
      --s.hc;
    }
  }
  esync(C);
  const double oldv = s.fval;
  s.value = v;
  ++s.acc;
  if (oldv - v <= C.o.ftol * fmax(1.0, fabs(oldv))) ++s.stag;
  else s.stag = 0;
  if (s.stag >= 2) s.status = ST_CONVERGED;
  if (s.itv && C.j == 0) s.itv[s.iters] = s.value;
  ++s.iters;
  if (s.status == ST_RUNNING && s.iters >= C.o.max_iters) s.status = ST_FAILED;
  s.phase = (s.status == ST_RUNNING) ? PH_DIR : PH_DONE;
}

template <int KW>
__device__ __forceinline__ Ctx make_ctx(const DModel& m, const DForces& f, const DSchedule& sc, const ChainLayout& L,
                                        double* cw, int* ci, long B, double* smem) {
  Ctx C;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  C.N = m.N;
  C.n = m.n;
  C.n8 = (m.n + 7) >> 3;
  C.nf = m.n >> 3;
  C.n4q = (m.n + 3) >> 2;
  C.e = lane >> 3;
  C.j = lane & 7;
  C.h = C.j >> 2;
  C.r = lane & 3;
  const long w = (long)blockIdx.x * KW + wib;
  C.ge = w * kE + C.e;
  C.B = B;
  C.valid = C.ge < B;
  C.em = 0xFFu << (lane & ~7);
  C.ws = smem + (long)wib * kWarpD;
  C.bar = reinterpret_cast<uint64_t*>(C.ws + kBar);
  C.mrec = smem + (long)KW * kWarpD;
  C.kind = reinterpret_cast<const int*>(C.mrec + 20L * m.N);
  C.roff = C.kind + m.N;
  C.rec = cw + L.rec + w * (long)C.roff[m.N];
  C.hist = cw + L.hist + w * (long)m.N * kE * kHistW;
  C.gh0 = cw + L.h0;
  C.gh1 = cw + L.h1;
  const long vl = w * (long)C.n8 * kGS + lane;
  C.x = cw + L.x + vl;
  C.g = cw + L.g + vl;
  C.cand = cw + L.cand + vl;
  C.dir = cw + L.dir + vl;
  C.q = cw + L.q + vl;
  C.evg = cw + L.evg + vl;
  C.tau = cw + L.tau + vl;
  C.hs = cw + L.hs + vl;
  C.hy = cw + L.hy + vl;
  C.VS = L.vstride;
  // per-env scalars; padded environments (ge >= B) point at env 0 and never write
  const long es = C.valid ? C.ge : 0;
  C.hsy = C.ws + kHsy + C.e * kHsyW;
  C.histc = cw + L.histc + es;
  C.ci = ci;
  C.dt = sc.dt;
  C.inv_dt2 = 1.0 / (sc.dt * sc.dt);
  C.wm = m.weighted_mass;
  C.gz[0] = f.gravity[0];
  C.gz[1] = f.gravity[1];
  C.gz[2] = f.gravity[2];
  C.gr = (C.r == 0) ? f.gravity[0] : (C.r == 1) ? f.gravity[1] : (C.r == 2) ? f.gravity[2] : 0.0;
  C.o = sc.opt;
  C.nload = 0;
  return C;
}

template <int KW>
__device__ __forceinline__ void stage(const DModel& m, double* smem) {
  double* rec = smem + (long)KW * kWarpD;
  int* kind = reinterpret_cast<int*>(rec + 20L * m.N);
  int* roff = kind + m.N;
  const double2* src = reinterpret_cast<const double2*>(m.crec);
  double2* dst = reinterpret_cast<double2*>(rec);
  for (int k = threadIdx.x; k < 10 * m.N; k += blockDim.x) dst[k] = __ldg(src + k);
  for (int k = threadIdx.x; k < m.N; k += blockDim.x) kind[k] = __ldg(m.ckind + k);
  // record offsets per 4-environment warp (the v4 offsets are per 8 environments)
  for (int k = threadIdx.x; k <= m.N; k += blockDim.x) roff[k] = __ldg(m.croff + k) / 2;
  if ((threadIdx.x & 31) == 0) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (long)(threadIdx.x >> 5) * kWarpD + kBar);
    for (int s = 0; s < kRing; ++s) mbar_init(bar + s);
    fence_mbar_init();
  }
  __syncthreads();
}

// One PBAD step for every environment of the warp: begin_step, L-BFGS to
// completion in lockstep rounds, finish_step (stepper.cpp:83-147).  A lane
// returns when its environment is done with the step.
template <int PAT>
__device__ __forceinline__ void env_step(Ctx& C, const DModel& m, const DForces& f, const DSchedule& sc, const Outputs& out) {
  // a warp with no running environment has nothing to do (warp-uniform exit)
  bool active = C.valid && ival(C, IS_RUN) == TR_RUNNING;
  if (!__any_sync(0xffffffffu, active)) return;
  const int n = m.n;
  const int step = C.valid ? ival(C, IS_STEP) : 0;
  if (active) {
    // StepObjective ctor validates the history (objective.cpp:176-177)
    if (!qallfinite(C, C.gh0) || !qallfinite(C, C.gh1)) {
      if (C.j == 0) ival(C, IS_RUN) = TR_NONFINITE_CFG;
      active = false;
    }
  }
  if (active) {
    // begin_step: actuation at the step end, warm start (stepper.cpp:83-115)
    tau_at(C, f, step * sc.dt + sc.times[2] * sc.dt);
    const double span = -sc.times[0];
    const double tau_m = sc.times[2];
    const bool ws = sc.warm_start != 0;
    for (int k = C.j; k < n; k += kL) {
      const double h1 = qv(C, C.gh1, k), h0 = qv(C, C.gh0, k);
      vat(C, C.x, k) = ws ? h1 + (tau_m / span) * (h1 - h0) : h1;
    }
    esync(C);
    hist_rotations_q(C, C.gh0, 0);
    hist_rotations_q(C, C.gh1, 1);
    const double hc = hist_const(C);
    if (C.j == 0) *C.histc = hc;
    esync(C);
    if (!eallfinite(C, C.x)) {
      if (C.j == 0) ival(C, IS_RUN) = TR_NONFINITE_CFG;
      active = false;
    }
  }
  __syncwarp();
  // LbfgsSolver ctor: first evaluation (warp-collective sweeps)
  Solver s{};
  s.status = ST_RUNNING;
  s.phase = PH_DIR;
  s.itv = (out.itv && C.valid) ? out.itv + out.rrow(C.ge, step) * out.itv_n : nullptr;
  double tdx0 = 0.0;
  if (active) {
    tdx0 = edot(C, C.tau, C.x);
    s.xinf = einfnorm(C, C.x);
  }
  __syncwarp();
  const double v0 = forward<PAT>(C, C.x, tdx0);
  reverse<PAT>(C, C.g);
  if (active && !isfinite(v0)) {
    if (C.j == 0) ival(C, IS_RUN) = TR_NONFINITE_INIT;
    active = false;
  }
  if (active) {
    s.value = v0;
    s.grad0 = einfnorm(C, C.g);
    s.ginf = s.grad0;
  } else {
    s.phase = PH_DONE;
  }
#ifdef PBAD_C6_STATS
  int st_eval = 0, st_acc = 0, st_acc0 = 0;
#endif
  for (;;) {
    if (s.phase == PH_DIR) begin_iteration(C, s);
    if (s.phase == PH_GEN) next_candidate(C, s);
    __syncwarp();
    const bool eval = s.phase == PH_EVAL;
    if (!__any_sync(0xffffffffu, eval)) break;
    const double v = forward<PAT>(C, C.cand, s.tdx);
    bool acc = false;
    if (eval) {
      if (isfinite(v) && v <= s.fval + C.o.armijo_c1 * s.t * s.slope && v < s.fval) {
        acc = true;
      } else {
        s.t *= C.o.backtrack_factor;
        ++s.trial;
        s.phase = PH_GEN;
      }
    }
    if (__any_sync(0xffffffffu, acc)) reverse<PAT>(C, C.evg);
#ifdef PBAD_C6_STATS
    if (eval) {
      ++st_eval;
      if (acc) {
        ++st_acc;
        if (s.trial == 0) ++st_acc0;
      }
    }
#endif
    if (acc) accept_step(C, s, v);
    __syncwarp();
  }
#ifdef PBAD_C6_STATS
  if (C.j == 0 && (C.ge % 512) == 0)
    printf("env %ld: evals %d accepted %d accepted-at-first-trial %d\n", C.ge, st_eval, st_acc, st_acc0);
#endif
  if (!active) return;
  // finish_step
  const bool converged = s.status == ST_CONVERGED;
  const double gnorm = einfnorm(C, C.g);
  if (C.j == 0) {
    if (out.iterations) out.iterations[out.rrow(C.ge, step)] = s.iters;
    if (out.converged) out.converged[out.rrow(C.ge, step)] = converged;
    if (out.accepted) out.accepted[out.rrow(C.ge, step)] = s.acc;
    if (out.final_value) out.final_value[out.rrow(C.ge, step)] = s.value;
    if (out.final_grad_norm) out.final_grad_norm[out.rrow(C.ge, step)] = gnorm;
    ival(C, IS_NREP) = step + 1;
  }
  const int fs = converged ? 0 : ival(C, IS_FAIL) + 1;
  esync(C);
  if (C.j == 0) ival(C, IS_FAIL) = fs;
  if (fs > sc.fail_limit) {
    if (C.j == 0) ival(C, IS_RUN) = TR_FAIL_LIMIT;
    return;
  }
  hist_rotations(C, C.x, 2);
  double ke, pe;
  step_energy(C, &ke, &pe);
  for (int k = C.j; k < n; k += kL) {
    const double xk = vat(C, C.x, k);
    qv(C, C.gh0, k) = qv(C, C.gh1, k);
    qv(C, C.gh1, k) = xk;
    if (out.q) out.q[out.qrow(C.ge, step + 1) * n + k] = xk;
  }
  if (C.j == 0) {
    if (out.energy) {
      out.energy[out.qrow(C.ge, step + 1) * 2] = ke;
      out.energy[out.qrow(C.ge, step + 1) * 2 + 1] = pe;
    }
    ival(C, IS_STEP) = step + 1;
    ival(C, IS_NSAMP) = step + 2;
    if (step + 1 >= sc.total_steps) ival(C, IS_RUN) = TR_OK;
  }
}

// nsteps PBAD steps in one launch (1 by default, launch_chain6_steps): a
// warp keeps its environments from step to step and runs its steps back to
// back, its TMA ring and mbarrier phases carrying over.
template <int PAT, int KW>
__global__ void __launch_bounds__(32 * KW) k_chain6_step(DModel m, DForces f, DSchedule sc, ChainLayout L,
                                                         double* cw, int* ci, long B, Outputs out, int nsteps) {
  extern __shared__ __align__(16) double smem[];
  stage<KW>(m, smem);
  Ctx C = make_ctx<KW>(m, f, sc, L, cw, ci, B, smem);
#pragma unroll 1
  for (int k = 0; k < nsteps; ++k) {
    __syncwarp();  // lanes that left the previous step early rejoin; its stores are visible to the warp
    env_step<PAT>(C, m, f, sc, out);
  }
}

template <int PAT, int KW>
cudaError_t launch_kw(const ChainArgs& a, const Outputs& out, int nsteps, cudaStream_t s) {
  const size_t sm = smem_bytes(a.m.N, KW);
  static SmemAttr attr_;
  size_t& configured = attr_.here();
  if (sm > configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_chain6_step<PAT, KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    configured = sm;
  }
  const long nw = (a.B + kE - 1) / kE;
  const unsigned grid = (unsigned)((nw + KW - 1) / KW);
  k_chain6_step<PAT, KW><<<grid, 32 * KW, sm, s>>>(a.m, a.f, a.sc, a.L, a.cw, a.ci, a.B, out, nsteps);
  return cudaGetLastError();
}

// Block size: the warps of the batch spread one block per SM where a block of
// 7 or 8 warps fits (shared model records, more L1), else blocks of 4 (two per
// SM).  PBAD_C6_WARPS = 4 / 7 / 8 forces one.
template <int PAT>
cudaError_t launch(const ChainArgs& a, const Outputs& out, int nsteps, cudaStream_t s) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  static const int forced = std::getenv("PBAD_C6_WARPS") ? std::atoi(std::getenv("PBAD_C6_WARPS")) : 0;
  const long nw = (a.B + kE - 1) / kE;
  int kw = forced;
  if (kw != 4 && kw != 7 && kw != 8) kw = nw <= 4L * sms ? 4 : nw <= 7L * sms ? 7 : 8;
  if (kw != 4 && smem_bytes(a.m.N, kw) > 227 * 1024) kw = 4;
  if (kw == 7) return launch_kw<PAT, 7>(a, out, nsteps, s);
  if (kw == 8) return launch_kw<PAT, 8>(a, out, nsteps, s);
  return launch_kw<PAT, 4>(a, out, nsteps, s);
}

constexpr int pat(int P, int K0, int K1) { return P | (K0 << 2) | (K1 << 5); }

}  // namespace c6

bool chain6_fits(int N, int mem) { return mem <= c6::kMaxMem && c6::smem_bytes(N, 4) <= 227 * 1024; }
// vector doubles per warp-group layout: ceil(B / 4) warps x ceil(n / 8) groups x 32
long chain6_vector_doubles(long B, int n) { return (B + c6::kE - 1) / c6::kE * (long)((n + 7) / 8) * c6::kGS; }

// One launch per step; with PBAD_C6_PERSIST=1 (A/B only) nsteps steps in one
// launch when the batch is one wave of resident warps (a warp then never
// waits on another).  Measured on C3: 93.4 vs 91.3 ms/step per step, so the
// per-step launches stay the default.  *launches: kernels
// launched.
cudaError_t launch_chain6_steps(const ChainArgs& a, int pattern, const Outputs& out, int nsteps, cudaStream_t s,
                                long* launches) {
  static const bool persist = std::getenv("PBAD_C6_PERSIST") && std::atoi(std::getenv("PBAD_C6_PERSIST")) == 1;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  // one wave: blocks of at most 8 warps, one block per SM (c6::launch)
  const bool one_wave = (a.B + c6::kE - 1) / c6::kE <= 8L * sms;
  const int per = (persist && one_wave) ? nsteps : 1;
  for (int k = 0; k < nsteps; k += per) {
    const int cnt = std::min(per, nsteps - k);
    cudaError_t e;
    switch (pattern) {
      case c6::pat(1, 6, 0): e = c6::launch<c6::pat(1, 6, 0)>(a, out, cnt, s); break;
      case c6::pat(2, 3, 6): e = c6::launch<c6::pat(2, 3, 6)>(a, out, cnt, s); break;
      default: e = c6::launch<0>(a, out, cnt, s); break;
    }
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  return cudaSuccess;
}

}  // namespace pbad_gpu
