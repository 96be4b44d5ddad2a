// pbad_chain.cu -- "quad" kernels for serial hinge chains (energy form, L-BFGS).
//
// Mapping: four lanes per environment ("quad"); lane r owns row r of every
// 4x4 transform (lane 3 carries the constant bottom row [0 0 0 1], which
// makes its contributions to the row-partial ddots come out exactly as the
// reference's).  Eight environments per warp.  Under the numeric contract
// everything the reference does per link is row-local:
//   FK          T_i[r,:]  = T_{i-1}[r,:] * L_i            (kinematics.cpp:171-181)
//   energy      ddot(A_i S_i, B_i) row partials           (adjoint.cpp:113-120)
//   seeds       ((T - 2T_k) + T_{k-1}) S / dt^2 per row   (objective.cpp:241-249)
//   lever       T_{i-1}[r,:] * dL_i/dq                    (adjoint.cpp:22-25)
//   adjoint     adj_{i-1}[r,:] = seed + adj_i[r,:] L_i^T  (adjoint.cpp:49-64)
// so the bit-exact serial recursions run on the row lanes with no data
// exchange; the per-link scalar reductions are batched through shared memory
// eight links at a time.  The forward sweep stores seeds, levers and joint
// rotations for the reverse (adjoint) sweep.  The L-BFGS vectors
// (optim.cpp:141-232) are quad-interleaved: element k of an environment lives
// on lane k%4, and the 32-partial dot of the numeric contract maps to eight
// partials per lane plus a two-level quad reduction.
//
// Performance structure: all addressing is per-lane base pointers plus
// strides kept in registers; per-link model data is one packed record read
// through the read-only path; the joint rotation of link i+1 (sqrt, sincos,
// two divisions: the longest dependent chain) is computed while link i's
// products run.
#include <cuda_runtime.h>

#include "pbad_kernels.cuh"
#include "pbad_launch.h"
#include "pbad_math.cuh"

namespace pbad_gpu {

namespace {

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_FAILED = 2 };
enum { TR_OK = 0, TR_FAIL_LIMIT = 1, TR_NONFINITE_INIT = 2, TR_NONFINITE_CFG = 3, TR_RUNNING = 4 };

constexpr int kEnvsPerWarp = 8;
constexpr int kWarpsPerBlock = 2;
constexpr int kThreads = 32 * kWarpsPerBlock;
constexpr int kEnvsPerBlock = kEnvsPerWarp * kWarpsPerBlock;
constexpr int kMaxMem = 16;
constexpr int kChunk = 8;          // links per shared-memory reduction batch
constexpr int kRed = kChunk * 16;  // doubles of reduction scratch per quad
constexpr int kU = 8;              // vector-loop unroll (groups per batch)
// Per-warp blocks of 8 environments with compile-time strides:
//   link arrays [warp][N][32 lanes][4]  -> link i of a lane at +kLS*i
//   vectors     [warp][n4][32 lanes]    -> group g of a lane at +kGS*g
constexpr long kLS = 128;
constexpr long kGS = 32;
#ifndef PBAD_CHAIN_PREFETCH_HIST
#define PBAD_CHAIN_PREFETCH_HIST 1
#endif

__device__ __forceinline__ void ld4(const double* p, double* v) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void st4(double* p, const double* v) {
  *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
}

// row of (a * B)
__device__ __forceinline__ void row_mul(const double* a, const M4& B, double* out) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double acc = a[0] * B.a[4 * c];
    acc = fma(a[1], B.a[1 + 4 * c], acc);
    acc = fma(a[2], B.a[2 + 4 * c], acc);
    acc = fma(a[3], B.a[3 + 4 * c], acc);
    out[c] = acc;
  }
}
// row of (a * S) with S a packed column-major record
__device__ __forceinline__ void row_mul_rec(const double* a, const double* S, double* out) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double acc = a[0] * S[4 * c];
    acc = fma(a[1], S[1 + 4 * c], acc);
    acc = fma(a[2], S[2 + 4 * c], acc);
    acc = fma(a[3], S[3 + 4 * c], acc);
    out[c] = acc;
  }
}
// row of (a * B^T)
__device__ __forceinline__ void row_mul_bt(const double* a, const M4& B, double* out) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double acc = a[0] * B.a[c];
    acc = fma(a[1], B.a[c + 4], acc);
    acc = fma(a[2], B.a[c + 8], acc);
    acc = fma(a[3], B.a[c + 12], acc);
    out[c] = acc;
  }
}

// row r of M without dynamic register indexing (keeps M out of local memory)
__device__ __forceinline__ void get_row(const M4& M, int r, double* v) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double a0 = M.a[4 * c], a1 = M.a[4 * c + 1], a2 = M.a[4 * c + 2], a3 = M.a[4 * c + 3];
    v[c] = (r == 0) ? a0 : (r == 1) ? a1 : (r == 2) ? a2 : a3;
  }
}

__device__ __forceinline__ void identity_row(int r, double* v) {
  v[0] = (r == 0) ? 1.0 : 0.0;
  v[1] = (r == 1) ? 1.0 : 0.0;
  v[2] = (r == 2) ? 1.0 : 0.0;
  v[3] = (r == 3) ? 1.0 : 0.0;
}

// --- per-link joint algebra ----------------------------------------------
// L = offset * [R(axis*q) 0; 0 1], d1 = offset * embed([axis]x R)
// (kinematics.cpp:119-129).  jk 1/2/3: axis exactly e_x/e_y/e_z and offset
// rotation block exactly I: R = I + A K + B K^2 then has two free entries
// (c, s) and each canonical product reduces to its non-zero terms (the
// dropped terms are fma(x, +-0, acc) with finite x: value unchanged).

// rotation_coeffs A, B (kinematics.cpp:20-45) for a unit-axis hinge angle q:
// n = sqrt(q*q); -K^2 has diagonal entries k2 = q*q.
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
  *s = A * q;         // (0 + A*K_ab) + B*(+-0)
  *c = 1.0 - B * k2;  // (1 + A*0) + B*(-k2)
}

struct GenJet {
  M4 L, d1;
};

__device__ __forceinline__ void general_jet(const DModel& m, int i, double qi, bool want_d1, GenJet* J) {
  const double* ax = m.axis + 3 * i;
  const double a0 = __ldg(ax), a1 = __ldg(ax + 1), a2 = __ldg(ax + 2);
  M4 o;
#pragma unroll
  for (int k = 0; k < 16; ++k) o.a[k] = __ldg(m.offset + 16 * i + k);
  const M3 R = rotation_vector_matrix(a0 * qi, a1 * qi, a2 * qi);
  J->L = mul(o, motion_rot(R));
  if (want_d1) J->d1 = mul(o, embed_rotation(mul3(skew(a0, a1, a2), R)));
}

// translation column: ((T0*t0 + T1*t1) + T2*t2) + T3
__device__ __forceinline__ double trans_col(const double* T, const double* t) {
  double acc = T[0] * t[0];
  acc = fma(T[1], t[1], acc);
  acc = fma(T[2], t[2], acc);
  return acc + T[3];
}

// row of (T * L): world = parent_world * value
__device__ __forceinline__ void fk_row(int jk, double c, double s, const double* t, const GenJet& G, const double* T,
                                       double* Tn) {
  switch (jk) {
    case 1:  // R = [1 0 0; 0 c -s; 0 s c]
      Tn[0] = T[0];
      Tn[1] = fma(T[2], s, T[1] * c);
      Tn[2] = fma(T[2], c, T[1] * (-s));
      Tn[3] = trans_col(T, t);
      return;
    case 2:  // R = [c 0 s; 0 1 0; -s 0 c]
      Tn[0] = fma(T[2], -s, T[0] * c);
      Tn[1] = T[1];
      Tn[2] = fma(T[2], c, T[0] * s);
      Tn[3] = trans_col(T, t);
      return;
    case 3:  // R = [c -s 0; s c 0; 0 0 1]
      Tn[0] = fma(T[1], s, T[0] * c);
      Tn[1] = fma(T[1], c, T[0] * (-s));
      Tn[2] = T[2];
      Tn[3] = trans_col(T, t);
      return;
    default:
      row_mul(T, G.L, Tn);
  }
}

// row of (T * d1): lever = parent_world * dL/dq; the specialised kinds keep
// their two non-zero columns in lev[0..1]
__device__ __forceinline__ void lever_row(int jk, double c, double s, const GenJet& G, const double* T, double* lev) {
  switch (jk) {
    case 1:  // [a]x R rows: 0; (0,-s,-c); (0,c,-s)        -> columns 1, 2
      lev[0] = fma(T[2], c, T[1] * (-s));
      lev[1] = fma(T[2], -s, T[1] * (-c));
      return;
    case 2:  // rows: (-s,0,c); 0; (-c,0,-s)                -> columns 0, 2
      lev[0] = fma(T[2], -c, T[0] * (-s));
      lev[1] = fma(T[2], -s, T[0] * c);
      return;
    case 3:  // rows: (-s,-c,0); (c,-s,0); 0                 -> columns 0, 1
      lev[0] = fma(T[1], c, T[0] * (-s));
      lev[1] = fma(T[1], -s, T[0] * (-c));
      return;
    default:
      row_mul(T, G.d1, lev);
  }
}

// ddot_row(lever_row, a) with the lever's zero columns dropped
__device__ __forceinline__ double lever_dot(int jk, const double* lev, const double* a) {
  switch (jk) {
    case 1: return fma(lev[1], a[2], lev[0] * a[1]);
    case 2: return fma(lev[1], a[2], lev[0] * a[0]);
    case 3: return fma(lev[1], a[1], lev[0] * a[0]);
    default: return ddot_row(lev, a);
  }
}

// row of (a * L^T): adjoint transport to the parent
__device__ __forceinline__ void transport_row(int jk, double c, double s, const double* t, const M4& L,
                                              const double* a, double* o) {
  switch (jk) {
    case 1:  // L rows (1,0,0,t0) (0,c,-s,t1) (0,s,c,t2)
      o[0] = fma(a[3], t[0], a[0]);
      o[1] = fma(a[3], t[1], fma(a[2], -s, a[1] * c));
      o[2] = fma(a[3], t[2], fma(a[2], c, a[1] * s));
      o[3] = a[3];
      return;
    case 2:  // (c,0,s,t0) (0,1,0,t1) (-s,0,c,t2)
      o[0] = fma(a[3], t[0], fma(a[2], s, a[0] * c));
      o[1] = fma(a[3], t[1], a[1]);
      o[2] = fma(a[3], t[2], fma(a[2], c, a[0] * (-s)));
      o[3] = a[3];
      return;
    case 3:  // (c,-s,0,t0) (s,c,0,t1) (0,0,1,t2)
      o[0] = fma(a[3], t[0], fma(a[1], -s, a[0] * c));
      o[1] = fma(a[3], t[1], fma(a[1], c, a[0] * s));
      o[2] = fma(a[3], t[2], a[2]);
      o[3] = a[3];
      return;
    default:
      row_mul_bt(a, L, o);
  }
}

// --- the per-quad context (register resident) ------------------------------
struct CK {
  DModel m;  // by value: taking a kernel parameter's address forces a local copy
  DOpt o;
  int N, n, n4, r;
  long B, e;
  unsigned qm;
  double* red;  // shared reduction scratch of this quad (kRed doubles)
  const double* rec;  // shared copy of the packed link records [N][20]
  const int* kind;    // shared copy of the link kinds [N]
  double* cw;
  int* ci;
  // link arrays: row r of link 0 of this env; link i at +i*LS
  double *tk, *tk1, *seed, *lev, *lmat, *lmat0;
  // vectors: this lane's group g at V + g*GS
  double *h0, *h1, *x, *g, *cand, *dir, *q, *evg, *tau, *hs, *hy;
  long VS;
  double* hsy;    // [cap][B]: this env at hsy[slot*B]
  double* histc;  // this env
  double wm, dt, inv_dt2;
  double gz[3];
};

__device__ __forceinline__ double qshfl(const CK& K, double v, int src) { return __shfl_sync(K.qm, v, src, 4); }
__device__ __forceinline__ void qsync(const CK& K) { __syncwarp(K.qm); }
__device__ __forceinline__ int& ival(const CK& K, int slot) { return K.ci[(long)slot * K.B + K.e]; }

// Dynamic shared memory: per-quad reduction scratch, then the packed link
// records and kinds (read by every lane at every link of every sweep: keeping
// them out of the L1/L2 path removes the dependent global load per link).
__host__ __device__ constexpr long smem_red_doubles() { return (long)kRed * kEnvsPerBlock; }
__host__ __device__ inline size_t chain_smem_bytes(int N) {
  return (size_t)(smem_red_doubles() + 20L * N) * sizeof(double) + (size_t)N * sizeof(int);
}
__device__ __forceinline__ void stage_model(const DModel& m, double* smem) {
  double* rec = smem + smem_red_doubles();
  int* kind = reinterpret_cast<int*>(rec + 20L * m.N);
  const double2* src = reinterpret_cast<const double2*>(m.crec);
  double2* dst = reinterpret_cast<double2*>(rec);
  for (int k = threadIdx.x; k < 10 * m.N; k += blockDim.x) dst[k] = __ldg(src + k);
  for (int k = threadIdx.x; k < m.N; k += blockDim.x) kind[k] = __ldg(m.ckind + k);
  __syncthreads();
}

__device__ __forceinline__ CK make_ck(const DModel& m, const DForces& f, const DSchedule& sc, const ChainLayout& L,
                                      double* cw, int* ci, long B, double* smem, bool* valid) {
  double* red_base = smem;
  CK K;
  const int lane = threadIdx.x & 31;
  const int quad_in_block = threadIdx.x >> 2;
  K.m = m;
  K.o = sc.opt;
  K.e = (long)blockIdx.x * kEnvsPerBlock + quad_in_block;
  *valid = K.e < B;
  K.r = lane & 3;
  K.qm = 0xFu << (lane & ~3);
  K.red = red_base + kRed * quad_in_block;
  K.rec = smem + smem_red_doubles();
  K.kind = reinterpret_cast<const int*>(K.rec + 20L * m.N);
  K.N = m.N;
  K.n = m.n;
  K.n4 = (m.n + 3) >> 2;
  K.B = B;
  K.cw = cw;
  K.ci = ci;
  const long w = K.e >> 3;
  const long lbase = w * (long)m.N * kLS + 4 * lane;
  K.tk = cw + L.tk + lbase;
  K.tk1 = cw + L.tk1 + lbase;
  K.seed = cw + L.seed + lbase;
  K.lev = cw + L.lev + lbase;
  K.lmat = cw + L.lmat + lbase;
  K.lmat0 = cw + L.lmat + w * (long)m.N * kLS + 4 * (lane & ~3);
  const long vl = w * (long)K.n4 * kGS + lane;
  K.h0 = cw + L.h0 + vl;
  K.h1 = cw + L.h1 + vl;
  K.x = cw + L.x + vl;
  K.g = cw + L.g + vl;
  K.cand = cw + L.cand + vl;
  K.dir = cw + L.dir + vl;
  K.q = cw + L.q + vl;
  K.evg = cw + L.evg + vl;
  K.tau = cw + L.tau + vl;
  K.hs = cw + L.hs + vl;
  K.hy = cw + L.hy + vl;
  K.VS = L.vstride;
  K.hsy = cw + L.hsy + K.e;
  K.histc = cw + L.histc + K.e;
  K.wm = m.weighted_mass;
  K.dt = sc.dt;
  K.inv_dt2 = 1.0 / (sc.dt * sc.dt);
  K.gz[0] = f.gravity[0];
  K.gz[1] = f.gravity[1];
  K.gz[2] = f.gravity[2];
  return K;
}

// element k (owned by any lane of the quad) of vector V
__device__ __forceinline__ double& vat(const CK& K, double* V, int k) {
  return V[(long)(k >> 2) * kGS + ((k & 3) - K.r)];
}

// --- vector ops (quad-interleaved, 32-partial canonical dot) --------------
// groups [0, nfull) are complete for every lane; the last group may be ragged
__device__ __forceinline__ int full_groups(const CK& K) { return K.n >> 2; }

__device__ __forceinline__ double qdot(const CK& K, const double* A, const double* Bv) {
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.0;
  const long GS = kGS;
  const int nf = full_groups(K);
  int g0 = 0;
  for (; g0 + kU <= nf; g0 += kU) {
    double a[kU], b[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      a[j] = A[(g0 + j) * GS];
      b[j] = Bv[(g0 + j) * GS];
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) acc[j] = fma(a[j], b[j], acc[j]);  // (g0+j)&7 == j
  }
  for (int gg = g0; gg < K.n4; ++gg) {
    if (4 * gg + K.r < K.n) acc[gg & 7] = fma(A[gg * GS], Bv[gg * GS], acc[gg & 7]);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = acc[j] + acc[j + 4];
  acc[0] = acc[0] + acc[2];
  acc[1] = acc[1] + acc[3];
  double v = acc[0] + acc[1];
  const double v2 = qshfl(K, v, (K.r + 2) & 3);
  if (K.r < 2) v = v + v2;
  const double v1 = qshfl(K, v, 1);
  if (K.r == 0) v = v + v1;
  return qshfl(K, v, 0);
}

// dst[k] = f(a[k], b[k]): eight groups of loads before any store
template <class F>
__device__ __forceinline__ void qmap2(const CK& K, double* dst, const double* A, const double* Bv, F f) {
  const long GS = kGS;
  const int nf = full_groups(K);
  int g0 = 0;
  for (; g0 + kU <= nf; g0 += kU) {
    double a[kU], b[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      a[j] = A[(g0 + j) * GS];
      b[j] = Bv[(g0 + j) * GS];
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) dst[(g0 + j) * GS] = f(a[j], b[j]);
  }
  for (int gg = g0; gg < K.n4; ++gg)
    if (4 * gg + K.r < K.n) dst[gg * GS] = f(A[gg * GS], Bv[gg * GS]);
}

__device__ __forceinline__ double qinfnorm(const CK& K, const double* A) {
  double mx = 0.0;
  const long GS = kGS;
  for (int g0 = 0; g0 < K.n4; g0 += kU) {
    double a[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int gg = g0 + j;
      a[j] = (gg < K.n4 && 4 * gg + K.r < K.n) ? A[gg * GS] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) mx = fmax(mx, fabs(a[j]));
  }
  mx = fmax(mx, qshfl(K, mx, K.r ^ 1));
  mx = fmax(mx, qshfl(K, mx, K.r ^ 2));
  return mx;
}
__device__ __forceinline__ bool qallfinite(const CK& K, const double* A) {
  bool ok = true;
  const long GS = kGS;
  for (int g0 = 0; g0 < K.n4; g0 += kU) {
    double a[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int gg = g0 + j;
      a[j] = (gg < K.n4 && 4 * gg + K.r < K.n) ? A[gg * GS] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) ok = ok && isfinite(a[j]);
  }
  return __all_sync(K.qm, ok);
}

// --- link records -----------------------------------------------------------
struct Rec {
  double S[16];
  double t[3];
};
__device__ __forceinline__ void load_rec(const CK& K, int i, Rec* R, bool want_S) {
  const double* p = K.rec + 20 * i;
  if (want_S) {
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      const double2 v = *reinterpret_cast<const double2*>(p + k);
      R->S[k] = v.x;
      R->S[k + 1] = v.y;
    }
  }
  const double2 t01 = *reinterpret_cast<const double2*>(p + 16);
  R->t[0] = t01.x;
  R->t[1] = t01.y;
  R->t[2] = p[18];
}

// --- forward kinematics of a configuration into a link array ---------------
// forward_pass (kinematics.cpp:171-181): the root's world is its local transform
__device__ __forceinline__ void chain_fk(const CK& K, double* V, double* dst) {
  const DModel& m = K.m;
  double T[4];
  identity_row(K.r, T);
  double* d = dst;
  for (int i = 0; i < K.N; ++i, d += kLS) {
    const int kind = K.kind[i];
    const int jk = kind & 3;
    const double qi = vat(K, V, i);
    Rec R;
    load_rec(K, i, &R, false);
    double c = 0.0, s = 0.0;
    GenJet G;
    if (jk) hinge_cs(qi, &c, &s);
    else general_jet(m, i, qi, false, &G);
    double Tn[4];
    fk_row(jk, c, s, R.t, G, T, Tn);
#pragma unroll
    for (int k = 0; k < 4; ++k) T[k] = Tn[k];
    st4(d, T);
  }
}

// correlation_value(A, B) over two link arrays (adjoint.cpp:113-120)
__device__ __forceinline__ double chain_cv(const CK& K, const double* A, const double* Bw) {
  double v = 0.0;
  for (int i = 0; i < K.N; ++i) {
    double a[4], b[4], as[4];
    ld4(A + i * kLS, a);
    ld4(Bw + i * kLS, b);
    Rec R;
    load_rec(K, i, &R, true);
    row_mul_rec(a, R.S, as);
    qsync(K);
    K.red[K.r] = ddot_row(as, b);
    qsync(K);
    v += ((K.red[0] + K.red[1]) + K.red[2]) + K.red[3];
  }
  return v - K.wm;
}

// --- the evaluation ---------------------------------------------------------
// Forward sweep at vector X (StepObjective::value, objective.cpp:215-239),
// storing seeds / levers / joint rotations for the reverse sweep when store.
// Per-link row partials of the four energy terms are reduced eight links at a
// time: lane t sums term t ((p0+p1)+p2)+p3 link after link (serial order).
__device__ __forceinline__ double chain_forward(const CK& K, double* X, bool store) {
  const DModel& m = K.m;
  const int N = K.N;
  const double inv_dt2 = K.inv_dt2;
  const double gr = (K.r == 0) ? K.gz[0] : (K.r == 1) ? K.gz[1] : (K.r == 2) ? K.gz[2] : 0.0;
  // phase A (link-parallel): the joint rotations (c, s) of all specialised
  // links; lane r owns links r, r+4, ... (its own elements of X), two at a
  // time for ILP.  Stored where the reverse sweep reads them.
  for (int g0 = 0; g0 < K.n4; g0 += 2) {
    const int i0 = 4 * g0 + K.r, i1 = i0 + 4;
    const bool ok0 = i0 < N, ok1 = g0 + 1 < K.n4 && i1 < N;
    const int k0 = ok0 ? K.kind[i0] : 0, k1 = ok1 ? K.kind[i1] : 0;
    const double q0 = ok0 ? X[(long)g0 * kGS] : 0.0, q1 = ok1 ? X[(long)(g0 + 1) * kGS] : 0.0;
    double c0, s0, c1, s1;
    hinge_cs(q0, &c0, &s0);
    hinge_cs(q1, &c1, &s1);
    if (ok0 && (k0 & 3)) *reinterpret_cast<double2*>(K.lmat0 + (long)i0 * kLS) = make_double2(c0, s0);
    if (ok1 && (k1 & 3)) *reinterpret_cast<double2*>(K.lmat0 + (long)i1 * kLS) = make_double2(c1, s1);
  }
  qsync(K);
  // phase B (serial over links): FK, levers, energy-term row partials, seeds
  double T[4];
  identity_row(K.r, T);
  double sum = 0.0;  // lane t: running sum of term t
  int nchunk = 0;
  int kind_n = K.kind[0];
  double2 cs_n = (kind_n & 3) ? *reinterpret_cast<const double2*>(K.lmat0) : make_double2(0.0, 0.0);
  long off = 0;
  // history rows of the next mass link, loaded one link ahead
  double tk_n[4] = {0.0, 0.0, 0.0, 0.0}, tk1_n[4] = {0.0, 0.0, 0.0, 0.0};
  if (kind_n >> 2) {
    ld4(K.tk, tk_n);
    ld4(K.tk1, tk1_n);
  }
  for (int i = 0; i < N; ++i, off += kLS) {
    const int kind = kind_n;
    const int jk = kind & 3, sk = kind >> 2;
    const double c = cs_n.x, s = cs_n.y;
    double tk[4], tk1[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      tk[k] = tk_n[k];
      tk1[k] = tk1_n[k];
    }
    if (!PBAD_CHAIN_PREFETCH_HIST && sk) {
      ld4(K.tk + off, tk);
      ld4(K.tk1 + off, tk1);
    }
    if (i + 1 < N) {
      kind_n = K.kind[i + 1];
      if (kind_n & 3) cs_n = *reinterpret_cast<const double2*>(K.lmat0 + off + kLS);
      if (PBAD_CHAIN_PREFETCH_HIST && (kind_n >> 2)) {
        ld4(K.tk + off + kLS, tk_n);
        ld4(K.tk1 + off + kLS, tk1_n);
      }
    }
    Rec R;
    load_rec(K, i, &R, sk != 0);
    GenJet G;
    if (!jk) general_jet(m, i, vat(K, X, i), store, &G);
    if (store) {
      double lv[4];
      lever_row(jk, c, s, G, T, lv);
      if (jk) {
        *reinterpret_cast<double2*>(K.lev + off) = make_double2(lv[0], lv[1]);
      } else {
        st4(K.lev + off, lv);
        double lr[4];
        get_row(G.L, K.r, lr);
        st4(K.lmat + off, lr);
      }
    }
    double Tn[4];
    fk_row(jk, c, s, R.t, G, T, Tn);
#pragma unroll
    for (int k = 0; k < 4; ++k) T[k] = Tn[k];
    if (sk) {
      double ts[4], p1[4], p2[4], cg[4];
      row_mul_rec(T, R.S, ts);
      row_mul_rec(tk, R.S, p1);
      row_mul_rec(tk1, R.S, p2);
#pragma unroll
      for (int k = 0; k < 4; ++k) cg[k] = (-gr) * R.S[12 + k];  // -ghat u^T, u = S e4
      double* slot = K.red + 16 * nchunk + 4 * K.r;
      const double pa = ddot_row(ts, T), pb = ddot_row(p1, T), pc = ddot_row(p2, T), pg = ddot_row(cg, T);
      *reinterpret_cast<double2*>(slot) = make_double2(pa, pb);
      *reinterpret_cast<double2*>(slot + 2) = make_double2(pc, pg);
      ++nchunk;
      if (store) {
        double dd[4], sd[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          dd[k] = T[k] - 2.0 * tk[k];
          dd[k] = dd[k] + tk1[k];
          dd[k] = inv_dt2 * dd[k];
        }
        row_mul_rec(dd, R.S, sd);
        st4(K.seed + off, sd);
      }
    }
    if (nchunk == kChunk || (i + 1 == N && nchunk > 0)) {
      qsync(K);
      for (int j = 0; j < nchunk; ++j) {
        const double* b = K.red + 16 * j + K.r;  // term K.r of link j, rows 0..3
        sum += ((b[0] + b[4]) + b[8]) + b[12];
      }
      qsync(K);
      nchunk = 0;
    }
  }
  const double sa = qshfl(K, sum, 0), sb = qshfl(K, sum, 1), sc2 = qshfl(K, sum, 2), sg = qshfl(K, sum, 3);
  const double wm = K.wm;
  const double cpp = sa - wm, c1p = sb - wm, c2p = sc2 - wm;
  const double inertial = 0.5 * inv_dt2 * (cpp - 4.0 * c1p + 2.0 * c2p + *K.histc);
  const double tdx = qdot(K, K.tau, X);
  return inertial + sg - tdx;
}

// Reverse sweep (functional_grad twice, adjoint.cpp:49-64): gradient =
// (inertial adjoint + gravity adjoint) - tau into Gv (objective.cpp:241-250).
// Per-link row partials are reduced eight links at a time; lane k writes the
// gradient entries it owns (index % 4 == k).
__device__ __forceinline__ void chain_reverse(const CK& K, double* Gv) {
  const int N = K.N;
  const double gr = (K.r == 0) ? K.gz[0] : (K.r == 1) ? K.gz[1] : (K.r == 2) ? K.gz[2] : 0.0;
  double cI[4] = {0.0, 0.0, 0.0, 0.0}, cG[4] = {0.0, 0.0, 0.0, 0.0};
  // loads one link ahead
  long off = (long)(N - 1) * kLS;
  int kind_n = K.kind[N - 1];
  double lev_n[4] = {0.0, 0.0, 0.0, 0.0}, seed_n[4] = {0.0, 0.0, 0.0, 0.0}, cs_n[2] = {0.0, 0.0};
  auto fetch = [&](int kind, long o, double* lv, double* sd, double* cs) {
    if (kind & 3) {
      const double2 v = *reinterpret_cast<const double2*>(K.lev + o);
      lv[0] = v.x;
      lv[1] = v.y;
      const double2 w = *reinterpret_cast<const double2*>(K.lmat0 + o);
      cs[0] = w.x;
      cs[1] = w.y;
    } else {
      ld4(K.lev + o, lv);
    }
    if (kind >> 2) ld4(K.seed + o, sd);
  };
  fetch(kind_n, off, lev_n, seed_n, cs_n);
  int nchunk = 0, chunk_top = N - 1;
  for (int i = N - 1; i >= 0; --i, off -= kLS) {
    const int kind = kind_n;
    const int jk = kind & 3, sk = kind >> 2;
    double lv[4], sd[4], cs[2];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      lv[k] = lev_n[k];
      sd[k] = seed_n[k];
    }
    cs[0] = cs_n[0];
    cs[1] = cs_n[1];
    if (i > 0) {
      kind_n = K.kind[i - 1];
      fetch(kind_n, off - kLS, lev_n, seed_n, cs_n);
    }
    double aI[4], aG[4];
    if (sk) {
      const double* p = K.rec + 20 * i + 12;
      const double2 u01 = *reinterpret_cast<const double2*>(p);
      const double2 u23 = *reinterpret_cast<const double2*>(p + 2);
      const double u[4] = {u01.x, u01.y, u23.x, u23.y};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        aI[k] = cI[k] + sd[k];
        aG[k] = cG[k] + (0.0 + (-gr) * u[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        aI[k] = cI[k];
        aG[k] = cG[k];
      }
    }
    double* slot = K.red + 8 * nchunk + 2 * K.r;
    *reinterpret_cast<double2*>(slot) = make_double2(lever_dot(jk, lv, aI), lever_dot(jk, lv, aG));
    ++nchunk;
    if (nchunk == kChunk || i == 0) {
      qsync(K);
      // links chunk_top - j for j in [0, nchunk)
      for (int j = 0; j < nchunk; ++j) {
        const int li = chunk_top - j;
        if ((li & 3) == K.r) {
          const double* b = K.red + 8 * j;
          const double gi = 0.0 + (((b[0] + b[2]) + b[4]) + b[6]);
          const double gp = 0.0 + (((b[1] + b[3]) + b[5]) + b[7]);
          vat(K, Gv, li) = (gi + gp) - vat(K, K.tau, li);
        }
      }
      qsync(K);
      nchunk = 0;
      chunk_top = i - 1;
    }
    if (i > 0) {
      double t3[3] = {0.0, 0.0, 0.0};
      M4 Lg;
      if (jk) {
        const double* p = K.rec + 20 * i + 16;
        const double2 t01 = *reinterpret_cast<const double2*>(p);
        t3[0] = t01.x;
        t3[1] = t01.y;
        t3[2] = p[2];
      } else {
        double rows[16];
        ld4(K.lmat0 + off, rows);
        ld4(K.lmat0 + off + 4, rows + 4);
        ld4(K.lmat0 + off + 8, rows + 8);
        ld4(K.lmat0 + off + 12, rows + 12);
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
          for (int k = 0; k < 4; ++k) Lg.a[rr + 4 * k] = rows[4 * rr + k];
      }
      double tI[4], tG[4];
      transport_row(jk, cs[0], cs[1], t3, Lg, aI, tI);
      transport_row(jk, cs[0], cs[1], t3, Lg, aG, tG);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cI[k] = 0.0 + tI[k];
        cG[k] = 0.0 + tG[k];
      }
    }
  }
  qsync(K);
}

// --- optimizer (LbfgsSolver, optim.cpp:141-232) -----------------------------
struct SolverState {
  double value, grad0;
  int status, iters, stag, acc, h0, hc;
  double* itv;  // per_iteration_values row of this step (lane 0 writes), or null
};

__device__ __forceinline__ bool grad_converged(const CK& K, const SolverState& s) {
  const DOpt& o = K.o;
  const double g = qinfnorm(K, K.g);
  if (g <= o.grad_tol * fmax(1.0, qinfnorm(K, K.x))) return true;
  if (o.grad_rtol > 0.0 && g <= o.grad_rtol * s.grad0) return true;
  return false;
}
__device__ __forceinline__ bool stagnation_update(const CK& K, SolverState& s, double oldv, double newv) {
  if (oldv - newv <= K.o.ftol * fmax(1.0, fabs(oldv))) ++s.stag;
  else s.stag = 0;
  return s.stag >= 2;
}

// two_loop (optim.cpp:213-229): q = H g
__device__ __forceinline__ void two_loop(const CK& K, const SolverState& s) {
  const int cap = K.o.mem + 1;
  qmap2(K, K.q, K.g, K.g, [](double a, double) { return a; });
  double alpha[kMaxMem];
  for (int i = s.hc - 1; i >= 0; --i) {
    const int slot = (s.h0 + i) % cap;
    const double* sv = K.hs + slot * K.VS;
    const double* yv = K.hy + slot * K.VS;
    const double a = qdot(K, sv, K.q) / K.hsy[slot * K.B];
    alpha[i] = a;
    qmap2(K, K.q, K.q, yv, [a](double qv, double y) { return qv - a * y; });
  }
  if (s.hc > 0) {
    const int slot = (s.h0 + s.hc - 1) % cap;
    const double* yv = K.hy + slot * K.VS;
    const double scl = K.hsy[slot * K.B] / qdot(K, yv, yv);
    qmap2(K, K.q, K.q, K.q, [scl](double qv, double) { return qv * scl; });
  }
  for (int i = 0; i < s.hc; ++i) {
    const int slot = (s.h0 + i) % cap;
    const double* sv = K.hs + slot * K.VS;
    const double* yv = K.hy + slot * K.VS;
    const double beta = qdot(K, yv, K.q) / K.hsy[slot * K.B];
    const double c = alpha[i] - beta;
    qmap2(K, K.q, K.q, sv, [c](double qv, double sv2) { return qv + c * sv2; });
  }
}

// LbfgsSolver::iterate (optim.cpp:152-205).  value(cand) and evaluate(cand)
// share one forward sweep (the value is bit-identical either way).
__device__ __forceinline__ int lbfgs_iterate(const CK& K, SolverState& s) {
  const DOpt& o = K.o;
  if (s.status != ST_RUNNING) return s.status;
  if (s.iters >= o.max_iters) return s.status = ST_FAILED;
  if (grad_converged(K, s)) return s.status = ST_CONVERGED;
  two_loop(K, s);
  qmap2(K, K.dir, K.q, K.q, [](double qv, double) { return -qv; });
  double slope = qdot(K, K.dir, K.g);
  if (!(slope < 0.0)) {
    s.hc = 0;
    s.h0 = 0;
    qmap2(K, K.dir, K.g, K.g, [](double gv, double) { return -gv; });
    slope = qdot(K, K.dir, K.g);
  }
  double t = 1.0;
  bool accepted = false;
  const double fval = s.value;
  const int cap = o.mem + 1;
  for (int trial = 0; trial < o.max_line_search; ++trial) {
    qmap2(K, K.cand, K.x, K.dir, [t](double xv, double dv) { return xv + t * dv; });
    if (qallfinite(K, K.cand)) {
      const double v = chain_forward(K, K.cand, true);
      if (isfinite(v) && v <= fval + o.armijo_c1 * t * slope && v < fval) {
        chain_reverse(K, K.evg);
        const int slot = (s.h0 + s.hc) % cap;
        double* sv = K.hs + slot * K.VS;
        double* yv = K.hy + slot * K.VS;
        qmap2(K, sv, K.dir, K.dir, [t](double dv, double) { return t * dv; });
        qmap2(K, yv, K.evg, K.g, [](double ev, double gv) { return ev - gv; });
        const double sy = qdot(K, sv, yv);
        if (sy > 1e-12) {
          if (K.r == 0) K.hsy[slot * K.B] = sy;
          ++s.hc;
          if (s.hc > o.mem) {
            s.h0 = (s.h0 + 1) % cap;
            --s.hc;
          }
        }
        qmap2(K, K.x, K.cand, K.cand, [](double cv, double) { return cv; });
        qmap2(K, K.g, K.evg, K.evg, [](double ev, double) { return ev; });
        qsync(K);
        s.value = v;
        accepted = true;
        ++s.acc;
        if (stagnation_update(K, s, fval, v)) s.status = ST_CONVERGED;
        break;
      }
    }
    t *= o.backtrack_factor;
  }
  if (!accepted) s.status = ST_FAILED;
  if (s.itv && K.r == 0) s.itv[s.iters] = s.value;
  ++s.iters;
  if (s.status == ST_RUNNING && s.iters >= o.max_iters) s.status = ST_FAILED;
  return s.status;
}

// ForceModel::tau_at (objective.hpp:28-58) into the tau vector
__device__ __forceinline__ void tau_at(const CK& K, const DForces& f, double t) {
  const int n = K.n;
  for (int i = K.r; i < n; i += 4) {
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
    vat(K, K.tau, i) = v;
  }
}

// fd_kinetic (stepper.cpp:14-22) + gravity_potential (baseline.cpp:219-229)
__device__ __forceinline__ void chain_energy(const CK& K, const double* Wp, const double* Wn, double dt, double* ke, double* pe) {
  double k = 0.0, p = 0.0;
  const double ghat[4] = {K.gz[0], K.gz[1], K.gz[2], 0.0};
  for (int i = 0; i < K.N; ++i) {
    double wp[4], wn[4], td[4], tds[4];
    ld4(Wp + i * kLS, wp);
    ld4(Wn + i * kLS, wn);
#pragma unroll
    for (int c = 0; c < 4; ++c) td[c] = (wn[c] - wp[c]) / dt;
    Rec R;
    load_rec(K, i, &R, true);
    row_mul_rec(td, R.S, tds);
    // u = S e4 (canonical product: exactly column 3 of S)
    double wu = wn[0] * R.S[12];
    wu = fma(wn[1], R.S[13], wu);
    wu = fma(wn[2], R.S[14], wu);
    wu = fma(wn[3], R.S[15], wu);
    qsync(K);
    K.red[K.r] = ddot_row(tds, td);
    K.red[4 + K.r] = wu;
    qsync(K);
    const double term = ((K.red[0] + K.red[1]) + K.red[2]) + K.red[3];
    double d = ghat[0] * K.red[4];
    d = fma(ghat[1], K.red[5], d);
    d = fma(ghat[2], K.red[6], d);
    d = fma(ghat[3], K.red[7], d);
    k += 0.5 * term;
    p -= d;
  }
  *ke = k;
  *pe = p;
}

}  // namespace

// init_pbad_run (stepper.cpp:62-80) for the chain path
__global__ void __launch_bounds__(kThreads) k_chain_init(DModel m, DForces f, DSchedule sc, ChainLayout L, double* cw,
                                                         int* ci, long B, const double* q0, const double* qdot0,
                                                         const double* hist0, Outputs out) {
  extern __shared__ __align__(16) double smem[];
  stage_model(m, smem);
  bool valid;
  const CK K = make_ck(m, f, sc, L, cw, ci, B, smem, &valid);
  if (!valid) return;
  const int n = m.n, N = m.N;
  bool finite = true;
  for (int k = K.r; k < n; k += 4) {
    const double q = q0[K.e * n + k];
    vat(K, K.h1, k) = q;
    vat(K, K.g, k) = qdot0[K.e * n + k];  // qdot scratch
    finite = finite && isfinite(q);
  }
  finite = __all_sync(K.qm, finite);
  if (K.r == 0) {
    ival(K, IS_STEP) = 0;
    ival(K, IS_FAIL) = 0;
    ival(K, IS_NSAMP) = 0;
    ival(K, IS_NREP) = 0;
  }
  if (!finite) {
    if (K.r == 0) ival(K, IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  const double tl = sc.times[0] * sc.dt;
  for (int k = K.r; k < n; k += 4)  // refined_bootstrap: precomputed (k_refined_bootstrap)
    vat(K, K.h0, k) = hist0 ? hist0[K.e * n + k] : vat(K, K.h1, k) + tl * vat(K, K.g, k);
  qsync(K);
  // kinetic_energy via the velocity pass (baseline.cpp:20-54,208-217) and
  // gravity_potential (baseline.cpp:219-229) at q0; general joint algebra
  // (this runs once per trajectory)
  double T[4], Td[4];
  identity_row(K.r, T);
  Td[0] = Td[1] = Td[2] = Td[3] = 0.0;
  double ke = 0.0, pe = 0.0;
  const double ghat[4] = {f.gravity[0], f.gravity[1], f.gravity[2], 0.0};
  for (int i = 0; i < N; ++i) {
    const double qi = vat(K, K.h1, i);
    GenJet G;
    general_jet(m, i, qi, true, &G);
    const double qd = vat(K, K.g, i);
    M4 ldot;
#pragma unroll
    for (int k = 0; k < 16; ++k) ldot.a[k] = 0.0 + qd * G.d1.a[k];
    double a[4], b[4], Tn[4], Tdn[4];
    if (i == 0) {
      const double z[4] = {0.0, 0.0, 0.0, 0.0};
      row_mul(z, G.L, a);  // parent_tdot = Zero
    } else {
      row_mul(Td, G.L, a);
    }
    row_mul(T, ldot, b);  // parent_world (Identity for the root) * ldot
#pragma unroll
    for (int c = 0; c < 4; ++c) Tdn[c] = a[c] + b[c];
    if (i == 0) {
      get_row(G.L, K.r, Tn);
    } else {
      row_mul(T, G.L, Tn);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      T[c] = Tn[c];
      Td[c] = Tdn[c];
    }
    Rec R;
    load_rec(K, i, &R, true);
    double tds[4];
    row_mul_rec(Td, R.S, tds);
    double wu = T[0] * R.S[12];
    wu = fma(T[1], R.S[13], wu);
    wu = fma(T[2], R.S[14], wu);
    wu = fma(T[3], R.S[15], wu);
    qsync(K);
    K.red[K.r] = ddot_row(tds, Td);
    K.red[4 + K.r] = wu;
    qsync(K);
    const double term = ((K.red[0] + K.red[1]) + K.red[2]) + K.red[3];
    double d = ghat[0] * K.red[4];
    d = fma(ghat[1], K.red[5], d);
    d = fma(ghat[2], K.red[6], d);
    d = fma(ghat[3], K.red[7], d);
    ke += 0.5 * term;
    pe -= d;
  }
  for (int k = K.r; k < n; k += 4)
    if (out.q) out.q[out.qrow(K.e, 0) * n + k] = vat(K, K.h1, k);
  if (K.r == 0) {
    if (out.energy) {
      out.energy[out.qrow(K.e, 0) * 2] = ke;
      out.energy[out.qrow(K.e, 0) * 2 + 1] = pe;
    }
    ival(K, IS_NSAMP) = 1;
    ival(K, IS_RUN) = (sc.total_steps > 0) ? TR_RUNNING : TR_OK;
  }
}

// One PBAD step per environment: begin_step, L-BFGS to completion,
// finish_step (stepper.cpp:83-147).
__global__ void __launch_bounds__(kThreads) k_chain_step(DModel m, DForces f, DSchedule sc, ChainLayout L, double* cw,
                                                         int* ci, long B, Outputs out) {
  extern __shared__ __align__(16) double smem[];
  stage_model(m, smem);
  bool valid;
  const CK K = make_ck(m, f, sc, L, cw, ci, B, smem, &valid);
  if (!valid) return;
  if (ival(K, IS_RUN) != TR_RUNNING) return;
  const int n = m.n;
  const int step = ival(K, IS_STEP);
  // StepObjective ctor validates the history (objective.cpp:176-177)
  if (!qallfinite(K, K.h0) || !qallfinite(K, K.h1)) {
    if (K.r == 0) ival(K, IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  // begin_step: actuation at the step end, warm start (stepper.cpp:83-115)
  tau_at(K, f, step * sc.dt + sc.times[2] * sc.dt);
  const double span = -sc.times[0];
  const double tau_m = sc.times[2];
  const bool ws = sc.warm_start != 0;
  qmap2(K, K.x, K.h1, K.h0,
        [tau_m, span, ws](double h1, double h0) { return ws ? h1 + (tau_m / span) * (h1 - h0) : h1; });
  qsync(K);
  // StepObjective ctor: history passes and hist_const (objective.cpp:162-185)
  chain_fk(K, K.h0, K.tk1);
  chain_fk(K, K.h1, K.tk);
  qsync(K);
  const double hc = 4.0 * chain_cv(K, K.tk, K.tk) + chain_cv(K, K.tk1, K.tk1) - 4.0 * chain_cv(K, K.tk, K.tk1);
  if (K.r == 0) *K.histc = hc;
  qsync(K);
  // LbfgsSolver ctor: first evaluation
  SolverState s{};
  s.status = ST_RUNNING;
  s.itv = out.itv ? out.itv + out.rrow(K.e, step) * out.itv_n : nullptr;
  if (!qallfinite(K, K.x)) {
    if (K.r == 0) ival(K, IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  const double v0 = chain_forward(K, K.x, true);
  if (!isfinite(v0)) {
    if (K.r == 0) ival(K, IS_RUN) = TR_NONFINITE_INIT;
    return;
  }
  chain_reverse(K, K.g);
  s.value = v0;
  s.grad0 = qinfnorm(K, K.g);
  while (lbfgs_iterate(K, s) == ST_RUNNING) {
  }
  // finish_step
  const long S = sc.total_steps;
  const bool converged = s.status == ST_CONVERGED;
  const double gnorm = qinfnorm(K, K.g);
  if (K.r == 0) {
    if (out.iterations) out.iterations[out.rrow(K.e, step)] = s.iters;
    if (out.converged) out.converged[out.rrow(K.e, step)] = converged;
    if (out.accepted) out.accepted[out.rrow(K.e, step)] = s.acc;
    if (out.final_value) out.final_value[out.rrow(K.e, step)] = s.value;
    if (out.final_grad_norm) out.final_grad_norm[out.rrow(K.e, step)] = gnorm;
    ival(K, IS_NREP) = step + 1;
  }
  const int fs = converged ? 0 : ival(K, IS_FAIL) + 1;
  qsync(K);
  if (K.r == 0) ival(K, IS_FAIL) = fs;
  if (fs > sc.fail_limit) {
    if (K.r == 0) ival(K, IS_RUN) = TR_FAIL_LIMIT;
    return;
  }
  qmap2(K, K.h0, K.h1, K.h1, [](double a, double) { return a; });
  qsync(K);
  qmap2(K, K.h1, K.x, K.x, [](double a, double) { return a; });
  qsync(K);
  chain_fk(K, K.h1, K.tk1);  // tk still holds forward_pass(old hist1)
  qsync(K);
  double ke, pe;
  chain_energy(K, K.tk, K.tk1, sc.dt, &ke, &pe);
  for (int k = K.r; k < n; k += 4)
    if (out.q) out.q[out.qrow(K.e, step + 1) * n + k] = vat(K, K.h1, k);
  if (K.r == 0) {
    if (out.energy) {
      out.energy[out.qrow(K.e, step + 1) * 2] = ke;
      out.energy[out.qrow(K.e, step + 1) * 2 + 1] = pe;
    }
    ival(K, IS_STEP) = step + 1;
    ival(K, IS_NSAMP) = step + 2;
    if (step + 1 >= S) ival(K, IS_RUN) = TR_OK;
  }
}

unsigned chain_grid(long B) { return (unsigned)((B + kEnvsPerBlock - 1) / kEnvsPerBlock); }

static cudaError_t chain_smem_attr(int N, size_t* bytes) {
  *bytes = chain_smem_bytes(N);
  static SmemAttr attr_;  // per device; raised monotonically
  size_t& configured = attr_.here();
  if (*bytes > configured) {
    cudaError_t e = cudaFuncSetAttribute(k_chain_init, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*bytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_chain_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*bytes);
    if (e != cudaSuccess) return e;
    configured = *bytes;
  }
  return cudaSuccess;
}

cudaError_t launch_chain_init(const ChainArgs& a, const double* q0, const double* qdot0, const double* hist0,
                              const Outputs& out, cudaStream_t s) {
  size_t sm;
  cudaError_t e = chain_smem_attr(a.m.N, &sm);
  if (e != cudaSuccess) return e;
  k_chain_init<<<chain_grid(a.B), kThreads, sm, s>>>(a.m, a.f, a.sc, a.L, a.cw, a.ci, a.B, q0, qdot0, hist0, out);
  return cudaGetLastError();
}
cudaError_t launch_chain_step(const ChainArgs& a, const Outputs& out, cudaStream_t s) {
  size_t sm;
  cudaError_t e = chain_smem_attr(a.m.N, &sm);
  if (e != cudaSuccess) return e;
  k_chain_step<<<chain_grid(a.B), kThreads, sm, s>>>(a.m, a.f, a.sc, a.L, a.cw, a.ci, a.B, out);
  return cudaGetLastError();
}
int chain_max_memory() { return kMaxMem; }
// links the shared-memory model copy admits (227 KB per block)
int chain_max_links() { return (int)((227L * 1024 - smem_red_doubles() * 8) / (20 * 8 + 4)); }

}  // namespace pbad_gpu
