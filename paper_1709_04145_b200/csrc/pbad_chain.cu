// pbad_chain.cu -- "quad" kernels for serial hinge chains (energy form, L-BFGS).
//
// Mapping: four lanes per environment ("quad"), lane r owns row r of every
// 4x4 transform (lane 3 carries the constant bottom row [0 0 0 1], which
// makes its contributions to the row-partial ddots come out exactly as the
// reference's).  Eight environments per warp.  Everything the reference does
// per link is row-local under the numeric contract:
//   FK          T_i[r,:]  = T_{i-1}[r,:] * L_i            (kinematics.cpp:171-181)
//   energy      ddot(A_i S_i, B_i) row partials           (adjoint.cpp:113-120)
//   seeds       ((T - 2T_k) + T_{k-1}) S / dt^2 per row   (objective.cpp:241-249)
//   lever       T_{i-1}[r,:] * dL_i/dq                    (adjoint.cpp:22-25)
//   adjoint     adj_{i-1}[r,:] = seed + adj_i[r,:] L_i^T  (adjoint.cpp:49-64)
// so the bit-exact serial recursions run on 3 lanes per environment with no
// data exchange except the per-link scalar reductions (through shared memory).
// The L-BFGS vectors (optim.cpp:141-232) are quad-interleaved: element k of an
// environment lives on lane k%4, and the 32-partial dot of the numeric
// contract maps to 8 partials per lane plus a 2-level quad reduction.
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

struct Q {
  const DModel* m;
  const DForces* f;
  const DSchedule* sc;
  const ChainLayout* L;
  double* cw;
  int* ci;
  long B;
  int e;       // environment
  int r;       // row / lane in quad
  unsigned qm; // quad lane mask
  double* red; // shared scratch for this quad: 16 doubles
};

__device__ __forceinline__ double qshfl(const Q& Z, double v, int src) { return __shfl_sync(Z.qm, v, src, 4); }
__device__ __forceinline__ void qsync(const Q& Z) { __syncwarp(Z.qm); }

// --- global layouts -------------------------------------------------------
// link arrays: [N][B][16], row r at +4r
__device__ __forceinline__ double* lrow(const Q& Z, long off, int i) {
  return Z.cw + off + ((long)i * Z.B + Z.e) * 16 + 4 * Z.r;
}
// quad-interleaved vectors: element k at ((k>>2)*B + e)*4 + (k&3)
__device__ __forceinline__ double* vel(const Q& Z, long off, int k) {
  return Z.cw + off + ((long)(k >> 2) * Z.B + Z.e) * 4 + (k & 3);
}
__device__ __forceinline__ double& scal(const Q& Z, long off) { return Z.cw[off + Z.e]; }
__device__ __forceinline__ int& ival(const Q& Z, int slot) { return Z.ci[(long)slot * Z.B + Z.e]; }

__device__ __forceinline__ void ld4(const double* p, double* v) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void st4(double* p, const double* v) {
  *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
}
__device__ __forceinline__ M4 ldS(const Q& Z, int i) {
  M4 m;
#pragma unroll
  for (int k = 0; k < 16; ++k) m.a[k] = __ldg(Z.m->S + 16 * i + k);
  return m;
}

// row r of (A * B) for a 4-vector row a
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
// row r of (A * B^T)
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

// --- per-link joint algebra ----------------------------------------------
// A link's local transform L = offset * [R(axis*q) 0; 0 1] and its
// derivative d1 = offset * embed([axis]x R) (kinematics.cpp:119-129).
// jkind 1/2/3: axis exactly e_x/e_y/e_z and offset rotation block exactly I.
// Then R = I + A K + B K^2 has two free entries (c, s) and every canonical
// product below reduces to its non-zero terms: the dropped terms are
// fma(x, +-0, acc) with finite x, which leave the value unchanged.
struct LinkJet {
  int jk;
  double c, s;   // specialised: R entries
  double t[3];   // offset translation
  M4 L, d1;      // general: full matrices
};

// rotation_coeffs A, B (kinematics.cpp:20-45) for a hinge of angle q about
// a unit axis: n = |q|, k2 = q*q is -K^2's diagonal entry.
__device__ __forceinline__ void hinge_cs(double q, double* c, double* s) {
  const double k2 = q * q;
  const double n = sqrt(k2);
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
  *s = A * q;           // (0 + A*K_ab) + B*(+-0)
  *c = 1.0 - B * k2;    // (1 + A*0) + B*(-k2)
}

__device__ __forceinline__ void link_jet(const Q& Z, int i, double qi, bool want_d1, LinkJet* J) {
  J->jk = __ldg(Z.m->jkind + i);
  const double* off = Z.m->offset + 16 * i;
  if (J->jk) {
    hinge_cs(qi, &J->c, &J->s);
    J->t[0] = __ldg(off + 12);
    J->t[1] = __ldg(off + 13);
    J->t[2] = __ldg(off + 14);
    return;
  }
  const double* ax = Z.m->axis + 3 * i;
  const double a0 = __ldg(ax), a1 = __ldg(ax + 1), a2 = __ldg(ax + 2);
  M4 o;
#pragma unroll
  for (int k = 0; k < 16; ++k) o.a[k] = __ldg(off + k);
  const M3 R = rotation_vector_matrix(a0 * qi, a1 * qi, a2 * qi);
  J->L = mul(o, motion_rot(R));
  if (want_d1) J->d1 = mul(o, embed_rotation(mul3(skew(a0, a1, a2), R)));
}

// translation column: T0*t0 + T1*t1 + T2*t2 + T3
__device__ __forceinline__ double trans_col(const double* T, const double* t) {
  double acc = T[0] * t[0];
  acc = fma(T[1], t[1], acc);
  acc = fma(T[2], t[2], acc);
  return acc + T[3];
}

// row of (T * L): forward kinematics world = parent_world * value
__device__ __forceinline__ void link_fk_row(const LinkJet& J, const double* T, double* Tn) {
  const double c = J.c, s = J.s;
  switch (J.jk) {
    case 1:  // R = [1 0 0; 0 c -s; 0 s c]
      Tn[0] = T[0];
      Tn[1] = fma(T[2], s, T[1] * c);
      Tn[2] = fma(T[2], c, T[1] * (-s));
      Tn[3] = trans_col(T, J.t);
      return;
    case 2:  // R = [c 0 s; 0 1 0; -s 0 c]
      Tn[0] = fma(T[2], -s, T[0] * c);
      Tn[1] = T[1];
      Tn[2] = fma(T[2], c, T[0] * s);
      Tn[3] = trans_col(T, J.t);
      return;
    case 3:  // R = [c -s 0; s c 0; 0 0 1]
      Tn[0] = fma(T[1], s, T[0] * c);
      Tn[1] = fma(T[1], c, T[0] * (-s));
      Tn[2] = T[2];
      Tn[3] = trans_col(T, J.t);
      return;
    default:
      row_mul(T, J.L, Tn);
  }
}

// row of (T * d1): lever = parent_world * dL/dq; compact storage lev[0..1]
// for the specialised kinds (the other two entries are +-0)
__device__ __forceinline__ void link_lever_row(const LinkJet& J, const double* T, double* lev) {
  const double c = J.c, s = J.s;
  switch (J.jk) {
    case 1:  // [a]x R rows: 0; (0,-s,-c); (0,c,-s)   -> columns 1, 2
      lev[0] = fma(T[2], c, T[1] * (-s));
      lev[1] = fma(T[2], -s, T[1] * (-c));
      return;
    case 2:  // rows: (-s,0,c); 0; (-c,0,-s)           -> columns 0, 2
      lev[0] = fma(T[2], -c, T[0] * (-s));
      lev[1] = fma(T[2], -s, T[0] * c);
      return;
    case 3:  // rows: (-s,-c,0); (c,-s,0); 0            -> columns 0, 1
      lev[0] = fma(T[1], c, T[0] * (-s));
      lev[1] = fma(T[1], -s, T[0] * (-c));
      return;
    default:
      row_mul(T, J.d1, lev);
  }
}

// ddot_row(lever_row, a) with the lever's zero columns dropped
__device__ __forceinline__ double link_lever_dot(int jk, const double* lev, const double* a) {
  switch (jk) {
    case 1: return fma(lev[1], a[2], lev[0] * a[1]);
    case 2: return fma(lev[1], a[2], lev[0] * a[0]);
    case 3: return fma(lev[1], a[1], lev[0] * a[0]);
    default: return ddot_row(lev, a);
  }
}

// row of (a * L^T): adjoint transport to the parent
__device__ __forceinline__ void link_transport_row(const LinkJet& J, const double* a, double* t) {
  const double c = J.c, s = J.s;
  switch (J.jk) {
    case 1:  // L rows (1,0,0,t0) (0,c,-s,t1) (0,s,c,t2)
      t[0] = fma(a[3], J.t[0], a[0]);
      t[1] = fma(a[3], J.t[1], fma(a[2], -s, a[1] * c));
      t[2] = fma(a[3], J.t[2], fma(a[2], c, a[1] * s));
      t[3] = a[3];
      return;
    case 2:  // (c,0,s,t0) (0,1,0,t1) (-s,0,c,t2)
      t[0] = fma(a[3], J.t[0], fma(a[2], s, a[0] * c));
      t[1] = fma(a[3], J.t[1], a[1]);
      t[2] = fma(a[3], J.t[2], fma(a[2], c, a[0] * (-s)));
      t[3] = a[3];
      return;
    case 3:  // (c,-s,0,t0) (s,c,0,t1) (0,0,1,t2)
      t[0] = fma(a[3], J.t[0], fma(a[1], -s, a[0] * c));
      t[1] = fma(a[3], J.t[1], fma(a[1], c, a[0] * s));
      t[2] = fma(a[3], J.t[2], a[2]);
      t[3] = a[3];
      return;
    default:
      row_mul_bt(a, J.L, t);
  }
}

__device__ __forceinline__ void identity_row(int r, double* v) {
  v[0] = (r == 0) ? 1.0 : 0.0;
  v[1] = (r == 1) ? 1.0 : 0.0;
  v[2] = (r == 2) ? 1.0 : 0.0;
  v[3] = (r == 3) ? 1.0 : 0.0;
}

// row r of the gravity cotangent c = -ghat u^T, u = S e4 (objective.cpp:48-58)
__device__ __forceinline__ void grav_row(const Q& Z, const M4& S, double* c) {
  const double e4[4] = {0.0, 0.0, 0.0, 1.0};
  double u[4];
  mul_vec4(S, e4, u);
  const double g = (Z.r < 3) ? Z.f->gravity[Z.r] : 0.0;
#pragma unroll
  for (int s = 0; s < 4; ++s) c[s] = (-g) * u[s];
}

// combine 4 row partials of each of K values: ((p0+p1)+p2)+p3, all lanes
template <int K>
__device__ __forceinline__ void quad_combine(const Q& Z, const double* p, double* out) {
  qsync(Z);
#pragma unroll
  for (int k = 0; k < K; ++k) Z.red[4 * k + Z.r] = p[k];
  qsync(Z);
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = ((Z.red[4 * k] + Z.red[4 * k + 1]) + Z.red[4 * k + 2]) + Z.red[4 * k + 3];
}

// --- vector ops (quad-interleaved, 32-partial canonical dot) --------------
// Element k of a vector lives on lane k%4 at group k>>2.  Loops run eight
// groups at a time with all loads issued first (memory-level parallelism:
// one resident warp per scheduler cannot hide a serial load chain).
constexpr int kU = 8;

__device__ double qdot(const Q& Z, long oa, long ob, int n) {
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.0;
  const int n4 = (n + 3) >> 2;
  for (int g0 = 0; g0 < n4; g0 += kU) {
    double a[kU], b[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int k = 4 * (g0 + j) + Z.r;
      const bool ok = (g0 + j < n4) && k < n;
      a[j] = ok ? *vel(Z, oa, k) : 0.0;
      b[j] = ok ? *vel(Z, ob, k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int k = 4 * (g0 + j) + Z.r;
      if ((g0 + j < n4) && k < n) acc[j] = fma(a[j], b[j], acc[j]);  // (g0+j)&7 == j
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = acc[j] + acc[j + 4];
  acc[0] = acc[0] + acc[2];
  acc[1] = acc[1] + acc[3];
  double v = acc[0] + acc[1];
  const double v2 = qshfl(Z, v, (Z.r + 2) & 3);
  if (Z.r < 2) v = v + v2;
  const double v1 = qshfl(Z, v, 1);
  if (Z.r == 0) v = v + v1;
  return qshfl(Z, v, 0);
}

// dst[k] = f(a[k], b[k]) for the lane's elements: loads of eight groups are
// issued before any store (the compiler cannot reorder across the stores)
template <class F>
__device__ __forceinline__ void qmap2(const Q& Z, int n, long dst, long oa, long ob, F f) {
  const int n4 = (n + 3) >> 2;
  for (int g0 = 0; g0 < n4; g0 += kU) {
    double a[kU], b[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int k = 4 * (g0 + j) + Z.r;
      const bool ok = (g0 + j < n4) && k < n;
      a[j] = ok ? *vel(Z, oa, k) : 0.0;
      b[j] = ok ? *vel(Z, ob, k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int k = 4 * (g0 + j) + Z.r;
      if ((g0 + j < n4) && k < n) *vel(Z, dst, k) = f(a[j], b[j]);
    }
  }
}

__device__ double qinfnorm(const Q& Z, long oa, int n) {
  double mx = 0.0;
  const int n4 = (n + 3) >> 2;
  for (int g0 = 0; g0 < n4; g0 += kU) {
    double a[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int k = 4 * (g0 + j) + Z.r;
      a[j] = (g0 + j < n4 && k < n) ? *vel(Z, oa, k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) mx = fmax(mx, fabs(a[j]));
  }
  mx = fmax(mx, qshfl(Z, mx, Z.r ^ 1));
  mx = fmax(mx, qshfl(Z, mx, Z.r ^ 2));
  return mx;
}
__device__ bool qallfinite(const Q& Z, long oa, int n) {
  bool ok = true;
  const int n4 = (n + 3) >> 2;
  for (int g0 = 0; g0 < n4; g0 += kU) {
    double a[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int k = 4 * (g0 + j) + Z.r;
      a[j] = (g0 + j < n4 && k < n) ? *vel(Z, oa, k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) ok = ok && isfinite(a[j]);
  }
  return __all_sync(Z.qm, ok);
}

// --- the per-step constants: T_k, T_{k-1} and hist_const -----------------
// forward_pass of the vector at `ov` into link array `olink`
__device__ void chain_fk(const Q& Z, long ov, long olink) {
  const int N = Z.m->N;
  double T[4];
  identity_row(Z.r, T);
  for (int i = 0; i < N; ++i) {
    LinkJet J;
    link_jet(Z, i, *vel(Z, ov, i), false, &J);
    double Tn[4];
    if (i == 0) {
      // forward_pass: the root's world transform is its local transform
      double I[4];
      identity_row(Z.r, I);
      link_fk_row(J, I, Tn);
    } else {
      link_fk_row(J, T, Tn);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) T[c] = Tn[c];
    st4(lrow(Z, olink, i), T);
  }
}

// correlation_value(A, B) over two link arrays (adjoint.cpp:113-120)
__device__ double chain_cv(const Q& Z, long oa, long ob) {
  const int N = Z.m->N;
  double v = 0.0;
  for (int i = 0; i < N; ++i) {
    double a[4], b[4], as[4];
    ld4(lrow(Z, oa, i), a);
    ld4(lrow(Z, ob, i), b);
    row_mul(a, ldS(Z, i), as);
    double p = ddot_row(as, b), t;
    quad_combine<1>(Z, &p, &t);
    v += t;
  }
  return v - Z.m->weighted_mass;
}

// --- the evaluation --------------------------------------------------------
// Forward sweep at vector `ox`: value (StepObjective::value,
// objective.cpp:215-239) and, with store, the seeds / levers / joint
// transforms the reverse sweep needs.
__device__ double chain_forward(const Q& Z, long ox, bool store) {
  const ChainLayout& L = *Z.L;
  const DSchedule& sc = *Z.sc;
  const int N = Z.m->N;
  const double inv_dt2 = 1.0 / (sc.dt * sc.dt);
  double T[4];
  identity_row(Z.r, T);
  double sa = 0.0, sb = 0.0, sc2 = 0.0, sg = 0.0;
  // software pipeline: the next link's per-env loads are issued one link early
  double qnext = *vel(Z, ox, 0);
  double ntk[4] = {0.0, 0.0, 0.0, 0.0}, ntk1[4] = {0.0, 0.0, 0.0, 0.0};
  int nsk = __ldg(Z.m->skind);
  if (nsk) {
    ld4(lrow(Z, L.tk, 0), ntk);
    ld4(lrow(Z, L.tk1, 0), ntk1);
  }
  for (int i = 0; i < N; ++i) {
    const double qi = qnext;
    const int sk = nsk;
    double tk[4], tk1[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      tk[c] = ntk[c];
      tk1[c] = ntk1[c];
    }
    if (i + 1 < N) {
      qnext = *vel(Z, ox, i + 1);
      nsk = __ldg(Z.m->skind + i + 1);
      if (nsk) {
        ld4(lrow(Z, L.tk, i + 1), ntk);
        ld4(lrow(Z, L.tk1, i + 1), ntk1);
      }
    }
    LinkJet J;
    link_jet(Z, i, qi, store, &J);
    if (store) {
      double lev[4];
      link_lever_row(J, T, lev);  // parent_world * d1 (identity row for the root)
      double* lp = lrow(Z, L.lev, i);
      if (J.jk) {
        *reinterpret_cast<double2*>(lp) = make_double2(lev[0], lev[1]);
        if (Z.r == 0)
          *reinterpret_cast<double2*>(Z.cw + L.lmat + ((long)i * Z.B + Z.e) * 16) = make_double2(J.c, J.s);
      } else {
        st4(lp, lev);
        double lr[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) lr[c] = J.L.a[Z.r + 4 * c];
        st4(lrow(Z, L.lmat, i), lr);
      }
    }
    double Tn[4];
    link_fk_row(J, T, Tn);  // world = parent_world * value
#pragma unroll
    for (int c = 0; c < 4; ++c) T[c] = Tn[c];
    if (!sk) continue;  // massless link: every term below is exactly +-0
    const M4 S = ldS(Z, i);
    double ts[4], p1[4], p2[4], cg[4];
    row_mul(T, S, ts);
    row_mul(tk, S, p1);
    row_mul(tk1, S, p2);
    grav_row(Z, S, cg);
    double part[4], term[4];
    part[0] = ddot_row(ts, T);
    part[1] = ddot_row(p1, T);
    part[2] = ddot_row(p2, T);
    part[3] = ddot_row(cg, T);
    quad_combine<4>(Z, part, term);
    sa += term[0];
    sb += term[1];
    sc2 += term[2];
    sg += term[3];
    if (store) {
      double d[4], sd[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        d[c] = T[c] - 2.0 * tk[c];
        d[c] = d[c] + tk1[c];
        d[c] = inv_dt2 * d[c];
      }
      row_mul(d, S, sd);
      st4(lrow(Z, L.seed, i), sd);
    }
  }
  const double wm = Z.m->weighted_mass;
  const double cpp = sa - wm, c1p = sb - wm, c2p = sc2 - wm;
  const double inertial = 0.5 * inv_dt2 * (cpp - 4.0 * c1p + 2.0 * c2p + scal(Z, L.histc));
  const double tdx = qdot(Z, L.tau, ox, Z.m->n);
  return inertial + sg - tdx;
}

// Reverse sweep (functional_grad twice, adjoint.cpp:49-64): gradient =
// (inertial adjoint + gravity adjoint) - tau into og (objective.cpp:241-250).
__device__ void chain_reverse(const Q& Z, long og) {
  const ChainLayout& L = *Z.L;
  const int N = Z.m->N;
  double cI[4] = {0.0, 0.0, 0.0, 0.0}, cG[4] = {0.0, 0.0, 0.0, 0.0};
  // per-link loads one link ahead (software pipeline)
  auto fetch = [&](int i, double* lev, double* seed, double* cs) {
    const int jk = __ldg(Z.m->jkind + i);
    const int sk = __ldg(Z.m->skind + i);
    const double* lp = lrow(Z, L.lev, i);
    if (jk) {
      const double2 v = *reinterpret_cast<const double2*>(lp);
      lev[0] = v.x;
      lev[1] = v.y;
      const double2 w = *reinterpret_cast<const double2*>(Z.cw + L.lmat + ((long)i * Z.B + Z.e) * 16);
      cs[0] = w.x;
      cs[1] = w.y;
    } else {
      ld4(lp, lev);
    }
    if (sk) ld4(lrow(Z, L.seed, i), seed);
  };
  double nlev[4], nseed[4], ncs[2];
  fetch(N - 1, nlev, nseed, ncs);
  for (int i = N - 1; i >= 0; --i) {
    const int jk = __ldg(Z.m->jkind + i);
    const int sk = __ldg(Z.m->skind + i);
    double lev[4], aI[4], aG[4], seed[4], cs[2];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      lev[c] = nlev[c];
      seed[c] = nseed[c];
    }
    cs[0] = ncs[0];
    cs[1] = ncs[1];
    if (i > 0) fetch(i - 1, nlev, nseed, ncs);
    if (sk) {
      double cg[4];
      const M4 S = ldS(Z, i);
      grav_row(Z, S, cg);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        aI[c] = cI[c] + seed[c];
        aG[c] = cG[c] + (0.0 + cg[c]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        aI[c] = cI[c];
        aG[c] = cG[c];
      }
    }
    double part[2], gg[2];
    part[0] = link_lever_dot(jk, lev, aI);
    part[1] = link_lever_dot(jk, lev, aG);
    quad_combine<2>(Z, part, gg);
    if ((i & 3) == Z.r) {
      const double gi = 0.0 + gg[0];
      const double gp = 0.0 + gg[1];
      *vel(Z, og, i) = (gi + gp) - *vel(Z, L.tau, i);
    }
    if (i > 0) {
      LinkJet J;
      J.jk = jk;
      const double* lm = Z.cw + L.lmat + ((long)i * Z.B + Z.e) * 16;
      if (jk) {
        J.c = cs[0];
        J.s = cs[1];
        const double* off = Z.m->offset + 16 * i;
        J.t[0] = __ldg(off + 12);
        J.t[1] = __ldg(off + 13);
        J.t[2] = __ldg(off + 14);
      } else {
        double rows[16];
        ld4(lm, rows);
        ld4(lm + 4, rows + 4);
        ld4(lm + 8, rows + 8);
        ld4(lm + 12, rows + 12);
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
          for (int c = 0; c < 4; ++c) J.L.a[rr + 4 * c] = rows[4 * rr + c];
      }
      double tI[4], tG[4];
      link_transport_row(J, aI, tI);
      link_transport_row(J, aG, tG);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        cI[c] = 0.0 + tI[c];
        cG[c] = 0.0 + tG[c];
      }
    }
  }
  qsync(Z);
}

// --- optimizer --------------------------------------------------------------
struct SolverState {
  double value, grad0;
  int status, iters, stag, acc, h0, hc;
};

__device__ __forceinline__ bool grad_converged(const Q& Z, const SolverState& s) {
  const DOpt& o = Z.sc->opt;
  const int n = Z.m->n;
  const double g = qinfnorm(Z, Z.L->g, n);
  if (g <= o.grad_tol * fmax(1.0, qinfnorm(Z, Z.L->x, n))) return true;
  if (o.grad_rtol > 0.0 && g <= o.grad_rtol * s.grad0) return true;
  return false;
}
__device__ __forceinline__ bool stagnation_update(const Q& Z, SolverState& s, double oldv, double newv) {
  if (oldv - newv <= Z.sc->opt.ftol * fmax(1.0, fabs(oldv))) ++s.stag;
  else s.stag = 0;
  return s.stag >= 2;
}

// LbfgsSolver::two_loop (optim.cpp:213-229): q = H g into L.q
__device__ void two_loop(const Q& Z, const SolverState& s) {
  const ChainLayout& L = *Z.L;
  const int n = Z.m->n;
  const int cap = Z.sc->opt.mem + 1;
  qmap2(Z, n, L.q, L.g, L.g, [](double a, double) { return a; });
  double alpha[kMaxMem];
  for (int i = s.hc - 1; i >= 0; --i) {
    const int slot = (s.h0 + i) % cap;
    const long os = L.hs + (long)slot * L.vstride, oy = L.hy + (long)slot * L.vstride;
    const double a = qdot(Z, os, L.q, n) / Z.cw[L.hsy + (long)slot * Z.B + Z.e];
    alpha[i] = a;
    qmap2(Z, n, L.q, L.q, oy, [a](double qv, double yv) { return qv - a * yv; });
  }
  if (s.hc > 0) {
    const int slot = (s.h0 + s.hc - 1) % cap;
    const long oy = L.hy + (long)slot * L.vstride;
    const double scl = Z.cw[L.hsy + (long)slot * Z.B + Z.e] / qdot(Z, oy, oy, n);
    qmap2(Z, n, L.q, L.q, L.q, [scl](double qv, double) { return qv * scl; });
  }
  for (int i = 0; i < s.hc; ++i) {
    const int slot = (s.h0 + i) % cap;
    const long os = L.hs + (long)slot * L.vstride, oy = L.hy + (long)slot * L.vstride;
    const double beta = qdot(Z, oy, L.q, n) / Z.cw[L.hsy + (long)slot * Z.B + Z.e];
    const double c = alpha[i] - beta;
    qmap2(Z, n, L.q, L.q, os, [c](double qv, double sv) { return qv + c * sv; });
  }
}

// LbfgsSolver::iterate (optim.cpp:152-205)
__device__ int lbfgs_iterate(const Q& Z, SolverState& s) {
  const DOpt& o = Z.sc->opt;
  const ChainLayout& L = *Z.L;
  const int n = Z.m->n;
  if (s.status != ST_RUNNING) return s.status;
  if (s.iters >= o.max_iters) return s.status = ST_FAILED;
  if (grad_converged(Z, s)) return s.status = ST_CONVERGED;
  two_loop(Z, s);
  qmap2(Z, n, L.dir, L.q, L.q, [](double qv, double) { return -qv; });
  double slope = qdot(Z, L.dir, L.g, n);
  if (!(slope < 0.0)) {
    s.hc = 0;
    s.h0 = 0;
    qmap2(Z, n, L.dir, L.g, L.g, [](double gv, double) { return -gv; });
    slope = qdot(Z, L.dir, L.g, n);
  }
  double t = 1.0;
  bool accepted = false;
  const double fval = s.value;
  const int cap = o.mem + 1;
  for (int trial = 0; trial < o.max_line_search; ++trial) {
    qmap2(Z, n, L.cand, L.x, L.dir, [t](double xv, double dv) { return xv + t * dv; });
    if (qallfinite(Z, L.cand, n)) {
      const double v = chain_forward(Z, L.cand, true);
      if (isfinite(v) && v <= fval + o.armijo_c1 * t * slope && v < fval) {
        chain_reverse(Z, L.evg);
        const int slot = (s.h0 + s.hc) % cap;
        const long os = L.hs + (long)slot * L.vstride, oy = L.hy + (long)slot * L.vstride;
        qmap2(Z, n, os, L.dir, L.dir, [t](double dv, double) { return t * dv; });
        qmap2(Z, n, oy, L.evg, L.g, [](double ev, double gv) { return ev - gv; });
        const double sy = qdot(Z, os, oy, n);
        if (sy > 1e-12) {
          if (Z.r == 0) Z.cw[L.hsy + (long)slot * Z.B + Z.e] = sy;
          ++s.hc;
          if (s.hc > o.mem) {
            s.h0 = (s.h0 + 1) % cap;
            --s.hc;
          }
        }
        qmap2(Z, n, L.x, L.cand, L.cand, [](double cv, double) { return cv; });
        qmap2(Z, n, L.g, L.evg, L.evg, [](double ev, double) { return ev; });
        qsync(Z);
        s.value = v;
        accepted = true;
        ++s.acc;
        if (stagnation_update(Z, s, fval, v)) s.status = ST_CONVERGED;
        break;
      }
    }
    t *= o.backtrack_factor;
  }
  if (!accepted) s.status = ST_FAILED;
  ++s.iters;
  if (s.status == ST_RUNNING && s.iters >= o.max_iters) s.status = ST_FAILED;
  return s.status;
}

// ForceModel::tau_at (objective.hpp:28-58) into the tau vector
__device__ void tau_at(const Q& Z, double t) {
  const DForces& f = *Z.f;
  const int n = Z.m->n;
  for (int i = Z.r; i < n; i += 4) {
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
    *vel(Z, Z.L->tau, i) = v;
  }
}

// fd_kinetic + gravity_potential of the new configuration (stepper.cpp:132-138)
__device__ void chain_energy(const Q& Z, long wprev, long wnext, double dt, double* ke, double* pe) {
  const int N = Z.m->N;
  double k = 0.0, p = 0.0;
  const double ghat[4] = {Z.f->gravity[0], Z.f->gravity[1], Z.f->gravity[2], 0.0};
  for (int i = 0; i < N; ++i) {
    double wp[4], wn[4], td[4], tds[4];
    ld4(lrow(Z, wprev, i), wp);
    ld4(lrow(Z, wnext, i), wn);
#pragma unroll
    for (int c = 0; c < 4; ++c) td[c] = (wn[c] - wp[c]) / dt;
    const M4 S = ldS(Z, i);
    row_mul(td, S, tds);
    const double e4[4] = {0.0, 0.0, 0.0, 1.0};
    double u[4];
    mul_vec4(S, e4, u);
    double part[2], out[2];
    part[0] = ddot_row(tds, td);
    double wu = wn[0] * u[0];
    wu = fma(wn[1], u[1], wu);
    wu = fma(wn[2], u[2], wu);
    wu = fma(wn[3], u[3], wu);
    part[1] = wu;  // row r of (W u)
    qsync(Z);
    Z.red[Z.r] = part[0];
    Z.red[4 + Z.r] = part[1];
    qsync(Z);
    out[0] = ((Z.red[0] + Z.red[1]) + Z.red[2]) + Z.red[3];
    double d = ghat[0] * Z.red[4];
    d = fma(ghat[1], Z.red[5], d);
    d = fma(ghat[2], Z.red[6], d);
    d = fma(ghat[3], Z.red[7], d);
    k += 0.5 * out[0];
    p -= d;
  }
  *ke = k;
  *pe = p;
}

__device__ __forceinline__ Q make_q(const DModel* m, const DForces* f, const DSchedule* sc, const ChainLayout* L,
                                    double* cw, int* ci, long B, double* red_base, bool* valid) {
  const int lane = threadIdx.x & 31;
  const int quad_in_block = threadIdx.x >> 2;
  const long e = (long)blockIdx.x * kEnvsPerBlock + quad_in_block;
  Q Z{m, f, sc, L, cw, ci, B, (int)e, lane & 3, 0xFu << (lane & ~3), red_base + 16 * quad_in_block};
  *valid = e < B;
  return Z;
}

}  // namespace

// init_pbad_run (stepper.cpp:62-80) for the chain path
__global__ void __launch_bounds__(kThreads) k_chain_init(DModel m, DForces f, DSchedule sc, ChainLayout L, double* cw,
                                                         int* ci, long B, const double* q0, const double* qdot0,
                                                         Outputs out) {
  __shared__ double red[16 * kEnvsPerBlock];
  bool valid;
  const Q Z = make_q(&m, &f, &sc, &L, cw, ci, B, red, &valid);
  if (!valid) return;
  const int n = m.n, N = m.N;
  bool finite = true;
  for (int k = Z.r; k < n; k += 4) {
    const double q = q0[(long)Z.e * n + k];
    *vel(Z, L.h1, k) = q;
    *vel(Z, L.g, k) = qdot0[(long)Z.e * n + k];  // qdot scratch
    finite = finite && isfinite(q);
  }
  finite = __all_sync(Z.qm, finite);
  if (Z.r == 0) {
    ival(Z, IS_STEP) = 0;
    ival(Z, IS_FAIL) = 0;
    ival(Z, IS_NSAMP) = 0;
    ival(Z, IS_NREP) = 0;
  }
  if (!finite) {
    if (Z.r == 0) ival(Z, IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  const double tl = sc.times[0] * sc.dt;
  for (int k = Z.r; k < n; k += 4) *vel(Z, L.h0, k) = *vel(Z, L.h1, k) + tl * *vel(Z, L.g, k);
  qsync(Z);
  // kinetic_energy via the velocity pass (baseline.cpp:20-54,208-217) and
  // gravity_potential (baseline.cpp:219-229) at q0
  double T[4], Td[4];
  identity_row(Z.r, T);
  Td[0] = Td[1] = Td[2] = Td[3] = 0.0;
  double ke = 0.0, pe = 0.0;
  const double ghat[4] = {f.gravity[0], f.gravity[1], f.gravity[2], 0.0};
  for (int i = 0; i < N; ++i) {
    // general joint algebra here (runs once per trajectory)
    M4 Lv, d1;
    {
      const double qi = *vel(Z, L.h1, i);
      const double* ax = m.axis + 3 * i;
      M4 o;
#pragma unroll
      for (int k = 0; k < 16; ++k) o.a[k] = __ldg(m.offset + 16 * i + k);
      const M3 R = rotation_vector_matrix(ax[0] * qi, ax[1] * qi, ax[2] * qi);
      Lv = mul(o, motion_rot(R));
      d1 = mul(o, embed_rotation(mul3(skew(ax[0], ax[1], ax[2]), R)));
    }
    const double qd = *vel(Z, L.g, i);
    M4 ldot;
#pragma unroll
    for (int k = 0; k < 16; ++k) ldot.a[k] = 0.0 + qd * d1.a[k];
    double a[4], b[4], Tn[4], Tdn[4];
    if (i == 0) {
      // parent_tdot = Zero, parent_world = Identity
      double z[4] = {0.0, 0.0, 0.0, 0.0};
      row_mul(z, Lv, a);
    } else {
      row_mul(Td, Lv, a);
    }
    row_mul(T, ldot, b);
#pragma unroll
    for (int c = 0; c < 4; ++c) Tdn[c] = a[c] + b[c];
    if (i == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) Tn[c] = Lv.a[Z.r + 4 * c];
    } else {
      row_mul(T, Lv, Tn);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      T[c] = Tn[c];
      Td[c] = Tdn[c];
    }
    st4(lrow(Z, L.tk, i), T);
    const M4 S = ldS(Z, i);
    double tds[4];
    row_mul(Td, S, tds);
    const double e4[4] = {0.0, 0.0, 0.0, 1.0};
    double u[4];
    mul_vec4(S, e4, u);
    double wu = T[0] * u[0];
    wu = fma(T[1], u[1], wu);
    wu = fma(T[2], u[2], wu);
    wu = fma(T[3], u[3], wu);
    qsync(Z);
    Z.red[Z.r] = ddot_row(tds, Td);
    Z.red[4 + Z.r] = wu;
    qsync(Z);
    const double term = ((Z.red[0] + Z.red[1]) + Z.red[2]) + Z.red[3];
    double d = ghat[0] * Z.red[4];
    d = fma(ghat[1], Z.red[5], d);
    d = fma(ghat[2], Z.red[6], d);
    d = fma(ghat[3], Z.red[7], d);
    ke += 0.5 * term;
    pe -= d;
  }
  const long S1 = sc.total_steps + 1;
  for (int k = Z.r; k < n; k += 4)
    if (out.q) out.q[((long)Z.e * S1) * n + k] = *vel(Z, L.h1, k);
  if (Z.r == 0) {
    if (out.energy) {
      out.energy[((long)Z.e * S1) * 2] = ke;
      out.energy[((long)Z.e * S1) * 2 + 1] = pe;
    }
    ival(Z, IS_NSAMP) = 1;
    ival(Z, IS_RUN) = (sc.total_steps > 0) ? TR_RUNNING : TR_OK;
  }
}

// One PBAD step per environment: begin_step, L-BFGS to completion,
// finish_step (stepper.cpp:83-147).
__global__ void __launch_bounds__(kThreads) k_chain_step(DModel m, DForces f, DSchedule sc, ChainLayout L, double* cw,
                                                         int* ci, long B, Outputs out) {
  __shared__ double red[16 * kEnvsPerBlock];
  bool valid;
  const Q Z = make_q(&m, &f, &sc, &L, cw, ci, B, red, &valid);
  if (!valid) return;
  if (ival(Z, IS_RUN) != TR_RUNNING) return;
  const int n = m.n;
  const int step = ival(Z, IS_STEP);
  // StepObjective ctor validates the history (objective.cpp:176-177)
  if (!qallfinite(Z, L.h0, n) || !qallfinite(Z, L.h1, n)) {
    if (Z.r == 0) ival(Z, IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  // begin_step
  tau_at(Z, step * sc.dt + sc.times[2] * sc.dt);
  const double span = -sc.times[0];
  const double tau_m = sc.times[2];
  for (int k = Z.r; k < n; k += 4) {
    const double h1 = *vel(Z, L.h1, k), h0 = *vel(Z, L.h0, k);
    *vel(Z, L.x, k) = sc.warm_start ? h1 + (tau_m / span) * (h1 - h0) : h1;
  }
  qsync(Z);
  // StepObjective ctor: history passes and hist_const (objective.cpp:162-185)
  chain_fk(Z, L.h0, L.tk1);
  chain_fk(Z, L.h1, L.tk);
  qsync(Z);
  const double hc = 4.0 * chain_cv(Z, L.tk, L.tk) + chain_cv(Z, L.tk1, L.tk1) - 4.0 * chain_cv(Z, L.tk, L.tk1);
  if (Z.r == 0) scal(Z, L.histc) = hc;
  qsync(Z);
  // LbfgsSolver ctor: first evaluation
  SolverState s{};
  s.status = ST_RUNNING;
  if (!qallfinite(Z, L.x, n)) {
    if (Z.r == 0) ival(Z, IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  const double v0 = chain_forward(Z, L.x, true);
  if (!isfinite(v0)) {
    if (Z.r == 0) ival(Z, IS_RUN) = TR_NONFINITE_INIT;
    return;
  }
  chain_reverse(Z, L.g);
  s.value = v0;
  s.grad0 = qinfnorm(Z, L.g, n);
  while (lbfgs_iterate(Z, s) == ST_RUNNING) {
  }
  // finish_step
  const long S = sc.total_steps;
  const bool converged = s.status == ST_CONVERGED;
  const double gnorm = qinfnorm(Z, L.g, n);
  if (Z.r == 0) {
    if (out.iterations) out.iterations[(long)Z.e * S + step] = s.iters;
    if (out.converged) out.converged[(long)Z.e * S + step] = converged;
    if (out.accepted) out.accepted[(long)Z.e * S + step] = s.acc;
    if (out.final_value) out.final_value[(long)Z.e * S + step] = s.value;
    if (out.final_grad_norm) out.final_grad_norm[(long)Z.e * S + step] = gnorm;
    ival(Z, IS_NREP) = step + 1;
  }
  const int fs = converged ? 0 : ival(Z, IS_FAIL) + 1;
  qsync(Z);
  if (Z.r == 0) ival(Z, IS_FAIL) = fs;
  if (fs > sc.fail_limit) {
    if (Z.r == 0) ival(Z, IS_RUN) = TR_FAIL_LIMIT;
    return;
  }
  for (int k = Z.r; k < n; k += 4) {
    *vel(Z, L.h0, k) = *vel(Z, L.h1, k);
    *vel(Z, L.h1, k) = *vel(Z, L.x, k);
  }
  qsync(Z);
  chain_fk(Z, L.h1, L.tk1);  // tk holds forward_pass(old hist1)
  qsync(Z);
  double ke, pe;
  chain_energy(Z, L.tk, L.tk1, sc.dt, &ke, &pe);
  const long S1 = S + 1;
  for (int k = Z.r; k < n; k += 4)
    if (out.q) out.q[((long)Z.e * S1 + step + 1) * n + k] = *vel(Z, L.h1, k);
  if (Z.r == 0) {
    if (out.energy) {
      out.energy[((long)Z.e * S1 + step + 1) * 2] = ke;
      out.energy[((long)Z.e * S1 + step + 1) * 2 + 1] = pe;
    }
    ival(Z, IS_STEP) = step + 1;
    ival(Z, IS_NSAMP) = step + 2;
    if (step + 1 >= S) ival(Z, IS_RUN) = TR_OK;
  }
}

unsigned chain_grid(long B) { return (unsigned)((B + kEnvsPerBlock - 1) / kEnvsPerBlock); }

cudaError_t launch_chain_init(const ChainArgs& a, const double* q0, const double* qdot0, const Outputs& out,
                              cudaStream_t s) {
  k_chain_init<<<chain_grid(a.B), kThreads, 0, s>>>(a.m, a.f, a.sc, a.L, a.cw, a.ci, a.B, q0, qdot0, out);
  return cudaGetLastError();
}
cudaError_t launch_chain_step(const ChainArgs& a, const Outputs& out, cudaStream_t s) {
  k_chain_step<<<chain_grid(a.B), kThreads, 0, s>>>(a.m, a.f, a.sc, a.L, a.cw, a.ci, a.B, out);
  return cudaGetLastError();
}
int chain_max_memory() { return kMaxMem; }

}  // namespace pbad_gpu
