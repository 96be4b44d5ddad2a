// pbad_resid.cu -- CTA-per-environment Newton (LM) kernel for the residual
// (high-order collocation) form of PBAD: the C5 workload (SURVEY.md §8 K6+K7).
//
// One thread block owns one environment for a whole PBAD step (begin_step, the
// Levenberg-Marquardt loop, finish_step; stepper.cpp:83-147, optim.cpp:80-139).
// The unknowns are the u = K-1 stacked configurations of the collocation window
// (U = u n); per accepted iterate the kernel builds the residual Jacobian J
// (objective.cpp:258-334: u functional_hess blocks, u^2 correlation_hess_ab
// blocks, the gravity potential Hessian) and the Gauss-Newton matrix 2 J^T J;
// every iteration factors the damped U x U matrix.  Layout per environment
// (env-major, HBM/L2): J, GN and the factor as column-major U x U matrices,
// the u link passes, the u^2 hess_ab walk states.  Shared memory holds the
// GEMM operand tiles, the panel of the blocked Cholesky and the solve vector.
//
//  * J^T J: 64 x 64 output tiles of the lower triangle, 4 x 4 per thread,
//    operand k-chunks staged in shared memory with 2 J pre-applied.  Because
//    2 J(k,a) J(k,b) is the same real number as 2 J(k,b) J(k,a) (doubling is
//    exact), the reference's ab1/ab2 chains are equal bit for bit and
//    0.5 (gn + gn^T) is gn itself: only one triangle is computed.
//  * Cholesky (optim.cpp:11-15): blocked left-looking with 32-wide block
//    columns -- a register-tiled update of the block column by all previous
//    columns (each element's fma chain runs over k ascending, exactly the
//    reference's right-looking order), the diagonal block factored by one warp
//    in registers, the rows below solved one thread per row.
//  * triangular solves blocked the same way (warp solves the diagonal block,
//    all threads apply it to the remaining rows).
// Every scalar follows the numeric contract (pbad_math.cuh); results are
// bit-identical to the reference build and the C oracle.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "pbad_joint.cuh"
#include "pbad_kernels.cuh"
#include "pbad_launch.h"
#include "pbad_math.cuh"

namespace pbad_gpu {
namespace resid {

#ifndef PBAD_RESID_CHOL_REG
#define PBAD_RESID_CHOL_REG 2  // 2: lookahead; 1: diagonal blocks and solve rows in registers (unrolled); 0: shared memory loops
#endif
#ifndef PBAD_RESID_NT
#define PBAD_RESID_NT 256
#endif
constexpr int NT = PBAD_RESID_NT;  // threads per environment (256 or 512)
constexpr int TG = NT / 256;       // concurrent J^T J tiles
constexpr unsigned FULL = 0xffffffffu;
enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_FAILED = 2 };
enum { TR_OK = 0, TR_FAIL_LIMIT = 1, TR_NONFINITE_INIT = 2, TR_NONFINITE_CFG = 3, TR_RUNNING = 4 };

// GEMM (J^T J) tiling
constexpr int GB = 64;       // output tile
constexpr int GK = 32;       // k chunk
constexpr int GP = GB + 1;   // padded smem row (odd: conflict-free staging stores)
// Cholesky tiling
constexpr int CB = 32;       // block column width
constexpr int LK = 16;       // k chunk of the block-column update
constexpr int MAXU = 400;       // U = u n; shared memory bounds it further (resid_eligible_sizes)
constexpr int SMS = 18;      // shared-memory stride of a 4x4 (16 + 2 pad: conflict-free per-link double2 access)
constexpr int LP = MAXU + 2; // padded smem row of the update panel
constexpr int LSCAP = 16384; // shared-memory doubles for the Cholesky update panel
constexpr int LSCAP_A = 12288;  // lookahead variant: panel of warps 1..7
constexpr int LSCAP_C = 10240;  // lookahead variant: panel of block J's columns

__device__ __forceinline__ M4 ldm4(const double* p) {
  M4 m;
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 v = q[k];
    m.a[2 * k] = v.x;
    m.a[2 * k + 1] = v.y;
  }
  return m;
}
__device__ __forceinline__ M4 ldgm4(const double* p) {
  M4 m;
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 v = __ldg(q + k);
    m.a[2 * k] = v.x;
    m.a[2 * k + 1] = v.y;
  }
  return m;
}
__device__ __forceinline__ void stm4(double* p, const M4& m) {
  double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
  for (int k = 0; k < 8; ++k) q[k] = make_double2(m.a[2 * k], m.a[2 * k + 1]);
}
__device__ __forceinline__ double trace_mul(const M4& X, const M4& F) {
  double d[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    double acc = X.a[p] * F.a[4 * p];
    acc = fma(X.a[p + 4], F.a[1 + 4 * p], acc);
    acc = fma(X.a[p + 8], F.a[2 + 4 * p], acc);
    acc = fma(X.a[p + 12], F.a[3 + 4 * p], acc);
    d[p] = acc;
  }
  return ((d[0] + d[1]) + d[2]) + d[3];
}
__device__ __forceinline__ M4 gravity_cot(const DForces& f, const M4& S) {
  const double ghat[4] = {f.gravity[0], f.gravity[1], f.gravity[2], 0.0};
  const double e4[4] = {0.0, 0.0, 0.0, 1.0};
  double u[4];
  mul_vec4(S, e4, u);
  M4 c;
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int r = 0; r < 4; ++r) c.a[r + 4 * s] = (-ghat[r]) * u[s];
  return c;
}

#ifndef PBAD_PHASE_TIMING
#define PBAD_PHASE_TIMING 0  // 1: per-phase clock64 totals printed by block 0 (diagnostic builds only)
#endif
struct Smem {
  long long pt[20];
  double red[NT];
  int flag;
  double scal[8];
  int parent[MAXU];
  short pk32[CB * (CB + 1) / 2];  // packed 32x32 lower triangle, column-major: row | col << 8
};

// Shared memory is addressed through these namespace-scope symbols (not through
// pointers stored in R) so the out-of-line phase functions keep LDS/STS
// addressing instead of generic loads.
__shared__ Smem rss;
extern __shared__ __align__(16) double rsm[];

#if PBAD_PHASE_TIMING
#define PT_START() long long pt_t0 = clock64()
#define PT_MARK(k)                                   \
  do {                                               \
    const long long pt_t1 = clock64();               \
    if (r.tid == 0) rss.pt[k] += pt_t1 - pt_t0;    \
    pt_t0 = pt_t1;                                   \
  } while (0)
#else
#define PT_START() \
  do {             \
  } while (0)
#define PT_MARK(k) \
  do {             \
  } while (0)
#endif


// per-environment context (identical in every thread)
struct R {
  const DModel* m;
  const DForces* f;
  const DSchedule* sc;
  const ResidDesc* rd;
  int tid, N, n, u, U, D, K1;
  bool grav;
  bool drag;      // residual form with drag (chains): per-instant cotangents, pot.hess adds 2 scale ab
  bool have_cot;  // potential cotangents exist (gravity or drag: PotentialEval::have_cot)
  bool contact;   // residual form with contact samples (hinge trees, walks path)
  bool cot_pi;    // cotangents per instant (drag or contact), else the gravity cotangent once
  double s2[8];   // drag: 2 D / (t_m dt)^2 per unknown instant (objective.cpp:62-68)
  bool energy;    // energy form (K = 2, u = 1): the large-n Newton path of the energy objective
  double histc;   // energy form: hist_const (objective.cpp:178-184)
  double inv_dt2;
  double *J, *GN, *DM, *FH, *PH, *pass, *hw0, *hw1, *HA, *FA, *seeds, *cot, *x, *grad, *cand, *res, *pg, *tau,
      *step, *CJ;
  __device__ __forceinline__ double* val(int mm) const { return pass + mm * rd->pstride; }
  __device__ __forceinline__ double* wld(int mm) const { return pass + mm * rd->pstride + 16L * N; }
  __device__ __forceinline__ double* dd1(int mm) const { return pass + mm * rd->pstride + 32L * N; }
  __device__ __forceinline__ double* dd2(int mm) const { return pass + mm * rd->pstride + 48L * N; }
  __device__ __forceinline__ double* lev(int mm) const { return pass + mm * rd->pstride + 64L * N; }
  // hess_ab state of pair (a, b): ai, fwd, bwd, Z
  __device__ __forceinline__ double* ha(int pair, int k) const { return HA + (pair * 4L + k) * 16L * N; }
  // functional_grad sweep sw (0..u-1 seeds of instant sw, u..2u-1 gravity at instant sw-u): a, X
  __device__ __forceinline__ double* fa(int sw, int k) const { return FA + (sw * 2L + k) * 16L * N; }
};

// ---- block reductions (result in every thread) ----
__device__ double block_max(const R& r, double v) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, s));
  __syncthreads();
  if ((r.tid & 31) == 0) rss.red[r.tid >> 5] = v;
  __syncthreads();
  double mx = 0.0;
  for (int w = 0; w < NT / 32; ++w) mx = fmax(mx, rss.red[w]);
  __syncthreads();
  return mx;
}
__device__ double infnorm(const R& r, const double* a, int len) {
  double mx = 0.0;
  for (int i = r.tid; i < len; i += NT) mx = fmax(mx, fabs(a[i]));
  return block_max(r, mx);
}
__device__ bool all_finite(const R& r, const double* a, int len) {
  bool ok = true;
  for (int i = r.tid; i < len; i += NT) ok = ok && isfinite(a[i]);
  return __syncthreads_and(ok) != 0;
}

// Serial chain recursions (rd.chain): one 16-lane group per recursion, lane
// e16 = row + 4 col holding that element of a 4x4, the operand rows/columns
// gathered by shuffles inside the group.  Every element keeps the contract's
// product sequence (pbad_math.cuh mul / mul_bt: first product, then fma in
// ascending k), so the values equal the level-synchronous block version; the
// chain depth no longer costs a block barrier per link.
// (the other half-warp may be outside any group: the mask names this group only)
__device__ __forceinline__ double gsh(double v, int src) {
  return __shfl_sync(0xFFFFu << (threadIdx.x & 16), v, src, 16);
}
// element (ri, cj) of A B, A held by the group (lane ri + 4 k), B(k, cj) = Bm[k + 4 cj]
__device__ __forceinline__ double g_mul_left(double a_el, const double* Bm, int ri, int cj) {
  const double a0 = gsh(a_el, ri), a1 = gsh(a_el, ri + 4), a2 = gsh(a_el, ri + 8), a3 = gsh(a_el, ri + 12);
  double acc = a0 * Bm[4 * cj];
  acc = fma(a1, Bm[1 + 4 * cj], acc);
  acc = fma(a2, Bm[2 + 4 * cj], acc);
  return fma(a3, Bm[3 + 4 * cj], acc);
}
// element (ri, cj) of A B^T, A held by the group, B(cj, k) = Bm[cj + 4 k]
__device__ __forceinline__ double g_mul_bt(double a_el, const double* Bm, int ri, int cj) {
  const double a0 = gsh(a_el, ri), a1 = gsh(a_el, ri + 4), a2 = gsh(a_el, ri + 8), a3 = gsh(a_el, ri + 12);
  double acc = a0 * Bm[cj];
  acc = fma(a1, Bm[cj + 4], acc);
  acc = fma(a2, Bm[cj + 8], acc);
  return fma(a3, Bm[cj + 12], acc);
}
// element (ri, cj) of A B, A(ri, k) = Am[ri + 4 k] in memory, B held by the group (lane k + 4 cj)
__device__ __forceinline__ double g_mul_right(const double* Am, double b_el, int ri, int cj) {
  const double b0 = gsh(b_el, 4 * cj), b1 = gsh(b_el, 1 + 4 * cj), b2 = gsh(b_el, 2 + 4 * cj),
               b3 = gsh(b_el, 3 + 4 * cj);
  double acc = Am[ri] * b0;
  acc = fma(Am[ri + 4], b1, acc);
  acc = fma(Am[ri + 8], b2, acc);
  return fma(Am[ri + 12], b3, acc);
}

// forward_pass (kinematics.cpp:171-181) of one configuration into world
__device__ __noinline__ void fk_config(const R& r, const double* q, double* world) {
  const DModel& m = *r.m;
  const ResidDesc& rd = *r.rd;
  for (int i = r.tid; i < r.N; i += NT)
    stm4(world + 16 * i, joint_transform(m.kind[i], m.axis + 3 * i, ldgm4(m.offset + 16 * i), q + m.dof_off[i]));
  __syncthreads();
  for (int d = 1; d <= r.D; ++d) {
    for (int t = rd.lvl_start[d] + r.tid; t < rd.lvl_start[d + 1]; t += NT) {
      const int i = rd.lvl_links[t];
      stm4(world + 16 * i, mul(ldm4(world + 16 * m.parent[i]), ldm4(world + 16 * i)));
    }
    __syncthreads();
  }
}

// ConfigPass::make (adjoint.cpp:9-27) for the u stacked configurations of xs.
// false = a non-finite entry (ModelError).
__device__ __noinline__ bool passes(const R& r, const double* xs, bool want_d2) {
  if (!all_finite(r, xs, r.U)) return false;
  const DModel& m = *r.m;
  const ResidDesc& rd = *r.rd;
  const int N = r.N;
  const long NS = (long)SMS * N;
  double* Vs = rsm;                 // values [u][N][16]
  double* Ws = rsm + r.u * NS;     // worlds [u][N][16]
  for (int t = r.tid; t < r.u * N; t += NT) {
    const int mm = t / N, i = t - mm * N;
    const double q = xs[mm * r.n + i];
    M4 v, d1, d2;
    joint_jet(0, m.axis + 3 * i, ldgm4(m.offset + 16 * i), &q, &v, &d1, &d2, want_d2);
    stm4(Vs + mm * NS + SMS * i, v);
    stm4(r.val(mm) + 16 * i, v);
    stm4(r.dd1(mm) + 16 * i, d1);
    if (want_d2) stm4(r.dd2(mm) + 16 * i, d2);
  }
  __syncthreads();
  if (rd.chain) {
    // W_i = W_{i-1} V_i, group mm = instant mm
    const int g = r.tid >> 4, e16 = r.tid & 15, ri = e16 & 3, cj = e16 >> 2;
    if (g < r.u) {
      double w = 0.0;
      for (int i = 0; i < N; ++i) {
        const double* V = Vs + g * NS + SMS * i;
        w = (i == 0) ? V[e16] : g_mul_left(w, V, ri, cj);
        Ws[g * NS + SMS * i + e16] = w;
      }
    }
    __syncthreads();
  } else {
    for (int d = 0; d <= r.D; ++d) {
      const int l0 = rd.lvl_start[d], cnt = rd.lvl_start[d + 1] - l0;
      for (int t = r.tid; t < r.u * cnt; t += NT) {
        const int mm = t / cnt;
        const int i = rd.lvl_links[l0 + t - mm * cnt];
        const int p = rss.parent[i];
        const M4 v = ldm4(Vs + mm * NS + SMS * i);
        stm4(Ws + mm * NS + SMS * i, p >= 0 ? mul(ldm4(Ws + mm * NS + SMS * p), v) : v);
      }
      __syncthreads();
    }
  }
  for (int t = r.tid; t < r.u * N; t += NT) {
    const int mm = t / N, i = t - mm * N;
    const int p = rss.parent[i];
    stm4(r.wld(mm) + 16 * i, ldm4(Ws + mm * NS + SMS * i));
    const M4 pw = p >= 0 ? ldm4(Ws + mm * NS + SMS * p) : m4_identity();
    stm4(r.lev(mm) + 16 * i, mul(pw, ldm4(r.dd1(mm) + 16 * i)));
  }
  __syncthreads();
  return true;
}

// second joint derivatives of the u configurations (joint_jet d2, kinematics.cpp:119-169);
// the rest of the pass is already current
__device__ __noinline__ void passes_d2(const R& r, const double* xs) {
  const DModel& m = *r.m;
  const int N = r.N;
  for (int t = r.tid; t < r.u * N; t += NT) {
    const int mm = t / N, i = t - mm * N;
    const double q = xs[mm * r.n + i];
    M4 v, d1, d2;
    joint_jet(0, m.axis + 3 * i, ldgm4(m.offset + 16 * i), &q, &v, &d1, &d2, true);
    stm4(r.dd2(mm) + 16 * i, d2);
  }
  __syncthreads();
}

// stage the u passes' values and levers into shared memory
__device__ void stage_vl(const R& r, double* Vs, double* Ls) {
  const int N8 = 8 * r.N;  // double2 per pass
  for (int t = r.tid; t < r.u * N8; t += NT) {
    const int mm = t / N8;
    const int e = t - mm * N8;
    const int link = e >> 3, k = 2 * (e & 7);
    const long dst = (long)mm * SMS * r.N + SMS * link + k;
    *reinterpret_cast<double2*>(Vs + dst) = *reinterpret_cast<const double2*>(r.val(mm) + 2 * e);
    *reinterpret_cast<double2*>(Ls + dst) = *reinterpret_cast<const double2*>(r.lev(mm) + 2 * e);
  }
}

__device__ __noinline__ void adjoint_sweeps(const R& r);

// contact sample sidx of link i at instant mm (objective.cpp:77-90, dt = t_m dt):
// false = inactive (depth <= 0); else ph, the projected velocity and depth
__device__ __forceinline__ bool contact_state(const R& r, int mm, int i, int sidx, double (&ph)[4], double (&pv)[3],
                                              double* depth_out) {
  const DModel& m = *r.m;
  const DForces& f = *r.f;
  const double* nrm = f.normal;
  ph[0] = m.samples[3 * sidx];
  ph[1] = m.samples[3 * sidx + 1];
  ph[2] = m.samples[3 * sidx + 2];
  ph[3] = 1.0;
  double x4[4], xp4[4];
  mul_vec4(ldm4(r.wld(mm) + 16 * i), ph, x4);
  const double depth = f.plane_offset - dot3(nrm, x4);
  if (depth <= 0.0) return false;
  const double dtm = r.sc->times[2 + mm] * r.sc->dt;
  mul_vec4(ldm4(r.hw1 + 16 * i), ph, xp4);
  double proj[9];
  for (int c = 0; c < 3; ++c)
    for (int rr = 0; rr < 3; ++rr) proj[rr + 3 * c] = ((rr == c) ? 1.0 : 0.0) - nrm[rr] * nrm[c];
  double v[3];
  for (int k = 0; k < 3; ++k) v[k] = (x4[k] - xp4[k]) / dtm;
  for (int rr = 0; rr < 3; ++rr) {
    double acc = proj[rr] * v[0];
    acc = fma(proj[rr + 3], v[1], acc);
    acc = fma(proj[rr + 6], v[2], acc);
    pv[rr] = acc;
  }
  *depth_out = depth;
  return true;
}

// residuals g_m (objective.cpp:281-308) of the configuration whose passes are
// current; returns value = sum_m |g_m|^2 (objective.cpp:323-324).  Leaves the
// adjoint sums a of every sweep in fa(sw, 0) for functional_hess.
__device__ __noinline__ double residual(const R& r) {
  const DModel& m = *r.m;
  const DSchedule& sc = *r.sc;
  const ResidDesc& rd = *r.rd;
  const int N = r.N, n = r.n, u = r.u;
  for (int t = r.tid; t < u * N; t += NT) {
    const int mm = t / N, i = t - mm * N;
    const double* st = sc.H2 + r.K1 * (2 + mm);
    M4 acc = m4_zero();
    for (int j = 0; j < r.K1; ++j) {
      const double* W = (j == 0) ? r.hw0 : (j == 1) ? r.hw1 : r.wld(j - 2);
      addto(acc, scale(st[j], ldm4(W + 16 * i)));
    }
    stm4(r.seeds + (long)mm * 16 * N + 16 * i, mul(scale(r.inv_dt2, acc), ldgm4(m.S + 16 * i)));
    if (r.cot_pi) {
      // potential_terms' cotangents at instant mm (objective.cpp:45-101):
      // cot = (0 + gravity) + (2 D / (t_m dt)^2) (T_m - T_hist1) S, then
      // + dqdx ph^T of every active contact sample of the link, in order
      const M4 S = ldgm4(m.S + 16 * i);
      M4 cot = r.grav ? add(m4_zero(), gravity_cot(*r.f, S)) : m4_zero();
      if (r.drag) {
        const M4 diff_s = mul(sub(ldm4(r.wld(mm) + 16 * i), ldm4(r.hw1 + 16 * i)), S);
        cot = add(cot, scale(r.s2[mm], diff_s));
      }
      if (r.contact) {
        const DForces& f = *r.f;
        const double dtm = sc.times[2 + mm] * sc.dt;
        for (int sidx = m.sample_off[i]; sidx < m.sample_off[i + 1]; ++sidx) {
          double ph[4], pv[3], depth;
          if (!contact_state(r, mm, i, sidx, ph, pv, &depth)) continue;
          const double pv2 = dot3(pv, pv);
          const double ca = -2.0 * f.d1 * depth - 2.0 * f.d2 * depth * pv2;
          const double cb = 2.0 * f.d2 * depth * depth / dtm;
          double dq[4];
          for (int k = 0; k < 3; ++k) dq[k] = ca * f.normal[k] + cb * pv[k];
          dq[3] = 0.0;
          M4 oc;
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) oc.a[rr + 4 * c] = dq[rr] * ph[c];
          cot = add(cot, oc);
        }
      }
      stm4(r.cot + (long)mm * 16 * N + 16 * i, cot);
    }
  }
  __syncthreads();
  adjoint_sweeps(r);
  for (int t = r.tid; t < r.U; t += NT) r.res[t] = r.res[t] + ((r.have_cot ? r.pg[t] : 0.0) - r.tau[t]);
  __syncthreads();
  // value: sum over instants of vdot32(g_m, g_m), warp mm computes instant mm
  const int warp = r.tid >> 5, lane = r.tid & 31;
  if (warp < u) {
    double p = 0.0;
    for (int i = lane; i < n; i += 32) p = fma(r.res[warp * n + i], r.res[warp * n + i], p);
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) p = p + __shfl_xor_sync(FULL, p, s);
    if (lane == 0) rss.scal[warp] = p;
  }
  __syncthreads();
  double v = 0.0;
  for (int mm = 0; mm < u; ++mm) v += rss.scal[mm];
  __syncthreads();
  return v;
}

// functional_grad (adjoint.cpp:49-64) of the u inertial seeds (r.seeds) and
// the u gravity cotangent sweeps, level-synchronous from the leaves: the
// inertial sums into r.res, the gravity sums into r.pg, the adjoints a of
// every sweep into fa(sw, 0)
__device__ __noinline__ void adjoint_sweeps(const R& r) {
  const ResidDesc& rd = *r.rd;
  const int N = r.N, n = r.n, u = r.u;
  const int nsw = r.have_cot ? 2 * u : u;
  const long NS = (long)SMS * N;
  double* Xs = rsm;                  // children contributions [2u][N][16]
  double* Ls = rsm + 2 * u * NS;    // levers [u][N][16]
  double* Vs = Ls + u * NS;          // values [u][N][16]
  stage_vl(r, Vs, Ls);
  __syncthreads();
  if (rd.chain) {
    // a_i = (0 + a_{i+1} V_{i+1}^T) + seed_i from the leaf, group sw = sweep sw;
    // the adjoints land in fa(sw, 0) and in shared memory (Xs, free here)
    // the seeds / cotangents staged in Xs first: the serial loop then reads
    // shared memory, not global loads ordered behind its own global stores
    for (int t = r.tid; t < nsw * N * 16; t += NT) {
      const int sw = t / (16 * N), k = t - sw * 16 * N;
      const double* src = sw < u ? r.seeds + (long)sw * 16 * N : r.cot + (r.cot_pi ? (long)(sw - u) * 16 * N : 0L);
      Xs[sw * NS + SMS * (k >> 4) + (k & 15)] = src[k];
    }
    __syncthreads();
    const int g = r.tid >> 4, e16 = r.tid & 15, ri = e16 & 3, cj = e16 >> 2;
    if (g < nsw) {
      const int mm = g < u ? g : g - u;
      double* fa = r.fa(g, 0);
      double* xg = Xs + g * NS + e16;
      double x = 0.0;  // element of a_{i+1} V_{i+1}^T
      for (int i = N - 1; i >= 0; --i) {
        const double adj = (i == N - 1) ? 0.0 : 0.0 + x;
        const double a = adj + xg[SMS * i];
        fa[16 * i + e16] = a;
        xg[SMS * i] = a;
        if (i > 0) x = g_mul_bt(a, Vs + mm * NS + SMS * i, ri, cj);
      }
    }
    __syncthreads();
    for (int t = r.tid; t < nsw * N; t += NT) {
      const int sw = t / N, i = t - sw * N;
      const int mm = sw < u ? sw : sw - u;
      const double gi = 0.0 + ddot(ldm4(Ls + mm * NS + SMS * i), ldm4(Xs + sw * NS + SMS * i));
      if (sw < u) r.res[mm * n + i] = gi;
      else r.pg[mm * n + i] = gi;
    }
    __syncthreads();
    return;
  }
  for (int d = r.D; d >= 0; --d) {
    const int l0 = rd.lvl_start[d], cnt = rd.lvl_start[d + 1] - l0;
    for (int t = r.tid; t < nsw * cnt; t += NT) {
      const int sw = t / cnt;
      const int i = rd.lvl_links[l0 + t - sw * cnt];
      const int mm = sw < u ? sw : sw - u;
      const double* src = sw < u ? r.seeds + (long)mm * 16 * N : r.cot + (r.cot_pi ? (long)mm * 16 * N : 0L);
      double* X = Xs + sw * NS;
      M4 adj = m4_zero();
      for (int c = rd.ch_start[i]; c < rd.ch_start[i + 1]; ++c) adj = add(adj, ldm4(X + SMS * rd.ch_list[c]));
      const M4 a = add(adj, ldm4(src + 16 * i));
      stm4(r.fa(sw, 0) + 16 * i, a);
      const double gi = 0.0 + ddot(ldm4(Ls + mm * NS + SMS * i), a);
      if (sw < u) r.res[mm * n + i] = gi;
      else r.pg[mm * n + i] = gi;
      stm4(X + SMS * i, mul_bt(a, ldm4(Vs + mm * NS + SMS * i)));
    }
    __syncthreads();
  }
}

// ---- energy form (objective.cpp:162-256), K = 2 (u = 1) --------------------
// The large-n Newton path of the energy objective on this kernel's CTA: the
// value from per-link correlation terms summed link by link by one thread
// (correlation_value's loop, adjoint.cpp:113-120), the gradient from the
// shared adjoint sweeps, the Gauss-Newton matrix from the hess_ab walks of
// jacobian() (pair (0, 0), scale inv_dt2) symmetrised like the reference.

// hist_const = 4 cv(A, A) + cv(H, H) - 4 cv(A, H), A = FK(hist1), H = FK(hist0)
// (objective.cpp:178-184); hw0/hw1 are current
__device__ __noinline__ double energy_hist_const(const R& r) {
  const DModel& m = *r.m;
  const int N = r.N;
  double* tt = rsm;  // [N][3]
  for (int i = r.tid; i < N; i += NT) {
    const M4 S = ldgm4(m.S + 16 * i);
    const M4 A = ldm4(r.hw1 + 16 * i), H = ldm4(r.hw0 + 16 * i);
    const M4 AS = mul(A, S);
    tt[3 * i] = ddot(AS, A);
    tt[3 * i + 1] = ddot(mul(H, S), H);
    tt[3 * i + 2] = ddot(AS, H);
  }
  __syncthreads();
  if (r.tid == 0) {
    double aa = 0.0, hh = 0.0, ah = 0.0;
    for (int i = 0; i < N; ++i) {
      aa += tt[3 * i];
      hh += tt[3 * i + 1];
      ah += tt[3 * i + 2];
    }
    const double wm = m.weighted_mass;
    rss.scal[0] = 4.0 * (aa - wm) + (hh - wm) - 4.0 * (ah - wm);
  }
  __syncthreads();
  const double hc = rss.scal[0];
  __syncthreads();
  return hc;
}

// StepObjective::value at xs (objective.cpp:215-239) from its current pass
__device__ __noinline__ double energy_value(const R& r, const double* xs) {
  const DModel& m = *r.m;
  const DForces& f = *r.f;
  const int N = r.N, n = r.n;
  double* tt = rsm;  // [N][4]
  for (int i = r.tid; i < N; i += NT) {
    const M4 S = ldgm4(m.S + 16 * i);
    const M4 T = ldm4(r.wld(0) + 16 * i);
    tt[4 * i] = ddot(mul(T, S), T);                            // cv(pass, pass)
    tt[4 * i + 1] = ddot(mul(ldm4(r.hw1 + 16 * i), S), T);     // cv(prev1, pass)
    tt[4 * i + 2] = ddot(mul(ldm4(r.hw0 + 16 * i), S), T);     // cv(prev2, pass)
    tt[4 * i + 3] = r.grav ? ddot(gravity_cot(f, S), T) : 0.0;  // gravity (objective.cpp:48-58)
  }
  // tau . x: the 32-partial dot (numeric contract) in warp 0
  if (r.tid < 32) {
    double p = 0.0;
    for (int i = r.tid; i < n; i += 32) p = fma(r.tau[i], xs[i], p);
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) p = p + __shfl_xor_sync(FULL, p, s);
    if (r.tid == 0) rss.scal[1] = p;
  }
  __syncthreads();
  if (r.tid == 0) {
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, pv = 0.0;
    for (int i = 0; i < N; ++i) {
      c0 += tt[4 * i];
      c1 += tt[4 * i + 1];
      c2 += tt[4 * i + 2];
    }
    if (r.grav)
      for (int i = 0; i < N; ++i) pv += tt[4 * i + 3];
    const double wm = m.weighted_mass;
    const double inertial = 0.5 * r.inv_dt2 * ((c0 - wm) - 4.0 * (c1 - wm) + 2.0 * (c2 - wm) + r.histc);
    rss.scal[0] = inertial + pv - rss.scal[1];
  }
  __syncthreads();
  const double v = rss.scal[0];
  __syncthreads();
  return v;
}

// gradient (objective.cpp:241-250): functional_grad of the seeds
// inv_dt2 (T - 2 A + H) S plus the gravity potential's, minus tau
__device__ __noinline__ void energy_grad(const R& r) {
  const DModel& m = *r.m;
  const int N = r.N;
  for (int i = r.tid; i < N; i += NT) {
    const M4 T = ldm4(r.wld(0) + 16 * i);
    const M4 d = add(sub(T, scale(2.0, ldm4(r.hw1 + 16 * i))), ldm4(r.hw0 + 16 * i));
    stm4(r.seeds + 16 * i, mul(scale(r.inv_dt2, d), ldgm4(m.S + 16 * i)));
  }
  __syncthreads();
  adjoint_sweeps(r);
  for (int t = r.tid; t < r.n; t += NT) r.grad[t] = (r.res[t] + (r.grav ? r.pg[t] : 0.0)) - r.tau[t];
  __syncthreads();
}

// gn_matrix = 0.5 (gn + gn^T), gn = inv_dt2 ab + pot.gn (pot.gn = 0 without
// drag / contact; objective.cpp:251-254), lower triangle into r.GN; jacobian()
// left J(l, i) = inv_dt2 ab(i, l)
__device__ __noinline__ void energy_gn(const R& r) {
  const int U = r.U;
  for (long t = r.tid; t < (long)U * U; t += NT) {
    const int b = (int)(t / U), a = (int)(t - (long)b * U);
    if (a >= b) {
      const double g_ab = r.J[b + (long)U * a] + 0.0, g_ba = r.J[a + (long)U * b] + 0.0;
      r.GN[a + (long)U * b] = 0.5 * (g_ab + g_ba);
    }
  }
  __syncthreads();
}

// ---- hinge-chain walk steps on the non-zero blocks ---------------------------
// Hinge levers are 3x3 (row 3 and column 3 exact zeros), link values affine
// (row 3 = e4^T).  The walk quantities of correlation_hess_ab / functional_hess
// are only ever read through 3x3 traces/ddots with levers, so only their
// top-left 3x3 is updated; the fourth row (fwd) / column (bwd, walk) is
// invariant under the affine products (exact copies) and the dropped terms
// are fma(+-0, x, acc) = acc.  Same values as the full 4x4 reference products.
struct L3 {
  double a[9];  // a[r + 3c]
};
__device__ __forceinline__ L3 ldl3(const double* p) {
  L3 m;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) m.a[r + 3 * c] = p[r + 4 * c];
  return m;
}
// trace(mul(mul_at(A, B), F)) over the non-zero 3x3 blocks (adjoint.cpp:150-165)
__device__ __forceinline__ double trace_at3(const L3& A, const L3& B, const M4& F) {
  double M[9];
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      double acc = A.a[3 * p] * B.a[3 * q];
      acc = fma(A.a[1 + 3 * p], B.a[1 + 3 * q], acc);
      acc = fma(A.a[2 + 3 * p], B.a[2 + 3 * q], acc);
      M[p + 3 * q] = acc;
    }
  double d[3];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    double acc = M[p] * F.a[4 * p];
    acc = fma(M[p + 3], F.a[1 + 4 * p], acc);
    acc = fma(M[p + 6], F.a[2 + 4 * p], acc);
    d[p] = acc;
  }
  return (d[0] + d[1]) + d[2];
}
// F <- V F on rows 0..2, columns 0..2 (V affine, smem)
__device__ __forceinline__ void fwd_step3(const double* V, M4& F) {
  double v[12];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) v[r + 3 * c] = V[r + 4 * c];
  double o[9];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double acc = v[r] * F.a[4 * c];
      acc = fma(v[r + 3], F.a[1 + 4 * c], acc);
      acc = fma(v[r + 6], F.a[2 + 4 * c], acc);
      acc = fma(v[r + 9], F.a[3 + 4 * c], acc);
      o[r + 3 * c] = acc;
    }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) F.a[r + 4 * c] = o[r + 3 * c];
}
// B <- B V^T on rows 0..2, columns 0..2 (V affine, smem)
__device__ __forceinline__ void bwd_step3(M4& Bm, const double* V) {
  double v[12];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) v[r + 3 * c] = V[r + 4 * c];
  double o[9];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double acc = Bm.a[r] * v[c];
      acc = fma(Bm.a[r + 4], v[c + 3], acc);
      acc = fma(Bm.a[r + 8], v[c + 6], acc);
      acc = fma(Bm.a[r + 12], v[c + 9], acc);
      o[r + 3 * c] = acc;
    }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) Bm.a[r + 4 * c] = o[r + 3 * c];
}
// ddot(lever, W) over the non-zero 3x3 block (adjoint.cpp:84-86)
__device__ __forceinline__ double ddot3(const L3& A, const M4& W) {
  double rs[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    double acc = A.a[r] * W.a[r];
    acc = fma(A.a[r + 3], W.a[r + 4], acc);
    acc = fma(A.a[r + 6], W.a[r + 8], acc);
    rs[r] = acc;
  }
  return (rs[0] + rs[1]) + rs[2];
}

// Jacobian of the residuals (objective.cpp:310-320) into r.J
// contact part of pot.hess (objective.cpp:104-123, flags.hess) at every
// instant: per (instant, sample) the Hessian hxx and the sample Jacobian jx
// (3 x n, zero off the sample's root path) into r.CJ; then every element of
// the instant's n x n block adds (jx^T hxx) jx of the active samples, in
// sample order, onto 0 (+ 2 scale ab with drag, PH's raw ab) -> PH.  The
// cotangent functional_hess walk adds its term last (objective.cpp:132-135).
__device__ __noinline__ void contact_hess(const R& r, const double* Vs, const double* Ls) {
  const DModel& m = *r.m;
  const DForces& f = *r.f;
  const int N = r.N, n = r.n, u = r.u, ns = r.rd->ns;
  const long NS = (long)SMS * N;
  const long cs = 3L * n + 10;
  const double* nrm = f.normal;
  for (int t = r.tid; t < u * ns; t += NT) {
    const int mm = t / ns, sidx = t - mm * ns;
    int i = 0;
    while (m.sample_off[i + 1] <= sidx) ++i;
    double* cj = r.CJ + (long)t * cs;
    double ph[4], pv[3], depth;
    if (!contact_state(r, mm, i, sidx, ph, pv, &depth)) {
      cj[9] = 0.0;
      continue;
    }
    const double dtm = r.sc->times[2 + mm] * r.sc->dt;
    const double pv2 = dot3(pv, pv);
    double hxx[9];
    for (int c = 0; c < 3; ++c)
      for (int rr = 0; rr < 3; ++rr) hxx[rr + 3 * c] = ((2.0 * f.d1) * nrm[rr]) * nrm[c];
    if (f.d2 > 0.0) {
      double proj[9];
      for (int c = 0; c < 3; ++c)
        for (int rr = 0; rr < 3; ++rr) proj[rr + 3 * c] = ((rr == c) ? 1.0 : 0.0) - nrm[rr] * nrm[c];
      const double k1 = (2.0 * f.d2) * pv2;
      const double k2 = 4.0 * f.d2 * depth / dtm;
      const double k3 = 2.0 * f.d2 * depth * depth / (dtm * dtm);
      for (int c = 0; c < 3; ++c)
        for (int rr = 0; rr < 3; ++rr) {
          const double t1 = (k1 * nrm[rr]) * nrm[c];
          const double t2 = k2 * (nrm[rr] * pv[c] + pv[rr] * nrm[c]);
          const double t3 = k3 * proj[rr + 3 * c];
          hxx[rr + 3 * c] = hxx[rr + 3 * c] + ((t1 - t2) + t3);
        }
    }
    for (int k = 0; k < 9; ++k) cj[k] = hxx[k];
    cj[9] = 1.0;
    double* jx = cj + 10;
    for (int k = 0; k < 3 * n; ++k) jx[k] = 0.0;
    double y[4] = {ph[0], ph[1], ph[2], ph[3]};
    for (int l = i; l >= 0; l = rss.parent[l]) {  // hinge: dof l = link l
      double t4[4], y2[4];
      mul_vec4(ldm4(Ls + mm * NS + SMS * l), y, t4);
      jx[3 * l] = t4[0];
      jx[3 * l + 1] = t4[1];
      jx[3 * l + 2] = t4[2];
      mul_vec4(ldm4(Vs + mm * NS + SMS * l), y, y2);
      for (int k = 0; k < 4; ++k) y[k] = y2[k];
    }
  }
  __syncthreads();
  const long nn = (long)n * n;
  for (long t = r.tid; t < u * nn; t += NT) {
    const int mm = (int)(t / nn);
    const long e = t - mm * nn;
    const int b = (int)(e / n), a = (int)(e - (long)b * n);
    double* P = r.PH + mm * nn + e;
    double acc = r.drag ? 0.0 + r.s2[mm] * *P : 0.0;
    for (int sidx = 0; sidx < ns; ++sidx) {
      const double* cj = r.CJ + ((long)mm * ns + sidx) * cs;
      if (cj[9] == 0.0) continue;
      const double* jx = cj + 10;
      double tmp[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double q = jx[3 * a] * cj[3 * c];
        q = fma(jx[3 * a + 1], cj[1 + 3 * c], q);
        q = fma(jx[3 * a + 2], cj[2 + 3 * c], q);
        tmp[c] = q;
      }
      double v = tmp[0] * jx[3 * b];
      v = fma(tmp[1], jx[3 * b + 1], v);
      v = fma(tmp[2], jx[3 * b + 2], v);
      acc = acc + v;
    }
    *P = acc;
  }
  __syncthreads();
}

__device__ __noinline__ void jacobian(const R& r) {
  const DModel& m = *r.m;
  const DSchedule& sc = *r.sc;
  const ResidDesc& rd = *r.rd;
  const int N = r.N, n = r.n, u = r.u, U = r.U;
  const long UU = (long)U * U;
  PT_START();
  if (!rd.chain) {
    for (long t = r.tid; t < UU; t += NT) r.J[t] = 0.0;
    if (!r.energy)
      for (long t = r.tid; t < (long)u * n * n; t += NT) {
        r.FH[t] = 0.0;
        r.PH[t] = 0.0;
      }
  }
  // pass values / levers of every instant and the composite-inertia
  // contributions Z live in shared memory for the walks below
  const long NS = (long)SMS * N;
  double* Vs = rsm;
  double* Ls = Vs + u * NS;
  double* Zs = Ls + u * NS;  // [u*u][N][16]
  stage_vl(r, Vs, Ls);
  __syncthreads();
  PT_MARK(18);
  // correlation_hess_ab(pass_a, pass_b) composite inertias for every pair
  // (a = instant l, b = instant mm), pair = a * u + b (adjoint.cpp:139-141,169-174)
  const int npair = u * u;
  if (rd.chain) {
    // ai = (0 + Z_{i+1}) + S_i, y = V_b ai, Z_i = y V_a^T from the leaf, group = pair
    const int g = r.tid >> 4, e16 = r.tid & 15, ri = e16 & 3, cj = e16 >> 2;
    if (g < npair) {
      const int a = g / u, b = g - a * u;
      double* h0 = r.ha(g, 0);
      double* h1 = r.ha(g, 1);
      double z = 0.0;
      for (int i = N - 1; i >= 0; --i) {
        const double acc = (i == N - 1) ? 0.0 : 0.0 + z;
        const double ai = acc + __ldg(m.S + 16 * i + e16);
        h0[16 * i + e16] = ai;
        const double y = g_mul_right(Vs + b * NS + SMS * i, ai, ri, cj);
        h1[16 * i + e16] = y;
        z = g_mul_bt(y, Vs + a * NS + SMS * i, ri, cj);
      }
    }
    __syncthreads();
    for (int t = r.tid; t < npair * N; t += NT) {
      const int pr = t / N, i = t - pr * N;
      const int a = pr / u;
      stm4(r.ha(pr, 2) + 16 * i, mul_bt(ldm4(r.ha(pr, 0) + 16 * i), ldm4(Vs + a * NS + SMS * i)));
    }
    __syncthreads();
  } else
  for (int d = r.D; d >= 0; --d) {
    const int l0 = rd.lvl_start[d], cnt = rd.lvl_start[d + 1] - l0;
    for (int t = r.tid; t < npair * cnt; t += NT) {
      const int pr = t / cnt;
      const int i = rd.lvl_links[l0 + t - pr * cnt];
      const int a = pr / u, b = pr - a * u;
      double* Z = Zs + pr * NS;
      M4 acc = m4_zero();
      for (int c = rd.ch_start[i]; c < rd.ch_start[i + 1]; ++c) acc = add(acc, ldm4(Z + SMS * rd.ch_list[c]));
      const M4 ai = add(acc, ldgm4(m.S + 16 * i));
      const M4 vb = ldm4(Vs + b * NS + SMS * i), va = ldm4(Vs + a * NS + SMS * i);
      stm4(r.ha(pr, 0) + 16 * i, ai);
      const M4 y = mul(vb, ai);
      stm4(r.ha(pr, 1) + 16 * i, y);
      stm4(r.ha(pr, 2) + 16 * i, mul_bt(ai, va));
      stm4(Z + SMS * i, mul_bt(y, va));
    }
    __syncthreads();
  }
  PT_MARK(14);
  // hess_ab entries: own block and the ancestor walk of every (pair, link),
  // written straight into J (transposed, scaled by inv_dt2 * stencil)
  for (int t = r.tid; t < npair * N; t += NT) {
    const int pr = t / N;
    const int i = rd.walk_order[t - pr * N];
    const int a = pr / u, b = pr - a * u;  // hess_ab(pass_a, pass_b) feeds J block (row b, col a)
    const double* stb = sc.H2 + r.K1 * (2 + b);
    const double ca = r.energy ? r.inv_dt2 : r.inv_dt2 * stb[2 + a];
    const double* la = Ls + a * NS;
    const double* lb = Ls + b * NS;
    const double* va = Vs + a * NS;
    const double* vb = Vs + b * NS;
    const long rowb = (long)b * n, cola = (long)a * n;
    if (rd.chain && !r.energy && a == b) {
      // chains, diagonal block (mm, mm): every entry of it is one (i, l) of
      // this walk, so the inertial and gravity functional_hess walks of
      // (mm, i) (adjoint.cpp:66-101) run here too and the block is finished
      // in registers, J = (fh + c_m ab^T) + ph, without a second pass over J
      const int mm = a;
      const double h = 0.0 + trace_mul(mul_at(ldm4(la + SMS * i), ldm4(lb + SMS * i)), ldm4(r.ha(pr, 0) + 16 * i));
      const M4 aF = ldm4(r.fa(mm, 0) + 16 * i);
      const M4 aP = r.have_cot ? ldm4(r.fa(u + mm, 0) + 16 * i) : m4_zero();
      const int p = rss.parent[i];
      const M4 pd = mul(p >= 0 ? ldm4(r.wld(mm) + 16 * p) : m4_identity(), ldm4(r.dd2(mm) + 16 * i));
      // pot.hess = (0 + 2 scale ab) + functional_hess(cot) with drag
      // (objective.cpp:70-71,131-134), functional_hess(cot) otherwise
      const double s2 = r.drag ? r.s2[mm] : 0.0;
      {
        const double hF = 0.0 + ddot(pd, aF);
        double hP = r.have_cot ? 0.0 + ddot(pd, aP) : 0.0;
        if (r.drag) hP = (0.0 + s2 * h) + hP;
        r.J[(rowb + i) + U * (cola + i)] = (hF + ca * h) + hP;
      }
      const L3 u_i = ldl3(la + SMS * i);
      M4 fwd = ldm4(r.ha(pr, 1) + 16 * i);
      M4 bwd = ldm4(r.ha(pr, 2) + 16 * i);
      const M4 d1 = ldm4(r.dd1(mm) + 16 * i);
      M4 wF = mul_bt(aF, d1);
      M4 wP = mul_bt(aP, d1);
      for (int l = p; l >= 0; l = rss.parent[l]) {
        const L3 u_l = ldl3(la + SMS * l);
        const double t1 = 0.0 + trace_at3(u_i, u_l, fwd);  // H(i, l)
        const double t2 = 0.0 + trace_at3(u_l, u_i, bwd);  // H(l, i)
        const double hF = 0.0 + ddot3(u_l, wF);
        const double hP = r.have_cot ? 0.0 + ddot3(u_l, wP) : 0.0;
        // J(l, i) takes pot.hess(l, i) = ... ab(l, i) = t2, J(i, l) ab(i, l) = t1
        const double p_li = r.drag ? (0.0 + s2 * t2) + hP : hP;
        const double p_il = r.drag ? (0.0 + s2 * t1) + hP : hP;
        r.J[(rowb + l) + U * (cola + i)] = (hF + ca * t1) + p_li;
        r.J[(rowb + i) + U * (cola + l)] = (hF + ca * t2) + p_il;
        fwd_step3(va + SMS * l, fwd);
        bwd_step3(bwd, va + SMS * l);
        bwd_step3(wF, va + SMS * l);
        if (r.have_cot) bwd_step3(wP, va + SMS * l);
      }
      continue;
    }
    // trees with drag: the diagonal pair's raw ab also lands in PH, where the
    // cotangent functional_hess walk below turns it into pot.hess
    double* abm = (r.drag && a == b) ? r.PH + (long)a * n * n : nullptr;
    {
      const double h = 0.0 + trace_mul(mul_at(ldm4(la + SMS * i), ldm4(lb + SMS * i)), ldm4(r.ha(pr, 0) + 16 * i));
      r.J[(rowb + i) + U * (cola + i)] = ca * h;
      if (abm) abm[i + (long)n * i] = h;
    }
    const L3 ua_i = ldl3(la + SMS * i), ub_i = ldl3(lb + SMS * i);
    M4 fwd = ldm4(r.ha(pr, 1) + 16 * i);
    M4 bwd = ldm4(r.ha(pr, 2) + 16 * i);
    for (int l = rss.parent[i]; l >= 0; l = rss.parent[l]) {
      const double t1 = 0.0 + trace_at3(ua_i, ldl3(lb + SMS * l), fwd);   // H(i, l)
      const double t2 = 0.0 + trace_at3(ldl3(la + SMS * l), ub_i, bwd);   // H(l, i)
      r.J[(rowb + l) + U * (cola + i)] = ca * t1;
      r.J[(rowb + i) + U * (cola + l)] = ca * t2;
      if (abm) {
        abm[i + (long)n * l] = t1;
        abm[l + (long)n * i] = t2;
      }
      fwd_step3(vb + SMS * l, fwd);
      bwd_step3(bwd, va + SMS * l);
    }
  }
  PT_MARK(15);
  // the chain walks below read J entries the hess_ab tasks above wrote, from
  // other threads (the two loops map tasks to threads differently)
  __syncthreads();
  if (r.energy) return;  // energy form: J holds inv_dt2 ab^T, no functional_hess terms
  if (rd.chain) {
    // chains: the functional_hess walks ran fused with the diagonal-block
    // hess_ab walks above
    PT_MARK(16);
  } else {
  if (r.contact) contact_hess(r, Vs, Ls);
  // functional_hess (adjoint.cpp:66-101) of the inertial seeds and of the
  // gravity cotangents at every instant
  const int nsw = r.have_cot ? 2 * u : u;
  for (int t = r.tid; t < nsw * N; t += NT) {
    const int sw = t / N;
    const int i = rd.walk_order[t - sw * N];
    const int mm = sw < u ? sw : sw - u;
    double* F = (sw < u ? r.FH : r.PH) + (long)mm * n * n;
    const double* lm = Ls + mm * NS;
    const double* vm = Vs + mm * NS;
    const M4 a = ldm4(r.fa(sw, 0) + 16 * i);
    const int p = rss.parent[i];
    const M4 pw = p >= 0 ? ldm4(r.wld(mm) + 16 * p) : m4_identity();
    // drag (cotangent sweeps): pot.hess = (0 + 2 scale ab) + functional_hess(cot),
    // ab left in PH by the hess_ab walk above; with contact PH already holds
    // everything before functional_hess (contact_hess)
    const bool pc = r.contact && sw >= u;
    const bool dr = r.drag && sw >= u && !pc;
    const double s2 = dr ? r.s2[mm] : 0.0;
    {
      const double h = 0.0 + ddot(mul(pw, ldm4(r.dd2(mm) + 16 * i)), a);
      F[i + (long)n * i] = pc ? F[i + (long)n * i] + h : dr ? (0.0 + s2 * F[i + (long)n * i]) + h : h;
    }
    M4 walk = mul_bt(a, ldm4(r.dd1(mm) + 16 * i));
    for (int l = p; l >= 0; l = rss.parent[l]) {
      const double h = 0.0 + ddot3(ldl3(lm + SMS * l), walk);
      if (pc) {
        F[l + (long)n * i] = F[l + (long)n * i] + h;
        F[i + (long)n * l] = F[i + (long)n * l] + h;
      } else if (dr) {
        F[l + (long)n * i] = (0.0 + s2 * F[l + (long)n * i]) + h;
        F[i + (long)n * l] = (0.0 + s2 * F[i + (long)n * l]) + h;
      } else {
        F[l + (long)n * i] = h;
        F[i + (long)n * l] = h;
      }
      bwd_step3(walk, vm + SMS * l);
    }
  }
  __syncthreads();
  PT_MARK(16);
  // diagonal blocks: (functional_hess + c_m ab_mm^T) + pot.hess; a warp per
  // pair of J columns, lanes down the rows (no index divisions, 24 loads in
  // flight per lane)
  {
    const int NW = NT / 32, wid = r.tid >> 5, lane = r.tid & 31;
    const int ncol = u * n;
    for (int c0 = 2 * wid; c0 < ncol; c0 += 2 * NW) {
      double fh[2][4], ph[2][4], jv[2][4];
      double* jc[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = min(c0 + h, ncol - 1);
        const int mm = col / n, cc = col - mm * n;
        const long fo = (long)mm * n * n + (long)cc * n;
        jc[h] = r.J + (long)mm * n + (long)U * ((long)mm * n + cc);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rr = lane + 32 * q;
          if (rr < n) {
            fh[h][q] = r.FH[fo + rr];
            ph[h][q] = r.have_cot ? 0.0 + r.PH[fo + rr] : 0.0;
            jv[h][q] = jc[h][rr];
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (c0 + h < ncol)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int rr = lane + 32 * q;
            if (rr < n) jc[h][rr] = (fh[h][q] + jv[h][q]) + ph[h][q];
          }
      for (int rb = 128; rb < n; rb += 32) {  // n > 128: remaining rows
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = c0 + h;
          const int rr = rb + lane;
          if (col < ncol && rr < n) {
            const int mm = col / n, cc = col - mm * n;
            const long fo = (long)mm * n * n + (long)cc * n;
            const double phv = r.have_cot ? 0.0 + r.PH[fo + rr] : 0.0;
            jc[h][rr] = (r.FH[fo + rr] + jc[h][rr]) + phv;
          }
        }
      }
    }
  }
  }
  __syncthreads();
  PT_MARK(17);
}

// grad = 2 J^T g (objective.cpp:326-327)
// 32-row chunk c of J into a shared tile (one column per 33-double row) by
// 8-byte cp.async, the warps column by column (coalesced)
__device__ __forceinline__ void grad_issue(const R& r, double* tile, int c) {
  constexpr int KC = 32, TS = KC + 1;
  const int U = r.U, k0 = c * KC, kc = min(KC, U - k0);
  const int warp = r.tid >> 5, lane = r.tid & 31;
  if (lane < kc)
    for (int a = warp; a < U; a += NT / 32) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(tile + a * TS + lane);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(r.J + (k0 + lane) + (long)U * a)
                   : "memory");
    }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __noinline__ void gradient(const R& r) {
  // Thread t owns columns t and t + NT (two independent fma chains, k
  // ascending: acc = (2 J(0,a)) g0, then fma(2 J(k,a), g_k, acc)); J arrives
  // in 32-row chunks, double-buffered, one chunk ahead of the products
  constexpr int KC = 32, TS = KC + 1;
  const int U = r.U;
  double* rs = rsm;
  const long tsz = (long)U * TS;
  double* tiles = rsm + ((U + 1) & ~1);
  for (int k = r.tid; k < U; k += NT) rs[k] = r.res[k];
  const int nc = (U + KC - 1) / KC;
  const int a0 = r.tid, a1 = r.tid + NT;
  double acc0 = 0.0, acc1 = 0.0;
  grad_issue(r, tiles, 0);
  for (int c = 0; c < nc; ++c) {
    const int k0 = c * KC, kc = min(KC, U - k0);
    if (c + 1 < nc) {
      grad_issue(r, tiles + ((c + 1) & 1) * tsz, c + 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // chunk c landed for every thread (and rs is written)
    const double* tile = tiles + (c & 1) * tsz;
    if (a0 < U) {
      const double* t = tile + a0 * TS;
      int kk = 0;
      if (c == 0) {
        acc0 = (2.0 * t[0]) * rs[0];
        kk = 1;
      }
      for (; kk < kc; ++kk) acc0 = fma(2.0 * t[kk], rs[k0 + kk], acc0);
    }
    if (a1 < U) {
      const double* t = tile + a1 * TS;
      int kk = 0;
      if (c == 0) {
        acc1 = (2.0 * t[0]) * rs[0];
        kk = 1;
      }
      for (; kk < kc; ++kk) acc1 = fma(2.0 * t[kk], rs[k0 + kk], acc1);
    }
    __syncthreads();  // chunk c consumed before its buffer takes chunk c + 2
  }
  if (a0 < U) r.grad[a0] = acc0;
  if (a1 < U) r.grad[a1] = acc1;
}

// GN = 0.5 (2 J^T J + (2 J^T J)^T) = 2 J^T J, lower triangle (objective.cpp:328-330).
// k-chunks of J land in shared memory by cp.async one chunk ahead of the
// multiply (no register staging); each thread doubles its own A elements
// (2 J exact) once its copies have arrived.
__device__ __forceinline__ void gn_cpa8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void gn_issue(const R& r, double* buf, int lt, int a0, int b0, int c) {
  const int U = r.U;
  double* As = buf + (c & 1) * 2 * GK * GP;
  double* Bs = As + GK * GP;
#pragma unroll
  for (int q = 0; q < GK * GB / 256; ++q) {
    const int t = lt + 256 * q;
    const int col = t / GK, kk = t - col * GK;
    const int k = c * GK + kk, a = a0 + col, b = b0 + col;
    if (k < U && a < U) gn_cpa8(As + kk * GP + col, r.J + k + (long)U * a);
    else As[kk * GP + col] = 0.0;
    if (k < U && b < U) gn_cpa8(Bs + kk * GP + col, r.J + k + (long)U * b);
    else Bs[kk * GP + col] = 0.0;
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// d += a b on the FP64 tensor cores (one 8x8x4 fragment per warp)
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

#ifndef PBAD_RESID_GN_DMMA
#define PBAD_RESID_GN_DMMA 1
#endif
#if PBAD_RESID_GN_DMMA
// FP64 tensor cores: mma.sync.m8n8k4.f64 computes d = fma(a3, b3, fma(a2, b2,
// fma(a1, b1, fma(a0, b0, c)))) -- the k-ascending fma chain of the numeric
// contract, bit for bit (scripts/micro/dmma.cu: 1.28 M random elements, 0
// mismatches) -- so 2 J^T J runs on DMMA unchanged: the chain starts from
// c = -0 (fma(a0, b0, -0) == a0 * b0, the product's first term) and padded k
// contribute (-0) * 0 = -0, which leaves every accumulator unchanged.
// Tile 64 x 64 per 256 threads; warp w owns rows 8w..8w+7 and all eight 8 x 8
// column blocks.  Staging k-fastest (column stride GQ = 36 = 4 mod 16 doubles:
// fragment loads and cp.async stores conflict-free).
#ifndef PBAD_RESID_GDK
#define PBAD_RESID_GDK 64
#endif
constexpr int GDK = PBAD_RESID_GDK;  // k chunk of the DMMA tiles
constexpr int GQ = GDK + 4;          // = 4 (mod 16)
static_assert(GQ % 16 == 4, "conflict-free fragment loads");
__device__ __forceinline__ void gnd_issue(const R& r, double* buf, int lt, int a0, int b0, int c) {
  const int U = r.U;
  double* As = buf + (c & 1) * 2 * GB * GQ;
  double* Bs = As + GB * GQ;
  if ((U & 1) == 0) {
    // k pairs: 16-byte copies (J column-major, U even: k-pairs are 16-byte aligned)
#pragma unroll
    for (int q = 0; q < GDK * GB / 512; ++q) {
      const int t = lt + 256 * q;
      const int col = t / (GDK / 2), kk = 2 * (t - col * (GDK / 2));
      const int k = c * GDK + kk, a = a0 + col, b = b0 + col;
      double* da = As + col * GQ + kk;
      double* db = Bs + col * GQ + kk;
      if (k < U && a < U) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(da)),
                     "l"(r.J + k + (long)U * a) : "memory");
      } else {
        da[0] = -0.0;
        da[1] = -0.0;
      }
      if (k < U && b < U) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(db)),
                     "l"(r.J + k + (long)U * b) : "memory");
      } else {
        db[0] = 0.0;
        db[1] = 0.0;
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < GDK * GB / 256; ++q) {
      const int t = lt + 256 * q;
      const int col = t / GDK, kk = t - col * GDK;
      const int k = c * GDK + kk, a = a0 + col, b = b0 + col;
      if (k < U && a < U) gn_cpa8(As + col * GQ + kk, r.J + k + (long)U * a);
      else As[col * GQ + kk] = -0.0;
      if (k < U && b < U) gn_cpa8(Bs + col * GQ + kk, r.J + k + (long)U * b);
      else Bs[col * GQ + kk] = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __noinline__ void gauss_newton(const R& r) {
  const int U = r.U;
  const int nb = (U + GB - 1) / GB;
  const int ntile = nb * (nb + 1) / 2;
  const int grp = r.tid >> 8, lt = r.tid & 255;
  const int w = lt >> 5, lane = lt & 31, g = lane >> 2, t4 = lane & 3;
  const int nkd = (U + GDK - 1) / GDK;
  double* buf = rsm + grp * 4 * GB * GQ;
  for (int t0 = 0; t0 < ntile; t0 += TG) {
    int tile = t0 + grp, bi = 0;
    const bool active = tile < ntile;
    if (!active) tile = ntile - 1;
    while (tile > bi) {
      tile -= bi + 1;
      ++bi;
    }
    const int bj = tile;
    const int a0 = bi * GB, b0 = bj * GB;
    double d[8][2];
#pragma unroll
    for (int cb = 0; cb < 8; ++cb) d[cb][0] = d[cb][1] = -0.0;
    gnd_issue(r, buf, lt, a0, b0, 0);
    for (int c = 0; c < nkd; ++c) {
      double* As = buf + (c & 1) * 2 * GB * GQ;
      double* Bs = As + GB * GQ;
      __syncthreads();
      if (c + 1 < nkd) {
        gnd_issue(r, buf, lt, a0, b0, c + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const double* ap = As + (8 * w + g) * GQ + t4;
      const double* bp = Bs + g * GQ + t4;
#pragma unroll
      for (int ks = 0; ks < GDK / 4; ++ks) {
        const double av = 2.0 * ap[4 * ks];  // 2 J (exact)
        double bv[8];
#pragma unroll
        for (int cb = 0; cb < 8; ++cb) bv[cb] = bp[cb * 8 * GQ + 4 * ks];
#pragma unroll
        for (int cb = 0; cb < 8; ++cb) dmma884(d[cb][0], d[cb][1], av, bv[cb]);
      }
    }
    if (active) {
      const int a = a0 + 8 * w + g;
#pragma unroll
      for (int cb = 0; cb < 8; ++cb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int b = b0 + 8 * cb + 2 * t4 + h;
          if (a < U && b <= a) r.GN[a + (long)U * b] = 0.5 * (d[cb][h] + d[cb][h]);
        }
    }
  }
  __syncthreads();
}
#else
__device__ __noinline__ void gauss_newton(const R& r) {
  const int U = r.U;
  const int nb = (U + GB - 1) / GB;
  const int nk = (U + GK - 1) / GK;
  const int ntile = nb * (nb + 1) / 2;
  const int grp = r.tid >> 8, lt = r.tid & 255;  // TG groups of 256 threads, one tile each
  const int tx = lt & 15, ty = lt >> 4;
  double* buf = rsm + grp * 4 * GK * GP;
  for (int t0 = 0; t0 < ntile; t0 += TG) {
    // tile t0 + grp of the lower triangle (row-major over block rows)
    int tile = t0 + grp, bi = 0;
    const bool active = tile < ntile;
    if (!active) tile = ntile - 1;
    while (tile > bi) {
      tile -= bi + 1;
      ++bi;
    }
    const int bj = tile;
    const int a0 = bi * GB, b0 = bj * GB;
    double acc[4][4];
    gn_issue(r, buf, lt, a0, b0, 0);
    for (int c = 0; c < nk; ++c) {
      double* As = buf + (c & 1) * 2 * GK * GP;
      double* Bs = As + GK * GP;
      __syncthreads();  // everyone is done with the buffer chunk c + 1 will overwrite
      if (c + 1 < nk) {
        gn_issue(r, buf, lt, a0, b0, c + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
#pragma unroll
      for (int q = 0; q < GK * GB / 256; ++q) {
        const int t = lt + 256 * q;
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
    if (active) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int a = a0 + ty + 16 * i, b = b0 + tx + 16 * j;
          if (a < U && b <= a) r.GN[a + (long)U * b] = 0.5 * (acc[i][j] + acc[i][j]);
        }
    }
  }
  __syncthreads();
}

#endif  // PBAD_RESID_GN_DMMA

// LLT of r.DM (lower, column-major), blocked left-looking; same per-element
// operation sequence as the right-looking reference (optim.cpp:11-15).
// The damped matrix gn + lambda I (optim.cpp:105-107) is read from r.GN at
// each element's first use (left-looking touches every original entry once).
// false = non-positive pivot.
#if PBAD_RESID_CHOL_REG == 2
// ---- lookahead variant ------------------------------------------------------
// Block column J+1's update by the columns left of block J (warps 1..7) runs
// while warp 0 factors the diagonal block J; then the rows below block J are
// solved (all threads) and block column J+1 receives block J's 32 columns.
// Every element still sees its k updates in ascending order.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void group_sync(int id, int nthreads) {
  if (id == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// acc(i, j) for rows i in [c0, U), cols j in [c0, c0 + bw), j <= i:
//   init (G + lambda I if fromG, else A), then acc = fma(-L(i,k), L(j,k), acc)
//   for k in [kb, ke) ascending; result to A.  Threads [NT - GS, NT) of the CTA,
//   thread tile NI rows (stride GS/8) x 4 columns (stride 8).
template <int GS, int NI>
__device__ __forceinline__ void bcu_tile(const R& r, double* A, const double* G, double lambda, bool fromG, int c0,
                                         int bw, int kb, int ke, double* panel, int cap, int bar) {
  constexpr int RY = GS / 8;
  const int U = r.U;
  const int t = r.tid - (NT - GS);
  const int tx = t & 7, ty = t >> 3;
  const int rows = U - c0;
  double acc[NI][4];
  int ri[NI];
#pragma unroll
  for (int ii = 0; ii < NI; ++ii) ri[ii] = min(ty + RY * ii, rows - 1);
  int cj[4];
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) cj[jj] = min(tx + 8 * jj, rows - 1);
#pragma unroll
  for (int ii = 0; ii < NI; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int i = c0 + ty + RY * ii, j = c0 + tx + 8 * jj;
      const long at = i + (long)U * j;
      acc[ii][jj] = (i < U && j < c0 + bw && j <= i) ? (fromG ? (i == j ? G[at] + lambda : G[at]) : A[at]) : 0.0;
    }
  const int kcap = cap / rows;
  for (int k0 = kb; k0 < ke; k0 += kcap) {
    const int kc = min(kcap, ke - k0);
    group_sync(bar, GS);
    for (int kk = 0; kk < kc; ++kk)
      for (int rr = t; rr < rows; rr += GS) cp_async8(panel + kk * rows + rr, A + (c0 + rr) + (long)U * (k0 + kk));
    asm volatile("cp.async.wait_all;" ::: "memory");
    group_sync(bar, GS);
#pragma unroll 4
    for (int kk = 0; kk < kc; ++kk) {
      const double* pk = panel + kk * rows;
      double bv[4], av[NI];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) bv[jj] = pk[cj[jj]];
#pragma unroll
      for (int ii = 0; ii < NI; ++ii) av[ii] = pk[ri[ii]];
#pragma unroll
      for (int ii = 0; ii < NI; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = fma(-av[ii], bv[jj], acc[ii][jj]);
    }
  }
#pragma unroll
  for (int ii = 0; ii < NI; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int i = c0 + ty + RY * ii, j = c0 + tx + 8 * jj;
      if (i < U && j < c0 + bw && j <= i) A[i + (long)U * j] = acc[ii][jj];
    }
}
#ifndef PBAD_RESID_BCU_DMMA
#define PBAD_RESID_BCU_DMMA 1
#endif
#if PBAD_RESID_BCU_DMMA
// The same update on FP64 tensor cores: per 8 x 8 block of the output,
// d = fma(-L(i,k+3), L(j,k+3), ... fma(-L(i,k), L(j,k), d)) is exactly one
// mma.m8n8k4 with A = -panel rows i, B = panel rows j (DMMA is the
// k-ascending fma chain).  Panel k-major with row stride RP = 4 (mod 16)
// doubles: staging stores and fragment loads are both conflict-free; k
// padded to a multiple of 4 with +0 (a (-0) * 0 product leaves the
// accumulator unchanged).  Warp wi of the group owns row blocks wi, wi + NW,
// ... and the four 8-column blocks of the block column.
template <int GS, int NRB>
__device__ __forceinline__ void bcu_dmma(const R& r, double* A, const double* G, double lambda, bool fromG, int c0,
                                         int bw, int kb, int ke, double* panel, int cap, int bar) {
  constexpr int NW = GS / 32;
  const int U = r.U;
  const int t = r.tid - (NT - GS);
  const int wi = t >> 5, lane = t & 31, g = lane >> 2, t4 = lane & 3;
  const int rows = U - c0;
  const int nrb = (rows + 7) >> 3;
  const int RP = rows + ((20 - (rows & 15)) & 15);  // >= rows, == 4 (mod 16)
  double d[NRB][4][2];
#pragma unroll
  for (int q = 0; q < NRB; ++q) {
    const int rb = wi + NW * q;
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = c0 + 8 * rb + g, j = c0 + 8 * cb + 2 * t4 + h;
        const long at = i + (long)U * j;
        d[q][cb][h] = (rb < nrb && i < U && j < c0 + bw && j <= i)
                          ? (fromG ? (i == j ? G[at] + lambda : G[at]) : A[at]) : 0.0;
      }
  }
  // two panel buffers: chunk c + 1 streams in (cp.async) while chunk c is
  // multiplied; 16-byte copies of row pairs when the column-major rows are
  // 16-byte aligned (U and c0 even)
  const int kcap = ((cap / 2) / RP) & ~3;
  const bool pairs = ((U | c0) & 1) == 0;
  auto stage = [&](int k0, double* buf) {
    const int kc = min(kcap, ke - k0);
    const int kc4 = (kc + 3) & ~3;
    if (pairs) {
      const int rp = (rows + 1) >> 1;
      for (int e = t; e < kc4 * rp; e += GS) {
        const int kk = e / rp, rr = 2 * (e - kk * rp);
        double* dst = buf + kk * RP + rr;
        if (kk < kc) {
          const double* src = A + (c0 + rr) + (long)U * (k0 + kk);
          if (rr + 1 < rows) {
            const unsigned da = (unsigned)__cvta_generic_to_shared(dst);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(da), "l"(src) : "memory");
          } else {
            cp_async8(dst, src);
          }
        } else {
          dst[0] = 0.0;
          if (rr + 1 < rows) dst[1] = 0.0;
        }
      }
    } else {
      for (int e = t; e < kc4 * rows; e += GS) {
        const int kk = e / rows, rr = e - kk * rows;
        if (kk < kc) cp_async8(buf + kk * RP + rr, A + (c0 + rr) + (long)U * (k0 + kk));
        else buf[kk * RP + rr] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double* pbuf[2] = {panel, panel + kcap * RP};
  if (kb < ke) {
    group_sync(bar, GS);  // the previous user of the panel is done with it
    stage(kb, pbuf[0]);
  }
  int ci = 0;
  for (int k0 = kb; k0 < ke; k0 += kcap, ++ci) {
    const int kc4 = (min(kcap, ke - k0) + 3) & ~3;
    if (k0 + kcap < ke) {
      stage(k0 + kcap, pbuf[(ci + 1) & 1]);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    group_sync(bar, GS);
    const double* cur = pbuf[ci & 1];
    for (int ks = 0; ks < kc4; ks += 4) {
      const double* pk = cur + (ks + t4) * RP + g;
      double bv[4];
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) bv[cb] = pk[8 * cb];
#pragma unroll
      for (int q = 0; q < NRB; ++q) {
        const int rb = wi + NW * q;
        if (rb < nrb) {
          const double av = -pk[8 * rb];
#pragma unroll
          for (int cb = 0; cb < 4; ++cb)
            if (cb <= rb) dmma884(d[q][cb][0], d[q][cb][1], av, bv[cb]);
        }
      }
    }
    group_sync(bar, GS);  // buffer ci & 1 is restaged two chunks later
  }
#pragma unroll
  for (int q = 0; q < NRB; ++q) {
    const int rb = wi + NW * q;
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = c0 + 8 * rb + g, j = c0 + 8 * cb + 2 * t4 + h;
        if (rb < nrb && i < U && j < c0 + bw && j <= i) A[i + (long)U * j] = d[q][cb][h];
      }
  }
}
// more than 6 row blocks per warp (U - c0 > 48 NW): its own function, so
// the larger accumulator tile does not set the register budget of the rest
template <int GS>
__device__ __noinline__ void block_col_update_big(const R& r, double* A, const double* G, double lambda, bool fromG,
                                                  int c0, int bw, int kb, int ke, double* panel, int cap, int bar) {
  constexpr int NW = GS / 32;
  bcu_dmma<GS, (MAXU / 8 + NW - 1) / NW>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
}
template <int GS>
__device__ __noinline__ void block_col_update(const R& r, double* A, const double* G, double lambda, bool fromG,
                                              int c0, int bw, int kb, int ke, double* panel, int cap, int bar) {
  constexpr int NW = GS / 32;
  const int q = ((r.U - c0 + 7) / 8 + NW - 1) / NW;  // row blocks per warp
  if (q <= 1) bcu_dmma<GS, 1>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else if (q <= 2) bcu_dmma<GS, 2>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else if (q <= 3) bcu_dmma<GS, 3>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else if (q <= 4) bcu_dmma<GS, 4>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else if (q <= 6) bcu_dmma<GS, 6>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else block_col_update_big<GS>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
}
#else
template <int GS>
__device__ __noinline__ void block_col_update(const R& r, double* A, const double* G, double lambda, bool fromG,
                                              int c0, int bw, int kb, int ke, double* panel, int cap, int bar) {
  constexpr int RY = GS / 8;
  const int ni = (r.U - c0 + RY - 1) / RY;
  if (ni <= 1) bcu_tile<GS, 1>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else if (ni <= 2) bcu_tile<GS, 2>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else if (ni <= 3) bcu_tile<GS, 3>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else if (ni <= 4) bcu_tile<GS, 4>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else if (ni <= 6) bcu_tile<GS, 6>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else if (ni <= 8) bcu_tile<GS, 8>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
  else bcu_tile<GS, (MAXU + RY - 1) / RY>(r, A, G, lambda, fromG, c0, bw, kb, ke, panel, cap, bar);
}

#endif  // PBAD_RESID_BCU_DMMA

constexpr int CS = CB + 4;  // = 4 (mod 16): conflict-free DMMA fragments of the diagonal block
__device__ __noinline__ bool cholesky(const R& r, double lambda) {
  const int U = r.U;
  double* A = r.DM;
  const double* G = r.GN;
  double* Lj = rsm;                       // [CB][CS] diagonal block
  double* panelA = Lj + CB * CS;           // lookahead update panel
  double* panelC = panelA + LSCAP_A;       // block-J update panel [CB][rows]
  const int warp = r.tid >> 5, lane = r.tid & 31;
  PT_START();
  for (int j0 = 0; j0 < U; j0 += CB) {
    const int bw = min(CB, U - j0);
    const int j1 = j0 + bw;                // next block column
    const int bw1 = min(CB, U - j1);
    // A) warp 0: diagonal block j0 | warps 1..7: block column j1 by k in [0, j0)
    if (warp == 0) {
#if PBAD_PHASE_TIMING
      const long long td0 = clock64();
#endif
      {
        // the block's rows, 16 loads in flight per lane (a dynamic loop here
        // exposed one L2 round trip per column)
        const double* src = (j0 > 0 ? A : G) + (j0 + lane) + (long)U * j0;
#pragma unroll
        for (int c0 = 0; c0 < CB; c0 += 16) {
          double v[16];
#pragma unroll
          for (int q = 0; q < 16; ++q)
            v[q] = (lane < bw && c0 + q < bw && c0 + q <= lane) ? src[(long)U * (c0 + q)] : 0.0;
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (lane < bw && c0 + q < bw && c0 + q <= lane)
              Lj[lane * CS + c0 + q] = (j0 == 0 && c0 + q == lane) ? v[q] + lambda : v[q];
        }
      }
      __syncwarp();
#ifndef PBAD_RESID_DIAG_DMMA
#define PBAD_RESID_DIAG_DMMA 1
#endif
#if PBAD_RESID_DIAG_DMMA
      // right-looking in 8-column sub-panels: pivots and the updates inside
      // the sub-panel are scalar (lane = row), the trailing update by the
      // sub-panel's 8 columns is one DMMA pair per 8 x 8 block (k ascending:
      // every element still receives its updates in k order)
      int ok = 1;
      const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
      for (int p = 0; p < CB / 8; ++p) {
        if (8 * p < bw && ok) {
          // lane = row: the sub-panel's 8 entries of the row in registers,
          // column k of the pivot step broadcast by shuffles
          double a[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) a[c] = Lj[lane * CS + 8 * p + c];
#pragma unroll
          for (int kq = 0; kq < 8; ++kq) {
            const int k = 8 * p + kq;
            if (k < bw && ok) {
              const double akk = __shfl_sync(FULL, a[kq], k);
              if (akk <= 0.0) {
                ok = 0;
              } else {
                const double d = sqrt(akk);
                if (lane == k) a[kq] = d;
                else if (lane > k) a[kq] = a[kq] / d;
#pragma unroll
                for (int c = kq + 1; c < 8; ++c) {
                  const double lck = __shfl_sync(FULL, a[kq], 8 * p + c);
                  if (lane > k && 8 * p + c <= lane) a[c] = fma(-a[kq], lck, a[c]);
                }
              }
            }
          }
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (8 * p + c <= lane) Lj[lane * CS + 8 * p + c] = a[c];
          __syncwarp();
          if (ok) {
#pragma unroll
            for (int rb = p + 1; rb < CB / 8; ++rb)
#pragma unroll
              for (int cb = p + 1; cb <= rb; ++cb) {
                if (8 * cb < bw) {
                  double* cp = Lj + (8 * rb + g) * CS + 8 * cb + 2 * t4;
                  double c0 = cp[0], c1 = cp[1];
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    const double a = -Lj[(8 * rb + g) * CS + 8 * p + 4 * h + t4];
                    const double b = Lj[(8 * cb + g) * CS + 8 * p + 4 * h + t4];
                    dmma884(c0, c1, a, b);
                  }
                  cp[0] = c0;
                  cp[1] = c1;
                }
              }
            __syncwarp();
          }
        }
      }
#else
      // right-looking, the trailing update spread over the packed 32x32
      // triangle (rss.pk32: row | col << 8, columns ascending)
      int ok = 1;
      for (int k = 0; k < bw; ++k) {
        const double akk = Lj[k * CS + k];
        if (akk <= 0.0) {
          ok = 0;
          break;
        }
        const double d = sqrt(akk);
        if (lane > k && lane < bw) Lj[lane * CS + k] = Lj[lane * CS + k] / d;
        __syncwarp();
        if (lane == k) Lj[k * CS + k] = d;
        const int e0 = (k + 1) * (2 * CB - k - 2) / 2 + k + 1;  // packed index of (k+1, k+1)
        for (int e = e0 + lane; e < CB * (CB + 1) / 2; e += 64) {
          const int p0 = rss.pk32[e];
          const int p1 = e + 32 < CB * (CB + 1) / 2 ? rss.pk32[e + 32] : -1;
          const int i0 = p0 & 255, c0 = p0 >> 8;
          const int i1 = p1 & 255, c1 = p1 >> 8;
          double u0 = 0.0, u1 = 0.0;
          if (i0 < bw) u0 = fma(-Lj[i0 * CS + k], Lj[c0 * CS + k], Lj[i0 * CS + c0]);
          if (p1 >= 0 && i1 < bw) u1 = fma(-Lj[i1 * CS + k], Lj[c1 * CS + k], Lj[i1 * CS + c1]);
          if (i0 < bw) Lj[i0 * CS + c0] = u0;
          if (p1 >= 0 && i1 < bw) Lj[i1 * CS + c1] = u1;
        }
        __syncwarp();
      }
#endif
      if (lane == 0) rss.flag = ok;
#if PBAD_PHASE_TIMING
      if (lane == 0) rss.pt[12] += clock64() - td0;
#endif
    } else if (j1 < U) {
#if PBAD_PHASE_TIMING
      const long long tu0 = clock64();
#endif
      block_col_update<NT - 32>(r, A, G, lambda, true, j1, bw1, 0, j0, panelA, LSCAP_A, 1);
#if PBAD_PHASE_TIMING
      if (r.tid == 32) rss.pt[13] += clock64() - tu0;
#endif
    }
    __syncthreads();
    PT_MARK(10);
    if (!rss.flag) {
      __syncthreads();
      return false;
    }
    // diagonal block to HBM
    for (int t = r.tid; t < bw * bw; t += NT) {
      const int rr = t / bw, c = t - rr * bw;
      if (c <= rr) A[(j0 + rr) + (long)U * (j0 + c)] = Lj[rr * CS + c];
    }
    // B) rows below the diagonal block: one thread per row, registers; the
    //    diagonal block's column k is read per step with explicit ld.shared
    //    (volatile: not hoisted across steps, no generic addressing)
    {
      const unsigned ljs = (unsigned)__cvta_generic_to_shared(Lj);
      for (int i = j1 + r.tid; i < U; i += NT) {
        double a[CB];
        const double* src = (j0 > 0 ? A : G) + i + (long)U * j0;
#pragma unroll
        for (int c = 0; c < CB; ++c) a[c] = c < bw ? src[(long)U * c] : 0.0;
        if (bw == CB) {
#pragma unroll
          for (int k = 0; k < CB; ++k) {
            a[k] = a[k] / lds_f64(ljs + 8u * (k * CS + k));
#pragma unroll
            for (int j0c = k + 1; j0c < CB; j0c += 8) {  // column k in chunks of 8 (register budget)
              double col[8];
#pragma unroll
              for (int q = 0; q < 8; ++q)
                if (j0c + q < CB) col[q] = lds_f64(ljs + 8u * ((j0c + q) * CS + k));
#pragma unroll
              for (int q = 0; q < 8; ++q)
                if (j0c + q < CB) a[j0c + q] = fma(-a[k], col[q], a[j0c + q]);
            }
          }
        } else {
          for (int k = 0; k < bw; ++k) {
            // short last block: dynamic k, row in registers through a rotation-free select
#pragma unroll
            for (int kk = 0; kk < CB; ++kk)
              if (kk == k) {
                a[kk] = a[kk] / lds_f64(ljs + 8u * (kk * CS + kk));
#pragma unroll
                for (int j = kk + 1; j < CB; ++j)
                  if (j < bw) a[j] = fma(-a[kk], lds_f64(ljs + 8u * (j * CS + kk)), a[j]);
              }
          }
        }
        double* dst = A + i + (long)U * j0;
#pragma unroll
        for (int c = 0; c < CB; ++c)
          if (c < bw) dst[(long)U * c] = a[c];
      }
    }
    __syncthreads();
    PT_MARK(11);
    // C) block column j1 by block j0's columns
    if (j1 < U) {
      block_col_update<NT>(r, A, G, lambda, false, j1, bw1, j0, j1, panelC, LSCAP_C, 0);
      __syncthreads();
    }
    PT_MARK(9);
  }
  return true;
}

// llt_solve (eigen_lite): x = L^-T L^-1 b in place on v (global, length U)
__device__ __noinline__ void llt_solve(const R& r, double* v) {
  const int U = r.U;
  const double* A = r.DM;
  const int warp = r.tid >> 5, lane = r.tid & 31;
  // forward: column-oriented, blocks ascending
  for (int j0 = 0; j0 < U; j0 += CB) {
    const int bw = min(CB, U - j0);
    if (warp == 0) {
      double x = lane < bw ? v[j0 + lane] : 0.0;
      double lrow[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) lrow[c] = (lane < bw && c <= lane) ? A[(j0 + lane) + (long)U * (j0 + c)] : 0.0;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (j < bw) {
          const double xj = __shfl_sync(FULL, x, j) / __shfl_sync(FULL, lrow[j], j);
          if (lane == j) x = xj;
          else if (lane > j && lane < bw) x = fma(-lrow[j], xj, x);
        }
      }
      if (lane < bw) v[j0 + lane] = x;
    }
    __syncthreads();
    for (int i = j0 + bw + r.tid; i < U; i += NT) {
      double x = v[i];
      for (int j = j0; j < j0 + bw; ++j) x = fma(-A[i + (long)U * j], v[j], x);
      v[i] = x;
    }
    __syncthreads();
  }
  // backward: for j descending, x_i -= L(j, i) x_j for i < j
  // The block row L(j0 .. j0+bw-1, 0 .. j0+bw-1) is staged in shared memory
  // first (warp per column, coalesced; column c at tile + 33 c), so the
  // per-column reads of the diagonal solve and of the update come from
  // shared memory instead of one L2 line per thread.
  constexpr int TS = CB + 1;
  double* tile = rsm;
  const int nbk = (U + CB - 1) / CB;
  for (int bk = nbk - 1; bk >= 0; --bk) {
    const int j0 = bk * CB;
    const int bw = min(CB, U - j0);
    if (lane < bw)
      for (int c = warp; c < j0 + bw; c += NT / 32) cp_async8(tile + c * TS + lane, A + (j0 + lane) + (long)U * c);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      double x = lane < bw ? v[j0 + lane] : 0.0;
      // lane l holds column j0 + l of the block: L(j0 + c, j0 + l) for c >= l
      double lcol[CB];
      const double* tc = tile + (j0 + lane) * TS;
#pragma unroll
      for (int c = 0; c < CB; ++c) lcol[c] = (lane < bw && c >= lane && c < bw) ? tc[c] : 0.0;
#pragma unroll
      for (int jr = CB - 1; jr >= 0; --jr) {
        if (jr < bw) {
          const double xj = __shfl_sync(FULL, x, jr) / __shfl_sync(FULL, lcol[jr], jr);
          if (lane == jr) x = xj;
          else if (lane < jr) x = fma(-lcol[jr], xj, x);
        }
      }
      if (lane < bw) v[j0 + lane] = x;
    }
    __syncthreads();
    for (int i = r.tid; i < j0; i += NT) {
      double x = v[i];
      const double* ti = tile + i * TS;
      for (int j = bw - 1; j >= 0; --j) x = fma(-ti[j], v[j0 + j], x);
      v[i] = x;
    }
    __syncthreads();
  }
}

#elif PBAD_RESID_CHOL_REG
constexpr int CS = CB + 1;  // smem row stride of the diagonal block / panel rows
__device__ __noinline__ bool cholesky(const R& r, double lambda) {
  const int U = r.U;
  double* A = r.DM;
  const double* G = r.GN;
  double* Lj = rsm;                 // [CB][CS] factored diagonal block
  double* Ls = rsm + CB * CS;       // [kc][rows] panel rows of the k-chunk (LSCAP doubles)
  const int warp = r.tid >> 5, lane = r.tid & 31;
  PT_START();
  for (int j0 = 0; j0 < U; j0 += CB) {
    const int bw = min(CB, U - j0);
    const int rows = U - j0;
    // 1) block-column update by columns [0, j0): acc over k ascending
    if (j0 > 0) {
      // thread (ty, tx): rows j0 + ty + 32 ii, cols j0 + tx + 8 jj
      const int tx = r.tid & 7, ty = r.tid >> 3;
      constexpr int MI = (MAXU + 31) / 32;
      double acc[MI][4];
      const int ni = (rows + 31) / 32;
#pragma unroll
      for (int ii = 0; ii < MI; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int i = j0 + ty + 32 * ii, j = j0 + tx + 8 * jj;
          acc[ii][jj] = (ii < ni && i < U && j < j0 + bw && j <= i)
                            ? (i == j ? G[i + (long)U * j] + lambda : G[i + (long)U * j])
                            : 0.0;
        }
      // k-chunks as long as the panel fits in shared memory (few, large chunks:
      // the late block columns have few rows and a long k range)
      const int kcap = LSCAP / rows;
      for (int k0 = 0; k0 < j0; k0 += kcap) {
        const int kc = min(kcap, j0 - k0);
        __syncthreads();
        // cp.async: every thread keeps all its copies in flight
        for (int kk = 0; kk < kc; ++kk)
          for (int rr = r.tid; rr < rows; rr += NT) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(Ls + kk * rows + rr);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(A + (j0 + rr) + (long)U * (k0 + kk))
                         : "memory");
          }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
          double bv[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) bv[jj] = Ls[kk * rows + min(tx + 8 * jj, rows - 1)];
#pragma unroll
          for (int ii = 0; ii < MI; ++ii) {
            if (ii < ni) {
              const double av = Ls[kk * rows + min(ty + 32 * ii, rows - 1)];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = fma(-av, bv[jj], acc[ii][jj]);
            }
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int ii = 0; ii < MI; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int i = j0 + ty + 32 * ii, j = j0 + tx + 8 * jj;
          if (ii < ni && i < U && j < j0 + bw && j <= i) A[i + (long)U * j] = acc[ii][jj];
        }
      __syncthreads();
    }
    PT_MARK(9);
    // 2) diagonal block: one warp, lane l owns row j0 + l
    if (warp == 0) {
      double a[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        const long at = (j0 + lane) + (long)U * (j0 + c);
        a[c] = (lane < bw && c <= lane) ? (j0 > 0 ? A[at] : (c == lane ? G[at] + lambda : G[at])) : 0.0;
      }
      int ok = 1;
#pragma unroll
      for (int k = 0; k < CB; ++k) {
        if (k < bw && ok) {
          const double akk = __shfl_sync(FULL, a[k], k);
          if (akk <= 0.0) {
            ok = 0;
          } else {
            const double d = sqrt(akk);
            if (lane == k) a[k] = d;
            else if (lane > k) a[k] = a[k] / d;
#pragma unroll
            for (int j = k + 1; j < CB; ++j) {
              const double ljk = __shfl_sync(FULL, a[k], j);
              if (j < bw && lane >= j) a[j] = fma(-a[k], ljk, a[j]);
            }
          }
        }
      }
      if (lane == 0) rss.flag = ok;
      if (ok) {
#pragma unroll
        for (int c = 0; c < CB; ++c)
          if (lane < bw && c <= lane) {
            A[(j0 + lane) + (long)U * (j0 + c)] = a[c];
            Lj[lane * CS + c] = a[c];
          }
      }
    }
    __syncthreads();
    if (!rss.flag) {
      __syncthreads();
      return false;
    }
    PT_MARK(10);
    // 3) rows below the diagonal block: one thread per row
    for (int i = j0 + bw + r.tid; i < U; i += NT) {
      double a[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) a[c] = c < bw ? (j0 > 0 ? A : G)[i + (long)U * (j0 + c)] : 0.0;
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
    PT_MARK(11);
  }
  return true;
}

// llt_solve (eigen_lite): x = L^-T L^-1 b in place on v (shared, length U)
__device__ __noinline__ void llt_solve(const R& r, double* v) {
  const int U = r.U;
  const double* A = r.DM;
  const int warp = r.tid >> 5, lane = r.tid & 31;
  // forward: column-oriented, blocks ascending
  for (int j0 = 0; j0 < U; j0 += CB) {
    const int bw = min(CB, U - j0);
    if (warp == 0) {
      double x = lane < bw ? v[j0 + lane] : 0.0;
      double lrow[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) lrow[c] = (lane < bw && c <= lane) ? A[(j0 + lane) + (long)U * (j0 + c)] : 0.0;
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (j < bw) {
          const double xj = __shfl_sync(FULL, x, j) / __shfl_sync(FULL, lrow[j], j);
          if (lane == j) x = xj;
          else if (lane > j && lane < bw) x = fma(-lrow[j], xj, x);
        }
      }
      if (lane < bw) v[j0 + lane] = x;
    }
    __syncthreads();
    for (int i = j0 + bw + r.tid; i < U; i += NT) {
      double x = v[i];
      for (int j = j0; j < j0 + bw; ++j) x = fma(-A[i + (long)U * j], v[j], x);
      v[i] = x;
    }
    __syncthreads();
  }
  // backward: for j descending, x_i -= L(j, i) x_j for i < j
  const int nbk = (U + CB - 1) / CB;
  for (int bk = nbk - 1; bk >= 0; --bk) {
    const int j0 = bk * CB;
    const int bw = min(CB, U - j0);
    if (warp == 0) {
      double x = lane < bw ? v[j0 + lane] : 0.0;
      // lane l holds column j0 + l of the block: L(j0 + c, j0 + l) for c >= l
      double lcol[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) lcol[c] = (lane < bw && c >= lane && c < bw) ? A[(j0 + c) + (long)U * (j0 + lane)] : 0.0;
#pragma unroll
      for (int jr = CB - 1; jr >= 0; --jr) {
        if (jr < bw) {
          const double xj = __shfl_sync(FULL, x, jr) / __shfl_sync(FULL, lcol[jr], jr);
          if (lane == jr) x = xj;
          else if (lane < jr) x = fma(-lcol[jr], xj, x);
        }
      }
      if (lane < bw) v[j0 + lane] = x;
    }
    __syncthreads();
    for (int i = r.tid; i < j0; i += NT) {
      double x = v[i];
      for (int j = j0 + bw - 1; j >= j0; --j) x = fma(-A[j + (long)U * i], v[j], x);
      v[i] = x;
    }
    __syncthreads();
  }
}

#else
constexpr int CS = CB + 1;
__device__ __noinline__ bool cholesky(const R& r, double lambda) {
  const int U = r.U;
  double* A = r.DM;
  const double* G = r.GN;
  double* Ls = rsm;                 // [LK][LP] panel rows of the k-chunk
  double* Lj = rsm + LK * LP;       // [CB][CS] diagonal block
  double* Rs = Lj + CB * CS;         // [MAXU][CS] rows below the diagonal block
  const int warp = r.tid >> 5, lane = r.tid & 31;
  for (int j0 = 0; j0 < U; j0 += CB) {
    const int bw = min(CB, U - j0);
    const int rows = U - j0;
    // 1) block-column update by columns [0, j0): acc over k ascending
    if (j0 > 0) {
      // thread (ty, tx): rows j0 + ty + 32 ii, cols j0 + tx + 8 jj
      const int tx = r.tid & 7, ty = r.tid >> 3;
      constexpr int MI = (MAXU + 31) / 32;
      double acc[MI][4];
      const int ni = (rows + 31) / 32;
#pragma unroll
      for (int ii = 0; ii < MI; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int i = j0 + ty + 32 * ii, j = j0 + tx + 8 * jj;
          acc[ii][jj] = (ii < ni && i < U && j < j0 + bw && j <= i)
                            ? (i == j ? G[i + (long)U * j] + lambda : G[i + (long)U * j])
                            : 0.0;
        }
      for (int k0 = 0; k0 < j0; k0 += LK) {
        const int kc = min(LK, j0 - k0);
        __syncthreads();
        for (int t = r.tid; t < LK * rows; t += NT) {
          const int kk = t / rows, rr = t - kk * rows;
          Ls[kk * LP + rr] = kk < kc ? A[(j0 + rr) + (long)U * (k0 + kk)] : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
          double bv[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) bv[jj] = Ls[kk * LP + tx + 8 * jj];
#pragma unroll
          for (int ii = 0; ii < MI; ++ii) {
            if (ii < ni) {
              const double av = Ls[kk * LP + min(ty + 32 * ii, rows - 1)];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = fma(-av, bv[jj], acc[ii][jj]);
            }
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int ii = 0; ii < MI; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int i = j0 + ty + 32 * ii, j = j0 + tx + 8 * jj;
          if (ii < ni && i < U && j < j0 + bw && j <= i) A[i + (long)U * j] = acc[ii][jj];
        }
      __syncthreads();
    }
    // 2) diagonal block: one warp in shared memory, lane l owns row j0 + l
    if (warp == 0) {
      for (int c = 0; c < bw; ++c)
        if (lane < bw && c <= lane) {
          const long at = (j0 + lane) + (long)U * (j0 + c);
          Lj[lane * CS + c] = j0 > 0 ? A[at] : (c == lane ? G[at] + lambda : G[at]);
        }
      __syncwarp();
      int ok = 1;
      for (int k = 0; k < bw; ++k) {
        const double akk = Lj[k * CS + k];
        if (akk <= 0.0) {
          ok = 0;
          break;
        }
        const double d = sqrt(akk);
        __syncwarp();
        if (lane == k) Lj[k * CS + k] = d;
        else if (lane > k && lane < bw) Lj[lane * CS + k] = Lj[lane * CS + k] / d;
        __syncwarp();
        if (lane > k && lane < bw) {
          const double lik = Lj[lane * CS + k];
          for (int j = k + 1; j <= lane; ++j) Lj[lane * CS + j] = fma(-lik, Lj[j * CS + k], Lj[lane * CS + j]);
        }
        __syncwarp();
      }
      if (lane == 0) rss.flag = ok;
      if (ok)
        for (int c = 0; c < bw; ++c)
          if (lane < bw && c <= lane) A[(j0 + lane) + (long)U * (j0 + c)] = Lj[lane * CS + c];
    }
    // stage the rows below the diagonal block meanwhile (other warps)
    const int nr = U - j0 - bw;
    for (int t = warp == 0 ? nr * bw : r.tid - 32; t < nr * bw; t += NT - 32) {
      const int c = t / nr, rr = t - c * nr;
      const long at = (j0 + bw + rr) + (long)U * (j0 + c);
      Rs[rr * CS + c] = j0 > 0 ? A[at] : G[at];
    }
    __syncthreads();
    if (!rss.flag) {
      __syncthreads();
      return false;
    }
    // 3) rows below the diagonal block: one thread per row (shared memory)
    for (int rr = r.tid; rr < nr; rr += NT) {
      double* row = Rs + rr * CS;
      for (int k = 0; k < bw; ++k) {
        const double lik = row[k] / Lj[k * CS + k];
        row[k] = lik;
        for (int j = k + 1; j < bw; ++j) row[j] = fma(-lik, Lj[j * CS + k], row[j]);
      }
    }
    __syncthreads();
    for (int t = r.tid; t < nr * bw; t += NT) {
      const int c = t / nr, rr = t - c * nr;
      A[(j0 + bw + rr) + (long)U * (j0 + c)] = Rs[rr * CS + c];
    }
    __syncthreads();
  }
  return true;
}

// llt_solve (eigen_lite): x = L^-T L^-1 b in place on v (global, length U),
// blocked: one warp solves each diagonal block, all threads apply it to the
// remaining rows (each element's fma chain keeps the reference order).
__device__ __noinline__ void llt_solve(const R& r, double* v) {
  const int U = r.U;
  const double* A = r.DM;
  double* Lj = rsm;            // [CB][CS]
  double* vs = Lj + CB * CS;    // [U]
  const int warp = r.tid >> 5, lane = r.tid & 31;
  for (int t = r.tid; t < U; t += NT) vs[t] = v[t];
  __syncthreads();
  // forward: x_i -= L(i, j) x_j for i > j, j ascending
  for (int j0 = 0; j0 < U; j0 += CB) {
    const int bw = min(CB, U - j0);
    if (warp == 0) {
      for (int c = 0; c < bw; ++c)
        if (lane < bw && c <= lane) Lj[lane * CS + c] = A[(j0 + lane) + (long)U * (j0 + c)];
      __syncwarp();
      for (int j = 0; j < bw; ++j) {
        const double xj = vs[j0 + j] / Lj[j * CS + j];
        __syncwarp();
        if (lane == j) vs[j0 + j] = xj;
        else if (lane > j && lane < bw) vs[j0 + lane] = fma(-Lj[lane * CS + j], xj, vs[j0 + lane]);
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = j0 + bw + r.tid; i < U; i += NT) {
      double x = vs[i];
#pragma unroll 8
      for (int j = j0; j < j0 + bw; ++j) x = fma(-A[i + (long)U * j], vs[j], x);
      vs[i] = x;
    }
    __syncthreads();
  }
  // backward: x_i -= L(j, i) x_j for i < j, j descending
  const int nbk = (U + CB - 1) / CB;
  for (int bk = nbk - 1; bk >= 0; --bk) {
    const int j0 = bk * CB;
    const int bw = min(CB, U - j0);
    if (warp == 0) {
      for (int c = 0; c < bw; ++c)
        if (lane < bw && c <= lane) Lj[lane * CS + c] = A[(j0 + lane) + (long)U * (j0 + c)];
      __syncwarp();
      for (int j = bw - 1; j >= 0; --j) {
        const double xj = vs[j0 + j] / Lj[j * CS + j];
        __syncwarp();
        if (lane == j) vs[j0 + j] = xj;
        else if (lane < j) vs[j0 + lane] = fma(-Lj[j * CS + lane], xj, vs[j0 + lane]);
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = r.tid; i < j0; i += NT) {
      double x = vs[i];
      const double* Ai = A + (long)U * i;
#pragma unroll 8
      for (int j = j0 + bw - 1; j >= j0; --j) x = fma(-Ai[j], vs[j], x);
      vs[i] = x;
    }
    __syncthreads();
  }
  for (int t = r.tid; t < U; t += NT) v[t] = vs[t];
  __syncthreads();
}

#endif

struct Solver {
  int status, iters, stag, acc;
  double value, lambda, grad0;
  double* itv;  // per_iteration_values row of this step (thread 0 writes), or null
};


// full evaluation at r.x: value, residual Jacobian, gradient, GN
__device__ __noinline__ int full_eval(const R& r, double* value) {
  if (r.energy) {
    if (!passes(r, r.x, false)) return TR_NONFINITE_CFG;
    const double v = energy_value(r, r.x);
    *value = v;
    if (!isfinite(v)) return TR_NONFINITE_INIT;
    energy_grad(r);
    jacobian(r);
    energy_gn(r);
    return 0;
  }
  PT_START();
  if (!passes(r, r.x, true)) return TR_NONFINITE_CFG;
  const double v = residual(r);
  *value = v;
  PT_MARK(5);
  if (!isfinite(v)) return TR_NONFINITE_INIT;
  jacobian(r);
  PT_MARK(6);
  gradient(r);
  __syncthreads();
  PT_MARK(7);
  gauss_newton(r);
  PT_MARK(8);
  return 0;
}

// LmSolver::iterate (optim.cpp:95-134).  Returns the status or -1 (ModelError).
__device__ int lm_iterate(const R& r, Solver& S) {
  const DOpt& o = r.sc->opt;
  if (S.status != ST_RUNNING) return S.status;
  if (S.iters >= o.max_iters) return S.status = ST_FAILED;
  PT_START();
  {
    const double g = infnorm(r, r.grad, r.U);
    const double xn = infnorm(r, r.x, r.U);
    bool conv = g <= o.grad_tol * fmax(1.0, xn);
    if (!conv && o.grad_rtol > 0.0 && g <= o.grad_rtol * S.grad0) conv = true;
    if (conv) return S.status = ST_CONVERGED;
  }
  const int U = r.U;
  double* v = r.step;
  for (int t = r.tid; t < U; t += NT) v[t] = -r.grad[t];
  __syncthreads();
  bool accepted = false;
  PT_MARK(0);
  const bool ok = cholesky(r, S.lambda);
  PT_MARK(1);
  bool finite = false;
  if (ok) {
    llt_solve(r, v);
    finite = all_finite(r, v, U);
  }
  PT_MARK(2);
  if (finite) {
    for (int t = r.tid; t < U; t += NT) r.cand[t] = r.x[t] + v[t];
    __syncthreads();
    if (!passes(r, r.cand, false)) return -1;
    PT_MARK(3);
    const double tv = r.energy ? energy_value(r, r.cand) : residual(r);
    PT_MARK(4);
    if (isfinite(tv) && tv < S.value) {
      const double oldv = S.value;
      for (int t = r.tid; t < U; t += NT) r.x[t] = r.cand[t];
      __syncthreads();
      // evaluate(x) at the accepted candidate: its passes, residuals and
      // adjoint sums are the trial's (same configuration, same operations),
      // only the second joint derivatives are new
      const double nv = tv;
      if (r.energy) {
        PT_START();
        energy_grad(r);
        PT_MARK(7);
        jacobian(r);
        PT_MARK(6);
        energy_gn(r);
        PT_MARK(8);
      } else {
        PT_START();
        passes_d2(r, r.x);
        PT_MARK(5);
        jacobian(r);
        PT_MARK(6);
        gradient(r);
        __syncthreads();
        PT_MARK(7);
        gauss_newton(r);
        PT_MARK(8);
      }
      S.value = nv;
      S.lambda = fmax(S.lambda / o.lm_lambda_factor, 1e-12);
      accepted = true;
      ++S.acc;
      if (oldv - nv <= o.ftol * fmax(1.0, fabs(oldv))) ++S.stag;
      else S.stag = 0;
      if (S.stag >= 2) S.status = ST_CONVERGED;
    }
  }
  if (!accepted) {
    S.lambda *= o.lm_lambda_factor;
    if (S.lambda > o.lm_lambda_max) S.status = ST_FAILED;
  }
  if (S.itv && r.tid == 0) S.itv[S.iters] = S.value;
  ++S.iters;
  if (S.status == ST_RUNNING && S.iters >= o.max_iters) S.status = ST_FAILED;
  return S.status;
}

// ForceModel::tau_at (objective.hpp:28-58) for instant mm into dst
__device__ __noinline__ void tau_at(const R& r, double t, double* dst) {
  const DForces& f = *r.f;
  const int n = r.n;
  for (int i = r.tid; i < n; i += NT) {
    double v = 0.0;
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
    }
    dst[i] = v;
  }
}

// One PBAD step of environment e by the whole CTA.  Every early return is
// CTA-uniform.
__device__ __forceinline__ void resid_env_step(const DModel& m, const DForces& f, const DSchedule& sc, const Layout& L,
                                               double* ws, int* iws, long B, const ResidDesc& rd, double* rws,
                                               const Outputs& out, const long e) {
  if (iws[(long)IS_RUN * B + e] != TR_RUNNING) return;
  R r;
  r.m = &m;
  r.f = &f;
  r.sc = &sc;
  r.rd = &rd;
  r.tid = threadIdx.x;
  r.N = rd.N;
  r.n = rd.n;
  r.u = rd.u;
  r.U = rd.U;
  r.D = rd.D;
  r.K1 = sc.K1;
  r.grav = f.gravity_nonzero != 0;
  r.drag = f.drag_d > 0.0;
  r.have_cot = r.grav || r.drag;  // contact runs only with one of them (resid_eligible)
  r.contact = rd.ns > 0;
  r.cot_pi = r.drag || r.contact;
  r.energy = sc.objective == 0;  // PBAD_ENERGY_FORM (include/pbad_gpu.h)
  for (int mm = 0; mm < 8; ++mm) {
    // potential_terms(..., dt = t_local dt): scale = D / (dt dt) (objective.cpp:62)
    const double dtl = mm < rd.u ? sc.times[2 + mm] * sc.dt : 1.0;
    r.s2[mm] = r.drag ? 2.0 * (f.drag_d / (dtl * dtl)) : 0.0;
  }
  r.histc = 0.0;
  const double dt = sc.dt;
  r.inv_dt2 = 1.0 / (dt * dt);
  {
    double* g = rws + e * rd.gstride;
    r.J = g + rd.oJ;
    r.GN = g + rd.oGN;
    r.DM = g + rd.oDM;
    r.FH = g + rd.oFH;
    r.PH = g + rd.oPH;
    r.pass = g + rd.oPass;
    r.hw0 = g + rd.oHW0;
    r.hw1 = g + rd.oHW1;
    r.HA = g + rd.oHA;
    r.FA = g + rd.oFA;
    r.seeds = g + rd.oSeeds;
    r.cot = g + rd.oCot;
    r.x = g + rd.oX;
    r.grad = g + rd.oGrad;
    r.cand = g + rd.oCand;
    r.res = g + rd.oRes;
    r.pg = g + rd.oPg;
    r.tau = g + rd.oTau;
    r.step = g + rd.oStep;
    r.CJ = g + rd.oCJ;
  }
  const int n = r.n, u = r.u, U = r.U, N = r.N;
  for (int i = r.tid; i < N; i += NT) rss.parent[i] = m.parent[i];
  for (int c = 0, e = 0; c < CB; ++c)
    for (int rr = c; rr < CB; ++rr, ++e)
      if (e % NT == r.tid) rss.pk32[e] = (short)(rr | (c << 8));
  if (r.tid < 20) rss.pt[r.tid] = 0;
  __syncthreads();
  int* const ivp = iws + e;
  auto iv = [&](int slot) -> int& { return ivp[(long)slot * B]; };
  const int step = iv(IS_STEP);

  // ---- begin_step (stepper.cpp:83-115) ----
  double* h0 = r.cand;      // scratch until the solver starts
  double* h1 = r.cand + n;
  for (int k = r.tid; k < n; k += NT) {
    h0[k] = ws[(L.hist0 + k) * B + e];
    h1[k] = ws[(L.hist1 + k) * B + e];
  }
  const double t0 = step * dt;
  for (int mm = 0; mm < u; ++mm) tau_at(r, t0 + sc.times[2 + mm] * dt, r.tau + (long)mm * n);
  __syncthreads();
  {
    const double span = -sc.times[0];
    for (int t = r.tid; t < U; t += NT) {
      const int mm = t / n, k = t - mm * n;
      const double tau_m = sc.times[2 + mm];
      r.x[t] = sc.warm_start ? h1[k] + (tau_m / span) * (h1[k] - h0[k]) : h1[k];
    }
  }
  __syncthreads();
  // StepObjective ctor (objective.cpp:162-185): history passes
  if (!all_finite(r, h0, n) || !all_finite(r, h1, n)) {
    if (r.tid == 0) iv(IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  fk_config(r, h0, r.hw0);
  fk_config(r, h1, r.hw1);
  if (r.energy) r.histc = energy_hist_const(r);
  // gravity cotangents (objective.cpp:48-58), the same at every instant
  if (r.grav && !r.cot_pi)
    for (int i = r.tid; i < N; i += NT) stm4(r.cot + 16 * i, add(m4_zero(), gravity_cot(f, ldgm4(m.S + 16 * i))));
  __syncthreads();
  // solver construction (optim.cpp:82-93)
  Solver S;
  S.status = ST_RUNNING;
  S.itv = out.itv ? out.itv + out.rrow(e, step) * out.itv_n : nullptr;
  S.iters = 0;
  S.stag = 0;
  S.acc = 0;
  S.lambda = sc.opt.lm_lambda0;
  {
    double v;
    const int rc = full_eval(r, &v);
    if (rc) {
      if (r.tid == 0) iv(IS_RUN) = rc;
      return;
    }
    S.value = v;
    S.grad0 = infnorm(r, r.grad, U);
  }
  int st;
  while ((st = lm_iterate(r, S)) == ST_RUNNING) {
  }
  if (st < 0) {
    if (r.tid == 0) iv(IS_RUN) = TR_NONFINITE_CFG;
    return;
  }

  // ---- finish_step (stepper.cpp:118-147) ----
  const bool converged = S.status == ST_CONVERGED;
  const double gnorm = infnorm(r, r.grad, U);
  const int fs = converged ? 0 : iv(IS_FAIL) + 1;
  __syncthreads();
  if (r.tid == 0) {
    if (out.iterations) out.iterations[out.rrow(e, step)] = S.iters;
    if (out.converged) out.converged[out.rrow(e, step)] = converged;
    if (out.accepted) out.accepted[out.rrow(e, step)] = S.acc;
    if (out.final_value) out.final_value[out.rrow(e, step)] = S.value;
    if (out.final_grad_norm) out.final_grad_norm[out.rrow(e, step)] = gnorm;
    iv(IS_NREP) = step + 1;
    iv(IS_ITERS) = S.iters;
    iv(IS_STATUS) = S.status;
    iv(IS_ACC) = S.acc;
    iv(IS_FAIL) = fs;
    if (fs > sc.fail_limit) iv(IS_RUN) = TR_FAIL_LIMIT;
  }
  if (fs > sc.fail_limit) return;
  // history shift: hist0 <- (K == 2 ? hist1 : x_{u-2}), hist1 <- x_{u-1}
  for (int k = r.tid; k < n; k += NT) {
    const double nh0 = (sc.order == 2) ? ws[(L.hist1 + k) * B + e] : r.x[(long)(u - 2) * n + k];
    ws[(L.hist0 + k) * B + e] = nh0;
    ws[(L.hist1 + k) * B + e] = r.x[(long)(u - 1) * n + k];
  }
  // energy audit on world(new hist1) (stepper.cpp:132-138); hw0 is free now
  const double* xq = r.x + (long)(u - 1) * n;
  fk_config(r, xq, r.hw0);
  for (int i = r.tid; i < N; i += NT) {
    const M4 S_i = ldgm4(m.S + 16 * i);
    const M4 wn = ldm4(r.hw0 + 16 * i);
    const M4 tdm = divs(sub(wn, ldm4(r.hw1 + 16 * i)), dt);
    r.FA[2 * i] = 0.5 * ddot(mul(tdm, S_i), tdm);
    const double ghat[4] = {f.gravity[0], f.gravity[1], f.gravity[2], 0.0};
    const double e4[4] = {0.0, 0.0, 0.0, 1.0};
    double uu[4], vv[4];
    mul_vec4(S_i, e4, uu);
    mul_vec4(wn, uu, vv);
    r.FA[2 * i + 1] = dot4(ghat, vv);
  }
  __syncthreads();
  if (r.tid == 0) {
    double ke = 0.0, pe = 0.0;
    for (int i = 0; i < N; ++i) {
      ke += r.FA[2 * i];
      pe -= r.FA[2 * i + 1];
    }
    if (out.energy) {
      out.energy[out.qrow(e, step + 1) * 2] = ke;
      out.energy[out.qrow(e, step + 1) * 2 + 1] = pe;
    }
    iv(IS_NSAMP) = step + 2;
    iv(IS_STEP) = step + 1;
    if (step + 1 >= sc.total_steps) iv(IS_RUN) = TR_OK;
  }
  if (out.q)
    for (int k = r.tid; k < n; k += NT) out.q[out.qrow(e, step + 1) * n + k] = xq[k];
#if PBAD_PHASE_TIMING
  if (e == 0 && r.tid == 0)
    printf("phase cycles (block 0, %d iterations, %d accepted): conv %lld chol %lld solve %lld tpass %lld tres %lld "
           "fpassres %lld jac %lld grad %lld gn %lld | chol: C %lld A %lld B %lld | diag-only %lld updA-only %lld | jac: acc %lld walks(t0) %lld fhess(t0)+sync %lld combine %lld stage %lld\n",
           S.iters, S.acc, rss.pt[0], rss.pt[1], rss.pt[2], rss.pt[3], rss.pt[4], rss.pt[5], rss.pt[6], rss.pt[7], rss.pt[8],
           rss.pt[9], rss.pt[10], rss.pt[11], rss.pt[12], rss.pt[13], rss.pt[14], rss.pt[15], rss.pt[16], rss.pt[17],
           rss.pt[18]);
#endif
}

__global__ void __launch_bounds__(NT, 1) k_resid_step(const __grid_constant__ DModel m,
                                                      const __grid_constant__ DForces f,
                                                      const __grid_constant__ DSchedule sc,
                                                      const __grid_constant__ Layout L, double* ws, int* iws, long B,
                                                      const __grid_constant__ ResidDesc rd, double* rws,
                                                      const __grid_constant__ Outputs out) {
  const long e = blockIdx.x;
  if (e >= B) return;
  resid_env_step(m, f, sc, L, ws, iws, B, rd, rws, out, e);
}

// nsteps PBAD steps of every environment in one persistent launch, one CTA
// per SM claiming env-steps t = s B + e in order (the tree kernel's scheme,
// pbad_tree.cu k_tree_steps): an env-step waits for its environment's
// previous step (release / acquire on a per-environment flag), so the SMs
// stay busy across step boundaries.  C5's 256 environments on 148 SMs need
// two waves per step with per-step launches (1.73 waves of work).
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void __launch_bounds__(NT, 1) k_resid_steps(const __grid_constant__ DModel m,
                                                       const __grid_constant__ DForces f,
                                                       const __grid_constant__ DSchedule sc,
                                                       const __grid_constant__ Layout L, double* ws, int* iws, long B,
                                                       const __grid_constant__ ResidDesc rd, double* rws,
                                                       const __grid_constant__ Outputs out, int nsteps,
                                                       unsigned long long* counter, int* done) {
  __shared__ unsigned long long task;
  const unsigned long long total = (unsigned long long)nsteps * (unsigned long long)B;
  for (;;) {
    if (threadIdx.x == 0) task = atomicAdd(counter, 1ull);
    __syncthreads();
    const unsigned long long t = task;
    if (t >= total) break;
    const long s = (long)(t / (unsigned long long)B), e = (long)(t - (unsigned long long)s * B);
    if (s > 0 && threadIdx.x == 0)
      while (ld_acquire_gpu(done + e) < s) __nanosleep(200);
    __syncthreads();  // thread 0's acquire orders the CTA's reads of the environment's state
    resid_env_step(m, f, sc, L, ws, iws, B, rd, rws, out, e);
    __syncthreads();  // every thread's stores of this env-step before the release; task reusable
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(done + e), "r"((int)s + 1) : "memory");
  }
}

}  // namespace resid

bool resid_eligible_sizes(int N, int u) {
  return N * u >= 1 && N * u <= resid::MAXU && resid_smem_bytes(N, u) + sizeof(resid::Smem) <= 227 * 1024;
}

size_t resid_smem_bytes(int N, int u) {
  const size_t N16 = resid::SMS * (size_t)N;
  size_t b = resid::TG * 4 * resid::GB * std::max(resid::GK + 4, resid::GQ);  // J^T J tiles (double-buffered, TG groups)
  b = std::max(b, (size_t)(resid::LK * resid::LP + resid::CB * (resid::CB + 1) + resid::MAXU * (resid::CB + 1)));  // Cholesky (smem variant)
  b = std::max(b, (size_t)(resid::CB * (resid::CB + 1) + resid::LSCAP));             // Cholesky update panel
  b = std::max(b, (size_t)(resid::CB * (resid::CB + 4) + resid::LSCAP_A + resid::LSCAP_C));  // lookahead panels
  b = std::max(b, 2 * u * N16);                                           // passes
  b = std::max(b, (size_t)(N * u + 2 + 2 * 33 * N * u));                  // gradient: g + two 32-row J tiles (covers the solve's 33 U block-row tile)
  b = std::max(b, 4 * u * N16);                                           // residual sweeps
  b = std::max(b, (2 * u + u * u) * N16);                                 // Jacobian walks
  return sizeof(double) * b;
}

cudaError_t launch_resid_step(const KernelArgs& a, const ResidDesc& rd, double* rws, const Outputs& out,
                              cudaStream_t s) {
  const size_t smem = resid_smem_bytes(rd.N, rd.u);
  static SmemAttr attr_;
  size_t& configured = attr_.here();
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(resid::k_resid_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  resid::k_resid_step<<<(unsigned)a.B, resid::NT, smem, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, rd, rws, out);
  return cudaGetLastError();
}

// nsteps steps: one persistent launch (k_resid_steps) unless
// PBAD_RESID_PERSIST=0, else one k_resid_step launch per step.  sync: 2 + B
// ints of device memory; *launches: kernels launched.
cudaError_t launch_resid_steps(const KernelArgs& a, const ResidDesc& rd, double* rws, const Outputs& out, int nsteps,
                               int* sync, cudaStream_t s, long* launches) {
  static const int mode = std::getenv("PBAD_RESID_PERSIST") ? std::atoi(std::getenv("PBAD_RESID_PERSIST")) : 1;
  if (mode == 0 || nsteps <= 1 || !sync) {
    for (int k = 0; k < nsteps; ++k) {
      const cudaError_t e = launch_resid_step(a, rd, rws, out, s);
      if (e != cudaSuccess) return e;
    }
    *launches += nsteps;
    return cudaSuccess;
  }
  const size_t smem = resid_smem_bytes(rd.N, rd.u);
  static SmemAttr attr_;
  size_t& configured = attr_.here();
  static int slots = 0;
  if (smem > configured || !slots) {
    cudaError_t e = cudaFuncSetAttribute(resid::k_resid_steps, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, resid::k_resid_steps, resid::NT, smem);
    if (e != cudaSuccess) return e;
    slots = per > 0 ? per * (sms > 0 ? sms : 148) : -1;  // -1: does not fit (its 8 extra bytes of shared memory)
  }
  if (slots < 0) {
    for (int k = 0; k < nsteps; ++k) {
      const cudaError_t e = launch_resid_step(a, rd, rws, out, s);
      if (e != cudaSuccess) return e;
    }
    *launches += nsteps;
    return cudaSuccess;
  }
  cudaError_t e = cudaMemsetAsync(sync, 0, sizeof(int) * (size_t)(2 + a.B), s);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)std::min<long>(a.B, slots);
  resid::k_resid_steps<<<grid, resid::NT, smem, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, rd, rws, out, nsteps,
                                                      reinterpret_cast<unsigned long long*>(sync), sync + 2);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace pbad_gpu
