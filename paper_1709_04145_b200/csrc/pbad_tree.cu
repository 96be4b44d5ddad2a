// pbad_tree.cu -- warp-per-environment Newton (LM) kernel for articulated trees.
//
// The Newton path of the north star (SURVEY.md §8 K4+K5): per PBAD step one
// warp owns one environment and runs begin_step, the whole Levenberg-Marquardt
// loop and finish_step (stepper.cpp:83-147, optim.cpp:80-139) without leaving
// the kernel.  Per evaluation:
//   * forward kinematics (kinematics.cpp:171-181, adjoint.cpp:9-27): joint
//     transforms link-parallel across lanes, world transforms level-synchronous
//     over the tree depth, levers dof-parallel;
//   * energy value (objective.cpp:215-226): the three correlation values and the
//     gravity potential are per-link ddots summed serially in link order, the
//     history factors T = hw S precomputed once per step;
//   * gradient (adjoint.cpp:49-64): both adjoint sweeps (inertial seeds and
//     gravity cotangents) run concurrently, level-synchronous from the leaves,
//     each parent summing its children's contributions in descending child index
//     (the reference's accumulation order);
//   * Gauss-Newton matrix (adjoint.cpp:132-176, objective.cpp:249-254):
//     composite inertias level-synchronous, then one lane per (link, ancestor,
//     dof pair) task evaluating both mixed traces from one A^T B product,
//     symmetrised on the fly into a lower-packed matrix;
//   * Cholesky (optim.cpp:11-15) right-looking in shared memory with the
//     trailing update spread over the packed triangle, and the two triangular
//     solves with the right-hand side in registers.
// Every scalar follows the numeric contract (pbad_math.cuh): the results are
// bit-identical to the reference build and the C oracle (tests/test_gpu_parity.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "pbad_joint.cuh"
#include "pbad_kernels.cuh"
#include "pbad_launch.h"
#include "pbad_math.cuh"

#ifndef PBAD_TREE_NOINLINE
#define PBAD_TREE_NOINLINE 0  // 1: phase functions kept out of line (smaller code, more registers)
#endif
#ifndef PBAD_TREE_GN_GLOBAL
#define PBAD_TREE_GN_GLOBAL 1  // 1: GN composite-inertia scratch in the per-env HBM/L2 block (smaller SMEM, more warps)
#endif
#ifndef PBAD_TREE_NOINLINE_COLD
#define PBAD_TREE_NOINLINE_COLD 0  // 1: multiply-called kinematics / cold phases out of line (I-cache)
#endif
#if PBAD_TREE_NOINLINE
#define TREE_NOINLINE __noinline__
#else
#define TREE_NOINLINE
#endif
#if PBAD_TREE_NOINLINE || PBAD_TREE_NOINLINE_COLD
#define TREE_COLD __noinline__
#else
#define TREE_COLD
#endif

namespace pbad_gpu {
// The L-BFGS translation unit (pbad_tree_lbfgs.cu) compiles this file again
// under its own namespace so the device functions' host stubs do not collide.
#ifdef PBAD_TREE_LBFGS_TU
#define PBAD_TREE_NS tree_lbfgs
#else
#define PBAD_TREE_NS tree
#endif
namespace PBAD_TREE_NS {

constexpr unsigned FULL = 0xffffffffu;
constexpr int MAXV = 3;  // dof vectors in registers: n <= 96
constexpr int MAXN = 96;
#ifndef PBAD_TREE_MS
#define PBAD_TREE_MS 18
#endif
constexpr int MS = PBAD_TREE_MS;
constexpr int TREE_SCR_ARRAYS = PBAD_TREE_GN_GLOBAL ? 2 : 4;  // link scratch arrays in SMEM  // shared-memory stride of a 4x4 (16 + 2 pad: conflict-free lane-per-link double2 access)
enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_FAILED = 2 };
enum { TR_OK = 0, TR_FAIL_LIMIT = 1, TR_NONFINITE_INIT = 2, TR_NONFINITE_CFG = 3, TR_RUNNING = 4 };

__device__ __forceinline__ M4 ld16(const double* p) {
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
__device__ __forceinline__ M4 ldg16(const double* p) {
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
__device__ __forceinline__ void st16(double* p, const M4& m) {
  double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
  for (int k = 0; k < 8; ++k) q[k] = make_double2(m.a[2 * k], m.a[2 * k + 1]);
}

// trace(mul(X, F)) and trace(mul(transpose(X), F)) from the diagonal only
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
__device__ __forceinline__ double trace_tmul(const M4& X, const M4& F) {
  double d[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    double acc = X.a[4 * p] * F.a[4 * p];
    acc = fma(X.a[1 + 4 * p], F.a[1 + 4 * p], acc);
    acc = fma(X.a[2 + 4 * p], F.a[2 + 4 * p], acc);
    acc = fma(X.a[3 + 4 * p], F.a[3 + 4 * p], acc);
    d[p] = acc;
  }
  return ((d[0] + d[1]) + d[2]) + d[3];
}

// gravity cotangent of one link (objective.cpp:48-58): c = -ghat (S e4)^T
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

__device__ __forceinline__ int pidx(int n, int row, int col) { return col * (2 * n - col - 1) / 2 + row; }

struct W {
  const DModel* m;
  const DForces* f;
  const DSchedule* sc;
  const TreeDesc* td;
  int lane, N, n, D, np;
  bool grav;
  double inv_dt2, histconst;
  // shared memory
  double *value, *world, *lever, *scr, *damped, *red;
  double *x, *grad, *cand, *vtau, *vtmp;
  double *q2, *dir, *evg;     // L-BFGS two-loop vector, direction, candidate gradient
  // global, this environment's block
  double *gn, *hw0, *hw1, *T0, *T1, *gs;
  // potentials: drag scale, contact flags / per-sample scratch
  bool drag, contact;
  double scl;                 // drag_d / dt^2
  double* ctv;                // [ns] contact value term of each sample (shared)
  int* cact;                  // [ns] sample active at the evaluated configuration (shared)
  int* clist;                 // [ns] ascending indices of the active samples (GN assembly)
  double* cdep;               // [ns][4]: depth, pv0..pv2 (shared)
  double *abl, *abu, *cs;     // global: packed ab(col,row), ab(row,col); sample dd / jr
  __device__ __forceinline__ double* scr_k(int k) const { return scr + (long)k * MS * N; }
};

// VecX dot (32 interleaved partials + pairwise tree, pbad_math.cuh vdot32):
// lane k owns partial k, the butterfly reproduces the tree (commutative adds)
__device__ __forceinline__ double vdot_warp(const W& w, const double* a, const double* b) {
  double p = 0.0;
  for (int i = w.lane; i < w.n; i += 32) p = fma(a[i], b[i], p);
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) p = p + __shfl_xor_sync(FULL, p, s);
  return p;
}
__device__ __forceinline__ double infnorm_warp(const W& w, const double* a) {
  double mx = 0.0;
  for (int i = w.lane; i < w.n; i += 32) mx = fmax(mx, fabs(a[i]));
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, s));
  return mx;
}
__device__ __forceinline__ bool all_finite_warp(const W& w, const double* a) {
  bool ok = true;
  for (int i = w.lane; i < w.n; i += 32) ok = ok && isfinite(a[i]);
  return __all_sync(FULL, ok);
}

// forward_pass / ConfigPass::make value+world part (kinematics.cpp:171-181,
// adjoint.cpp:9-27).  false = non-finite configuration (ModelError).
__device__ TREE_COLD bool fk_world(const W& w, const double* q) {
  if (!all_finite_warp(w, q)) return false;
  const DModel& m = *w.m;
  for (int i = w.lane; i < w.N; i += 32) {
    double ql[6];
    const int off = m.dof_off[i], cnt = m.dof_cnt[i];
    for (int j = 0; j < cnt; ++j) ql[j] = q[off + j];
    st16(w.value + MS * i, joint_transform(m.kind[i], m.axis + 3 * i, ldg16(m.offset + 16 * i), ql));
  }
  __syncwarp();
  const TreeDesc& td = *w.td;
  for (int d = 0; d <= w.D; ++d) {
    for (int t = td.lvl_start[d] + w.lane; t < td.lvl_start[d + 1]; t += 32) {
      const int i = td.lvl_links[t];
      const int p = m.parent[i];
      const M4 v = ld16(w.value + MS * i);
      st16(w.world + MS * i, p >= 0 ? mul(ld16(w.world + MS * p), v) : v);
    }
    __syncwarp();
  }
  return true;
}

// levers of ConfigPass::make (adjoint.cpp:20-24): lever = parent_world * d1
__device__ TREE_COLD void fk_levers(const W& w, const double* q) {
  const DModel& m = *w.m;
  double* d1s = w.scr;  // n x 16 scratch
  for (int i = w.lane; i < w.N; i += 32) {
    double ql[6];
    const int off = m.dof_off[i], cnt = m.dof_cnt[i];
    for (int j = 0; j < cnt; ++j) ql[j] = q[off + j];
    // joint_jet's d1 (kinematics.cpp:119-169), written straight to shared memory
    const M4 offm = ldg16(m.offset + 16 * i);
    const int kind = m.kind[i];
    double* dst = d1s + MS * off;
    if (kind == 0) {
      const double* ax = m.axis + 3 * i;
      const M3 Ka = skew(ax[0], ax[1], ax[2]);
      const M3 R = rotation_vector_matrix(ax[0] * ql[0], ax[1] * ql[0], ax[2] * ql[0]);
      st16(dst, mul(offm, embed_rotation(mul3(Ka, R))));
    } else {
      const int r0 = kind == 1 ? 0 : 3;
      M3 R, dR[3];
      rotation_vector_jet(ql + r0, &R, dR, nullptr, false);
      if (kind == 2) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          M4 dtj = m4_zero();
          dtj.a[j + 12] = 1.0;
          st16(dst + MS * j, mul(offm, dtj));
        }
      }
#pragma unroll
      for (int j = 0; j < 3; ++j) st16(dst + MS * (r0 + j), mul(offm, embed_rotation(dR[j])));
    }
  }
  __syncwarp();
  for (int k = w.lane; k < w.n; k += 32) {
    const int p = m.parent[w.td->dof_link[k]];
    const M4 pw = p >= 0 ? ld16(w.world + MS * p) : m4_identity();
    st16(w.lever + MS * k, mul(pw, ld16(d1s + MS * k)));
  }
  __syncwarp();
}


// contact sample s of link i at the configuration in w.world (objective.cpp:74-101):
// active flag, value term, depth and projected velocity
__device__ void contact_sample(const W& w, int i, int sidx) {
  const DModel& m = *w.m;
  const DForces& f = *w.f;
  const double* nrm = f.normal;
  const M4 wi = ld16(w.world + MS * i);
  const double ph[4] = {m.samples[3 * sidx], m.samples[3 * sidx + 1], m.samples[3 * sidx + 2], 1.0};
  double x4[4], xp4[4];
  mul_vec4(wi, ph, x4);
  const double depth = f.plane_offset - dot3(nrm, x4);
  if (depth <= 0.0) {
    w.cact[sidx] = 0;
    return;
  }
  const double dt = w.sc->dt;
  mul_vec4(ld16(w.hw1 + 16 * i), ph, xp4);
  double proj[9];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) proj[r + 3 * c] = ((r == c) ? 1.0 : 0.0) - nrm[r] * nrm[c];
  double v[3], pv[3];
  for (int k = 0; k < 3; ++k) v[k] = (x4[k] - xp4[k]) / dt;
  for (int r = 0; r < 3; ++r) {
    double acc = proj[r] * v[0];
    acc = fma(proj[r + 3], v[1], acc);
    acc = fma(proj[r + 6], v[2], acc);
    pv[r] = acc;
  }
  const double pv2 = dot3(pv, pv);
  w.cact[sidx] = 1;
  w.ctv[sidx] = f.d1 * depth * depth + f.d2 * depth * depth * pv2;
  w.cdep[4 * sidx] = depth;
  w.cdep[4 * sidx + 1] = pv[0];
  w.cdep[4 * sidx + 2] = pv[1];
  w.cdep[4 * sidx + 3] = pv[2];
}
// all samples, lane-parallel; then the drag / contact part of pot.value in
// the reference order (gravity over links, drag over links, contact samples)
__device__ void contact_all(const W& w) {
  const DModel& m = *w.m;
  for (int i = 0; i < w.N; ++i)
    for (int sidx = m.sample_off[i] + w.lane; sidx < m.sample_off[i + 1]; sidx += 32) contact_sample(w, i, sidx);
  __syncwarp();
}

// StepObjective energy value (objective.cpp:215-226, 237) at the configuration
// whose world transforms are in w.world; q is that configuration.
__device__ TREE_NOINLINE double value_at(const W& w, const double* q) {
  const DModel& m = *w.m;
  for (int i = w.lane; i < w.N; i += 32) {
    const M4 wi = ld16(w.world + MS * i);
    const M4 S = ldg16(m.S + 16 * i);
    w.red[4 * i] = ddot(mul(wi, S), wi);
    w.red[4 * i + 1] = ddot(ld16(w.T1 + 16 * i), wi);
    w.red[4 * i + 2] = ddot(ld16(w.T0 + 16 * i), wi);
    if (w.grav) w.red[4 * i + 3] = ddot(gravity_cot(*w.f, S), wi);
    if (w.drag) {
      const M4 diff = sub(wi, ld16(w.hw1 + 16 * i));
      w.red[4 * w.N + i] = w.scl * ddot(mul(diff, S), diff);
    }
  }
  if (w.contact) contact_all(w);
  __syncwarp();
  double s = 0.0;
  if (w.lane < 4) {
    if (w.lane < 3 || w.grav)
      for (int i = 0; i < w.N; ++i) s += w.red[4 * i + w.lane];
    if (w.lane == 3) {
      if (w.drag)
        for (int i = 0; i < w.N; ++i) s += w.red[4 * w.N + i];
      if (w.contact)
        for (int k = 0; k < w.td->ns; ++k)
          if (w.cact[k]) s += w.ctv[k];
    }
  }
  const double cpp = __shfl_sync(FULL, s, 0) - m.weighted_mass;
  const double c1 = __shfl_sync(FULL, s, 1) - m.weighted_mass;
  const double c0 = __shfl_sync(FULL, s, 2) - m.weighted_mass;
  const double pot = (w.grav || w.drag || w.contact) ? __shfl_sync(FULL, s, 3) : 0.0;
  const double inertial = 0.5 * w.inv_dt2 * (cpp - 4.0 * c1 + 2.0 * c0 + w.histconst);
  const double tdot = vdot_warp(w, w.vtau, q);
  return inertial + pot - tdot;
}

// energy gradient (objective.cpp:227-248): inertial seeds and gravity
// cotangents through functional_grad (adjoint.cpp:49-64), then (g + pg) - tau.
__device__ TREE_NOINLINE void gradient(const W& w, double* g) {
  const DModel& m = *w.m;
  const TreeDesc& td = *w.td;
  double* sA = w.scr_k(0);  // inertial seeds -> children contributions
  double* sB = w.scr_k(1);  // gravity cotangents -> children contributions
  for (int i = w.lane; i < w.N; i += 32) {
    const M4 S = ldg16(m.S + 16 * i);
    M4 d = sub(ld16(w.world + MS * i), scale(2.0, ld16(w.hw1 + 16 * i)));
    d = add(d, ld16(w.hw0 + 16 * i));
    d = scale(w.inv_dt2, d);
    st16(sA + MS * i, mul(d, S));
    if (w.grav || w.drag || w.contact) {
      M4 cot = m4_zero();
      if (w.grav) cot = add(cot, gravity_cot(*w.f, S));
      if (w.drag) {
        const M4 diff = sub(ld16(w.world + MS * i), ld16(w.hw1 + 16 * i));
        cot = add(cot, scale(2.0 * w.scl, mul(diff, S)));
      }
      if (w.contact) {
        const DForces& f = *w.f;
        const double dtc = w.sc->dt;
        for (int sidx = m.sample_off[i]; sidx < m.sample_off[i + 1]; ++sidx) {
          if (!w.cact[sidx]) continue;
          const double depth = w.cdep[4 * sidx];
          const double pv[3] = {w.cdep[4 * sidx + 1], w.cdep[4 * sidx + 2], w.cdep[4 * sidx + 3]};
          const double pv2 = dot3(pv, pv);
          const double a = -2.0 * f.d1 * depth - 2.0 * f.d2 * depth * pv2;
          const double b = 2.0 * f.d2 * depth * depth / dtc;
          double dq[4];
          for (int k = 0; k < 3; ++k) dq[k] = a * f.normal[k] + b * pv[k];
          dq[3] = 0.0;
          const double ph[4] = {m.samples[3 * sidx], m.samples[3 * sidx + 1], m.samples[3 * sidx + 2], 1.0};
          M4 oc;
          for (int c = 0; c < 4; ++c)
            for (int r = 0; r < 4; ++r) oc.a[r + 4 * c] = dq[r] * ph[c];
          cot = add(cot, oc);
        }
      }
      st16(sB + MS * i, cot);
    }
  }
  __syncwarp();
  // the potential sweep runs when the reference builds a cotangent
  // (objective.cpp:132-137: gravity, drag, or an active contact sample)
  bool have_cot = w.grav || w.drag;
  if (!have_cot && w.contact) {
    bool any = false;
    for (int k = w.lane; k < w.td->ns; k += 32) any = any || w.cact[k];
    have_cot = __any_sync(FULL, any);
  }
  const int nsw = have_cot ? 2 : 1;
  for (int d = w.D; d >= 0; --d) {
    const int l0 = td.lvl_start[d], cnt = td.lvl_start[d + 1] - l0;
    for (int t = w.lane; t < nsw * cnt; t += 32) {
      const int sw = t / cnt;
      const int i = td.lvl_links[l0 + t - sw * cnt];
      double* seeds = sw ? sB : sA;
      double* gout = sw ? w.vtmp : g;
      M4 adj = m4_zero();
      for (int c = td.ch_start[i]; c < td.ch_start[i + 1]; ++c) adj = add(adj, ld16(seeds + MS * td.ch_list[c]));
      const M4 a = add(adj, ld16(seeds + MS * i));
      const int off = m.dof_off[i];
      for (int j = 0; j < m.dof_cnt[i]; ++j) gout[off + j] = 0.0 + ddot(ld16(w.lever + MS * (off + j)), a);
      st16(seeds + MS * i, mul_bt(a, ld16(w.value + MS * i)));
    }
    __syncwarp();
  }
  for (int k = w.lane; k < w.n; k += 32) g[k] = (g[k] + (have_cot ? w.vtmp[k] : 0.0)) - w.vtau[k];
  __syncwarp();
}

// Gauss-Newton matrix gn = sym(hess_ab(x, x) / dt^2 + pot.gn) (objective.cpp:
// 249-254, adjoint.cpp:132-176), lower-packed into w.gn (global).
__device__ TREE_COLD void gn_assemble(const W& w) {
  const DModel& m = *w.m;
  const TreeDesc& td = *w.td;
#if PBAD_TREE_GN_GLOBAL
  constexpr int GS_ = MS;
  double* ai = w.gs;
  double* fwd = w.gs + (long)GS_ * w.N;
  double* bwd = w.gs + 2L * GS_ * w.N;
  double* Z = w.gs + 3L * GS_ * w.N;
#else
  double* ai = w.scr_k(0);
  double* fwd = w.scr_k(1);
  double* bwd = w.scr_k(2);
  double* Z = w.scr_k(3);
#endif
  for (int d = w.D; d >= 0; --d) {
    for (int t = td.lvl_start[d] + w.lane; t < td.lvl_start[d + 1]; t += 32) {
      const int i = td.lvl_links[t];
      M4 acc = m4_zero();
      for (int c = td.ch_start[i]; c < td.ch_start[i + 1]; ++c) acc = add(acc, ld16(Z + MS * td.ch_list[c]));
      const M4 a = add(acc, ldg16(m.S + 16 * i));
      const M4 v = ld16(w.value + MS * i);
      st16(ai + MS * i, a);
      const M4 y = mul(v, a);
      st16(fwd + MS * i, y);
      st16(bwd + MS * i, mul_bt(a, v));
      st16(Z + MS * i, mul_bt(y, v));
    }
    __syncwarp();
  }
  for (int t = w.lane; t < w.np; t += 32) {
    if (w.drag || w.contact) {
      w.abl[t] = 0.0;
      w.abu[t] = 0.0;
    } else {
      w.gn[t] = 0.0;
    }
  }
  __syncwarp();
  const int n = w.n;
  for (int s = 0; s <= w.D; ++s) {
    for (int t = td.task_start[s] + w.lane; t < td.task_start[s + 1]; t += 32) {
      const int code = td.tasks[t];
      const int i = code & 255, l = (code >> 8) & 255, j = (code >> 16) & 15, k = (code >> 20) & 15;
      const int offi = m.dof_off[i], offl = m.dof_off[l];
      const M4 M = mul_at(ld16(w.lever + MS * (offi + j)), ld16(w.lever + MS * (offl + k)));
      double a1, a2;  // ab(col, row), ab(row, col)
      int row, col;
      if (s == 0) {
        const M4 F = ld16(ai + MS * i);
        const double tjk = trace_mul(M, F);
        a1 = tjk;
        a2 = (j == k) ? tjk : trace_tmul(M, F);
        row = offi + k;
        col = offi + j;
      } else {
        a1 = trace_tmul(M, ld16(bwd + MS * i));
        a2 = trace_mul(M, ld16(fwd + MS * i));
        row = offi + j;
        col = offl + k;
      }
      const int e = pidx(n, row, col);
      if (w.drag || w.contact) {
        w.abl[e] = 0.0 + a1;
        w.abu[e] = 0.0 + a2;
      } else {
        const double grc = w.inv_dt2 * a1 + 0.0;
        const double gcr = w.inv_dt2 * a2 + 0.0;
        w.gn[e] = 0.5 * (grc + gcr);
      }
    }
    __syncwarp();
    if (s >= 1 && s < w.D) {
      for (int i = w.lane; i < w.N; i += 32) {
        if (td.depth[i] <= s) continue;
        const M4 vl = ld16(w.value + MS * td.anc[i * (w.D + 1) + s]);
        st16(fwd + MS * i, mul(vl, ld16(fwd + MS * i)));
        st16(bwd + MS * i, mul_bt(ld16(bwd + MS * i), vl));
      }
      __syncwarp();
    }
  }
  if (!(w.drag || w.contact)) return;
  __syncwarp();
  // contact Jacobian rows of the samples active at x (objective.cpp:103-129):
  // dd = -n^T jx, jr = pv dd^T + (depth/dt) P jx, one lane per sample
  const DForces& f = *w.f;
  if (w.contact) {
    const double* nrm = f.normal;
    double proj[9];
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) proj[r + 3 * c] = ((r == c) ? 1.0 : 0.0) - nrm[r] * nrm[c];
    for (int i = 0; i < w.N; ++i)
      for (int sidx = m.sample_off[i] + w.lane; sidx < m.sample_off[i + 1]; sidx += 32) {
        if (!w.cact[sidx]) continue;
        double* dd = w.cs + (long)sidx * 4 * n;
        double* jr = dd + n;  // holds jx first
        for (int k = 0; k < 3 * n; ++k) jr[k] = 0.0;
        double y[4] = {m.samples[3 * sidx], m.samples[3 * sidx + 1], m.samples[3 * sidx + 2], 1.0};
        for (int l = i; l >= 0; l = m.parent[l]) {
          const int off = m.dof_off[l];
          for (int j = 0; j < m.dof_cnt[l]; ++j) {
            double t4[4];
            mul_vec4(ld16(w.lever + MS * (off + j)), y, t4);
            for (int r = 0; r < 3; ++r) jr[r + 3 * (off + j)] = t4[r];
          }
          double y2[4];
          mul_vec4(ld16(w.value + MS * l), y, y2);
          for (int r = 0; r < 4; ++r) y[r] = y2[r];
        }
        for (int k = 0; k < n; ++k) {
          double acc = nrm[0] * jr[3 * k];
          acc = fma(nrm[1], jr[1 + 3 * k], acc);
          acc = fma(nrm[2], jr[2 + 3 * k], acc);
          dd[k] = -acc;
        }
        if (f.d2 > 0.0) {
          const double ddt = w.cdep[4 * sidx] / w.sc->dt;
          const double pv[3] = {w.cdep[4 * sidx + 1], w.cdep[4 * sidx + 2], w.cdep[4 * sidx + 3]};
          for (int k = 0; k < n; ++k) {
            double tmp[3];
            for (int r = 0; r < 3; ++r) {
              double acc = proj[r] * jr[3 * k];
              acc = fma(proj[r + 3], jr[1 + 3 * k], acc);
              acc = fma(proj[r + 6], jr[2 + 3 * k], acc);
              tmp[r] = acc;
            }
            for (int r = 0; r < 3; ++r) jr[r + 3 * k] = pv[r] * dd[k] + ddt * tmp[r];
          }
        }
      }
  }
  __syncwarp();
  // gn = sym(inv_dt2 ab + pot.gn), pot.gn = 2 scl ab (drag) + contact terms in
  // sample order (objective.cpp:69-70, 111-126, 249-254)
  const double s2 = 2.0 * w.scl;
  const double c2 = 2.0 * f.d1, c3 = 2.0 * f.d2;
  // active samples compacted once (ascending: the reference's sample order),
  // instead of every GN element scanning all samples
  int nact = 0;
  if (w.contact) {
    for (int base = 0; base < td.ns; base += 32) {
      const int k = base + w.lane;
      const bool on = k < td.ns && w.cact[k];
      const unsigned msk = __ballot_sync(FULL, on);
      if (on) w.clist[nact + __popc(msk & ((1u << w.lane) - 1u))] = k;
      nact += __popc(msk);
    }
    __syncwarp();
  }
  for (int t = w.lane; t < w.np; t += 32) {
    const int rc = __ldg(td.pk + t);
    const int row = rc & 0xffff, col = rc >> 16;
    const double a1 = w.abl[t], a2 = w.abu[t];
    double p1 = w.drag ? 0.0 + s2 * a1 : 0.0;  // pot.gn(col, row)
    double p2 = w.drag ? 0.0 + s2 * a2 : 0.0;  // pot.gn(row, col)
    for (int q = 0; q < nact; ++q) {
        const int k = w.clist[q];
        const double* dd = w.cs + (long)k * 4 * n;
        const double* jr = dd + n;
        p1 = p1 + (c2 * dd[col]) * dd[row];
        p2 = p2 + (c2 * dd[row]) * dd[col];
        if (f.d2 > 0.0) {
          double q1 = (c3 * jr[3 * col]) * jr[3 * row];
          q1 = fma(c3 * jr[1 + 3 * col], jr[1 + 3 * row], q1);
          q1 = fma(c3 * jr[2 + 3 * col], jr[2 + 3 * row], q1);
          double q2 = (c3 * jr[3 * row]) * jr[3 * col];
          q2 = fma(c3 * jr[1 + 3 * row], jr[1 + 3 * col], q2);
          q2 = fma(c3 * jr[2 + 3 * row], jr[2 + 3 * col], q2);
          p1 = p1 + q1;
          p2 = p2 + q2;
        }
      }
    const double grc = w.inv_dt2 * a1 + p1;
    const double gcr = w.inv_dt2 * a2 + p2;
    w.gn[t] = 0.5 * (grc + gcr);
  }
  __syncwarp();
}

// LLT (optim.cpp:11-15, eigen_lite right-looking) on the lower-packed damped
// matrix in shared memory.  false = non-positive pivot.
__device__ TREE_NOINLINE bool llt_factor_w(const W& w) {
  double* A = w.damped;
  const int n = w.n;
  for (int k = 0; k < n; ++k) {
    const int cb = pidx(n, 0, k);
    const double x = A[cb + k];
    if (x <= 0.0) return false;
    const double d = sqrt(x);
    __syncwarp();
    for (int i = k + 1 + w.lane; i < n; i += 32) A[cb + i] = A[cb + i] / d;
    if (w.lane == 0) A[cb + k] = d;
    __syncwarp();
    if (k + 1 < n) {
      // trailing update over the packed triangle, 4 elements per lane in flight
      // (column k is not written here, so the loads may run ahead of the stores)
      for (int t = pidx(n, k + 1, k + 1) + w.lane; t < w.np; t += 128) {
        int rc[4];
        double a[4], li[4], lj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) rc[u] = (t + 32 * u < w.np) ? __ldg(w.td->pk + t + 32 * u) : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = (t + 32 * u < w.np) ? A[t + 32 * u] : 0.0;
          li[u] = A[cb + (rc[u] & 0xffff)];
          lj[u] = A[cb + (rc[u] >> 16)];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (t + 32 * u < w.np) A[t + 32 * u] = fma(-li[u], lj[u], a[u]);
      }
    }
    __syncwarp();
  }
  return true;
}

__device__ __forceinline__ double sel(const double (&v)[MAXV], int s) {
  return s == 0 ? v[0] : (s == 1 ? v[1] : v[2]);
}

// llt_solve (eigen_lite): forward then backward substitution, column-oriented;
// v holds the right-hand side for rows lane + 32 s on entry, the solution on exit.
__device__ TREE_NOINLINE void llt_solve_w(const W& w, double (&v)[MAXV]) {
  const double* A = w.damped;
  const int n = w.n;
  const int nv = (n + 31) >> 5;  // live register slots (warp-uniform)
  // forward: column j of the packed factor starts at pidx(n, 0, j)
  for (int j = 0; j < n; ++j) {
    const int cs = j * (2 * n - j - 1) / 2;
    const double xj = __shfl_sync(FULL, sel(v, j >> 5), j & 31) / A[cs + j];
#pragma unroll
    for (int s = 0; s < MAXV; ++s) {
      if (s < nv) {
        const int i = w.lane + 32 * s;
        if (i == j) v[s] = xj;
        else if (i > j && i < n) v[s] = fma(-A[cs + i], xj, v[s]);
      }
    }
  }
  // backward: L(j, i) of this lane's rows i = lane + 32 s lies in column i
  int ci[MAXV];
#pragma unroll
  for (int s = 0; s < MAXV; ++s) {
    const int i = w.lane + 32 * s;
    ci[s] = i * (2 * n - i - 1) / 2;
  }
  for (int j = n - 1; j >= 0; --j) {
    const double xj = __shfl_sync(FULL, sel(v, j >> 5), j & 31) / A[pidx(n, j, j)];
#pragma unroll
    for (int s = 0; s < MAXV; ++s) {
      if (s < nv) {
        const int i = w.lane + 32 * s;
        if (i == j) v[s] = xj;
        else if (i < j) v[s] = fma(-A[ci[s] + j], xj, v[s]);
      }
    }
  }
}

// full evaluation at w.x (value, levers, gradient, GN); false = ModelError
__device__ bool full_eval(const W& w, double* value) {
  if (!fk_world(w, w.x)) return false;
  *value = value_at(w, w.x);
  return true;
}
__device__ TREE_COLD void derivatives(const W& w) {
  fk_levers(w, w.x);
  gradient(w, w.grad);
  gn_assemble(w);
}

struct Solver {
  int status, iters, stag, acc;
  double value, lambda, grad0;
  double* itv;  // per_iteration_values row of this step (lane 0 writes), or null
};

__device__ __forceinline__ bool grad_converged(const W& w, const Solver& S) {
  const DOpt& o = w.sc->opt;
  const double g = infnorm_warp(w, w.grad);
  if (g <= o.grad_tol * fmax(1.0, infnorm_warp(w, w.x))) return true;
  if (o.grad_rtol > 0.0 && g <= o.grad_rtol * S.grad0) return true;
  return false;
}

// LmSolver::iterate (optim.cpp:95-134).  Returns the status or -1 (ModelError).
__device__ int lm_iterate(const W& w, Solver& S) {
  const DOpt& o = w.sc->opt;
  if (S.status != ST_RUNNING) return S.status;
  if (S.iters >= o.max_iters) return S.status = ST_FAILED;
  if (grad_converged(w, S)) return S.status = ST_CONVERGED;
  const int n = w.n;
  for (int t = w.lane; t < w.np; t += 32) {
    const int rc = __ldg(w.td->pk + t);
    const double g = w.gn[t];
    w.damped[t] = ((rc & 0xffff) == (rc >> 16)) ? g + S.lambda : g;
  }
  double v[MAXV];
#pragma unroll
  for (int s = 0; s < MAXV; ++s) {
    const int i = w.lane + 32 * s;
    v[s] = i < n ? -w.grad[i] : 0.0;
  }
  __syncwarp();
  bool accepted = false;
  const bool ok = llt_factor_w(w);
  bool finite = false;
  if (ok) {
    llt_solve_w(w, v);
    bool f = true;
#pragma unroll
    for (int s = 0; s < MAXV; ++s)
      if (w.lane + 32 * s < n) f = f && isfinite(v[s]);
    finite = __all_sync(FULL, f);
  }
  if (finite) {
#pragma unroll
    for (int s = 0; s < MAXV; ++s) {
      const int i = w.lane + 32 * s;
      if (i < n) w.cand[i] = w.x[i] + v[s];
    }
    __syncwarp();
    if (!fk_world(w, w.cand)) return -1;
    const double tv = value_at(w, w.cand);
    if (isfinite(tv) && tv < S.value) {
      const double oldv = S.value;
      for (int i = w.lane; i < n; i += 32) w.x[i] = w.cand[i];
      __syncwarp();
      derivatives(w);
      const double nv = tv;  // evaluate(x) repeats value(cand) bit for bit
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
  if (S.itv && w.lane == 0) S.itv[S.iters] = S.value;
  ++S.iters;
  if (S.status == ST_RUNNING && S.iters >= o.max_iters) S.status = ST_FAILED;
  return S.status;
}

// ForceModel::tau_at (objective.hpp:28-58), element-parallel
__device__ TREE_COLD void tau_at(const W& w, double t, double* dst) {
  const DForces& f = *w.f;
  const int n = w.n;
  for (int i = w.lane; i < n; i += 32) {
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

// copy w.world into a history block and its body products T = hw S
__device__ TREE_COLD void store_history(const W& w, double* hw, double* T) {
  for (int i = w.lane; i < w.N; i += 32) {
    const M4 wi = ld16(w.world + MS * i);
    st16(hw + 16 * i, wi);
    st16(T + 16 * i, mul(wi, ldg16(w.m->S + 16 * i)));
  }
  __syncwarp();
}

#ifndef PBAD_TREE_LBFGS_TU
template <bool POT>
#ifndef PBAD_TREE_MINB
#define PBAD_TREE_MINB 11  // 168 registers: 12 single-warp blocks per SM by registers, ~10 by shared memory
#endif
__device__ __forceinline__ void tree_env_step(const DModel& m, const DForces& f, const DSchedule& sc, const Layout& L,
                                              double* ws, int* iws, long B, const TreeDesc& td, double* tws,
                                              const Outputs& out, long e, double* smem) {
  if (iws[(long)IS_RUN * B + e] != TR_RUNNING) return;
  W w;
  w.m = &m;
  w.f = &f;
  w.sc = &sc;
  w.td = &td;
  w.lane = threadIdx.x;
  w.N = td.N;
  w.n = td.n;
  w.D = td.D;
  w.np = td.np;
  w.grav = f.gravity_nonzero != 0;
  const double dt = sc.dt;
  w.inv_dt2 = 1.0 / (dt * dt);
  // POT = false compiles the drag / contact code out (lean fast path)
  w.drag = POT && f.drag_d > 0.0;
  w.scl = w.drag ? f.drag_d / (dt * dt) : 0.0;
  w.contact = POT && f.has_contact && (f.d1 > 0.0 || f.d2 > 0.0) && td.ns > 0;
  {
    const int N16 = MS * td.N, nv = (td.n + 1) & ~1;
    const int scr = (TREE_SCR_ARRAYS * N16 > MS * td.n) ? TREE_SCR_ARRAYS * N16 : MS * td.n;
    double* p = smem;
    w.value = p; p += N16;
    w.world = p; p += N16;
    // the damped matrix is live only from its rebuild to the end of the
    // solve, the levers and the link scratch only inside the derivatives
    // (fk_levers, gradient, GN assembly): one region serves both
    w.lever = p;
    w.scr = p + MS * td.n;
    w.damped = p;
    // the per-link value terms (value_at, hist_const, the energy audit) are
    // consumed before the derivatives run and after the solve: same region
    w.red = p;
    {
      int rs = MS * td.n + scr;
      if (((td.np + 1) & ~1) > rs) rs = (td.np + 1) & ~1;
      if (5 * td.N + 32 > rs) rs = 5 * td.N + 32;
      p += rs;
    }
    w.x = p; p += nv;
    w.grad = p; p += nv;
    w.cand = p; p += nv;
    w.vtau = p; p += nv;
    w.vtmp = p; p += nv;
    w.ctv = p; p += (td.ns + 1) & ~1;
    w.cdep = p; p += 4 * td.ns;
    w.cact = reinterpret_cast<int*>(p);
    w.clist = w.cact + ((td.ns + 1) & ~1);
    double* g = tws + e * td.gstride;
    w.gn = g;
    w.hw0 = g + td.o_hw0;
    w.hw1 = g + td.o_hw1;
    w.T0 = g + td.o_t0;
    w.T1 = g + td.o_t1;
    w.gs = g + td.o_gs;
    w.abl = g + td.o_abl;
    w.abu = g + td.o_abu;
    w.cs = g + td.o_cs;
  }
  const int n = td.n;
  int* const ivp = iws + e;
  auto iv = [&](int slot) -> int& { return ivp[(long)slot * B]; };
  const int step = iv(IS_STEP);

  // ---- begin_step (stepper.cpp:83-115) ----
  double* h0 = w.cand;
  double* h1 = w.vtmp;
  for (int k = w.lane; k < n; k += 32) {
    h0[k] = ws[(L.hist0 + k) * B + e];
    h1[k] = ws[(L.hist1 + k) * B + e];
  }
  const double t0 = step * dt;
  tau_at(w, t0 + sc.times[2] * dt, w.vtau);
  {
    const double span = -sc.times[0];
    const double tau_m = sc.times[2];
    for (int k = w.lane; k < n; k += 32) w.x[k] = sc.warm_start ? h1[k] + (tau_m / span) * (h1[k] - h0[k]) : h1[k];
  }
  __syncwarp();
  // StepObjective ctor (objective.cpp:162-185)
  if (!all_finite_warp(w, h0) || !all_finite_warp(w, h1)) {
    if (w.lane == 0) iv(IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
#pragma unroll 1
  for (int hs = 0; hs < 2; ++hs) {  // one inlined copy of the kinematics for both history configurations
    fk_world(w, hs ? h1 : h0);
    store_history(w, hs ? w.hw1 : w.hw0, hs ? w.T1 : w.T0);
  }
  {
    for (int i = w.lane; i < w.N; i += 32) {
      const M4 w0 = ld16(w.hw0 + 16 * i), w1 = ld16(w.hw1 + 16 * i);
      const M4 T1 = ld16(w.T1 + 16 * i);
      w.red[4 * i] = ddot(T1, w1);
      w.red[4 * i + 1] = ddot(ld16(w.T0 + 16 * i), w0);
      w.red[4 * i + 2] = ddot(T1, w0);
    }
    __syncwarp();
    double s = 0.0;
    if (w.lane < 3)
      for (int i = 0; i < w.N; ++i) s += w.red[4 * i + w.lane];
    const double c11 = __shfl_sync(FULL, s, 0) - m.weighted_mass;
    const double c00 = __shfl_sync(FULL, s, 1) - m.weighted_mass;
    const double c10 = __shfl_sync(FULL, s, 2) - m.weighted_mass;
    w.histconst = 4.0 * c11 + c00 - 4.0 * c10;
    __syncwarp();
  }
  // solver construction (optim.cpp:82-93) and LmSolver::iterate (optim.cpp:95-134)
  // share one loop body, so the kinematics / value / derivative code is inlined
  // once (instruction-cache footprint): pass 0 evaluates x0 with the GN matrix,
  // later passes solve the damped system and evaluate the candidate.
  Solver S;
  S.status = ST_RUNNING;
  S.itv = out.itv ? out.itv + out.rrow(e, step) * out.itv_n : nullptr;
  S.iters = 0;
  S.stag = 0;
  S.acc = 0;
  S.lambda = sc.opt.lm_lambda0;
  S.value = 0.0;
  S.grad0 = 0.0;
  {
    const DOpt& o = sc.opt;
    int err = 0;
    bool first = true;
#pragma unroll 1
    for (;;) {
      double* q = w.x;
      bool do_eval = true;
      if (!first) {
        if (S.status != ST_RUNNING) break;
        if (S.iters >= o.max_iters) {
          S.status = ST_FAILED;
          break;
        }
        if (grad_converged(w, S)) {
          S.status = ST_CONVERGED;
          break;
        }
        for (int t = w.lane; t < w.np; t += 32) {
          const int rc = __ldg(w.td->pk + t);
          const double g = w.gn[t];
          w.damped[t] = ((rc & 0xffff) == (rc >> 16)) ? g + S.lambda : g;
        }
        double v[MAXV];
#pragma unroll
        for (int s = 0; s < MAXV; ++s) {
          const int i = w.lane + 32 * s;
          v[s] = i < n ? -w.grad[i] : 0.0;
        }
        __syncwarp();
        bool finite = false;
        if (llt_factor_w(w)) {
          llt_solve_w(w, v);
          bool fin = true;
#pragma unroll
          for (int s = 0; s < MAXV; ++s)
            if (w.lane + 32 * s < n) fin = fin && isfinite(v[s]);
          finite = __all_sync(FULL, fin);
        }
        if (finite) {
#pragma unroll
          for (int s = 0; s < MAXV; ++s) {
            const int i = w.lane + 32 * s;
            if (i < n) w.cand[i] = w.x[i] + v[s];
          }
          __syncwarp();
          q = w.cand;
        } else {
          do_eval = false;
        }
      }
      bool accepted = false;
      if (do_eval) {
        if (!fk_world(w, q)) {
          err = TR_NONFINITE_CFG;
          break;
        }
        const double tv = value_at(w, q);
        bool take = false;
        if (first) {
          if (!isfinite(tv)) {
            err = TR_NONFINITE_INIT;
            break;
          }
          take = true;
        } else {
          take = isfinite(tv) && tv < S.value;
        }
        if (take) {
          const double oldv = S.value;
          if (!first) {
            for (int i = w.lane; i < n; i += 32) w.x[i] = w.cand[i];
            __syncwarp();
          }
          derivatives(w);
          S.value = tv;  // evaluate(x) repeats value(cand) bit for bit
          if (first) {
            S.grad0 = infnorm_warp(w, w.grad);
          } else {
            S.lambda = fmax(S.lambda / o.lm_lambda_factor, 1e-12);
            accepted = true;
            ++S.acc;
            if (oldv - tv <= o.ftol * fmax(1.0, fabs(oldv))) ++S.stag;
            else S.stag = 0;
            if (S.stag >= 2) S.status = ST_CONVERGED;
          }
        }
      }
      if (!first) {
        if (!accepted) {
          S.lambda *= o.lm_lambda_factor;
          if (S.lambda > o.lm_lambda_max) S.status = ST_FAILED;
        }
        if (S.itv && w.lane == 0) S.itv[S.iters] = S.value;
        ++S.iters;
        if (S.status == ST_RUNNING && S.iters >= o.max_iters) S.status = ST_FAILED;
      }
      first = false;
    }
    if (err) {
      if (w.lane == 0) iv(IS_RUN) = err;
      return;
    }
  }

  // ---- finish_step (stepper.cpp:118-147) ----
  const bool converged = S.status == ST_CONVERGED;
  const double gnorm = infnorm_warp(w, w.grad);
  if (w.lane == 0) {
    if (out.iterations) out.iterations[out.rrow(e, step)] = S.iters;
    if (out.converged) out.converged[out.rrow(e, step)] = converged;
    if (out.accepted) out.accepted[out.rrow(e, step)] = S.acc;
    if (out.final_value) out.final_value[out.rrow(e, step)] = S.value;
    if (out.final_grad_norm) out.final_grad_norm[out.rrow(e, step)] = gnorm;
    iv(IS_NREP) = step + 1;
    iv(IS_ITERS) = S.iters;
    iv(IS_STATUS) = S.status;
    iv(IS_ACC) = S.acc;
  }
  const int fs = converged ? 0 : iv(IS_FAIL) + 1;
  __syncwarp();
  if (w.lane == 0) iv(IS_FAIL) = fs;
  if (fs > sc.fail_limit) {
    if (w.lane == 0) iv(IS_RUN) = TR_FAIL_LIMIT;
    return;
  }
  // history shift (order 2): hist0 <- hist1, hist1 <- x
  for (int k = w.lane; k < n; k += 32) {
    const double h1k = ws[(L.hist1 + k) * B + e];  // (h1 scratch was reused by the solver)
    ws[(L.hist0 + k) * B + e] = h1k;
    ws[(L.hist1 + k) * B + e] = w.x[k];
  }
  // energy audit: fd_kinetic(world(hist1_old), world(x)), gravity_potential(world(x))
  fk_world(w, w.x);
  for (int i = w.lane; i < w.N; i += 32) {
    const M4 S_i = ldg16(m.S + 16 * i);
    const M4 wn = ld16(w.world + MS * i);
    const M4 td_ = divs(sub(wn, ld16(w.hw1 + 16 * i)), dt);
    w.red[4 * i] = 0.5 * ddot(mul(td_, S_i), td_);
    const double ghat[4] = {f.gravity[0], f.gravity[1], f.gravity[2], 0.0};
    const double e4[4] = {0.0, 0.0, 0.0, 1.0};
    double u[4], vv[4];
    mul_vec4(S_i, e4, u);
    mul_vec4(wn, u, vv);
    w.red[4 * i + 1] = dot4(ghat, vv);
  }
  __syncwarp();
  if (w.lane == 0) {
    double ke = 0.0, pe = 0.0;
    for (int i = 0; i < w.N; ++i) {
      ke += w.red[4 * i];
      pe -= w.red[4 * i + 1];
    }
    if (out.energy) {
      out.energy[out.qrow(e, step + 1) * 2] = ke;
      out.energy[out.qrow(e, step + 1) * 2 + 1] = pe;
    }
    iv(IS_NSAMP) = step + 2;
    iv(IS_STEP) = step + 1;
    if (step + 1 >= sc.total_steps) iv(IS_RUN) = TR_OK;
  }
  if (out.q) {
    for (int k = w.lane; k < n; k += 32) out.q[out.qrow(e, step + 1) * n + k] = w.x[k];
  }
}

// One PBAD step of environment blockIdx.x (one launch per step).
template <bool POT>
__global__ void __launch_bounds__(32, PBAD_TREE_MINB) k_tree_step(const __grid_constant__ DModel m, const __grid_constant__ DForces f,
                                                  const __grid_constant__ DSchedule sc, const __grid_constant__ Layout L,
                                                  double* ws, int* iws, long B, const __grid_constant__ TreeDesc td,
                                                  double* tws, const __grid_constant__ Outputs out) {
  extern __shared__ __align__(16) double smem[];
  const long e = blockIdx.x;
  if (e >= B) return;
  tree_env_step<POT>(m, f, sc, L, ws, iws, B, td, tws, out, e, smem);
}

// nsteps PBAD steps of every environment in one persistent launch.  Warps
// claim env-steps t = s B + e in order from a counter; an env-step waits (in
// practice never: its predecessor was claimed B tasks earlier) until its
// environment's previous step is done, so an environment starts its next
// step as soon as its current one ends and the per-step tail -- the last
// resident warps of a step running while the SMs drain -- is paid once per
// launch instead of once per step.  The predecessor is always held by a
// running warp, so the wait cannot deadlock.  Every env-step runs the same
// code as k_tree_step, so results are bit-identical.
#ifndef PBAD_TREE_STEP_CALL
#define PBAD_TREE_STEP_CALL 0  // 1: the persistent kernel calls the env-step body out of line
#endif
template <bool POT>
__device__ __noinline__ void tree_env_step_call(const DModel& m, const DForces& f, const DSchedule& sc, const Layout& L,
                                                double* ws, int* iws, long B, const TreeDesc& td, double* tws,
                                                const Outputs& out, long e, double* smem) {
  tree_env_step<POT>(m, f, sc, L, ws, iws, B, td, tws, out, e, smem);
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <bool POT>
__global__ void __launch_bounds__(32, PBAD_TREE_MINB) k_tree_steps(const __grid_constant__ DModel m, const __grid_constant__ DForces f,
                                                   const __grid_constant__ DSchedule sc, const __grid_constant__ Layout L,
                                                   double* ws, int* iws, long B, const __grid_constant__ TreeDesc td,
                                                   double* tws, const __grid_constant__ Outputs out, int nsteps,
                                                   unsigned long long* counter, int* done, int chunk) {
  extern __shared__ __align__(16) double smem[];
  // a task is `chunk` consecutive steps of one environment (one acquire per task)
  const int nchunks = (nsteps + chunk - 1) / chunk;
  const unsigned long long total = (unsigned long long)nchunks * (unsigned long long)B;
  for (;;) {
    unsigned long long t = 0;
    if (threadIdx.x == 0) t = atomicAdd(counter, 1ull);
    t = __shfl_sync(FULL, t, 0);
    if (t >= total) break;
    const long s = (long)(t / (unsigned long long)B), e = (long)(t - (unsigned long long)s * B);
    // lane 0's acquire (which also drops this SM's L1 lines) then the warp
    // barrier order the other lanes' reads of the environment's state after
    // the release below of the SM that ran its previous step
    if (s > 0 && threadIdx.x == 0)
      while (ld_acquire_gpu(done + e) < s) __nanosleep(100);
    __syncwarp();
#pragma unroll 1
    for (int k = 0; k < chunk && s * chunk + k < nsteps; ++k) {
      if (k) __syncwarp();
#if PBAD_TREE_STEP_CALL
      tree_env_step_call<POT>(m, f, sc, L, ws, iws, B, td, tws, out, e, smem);
#else
      tree_env_step<POT>(m, f, sc, L, ws, iws, B, td, tws, out, e, smem);
#endif
    }
    __syncwarp();  // every lane's stores of this env-step before lane 0's release
    if (threadIdx.x == 0) st_release_gpu(done + e, (int)s + 1);
  }
}

#else
template <bool POT>
__global__ void __launch_bounds__(32) k_tree_lbfgs(const __grid_constant__ DModel m, const __grid_constant__ DForces f,
                                                  const __grid_constant__ DSchedule sc, const __grid_constant__ Layout L,
                                                  double* ws, int* iws, long B, const __grid_constant__ TreeDesc td,
                                                  double* tws, const __grid_constant__ Outputs out) {
  extern __shared__ __align__(16) double smem[];
  const long e = blockIdx.x;
  if (e >= B) return;
  if (iws[(long)IS_RUN * B + e] != TR_RUNNING) return;
  W w;
  w.m = &m;
  w.f = &f;
  w.sc = &sc;
  w.td = &td;
  w.lane = threadIdx.x;
  w.N = td.N;
  w.n = td.n;
  w.D = td.D;
  w.np = td.np;
  w.grav = f.gravity_nonzero != 0;
  const double dt = sc.dt;
  w.inv_dt2 = 1.0 / (dt * dt);
  // POT = false compiles the drag / contact code out (lean fast path)
  w.drag = POT && f.drag_d > 0.0;
  w.scl = w.drag ? f.drag_d / (dt * dt) : 0.0;
  w.contact = POT && f.has_contact && (f.d1 > 0.0 || f.d2 > 0.0) && td.ns > 0;
  {
    const int N16 = MS * td.N, nv = (td.n + 1) & ~1;
    const int scr = (TREE_SCR_ARRAYS * N16 > MS * td.n) ? TREE_SCR_ARRAYS * N16 : MS * td.n;
    double* p = smem;
    w.value = p; p += N16;
    w.world = p; p += N16;
    // the damped matrix is live only from its rebuild to the end of the
    // solve, the levers and the link scratch only inside the derivatives
    // (fk_levers, gradient, GN assembly): one region serves both
    w.lever = p;
    w.scr = p + MS * td.n;
    w.damped = p;
    p += (MS * td.n + scr) > ((td.np + 1) & ~1) ? (MS * td.n + scr) : ((td.np + 1) & ~1);
    w.x = p; p += nv;
    w.grad = p; p += nv;
    w.cand = p; p += nv;
    w.vtau = p; p += nv;
    w.vtmp = p; p += nv;
    w.q2 = p; p += nv;
    w.dir = p; p += nv;
    w.evg = p; p += nv;
    w.red = p; p += 5 * td.N + 32;
    w.ctv = p; p += (td.ns + 1) & ~1;
    w.cdep = p; p += 4 * td.ns;
    w.cact = reinterpret_cast<int*>(p);
    w.clist = w.cact + ((td.ns + 1) & ~1);
    double* g = tws + e * td.gstride;
    w.gn = g;
    w.hw0 = g + td.o_hw0;
    w.hw1 = g + td.o_hw1;
    w.T0 = g + td.o_t0;
    w.T1 = g + td.o_t1;
    w.gs = g + td.o_gs;
    w.abl = g + td.o_abl;
    w.abu = g + td.o_abu;
    w.cs = g + td.o_cs;
  }
  const int n = td.n;
  int* const ivp = iws + e;
  auto iv = [&](int slot) -> int& { return ivp[(long)slot * B]; };
  const int step = iv(IS_STEP);

  // ---- begin_step (stepper.cpp:83-115) ----
  double* h0 = w.cand;
  double* h1 = w.vtmp;
  for (int k = w.lane; k < n; k += 32) {
    h0[k] = ws[(L.hist0 + k) * B + e];
    h1[k] = ws[(L.hist1 + k) * B + e];
  }
  const double t0 = step * dt;
  tau_at(w, t0 + sc.times[2] * dt, w.vtau);
  {
    const double span = -sc.times[0];
    const double tau_m = sc.times[2];
    for (int k = w.lane; k < n; k += 32) w.x[k] = sc.warm_start ? h1[k] + (tau_m / span) * (h1[k] - h0[k]) : h1[k];
  }
  __syncwarp();
  // StepObjective ctor (objective.cpp:162-185)
  if (!all_finite_warp(w, h0) || !all_finite_warp(w, h1)) {
    if (w.lane == 0) iv(IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
#pragma unroll 1
  for (int hs = 0; hs < 2; ++hs) {  // one inlined copy of the kinematics for both history configurations
    fk_world(w, hs ? h1 : h0);
    store_history(w, hs ? w.hw1 : w.hw0, hs ? w.T1 : w.T0);
  }
  {
    for (int i = w.lane; i < w.N; i += 32) {
      const M4 w0 = ld16(w.hw0 + 16 * i), w1 = ld16(w.hw1 + 16 * i);
      const M4 T1 = ld16(w.T1 + 16 * i);
      w.red[4 * i] = ddot(T1, w1);
      w.red[4 * i + 1] = ddot(ld16(w.T0 + 16 * i), w0);
      w.red[4 * i + 2] = ddot(T1, w0);
    }
    __syncwarp();
    double s = 0.0;
    if (w.lane < 3)
      for (int i = 0; i < w.N; ++i) s += w.red[4 * i + w.lane];
    const double c11 = __shfl_sync(FULL, s, 0) - m.weighted_mass;
    const double c00 = __shfl_sync(FULL, s, 1) - m.weighted_mass;
    const double c10 = __shfl_sync(FULL, s, 2) - m.weighted_mass;
    w.histconst = 4.0 * c11 + c00 - 4.0 * c10;
    __syncwarp();
  }
  // LbfgsSolver (optim.cpp:141-232): construction evaluates value + gradient,
  // every iterate runs the two-loop recursion and the Armijo backtracking
  Solver S;
  S.status = ST_RUNNING;
  S.itv = out.itv ? out.itv + out.rrow(e, step) * out.itv_n : nullptr;
  S.iters = 0;
  S.stag = 0;
  S.acc = 0;
  S.lambda = 0.0;
  S.value = 0.0;
  S.grad0 = 0.0;
  {
    // LbfgsSolver (optim.cpp:141-232): construction evaluates value + gradient,
    // every iterate runs the two-loop recursion and the Armijo backtracking
    const DOpt& o = sc.opt;
    const int cap = o.mem + 1;
    double* gtw = tws + e * td.gstride;
    double* hs = gtw + td.o_hs;
    double* hy = gtw + td.o_hy;
    double* hsy = gtw + td.o_hsy;
    double* alpha = gtw + td.o_alpha;
    int err = 0;
    if (!fk_world(w, w.x)) {
      err = TR_NONFINITE_CFG;
    } else {
      const double v0 = value_at(w, w.x);
      if (!isfinite(v0)) {
        err = TR_NONFINITE_INIT;
      } else {
        S.value = v0;
        fk_levers(w, w.x);
        gradient(w, w.grad);
        S.grad0 = infnorm_warp(w, w.grad);
      }
    }
    int h0 = 0, hc = 0;
#pragma unroll 1
    while (!err) {
      if (S.status != ST_RUNNING) break;
      if (S.iters >= o.max_iters) {
        S.status = ST_FAILED;
        break;
      }
      if (grad_converged(w, S)) {
        S.status = ST_CONVERGED;
        break;
      }
      // two_loop (optim.cpp:213-229): q = H g
      for (int k = w.lane; k < n; k += 32) w.q2[k] = w.grad[k];
      __syncwarp();
      for (int i = hc - 1; i >= 0; --i) {
        const int slot = (h0 + i) % cap;
        const double* si = hs + (long)slot * n;
        const double* yi = hy + (long)slot * n;
        const double a = vdot_warp(w, si, w.q2) / hsy[slot];
        if (w.lane == 0) alpha[i] = a;
        for (int k = w.lane; k < n; k += 32) w.q2[k] = w.q2[k] - a * yi[k];
        __syncwarp();
      }
      if (hc > 0) {
        const int slot = (h0 + hc - 1) % cap;
        const double* yl = hy + (long)slot * n;
        const double scl = hsy[slot] / vdot_warp(w, yl, yl);
        for (int k = w.lane; k < n; k += 32) w.q2[k] = w.q2[k] * scl;
        __syncwarp();
      }
      for (int i = 0; i < hc; ++i) {
        const int slot = (h0 + i) % cap;
        const double* si = hs + (long)slot * n;
        const double* yi = hy + (long)slot * n;
        const double beta = vdot_warp(w, yi, w.q2) / hsy[slot];
        const double c = alpha[i] - beta;
        for (int k = w.lane; k < n; k += 32) w.q2[k] = w.q2[k] + c * si[k];
        __syncwarp();
      }
      for (int k = w.lane; k < n; k += 32) w.dir[k] = -w.q2[k];
      __syncwarp();
      double slope = vdot_warp(w, w.dir, w.grad);
      if (!(slope < 0.0)) {
        hc = 0;
        h0 = 0;
        for (int k = w.lane; k < n; k += 32) w.dir[k] = -w.grad[k];
        __syncwarp();
        slope = vdot_warp(w, w.dir, w.grad);
      }
      // Armijo backtracking (optim.cpp:171-205)
      double t = 1.0;
      bool accepted = false;
      const double fval = S.value;
      for (int trial = 0; trial < o.max_line_search; ++trial) {
        for (int k = w.lane; k < n; k += 32) w.cand[k] = w.x[k] + t * w.dir[k];
        __syncwarp();
        if (all_finite_warp(w, w.cand)) {
          if (!fk_world(w, w.cand)) {
            err = TR_NONFINITE_CFG;
            break;
          }
          const double v = value_at(w, w.cand);
          if (isfinite(v) && v <= fval + o.armijo_c1 * t * slope && v < fval) {
            fk_levers(w, w.cand);
            gradient(w, w.evg);  // evaluate(cand): the value repeats v bit for bit
            const int slot = (h0 + hc) % cap;
            double* sn = hs + (long)slot * n;
            double* yn = hy + (long)slot * n;
            for (int k = w.lane; k < n; k += 32) {
              sn[k] = t * w.dir[k];
              yn[k] = w.evg[k] - w.grad[k];
            }
            __syncwarp();
            const double sy = vdot_warp(w, sn, yn);
            if (sy > 1e-12) {
              if (w.lane == 0) hsy[slot] = sy;
              ++hc;
              if (hc > o.mem) {
                h0 = (h0 + 1) % cap;
                --hc;
              }
            }
            for (int k = w.lane; k < n; k += 32) {
              w.x[k] = w.cand[k];
              w.grad[k] = w.evg[k];
            }
            __syncwarp();
            S.value = v;
            accepted = true;
            ++S.acc;
            if (fval - v <= o.ftol * fmax(1.0, fabs(fval))) ++S.stag;
            else S.stag = 0;
            if (S.stag >= 2) S.status = ST_CONVERGED;
            break;
          }
        }
        t *= o.backtrack_factor;
      }
      if (err) break;
      if (!accepted) S.status = ST_FAILED;
      if (S.itv && w.lane == 0) S.itv[S.iters] = S.value;
      ++S.iters;
      if (S.status == ST_RUNNING && S.iters >= o.max_iters) S.status = ST_FAILED;
    }
    if (err) {
      if (w.lane == 0) iv(IS_RUN) = err;
      return;
    }
  }

  // ---- finish_step (stepper.cpp:118-147) ----
  const bool converged = S.status == ST_CONVERGED;
  const double gnorm = infnorm_warp(w, w.grad);
  if (w.lane == 0) {
    if (out.iterations) out.iterations[out.rrow(e, step)] = S.iters;
    if (out.converged) out.converged[out.rrow(e, step)] = converged;
    if (out.accepted) out.accepted[out.rrow(e, step)] = S.acc;
    if (out.final_value) out.final_value[out.rrow(e, step)] = S.value;
    if (out.final_grad_norm) out.final_grad_norm[out.rrow(e, step)] = gnorm;
    iv(IS_NREP) = step + 1;
    iv(IS_ITERS) = S.iters;
    iv(IS_STATUS) = S.status;
    iv(IS_ACC) = S.acc;
  }
  const int fs = converged ? 0 : iv(IS_FAIL) + 1;
  __syncwarp();
  if (w.lane == 0) iv(IS_FAIL) = fs;
  if (fs > sc.fail_limit) {
    if (w.lane == 0) iv(IS_RUN) = TR_FAIL_LIMIT;
    return;
  }
  // history shift (order 2): hist0 <- hist1, hist1 <- x
  for (int k = w.lane; k < n; k += 32) {
    const double h1k = ws[(L.hist1 + k) * B + e];  // (h1 scratch was reused by the solver)
    ws[(L.hist0 + k) * B + e] = h1k;
    ws[(L.hist1 + k) * B + e] = w.x[k];
  }
  // energy audit: fd_kinetic(world(hist1_old), world(x)), gravity_potential(world(x))
  fk_world(w, w.x);
  for (int i = w.lane; i < w.N; i += 32) {
    const M4 S_i = ldg16(m.S + 16 * i);
    const M4 wn = ld16(w.world + MS * i);
    const M4 td_ = divs(sub(wn, ld16(w.hw1 + 16 * i)), dt);
    w.red[4 * i] = 0.5 * ddot(mul(td_, S_i), td_);
    const double ghat[4] = {f.gravity[0], f.gravity[1], f.gravity[2], 0.0};
    const double e4[4] = {0.0, 0.0, 0.0, 1.0};
    double u[4], vv[4];
    mul_vec4(S_i, e4, u);
    mul_vec4(wn, u, vv);
    w.red[4 * i + 1] = dot4(ghat, vv);
  }
  __syncwarp();
  if (w.lane == 0) {
    double ke = 0.0, pe = 0.0;
    for (int i = 0; i < w.N; ++i) {
      ke += w.red[4 * i];
      pe -= w.red[4 * i + 1];
    }
    if (out.energy) {
      out.energy[out.qrow(e, step + 1) * 2] = ke;
      out.energy[out.qrow(e, step + 1) * 2 + 1] = pe;
    }
    iv(IS_NSAMP) = step + 2;
    iv(IS_STEP) = step + 1;
    if (step + 1 >= sc.total_steps) iv(IS_RUN) = TR_OK;
  }
  if (out.q) {
    for (int k = w.lane; k < n; k += 32) out.q[out.qrow(e, step + 1) * n + k] = w.x[k];
  }
}
#endif

}  // namespace PBAD_TREE_NS

#ifndef PBAD_TREE_LBFGS_TU
bool tree_eligible_sizes(int N, int n) { return N >= 1 && N <= 255 && n >= 1 && n <= tree::MAXN; }

static int tree_smem_doubles(const TreeDesc& td) {
  const int N16 = tree::MS * td.N, nv = (td.n + 1) & ~1;
  const int scr = (tree::TREE_SCR_ARRAYS * N16 > tree::MS * td.n) ? tree::TREE_SCR_ARRAYS * N16 : tree::MS * td.n;
  const int np2 = (td.np + 1) & ~1, ls = tree::MS * td.n + scr, rd = 5 * td.N + 32;
  // one region for the damped matrix, the levers + link scratch and (LM) the
  // value terms; dof vectors x, grad, cand, vtau, vtmp (+ q2, dir, evg for L-BFGS)
  int region = ls > np2 ? ls : np2;
  if (!td.lb && rd > region) region = rd;
  return 2 * N16 + region + (td.lb ? 8 * nv + rd : 5 * nv) + ((td.ns + 1) & ~1) +
         4 * td.ns + td.ns + 2;  // cact + clist ints
}

size_t tree_smem_bytes(const TreeDesc& td) { return sizeof(double) * (size_t)tree_smem_doubles(td); }

cudaError_t launch_tree_step(const KernelArgs& a, const TreeDesc& td, double* tws, const Outputs& out,
                             cudaStream_t s) {
  const size_t smem = tree_smem_bytes(td);
  if (td.lb) return launch_tree_lbfgs(a, td, tws, out, s);
  static SmemAttr attr_[2];
  const int pot = td.pot ? 1 : 0;
  if (smem > 48 * 1024 && smem > attr_[pot].here()) {
    cudaError_t e = pot ? cudaFuncSetAttribute(tree::k_tree_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                        : cudaFuncSetAttribute(tree::k_tree_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_[pot].here() = smem;
  }
  if (pot) tree::k_tree_step<true><<<(unsigned)a.B, 32, smem, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, td, tws, out);
  else tree::k_tree_step<false><<<(unsigned)a.B, 32, smem, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, td, tws, out);
  return cudaGetLastError();
}

// Persistent launches pay where an env-step's LM iteration count varies a
// lot across the batch (ground contact: 6 to 512 iterations, C4b 120 -> 113
// ms/step); for smooth scenes the per-step launches are faster (C4 3.46 vs
// 3.62 ms/step: the acquire's L1 invalidation per env-step costs more than
// the short per-step tail).  PBAD_TREE_PERSIST: 0 never, 1 (default)
// contact scenes, 2 always.
static bool tree_persistent(const TreeDesc& td, int nsteps) {
  static const int mode = std::getenv("PBAD_TREE_PERSIST") ? std::atoi(std::getenv("PBAD_TREE_PERSIST")) : 1;
  if (td.lb || nsteps <= 1 || mode == 0) return false;
  return mode == 2 || (td.pot && td.ns > 0);
}

// nsteps steps: one persistent launch (k_tree_steps) where tree_persistent(),
// else one k_tree_step launch per step.  sync: 2 + B ints of device memory.
// *launches: kernels launched.
cudaError_t launch_tree_steps(const KernelArgs& a, const TreeDesc& td, double* tws, const Outputs& out, int nsteps,
                              int* sync, cudaStream_t s, long* launches) {
  if (!tree_persistent(td, nsteps) || !sync) {
    *launches += nsteps;
    for (int k = 0; k < nsteps; ++k) {
      const cudaError_t e = launch_tree_step(a, td, tws, out, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const size_t smem = tree_smem_bytes(td);
  const int pot = td.pot ? 1 : 0;
  static SmemAttr attr_[2];
  static int slots[2] = {0, 0};
  if (smem > attr_[pot].here() || !slots[pot]) {
    if (smem > 48 * 1024) {
      cudaError_t e = pot ? cudaFuncSetAttribute(tree::k_tree_steps<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                          : cudaFuncSetAttribute(tree::k_tree_steps<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    attr_[pot].here() = smem;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = pot ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tree::k_tree_steps<true>, 32, smem)
                        : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tree::k_tree_steps<false>, 32, smem);
    if (e != cudaSuccess) return e;
    slots[pot] = per > 0 ? per * (sms > 0 ? sms : 148) : -1;  // -1: does not fit
  }
  if (slots[pot] < 0) {
    for (int k = 0; k < nsteps; ++k) {
      const cudaError_t e = launch_tree_step(a, td, tws, out, s);
      if (e != cudaSuccess) return e;
    }
    *launches += nsteps;
    return cudaSuccess;
  }
  cudaError_t e = cudaMemsetAsync(sync, 0, sizeof(int) * (size_t)(2 + a.B), s);
  if (e != cudaSuccess) return e;
  *launches += 1;
  // steps per task (one acquire per task): C4b 112.5 (1) -> 103.5 (4) ms/step in one
  // run; 97.7 (4), 96.3 (8), 95.0 (16) in another
  static const int chunk = std::getenv("PBAD_TREE_CHUNK") ? std::max(1, std::atoi(std::getenv("PBAD_TREE_CHUNK"))) : 16;
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(sync);
  int* done = sync + 2;
  const unsigned grid = (unsigned)std::min<long>(a.B, slots[pot]);
  if (pot)
    tree::k_tree_steps<true><<<grid, 32, smem, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, td, tws, out, nsteps, counter, done,
                                                     chunk);
  else
    tree::k_tree_steps<false><<<grid, 32, smem, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, td, tws, out, nsteps, counter,
                                                      done, chunk);
  return cudaGetLastError();
}

}  // namespace pbad_gpu

#else  // PBAD_TREE_LBFGS_TU

cudaError_t launch_tree_lbfgs(const KernelArgs& a, const TreeDesc& td, double* tws, const Outputs& out,
                              cudaStream_t s) {
  const size_t smem = tree_smem_bytes(td);
  static SmemAttr attr_[2];
  const int pot = td.pot ? 1 : 0;
  if (smem > 48 * 1024 && smem > attr_[pot].here()) {
    cudaError_t e = pot ? cudaFuncSetAttribute(PBAD_TREE_NS::k_tree_lbfgs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                        : cudaFuncSetAttribute(PBAD_TREE_NS::k_tree_lbfgs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_[pot].here() = smem;
  }
  if (pot) PBAD_TREE_NS::k_tree_lbfgs<true><<<(unsigned)a.B, 32, smem, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, td, tws, out);
  else PBAD_TREE_NS::k_tree_lbfgs<false><<<(unsigned)a.B, 32, smem, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, td, tws, out);
  return cudaGetLastError();
}
}  // namespace pbad_gpu
#endif
