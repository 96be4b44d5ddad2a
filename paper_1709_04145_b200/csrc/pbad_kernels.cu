// pbad_kernels.cu -- sm_100a kernels of the PBAD hot path (general path).
//
// One thread = one trajectory.  Each function below restates the reference
// routine named in its comment with the same floating-point operation
// sequence (numeric contract in pbad_math.cuh), so results are bit-identical
// to the reference / oracle.  Structural zeros of the 4x4 affine matrices are
// kept here (this is the general kernel for trees, ball/free joints, drag,
// contact, residual form and LM); the specialised chain kernel in
// pbad_chain.cu drops them.
#include <cuda_runtime.h>

#include "pbad_kernels.cuh"
#include "pbad_math.cuh"
#include "pbad_joint.cuh"

namespace pbad_gpu {

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_FAILED = 2 };
enum { TR_OK = 0, TR_FAIL_LIMIT = 1, TR_NONFINITE_INIT = 2, TR_NONFINITE_CFG = 3, TR_RUNNING = 4 };

struct Arr {
  double* p;
  long s;
  __device__ __forceinline__ double& operator[](long k) const { return p[k * s]; }
};

struct Env {
  const DModel* m;
  const DForces* f;
  const DSchedule* sc;
  const Layout* L;
  double* ws;
  int* iws;
  long B;
  int e;
  double* itv = nullptr;  // this step's per_iteration_values row, or null
  __device__ __forceinline__ Arr arr(long off) const { return Arr{ws + off * B + e, B}; }
  __device__ __forceinline__ int& iv(int slot) const { return iws[(long)slot * B + e]; }
  __device__ __forceinline__ double& sv(int slot) const { return ws[(L->scal + slot) * B + e]; }
};

__device__ __forceinline__ M4 ldm(const Arr& a, long idx) {
  M4 m;
#pragma unroll
  for (int k = 0; k < 16; ++k) m.a[k] = a[idx * 16 + k];
  return m;
}
__device__ __forceinline__ void stm(const Arr& a, long idx, const M4& m) {
#pragma unroll
  for (int k = 0; k < 16; ++k) a[idx * 16 + k] = m.a[k];
}
__device__ __forceinline__ M4 ldg4(const double* p) {
  M4 m;
#pragma unroll
  for (int k = 0; k < 16; ++k) m.a[k] = __ldg(p + k);
  return m;
}

struct Pass {
  Arr value, d1, d2, world, lever;
};
__device__ __forceinline__ Pass pass_at(const Env& E, int idx) {
  const long base = E.L->pass + idx * E.L->pass_stride;
  return Pass{E.arr(base + E.L->p_value), E.arr(base + E.L->p_d1), E.arr(base + E.L->p_d2),
              E.arr(base + E.L->p_world), E.arr(base + E.L->p_lever)};
}

__device__ __forceinline__ bool all_finite(const Arr& a, int n) {
  for (int k = 0; k < n; ++k)
    if (!isfinite(a[k])) return false;
  return true;
}

// forward_pass (kinematics.cpp:171-181) into world (validation by caller)
__device__ void forward_pass(const Env& E, const Arr& q, const Arr& world) {
  const DModel& m = *E.m;
  for (int i = 0; i < m.N; ++i) {
    double ql[6];
    const int off = m.dof_off[i];
    for (int j = 0; j < m.dof_cnt[i]; ++j) ql[j] = q[off + j];
    const M4 local = joint_transform(m.kind[i], m.axis + 3 * i, ldg4(m.offset + 16 * i), ql);
    const int p = m.parent[i];
    stm(world, i, (p >= 0) ? mul(ldm(world, p), local) : local);
  }
}

// ConfigPass::make (adjoint.cpp:9-27); returns false for a non-finite q
__device__ bool pass_make(const Env& E, const Arr& q, const Pass& P, bool want_d2, bool check_finite = true) {
  const DModel& m = *E.m;
  if (check_finite && !all_finite(q, m.n)) return false;
  for (int i = 0; i < m.N; ++i) {
    double ql[6];
    const int off = m.dof_off[i];
    const int dof = m.dof_cnt[i];
    for (int j = 0; j < dof; ++j) ql[j] = q[off + j];
    M4 value, d1[6], d2[21];
    joint_jet(m.kind[i], m.axis + 3 * i, ldg4(m.offset + 16 * i), ql, &value, d1, d2, want_d2);
    stm(P.value, i, value);
    const int p = m.parent[i];
    const M4 pw = (p >= 0) ? ldm(P.world, p) : m4_identity();
    stm(P.world, i, mul(pw, value));
    for (int j = 0; j < dof; ++j) {
      stm(P.d1, off + j, d1[j]);
      stm(P.lever, off + j, mul(pw, d1[j]));
    }
    if (want_d2)
      for (int j = 0; j < dof * (dof + 1) / 2; ++j) stm(P.d2, m.d2_off[i] + j, d2[j]);
  }
  return true;
}

__device__ __forceinline__ M4 pworld(const Env& E, const Pass& P, int i) {
  const int p = E.m->parent[i];
  return (p >= 0) ? ldm(P.world, p) : m4_identity();
}

// correlation_value (adjoint.cpp:113-120) with pass_a given by world array
__device__ double correlation_value(const Env& E, const Arr& wa, const Arr& wb) {
  const DModel& m = *E.m;
  double v = 0.0;
  for (int i = 0; i < m.N; ++i) {
    const M4 ts = mul(ldm(wa, i), ldg4(m.S + 16 * i));
    v += ddot(ts, ldm(wb, i));
  }
  return v - m.weighted_mass;
}

// functional_grad (adjoint.cpp:49-64)
__device__ void functional_grad(const Env& E, const Arr& seeds, const Pass& P, const Arr& grad) {
  const DModel& m = *E.m;
  const Arr adj = E.arr(E.L->adj);
  for (int k = 0; k < m.n; ++k) grad[k] = 0.0;
  for (int k = 0; k < m.N * 16; ++k) adj[k] = 0.0;
  for (int i = m.N - 1; i >= 0; --i) {
    M4 a = add(ldm(adj, i), ldm(seeds, i));
    const int off = m.dof_off[i];
    for (int j = 0; j < m.dof_cnt[i]; ++j) grad[off + j] = grad[off + j] + ddot(ldm(P.lever, off + j), a);
    const int p = m.parent[i];
    if (p >= 0) stm(adj, p, add(ldm(adj, p), mul_bt(a, ldm(P.value, i))));
  }
}

// functional_hess (adjoint.cpp:66-101); hess column-major n x n
__device__ void functional_hess(const Env& E, const Arr& seeds, const Pass& P, const Arr& hess) {
  const DModel& m = *E.m;
  const int n = m.n;
  const Arr adj = E.arr(E.L->adj);
  for (long k = 0; k < (long)n * n; ++k) hess[k] = 0.0;
  for (int k = 0; k < m.N * 16; ++k) adj[k] = 0.0;
  for (int i = m.N - 1; i >= 0; --i) {
    const M4 a = add(ldm(adj, i), ldm(seeds, i));
    stm(adj, i, a);
    const int off = m.dof_off[i];
    const int dof = m.dof_cnt[i];
    const M4 pw = pworld(E, P, i);
    for (int l = 0; l < dof; ++l)
      for (int j = 0; j <= l; ++j) {
        const M4 pd = mul(pw, ldm(P.d2, m.d2_off[i] + l * (l + 1) / 2 + j));
        const double h = ddot(pd, a);
        hess[(off + j) + (long)n * (off + l)] = hess[(off + j) + (long)n * (off + l)] + h;
        if (j != l) hess[(off + l) + (long)n * (off + j)] = hess[(off + l) + (long)n * (off + j)] + h;
      }
    M4 walk[6];
    for (int j = 0; j < dof; ++j) walk[j] = mul_bt(a, ldm(P.d1, off + j));
    for (int l = m.parent[i]; l >= 0; l = m.parent[l]) {
      const int offl = m.dof_off[l];
      for (int k = 0; k < m.dof_cnt[l]; ++k) {
        const M4 lev = ldm(P.lever, offl + k);
        for (int j = 0; j < dof; ++j) {
          const double h = ddot(lev, walk[j]);
          hess[(offl + k) + (long)n * (off + j)] = hess[(offl + k) + (long)n * (off + j)] + h;
          hess[(off + j) + (long)n * (offl + k)] = hess[(off + j) + (long)n * (offl + k)] + h;
        }
      }
      const M4 vl = ldm(P.value, l);
      for (int j = 0; j < dof; ++j) walk[j] = mul_bt(walk[j], vl);
    }
    const int p = m.parent[i];
    if (p >= 0) stm(adj, p, add(ldm(adj, p), mul_bt(a, ldm(P.value, i))));
  }
}

// correlation_hess_ab (adjoint.cpp:132-176); uses E.adj as the acc array
__device__ void correlation_hess_ab(const Env& E, const Pass& pa, const Pass& pb, const Arr& hess) {
  const DModel& m = *E.m;
  const int n = m.n;
  const Arr acc = E.arr(E.L->adj);
  for (long k = 0; k < (long)n * n; ++k) hess[k] = 0.0;
  for (int k = 0; k < m.N * 16; ++k) acc[k] = 0.0;
  for (int i = m.N - 1; i >= 0; --i) {
    const M4 ai = add(ldm(acc, i), ldg4(m.S + 16 * i));
    stm(acc, i, ai);
    const int off = m.dof_off[i];
    const int dof = m.dof_cnt[i];
    for (int j = 0; j < dof; ++j) {
      const M4 ua = ldm(pa.lever, off + j);
      for (int k = 0; k < dof; ++k) {
        const double t = trace(mul(mul_at(ua, ldm(pb.lever, off + k)), ai));
        hess[(off + j) + (long)n * (off + k)] = hess[(off + j) + (long)n * (off + k)] + t;
      }
    }
    M4 fwd = mul(ldm(pb.value, i), ai);
    M4 bwd = mul_bt(ai, ldm(pa.value, i));
    for (int l = m.parent[i]; l >= 0; l = m.parent[l]) {
      const int offl = m.dof_off[l];
      for (int j = 0; j < dof; ++j) {
        const M4 ua = ldm(pa.lever, off + j);
        const M4 vb = ldm(pb.lever, off + j);
        for (int k = 0; k < m.dof_cnt[l]; ++k) {
          const double t1 = trace(mul(mul_at(ua, ldm(pb.lever, offl + k)), fwd));
          hess[(off + j) + (long)n * (offl + k)] = hess[(off + j) + (long)n * (offl + k)] + t1;
          const double t2 = trace(mul(mul(transpose(ldm(pa.lever, offl + k)), vb), bwd));
          hess[(offl + k) + (long)n * (off + j)] = hess[(offl + k) + (long)n * (off + j)] + t2;
        }
      }
      fwd = mul(ldm(pb.value, l), fwd);
      bwd = mul_bt(bwd, ldm(pa.value, l));
    }
    const int p = m.parent[i];
    if (p >= 0) stm(acc, p, add(ldm(acc, p), mul_bt(mul(ldm(pb.value, i), ai), ldm(pa.value, i))));
  }
}

// ---------------------------------------------------------------------------
// potentials (objective.cpp:25-138)
// ---------------------------------------------------------------------------
struct PotOut {
  double value;
};

__device__ void potential_terms(const Env& E, const Pass& pn, const Arr& world_prev, double dt,
                                bool want_grad, bool want_gn, bool want_hess, const Arr* ab_next,
                                PotOut* out) {
  const DModel& m = *E.m;
  const DForces& f = *E.f;
  const int N = m.N, n = m.n;
  const Layout& L = *E.L;
  const Arr grad = E.arr(L.potgrad);
  const Arr gn = E.arr(L.potgn);
  const Arr hess = E.arr(L.pothess);
  const Arr cot = E.arr(L.cot);
  out->value = 0.0;
  for (int k = 0; k < n; ++k) grad[k] = 0.0;
  if (want_gn)
    for (long k = 0; k < (long)n * n; ++k) gn[k] = 0.0;
  if (want_hess)
    for (long k = 0; k < (long)n * n; ++k) hess[k] = 0.0;
  const bool needs_ab = (want_gn || want_hess) && f.drag_d > 0.0;
  Arr ab = E.arr(L.ab);
  if (needs_ab) {
    if (ab_next) ab = *ab_next;
    else correlation_hess_ab(E, pn, pn, ab);
  }
  for (int k = 0; k < N * 16; ++k) cot[k] = 0.0;
  bool have_cot = false;

  if (f.gravity_nonzero) {
    const double ghat[4] = {f.gravity[0], f.gravity[1], f.gravity[2], 0.0};
    const double e4[4] = {0.0, 0.0, 0.0, 1.0};
    for (int i = 0; i < N; ++i) {
      double u[4];
      mul_vec4(ldg4(m.S + 16 * i), e4, u);
      M4 c;
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int r = 0; r < 4; ++r) c.a[r + 4 * s] = (-ghat[r]) * u[s];
      out->value += ddot(c, ldm(pn.world, i));
      stm(cot, i, add(ldm(cot, i), c));
    }
    have_cot = true;
  }
  if (f.drag_d > 0.0) {
    const double scl = f.drag_d / (dt * dt);
    for (int i = 0; i < N; ++i) {
      const M4 diff = sub(ldm(pn.world, i), ldm(world_prev, i));
      const M4 diff_s = mul(diff, ldg4(m.S + 16 * i));
      out->value += scl * ddot(diff_s, diff);
      stm(cot, i, add(ldm(cot, i), scale(2.0 * scl, diff_s)));
    }
    have_cot = true;
    const double s2 = 2.0 * scl;
    if (want_gn)
      for (long k = 0; k < (long)n * n; ++k) gn[k] = gn[k] + s2 * ab[k];
    if (want_hess)
      for (long k = 0; k < (long)n * n; ++k) hess[k] = hess[k] + s2 * ab[k];
  }
  if (f.has_contact && (f.d1 > 0.0 || f.d2 > 0.0)) {
    const double* nrm = f.normal;
    const double d1c = f.d1, d2c = f.d2;
    double proj[9];
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) proj[r + 3 * c] = ((r == c) ? 1.0 : 0.0) - nrm[r] * nrm[c];
    const bool need_jx = want_gn || want_hess;
    const Arr jx = E.arr(L.jx), dd = E.arr(L.dd), jr = E.arr(L.jr), tmp = E.arr(L.tmp3);
    for (int i = 0; i < N; ++i) {
      const M4 wi = ldm(pn.world, i);
      for (int sidx = m.sample_off[i]; sidx < m.sample_off[i + 1]; ++sidx) {
        const double ph[4] = {m.samples[3 * sidx], m.samples[3 * sidx + 1], m.samples[3 * sidx + 2], 1.0};
        double x4[4], xp4[4];
        mul_vec4(wi, ph, x4);
        const double depth = f.plane_offset - dot3(nrm, x4);
        if (depth <= 0.0) continue;
        mul_vec4(ldm(world_prev, i), ph, xp4);
        double v[3], pv[3];
        for (int k = 0; k < 3; ++k) v[k] = (x4[k] - xp4[k]) / dt;
        for (int r = 0; r < 3; ++r) {
          double acc = proj[r] * v[0];
          acc = fma(proj[r + 3], v[1], acc);
          acc = fma(proj[r + 6], v[2], acc);
          pv[r] = acc;
        }
        const double pv2 = dot3(pv, pv);
        out->value += d1c * depth * depth + d2c * depth * depth * pv2;
        const double a = -2.0 * d1c * depth - 2.0 * d2c * depth * pv2;
        const double b = 2.0 * d2c * depth * depth / dt;
        double dq[4];
        for (int k = 0; k < 3; ++k) dq[k] = a * nrm[k] + b * pv[k];
        dq[3] = 0.0;
        M4 oc;
        for (int s = 0; s < 4; ++s)
          for (int r = 0; r < 4; ++r) oc.a[r + 4 * s] = dq[r] * ph[s];
        stm(cot, i, add(ldm(cot, i), oc));
        have_cot = true;
        if (need_jx) {
          for (int k = 0; k < 3 * n; ++k) jx[k] = 0.0;
          double y[4] = {ph[0], ph[1], ph[2], ph[3]};
          for (int l = i; l >= 0; l = m.parent[l]) {
            const int off = m.dof_off[l];
            for (int j = 0; j < m.dof_cnt[l]; ++j) {
              double t4[4];
              mul_vec4(ldm(pn.lever, off + j), y, t4);
              for (int r = 0; r < 3; ++r) jx[r + 3 * (off + j)] = t4[r];
            }
            double y2[4];
            mul_vec4(ldm(pn.value, l), y, y2);
            for (int r = 0; r < 4; ++r) y[r] = y2[r];
          }
          for (int k = 0; k < n; ++k) {
            double acc = nrm[0] * jx[3 * k];
            acc = fma(nrm[1], jx[1 + 3 * k], acc);
            acc = fma(nrm[2], jx[2 + 3 * k], acc);
            dd[k] = -acc;
          }
          if (want_gn) {
            const double c2 = 2.0 * d1c;
            for (int bb = 0; bb < n; ++bb)
              for (int aa = 0; aa < n; ++aa)
                gn[aa + (long)n * bb] = gn[aa + (long)n * bb] + (c2 * dd[aa]) * dd[bb];
            if (d2c > 0.0) {
              const double ddt = depth / dt;
              for (int k = 0; k < n; ++k)
                for (int r = 0; r < 3; ++r) {
                  double acc = proj[r] * jx[3 * k];
                  acc = fma(proj[r + 3], jx[1 + 3 * k], acc);
                  acc = fma(proj[r + 6], jx[2 + 3 * k], acc);
                  tmp[r + 3 * k] = acc;
                }
              for (int k = 0; k < n; ++k)
                for (int r = 0; r < 3; ++r) jr[r + 3 * k] = pv[r] * dd[k] + ddt * tmp[r + 3 * k];
              const double c3 = 2.0 * d2c;
              for (int bb = 0; bb < n; ++bb)
                for (int aa = 0; aa < n; ++aa) {
                  double acc = (c3 * jr[3 * aa]) * jr[3 * bb];
                  acc = fma(c3 * jr[1 + 3 * aa], jr[1 + 3 * bb], acc);
                  acc = fma(c3 * jr[2 + 3 * aa], jr[2 + 3 * bb], acc);
                  gn[aa + (long)n * bb] = gn[aa + (long)n * bb] + acc;
                }
            }
          }
          if (want_hess) {
            double hxx[9];
            for (int c = 0; c < 3; ++c)
              for (int r = 0; r < 3; ++r) hxx[r + 3 * c] = ((2.0 * d1c) * nrm[r]) * nrm[c];
            if (d2c > 0.0) {
              const double k1 = (2.0 * d2c) * pv2;
              const double k2 = 4.0 * d2c * depth / dt;
              const double k3 = 2.0 * d2c * depth * depth / (dt * dt);
              for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r) {
                  const double t1 = (k1 * nrm[r]) * nrm[c];
                  const double t2 = k2 * (nrm[r] * pv[c] + pv[r] * nrm[c]);
                  const double t3 = k3 * proj[r + 3 * c];
                  hxx[r + 3 * c] = hxx[r + 3 * c] + ((t1 - t2) + t3);
                }
            }
            // (jx^T hxx) jx ; tmp holds n x 3 column-major (needs 3n slots)
            for (int k = 0; k < n; ++k)
              for (int c = 0; c < 3; ++c) {
                double acc = jx[3 * k] * hxx[3 * c];
                acc = fma(jx[1 + 3 * k], hxx[1 + 3 * c], acc);
                acc = fma(jx[2 + 3 * k], hxx[2 + 3 * c], acc);
                tmp[k + (long)n * c] = acc;
              }
            for (int bb = 0; bb < n; ++bb)
              for (int aa = 0; aa < n; ++aa) {
                double acc = tmp[aa] * jx[3 * bb];
                acc = fma(tmp[aa + (long)n], jx[1 + 3 * bb], acc);
                acc = fma(tmp[aa + 2 * (long)n], jx[2 + 3 * bb], acc);
                hess[aa + (long)n * bb] = hess[aa + (long)n * bb] + acc;
              }
          }
        }
      }
    }
  }
  if (have_cot) {
    if (want_grad) functional_grad(E, cot, pn, grad);
    if (want_hess) {
      const Arr fh = E.arr(L.fh);
      functional_hess(E, cot, pn, fh);
      for (long k = 0; k < (long)n * n; ++k) hess[k] = hess[k] + fh[k];
    }
  }
}

// ---------------------------------------------------------------------------
// StepObjective (objective.cpp:155-343)
// ---------------------------------------------------------------------------
// actuation_at (objective.cpp:195-204): tau for instant m into out
__device__ void actuation_at(const Env& E, bool have_tau, int instant, double* out_unused,
                             const Arr& dst) {
  const int n = E.m->n;
  if (have_tau) {
    const Arr tau = E.arr(E.L->tau + (long)instant * n);
    for (int k = 0; k < n; ++k) dst[k] = tau[k];
    return;
  }
  if (E.f->tau_len == n) {
    for (int k = 0; k < n; ++k) dst[k] = E.f->tau[k];
    return;
  }
  for (int k = 0; k < n; ++k) dst[k] = 0.0;
}

// StepObjective ctor (objective.cpp:162-185): history passes + hist_const.
// Returns false when a history configuration is non-finite.
__device__ bool obj_init(const Env& E) {
  const DModel& m = *E.m;
  const Arr h0 = E.arr(E.L->hist0), h1 = E.arr(E.L->hist1);
  if (!all_finite(h0, m.n) || !all_finite(h1, m.n)) return false;
  const Arr w0 = E.arr(E.L->hw0), w1 = E.arr(E.L->hw1);
  forward_pass(E, h0, w0);
  forward_pass(E, h1, w1);
  if (E.sc->objective == 0) {
    E.sv(SC_HISTCONST) = 4.0 * correlation_value(E, w1, w1) + correlation_value(E, w0, w0) -
                         4.0 * correlation_value(E, w1, w0);
  }
  return true;
}

// StepObjective::evaluate_impl (objective.cpp:206-334) at x (array offset).
// Writes value to *value, grad to E.evgrad, GN to E.evgn.  false = ModelError.
__device__ bool obj_evaluate(const Env& E, const Arr& x, bool want_grad, bool want_gn, bool have_tau,
                             double* value) {
  const DModel& m = *E.m;
  const DSchedule& sc = *E.sc;
  const Layout& L = *E.L;
  const int N = m.N, n = m.n;
  const double dt = sc.dt;
  const double inv_dt2 = 1.0 / (dt * dt);
  const Arr hw0 = E.arr(L.hw0), hw1 = E.arr(L.hw1);
  const Arr evgrad = E.arr(L.evgrad);
  const Arr evgn = E.arr(L.evgn);
  const Arr tauv = E.arr(L.g);  // scratch n

  if (sc.objective == 0) {
    const Pass P = pass_at(E, 0);
    if (!pass_make(E, x, P, false)) return false;
    const double inertial =
        0.5 * inv_dt2 *
        (correlation_value(E, P.world, P.world) - 4.0 * correlation_value(E, hw1, P.world) +
         2.0 * correlation_value(E, hw0, P.world) + E.sv(SC_HISTCONST));
    const Arr ab = E.arr(L.ab);
    if (want_gn) correlation_hess_ab(E, P, P, ab);
    PotOut pot;
    potential_terms(E, P, hw1, dt, want_grad, want_gn, false, want_gn ? &ab : nullptr, &pot);
    actuation_at(E, have_tau, 0, nullptr, tauv);
    *value = inertial + pot.value - vdot32(tauv, x, n);
    if (want_grad) {
      const Arr seeds = E.arr(L.seeds);
      for (int i = 0; i < N; ++i) {
        M4 d = sub(ldm(P.world, i), scale(2.0, ldm(hw1, i)));
        d = add(d, ldm(hw0, i));
        d = scale(inv_dt2, d);
        stm(seeds, i, mul(d, ldg4(m.S + 16 * i)));
      }
      functional_grad(E, seeds, P, evgrad);
      const Arr pg = E.arr(L.potgrad);
      for (int k = 0; k < n; ++k) evgrad[k] = (evgrad[k] + pg[k]) - tauv[k];
    }
    if (want_gn) {
      const Arr pgn = E.arr(L.potgn);
      // gn = inv_dt2*ab + pot.gn, then 0.5*(gn + gn^T)
      for (int c = 0; c < n; ++c)
        for (int r = 0; r <= c; ++r) {
          const double grc = inv_dt2 * ab[r + (long)n * c] + pgn[r + (long)n * c];
          const double gcr = inv_dt2 * ab[c + (long)n * r] + pgn[c + (long)n * r];
          const double s = 0.5 * (grc + gcr);
          evgn[r + (long)n * c] = s;
          evgn[c + (long)n * r] = 0.5 * (gcr + grc);
        }
    }
    return true;
  }

  // residual form
  const int u = sc.u, U = sc.U, K1 = sc.K1;
  for (int mm = 0; mm < u; ++mm) {
    const Arr xm = Arr{x.p + (long)mm * n * x.s, x.s};
    if (!pass_make(E, xm, pass_at(E, mm), want_grad)) return false;
  }
  const Arr resid = E.arr(L.resid);
  const Arr J = E.arr(L.J);
  const Arr ab_mm = E.arr(L.ab);
  const Arr fh = E.arr(L.fh);
  const Arr seeds = E.arr(L.seeds);
  const Arr pg = E.arr(L.potgrad);
  const Arr ph = E.arr(L.pothess);
  for (int mm = 0; mm < u; ++mm) {
    const Pass Pm = pass_at(E, mm);
    const double* stencil = sc.H2 + K1 * (2 + mm);
    for (int i = 0; i < N; ++i) {
      M4 acc = m4_zero();
      for (int j = 0; j < K1; ++j) {
        const M4 wj = (j == 0) ? ldm(hw0, i) : (j == 1) ? ldm(hw1, i) : ldm(pass_at(E, j - 2).world, i);
        addto(acc, scale(stencil[j], wj));
      }
      stm(seeds, i, mul(scale(inv_dt2, acc), ldg4(m.S + 16 * i)));
    }
    const Arr g = Arr{resid.p + (long)mm * n * resid.s, resid.s};
    functional_grad(E, seeds, Pm, g);
    if (want_grad) correlation_hess_ab(E, Pm, Pm, ab_mm);
    const double t_local = sc.times[2 + mm];
    PotOut pot;
    potential_terms(E, Pm, hw1, t_local * dt, true, false, want_grad, want_grad ? &ab_mm : nullptr, &pot);
    actuation_at(E, have_tau, mm, nullptr, tauv);
    for (int k = 0; k < n; ++k) g[k] = g[k] + (pg[k] - tauv[k]);
    if (want_grad) {
      functional_hess(E, seeds, Pm, fh);
      const double cm = inv_dt2 * stencil[2 + mm];
      for (int c = 0; c < n; ++c)
        for (int r = 0; r < n; ++r)
          J[(mm * n + r) + (long)U * (mm * n + c)] =
              (fh[r + (long)n * c] + cm * ab_mm[c + (long)n * r]) + ph[r + (long)n * c];
      for (int l = 0; l < u; ++l) {
        if (l == mm) continue;
        correlation_hess_ab(E, pass_at(E, l), Pm, fh);
        const double cl = inv_dt2 * stencil[2 + l];
        for (int c = 0; c < n; ++c)
          for (int r = 0; r < n; ++r) J[(mm * n + r) + (long)U * (l * n + c)] = cl * fh[c + (long)n * r];
      }
    }
  }
  double v = 0.0;
  for (int mm = 0; mm < u; ++mm) v += vdot32(Arr{resid.p + (long)mm * n * resid.s, resid.s},
                                             Arr{resid.p + (long)mm * n * resid.s, resid.s}, n);
  *value = v;
  if (want_grad) {
    for (int a = 0; a < U; ++a) {
      double acc = (2.0 * J[(long)U * a]) * resid[0];
      for (int k = 1; k < U; ++k) acc = fma(2.0 * J[k + (long)U * a], resid[k], acc);
      evgrad[a] = acc;
    }
    if (want_gn) {
      for (int b = 0; b < U; ++b)
        for (int a = 0; a <= b; ++a) {
          double ab1 = (2.0 * J[(long)U * a]) * J[(long)U * b];
          double ab2 = (2.0 * J[(long)U * b]) * J[(long)U * a];
          for (int k = 1; k < U; ++k) {
            ab1 = fma(2.0 * J[k + (long)U * a], J[k + (long)U * b], ab1);
            ab2 = fma(2.0 * J[k + (long)U * b], J[k + (long)U * a], ab2);
          }
          evgn[a + (long)U * b] = 0.5 * (ab1 + ab2);
          evgn[b + (long)U * a] = 0.5 * (ab2 + ab1);
        }
    }
  }
  return true;
}

// ---------------------------------------------------------------------------
// optim (optim.cpp:11-250)
// ---------------------------------------------------------------------------
__device__ double infnorm(const Arr& a, int n) {
  double mx = 0.0;
  for (int k = 0; k < n; ++k) mx = fmax(mx, fabs(a[k]));
  return mx;
}

// LLT (eigen_lite definition, optim.cpp:11-15)
__device__ bool llt_factor(const Arr& A, int n) {
  for (int k = 0; k < n; ++k) {
    const double x = A[k + (long)n * k];
    if (x <= 0.0) return false;
    const double d = sqrt(x);
    A[k + (long)n * k] = d;
    for (int i = k + 1; i < n; ++i) A[i + (long)n * k] = A[i + (long)n * k] / d;
    for (int j = k + 1; j < n; ++j) {
      const double ljk = A[j + (long)n * k];
      for (int i = j; i < n; ++i) A[i + (long)n * j] = fma(-A[i + (long)n * k], ljk, A[i + (long)n * j]);
    }
  }
  return true;
}
__device__ void llt_solve(const Arr& Lm, int n, const Arr& b, const Arr& x) {
  for (int i = 0; i < n; ++i) x[i] = b[i];
  for (int j = 0; j < n; ++j) {
    const double xj = x[j] / Lm[j + (long)n * j];
    x[j] = xj;
    for (int i = j + 1; i < n; ++i) x[i] = fma(-Lm[i + (long)n * j], xj, x[i]);
  }
  for (int j = n - 1; j >= 0; --j) {
    const double xj = x[j] / Lm[j + (long)n * j];
    x[j] = xj;
    for (int i = 0; i < j; ++i) x[i] = fma(-Lm[j + (long)n * i], xj, x[i]);
  }
}

__device__ __forceinline__ bool grad_converged(const Env& E) {
  const DOpt& o = E.sc->opt;
  const int U = E.sc->U;
  const double g = infnorm(E.arr(E.L->grad), U);
  if (g <= o.grad_tol * fmax(1.0, infnorm(E.arr(E.L->x), U))) return true;
  if (o.grad_rtol > 0.0 && g <= o.grad_rtol * E.sv(SC_GRAD0)) return true;
  return false;
}
__device__ __forceinline__ bool stagnation_update(const Env& E, double oldv, double newv) {
  int& st = E.iv(IS_STAG);
  if (oldv - newv <= E.sc->opt.ftol * fmax(1.0, fabs(oldv))) ++st;
  else st = 0;
  return st >= 2;
}

// solver construction: first evaluation (optim.cpp:82-93,143-150).
// Returns 0 ok, TR_NONFINITE_INIT / TR_NONFINITE_CFG on error.
__device__ int solver_init(const Env& E, bool have_tau) {
  const DOpt& o = E.sc->opt;
  const int U = E.sc->U;
  const bool lm = o.kind == 1;
  E.iv(IS_STATUS) = ST_RUNNING;
  E.iv(IS_ITERS) = 0;
  E.iv(IS_STAG) = 0;
  E.iv(IS_ACC) = 0;
  E.iv(IS_HSTART) = 0;
  E.iv(IS_HCOUNT) = 0;
  E.sv(SC_LAMBDA) = o.lm_lambda0;
  double v;
  if (!obj_evaluate(E, E.arr(E.L->x), true, lm, have_tau, &v)) return TR_NONFINITE_CFG;
  if (!isfinite(v)) return TR_NONFINITE_INIT;
  E.sv(SC_VALUE) = v;
  const Arr grad = E.arr(E.L->grad), evg = E.arr(E.L->evgrad);
  for (int k = 0; k < U; ++k) grad[k] = evg[k];
  if (lm) {
    const Arr gn = E.arr(E.L->gn), evgn = E.arr(E.L->evgn);
    for (long k = 0; k < (long)U * U; ++k) gn[k] = evgn[k];
  }
  E.sv(SC_GRAD0) = infnorm(grad, U);
  return 0;
}

// SolverBase::finish_iteration (optim.cpp:64-67): count, record the value
__device__ __forceinline__ void finish_iteration(const Env& E) {
  if (E.itv) E.itv[E.iv(IS_ITERS)] = E.sv(SC_VALUE);
  ++E.iv(IS_ITERS);
}

// LmSolver::iterate (optim.cpp:95-134). Returns status or -1 on ModelError.
__device__ int lm_iterate(const Env& E, bool have_tau) {
  const DOpt& o = E.sc->opt;
  int& status = E.iv(IS_STATUS);
  if (status != ST_RUNNING) return status;
  if (E.iv(IS_ITERS) >= o.max_iters) return status = ST_FAILED;
  if (grad_converged(E)) return status = ST_CONVERGED;
  const int n = E.sc->U;
  const Layout& L = *E.L;
  const Arr gn = E.arr(L.gn), damped = E.arr(L.damped), grad = E.arr(L.grad), tmp = E.arr(L.tmp),
            step = E.arr(L.step), x = E.arr(L.x), cand = E.arr(L.cand);
  double& lambda = E.sv(SC_LAMBDA);
  for (long k = 0; k < (long)n * n; ++k) damped[k] = gn[k];
  for (int k = 0; k < n; ++k) damped[k + (long)n * k] = damped[k + (long)n * k] + lambda;
  for (int k = 0; k < n; ++k) tmp[k] = -grad[k];
  bool accepted = false;
  const bool ok = llt_factor(damped, n);
  if (ok) llt_solve(damped, n, tmp, step);
  if (ok && all_finite(step, n)) {
    for (int k = 0; k < n; ++k) cand[k] = x[k] + step[k];
    double tv;
    if (!obj_evaluate(E, cand, false, false, have_tau, &tv)) return -1;
    if (isfinite(tv) && tv < E.sv(SC_VALUE)) {
      const double oldv = E.sv(SC_VALUE);
      for (int k = 0; k < n; ++k) x[k] = cand[k];
      double nv;
      if (!obj_evaluate(E, x, true, true, have_tau, &nv)) return -1;
      E.sv(SC_VALUE) = nv;
      const Arr evg = E.arr(L.evgrad), evgn = E.arr(L.evgn);
      for (int k = 0; k < n; ++k) grad[k] = evg[k];
      for (long k = 0; k < (long)n * n; ++k) gn[k] = evgn[k];
      lambda = fmax(lambda / o.lm_lambda_factor, 1e-12);
      accepted = true;
      ++E.iv(IS_ACC);
      if (stagnation_update(E, oldv, nv)) status = ST_CONVERGED;
    }
  }
  if (!accepted) {
    lambda *= o.lm_lambda_factor;
    if (lambda > o.lm_lambda_max) status = ST_FAILED;
  }
  finish_iteration(E);
  if (status == ST_RUNNING && E.iv(IS_ITERS) >= o.max_iters) status = ST_FAILED;
  return status;
}

// LbfgsSolver::two_loop (optim.cpp:213-229): q = H g (q, g arrays)
__device__ void two_loop(const Env& E, const Arr& g, const Arr& q) {
  const int n = E.sc->U;
  const int cap = E.sc->opt.mem + 1;
  const Layout& L = *E.L;
  const int H = E.iv(IS_HCOUNT), h0 = E.iv(IS_HSTART);
  const Arr alpha = E.arr(L.alpha), hsy = E.arr(L.hsy);
  for (int k = 0; k < n; ++k) q[k] = g[k];
  for (int i = H - 1; i >= 0; --i) {
    const int slot = (h0 + i) % cap;
    const Arr si = E.arr(L.hs + (long)slot * n), yi = E.arr(L.hy + (long)slot * n);
    const double a = vdot32(si, q, n) / hsy[slot];
    alpha[i] = a;
    for (int k = 0; k < n; ++k) q[k] = q[k] - a * yi[k];
  }
  if (H > 0) {
    const int slot = (h0 + H - 1) % cap;
    const Arr yl = E.arr(L.hy + (long)slot * n);
    const double scl = hsy[slot] / vdot32(yl, yl, n);
    for (int k = 0; k < n; ++k) q[k] = q[k] * scl;
  }
  for (int i = 0; i < H; ++i) {
    const int slot = (h0 + i) % cap;
    const Arr si = E.arr(L.hs + (long)slot * n), yi = E.arr(L.hy + (long)slot * n);
    const double beta = vdot32(yi, q, n) / hsy[slot];
    const double c = alpha[i] - beta;
    for (int k = 0; k < n; ++k) q[k] = q[k] + c * si[k];
  }
}

// LbfgsSolver::iterate (optim.cpp:152-205). value(cand) and
// evaluate(cand) share one pass: the value is bit-identical either way.
__device__ int lbfgs_iterate(const Env& E, bool have_tau) {
  const DOpt& o = E.sc->opt;
  int& status = E.iv(IS_STATUS);
  if (status != ST_RUNNING) return status;
  if (E.iv(IS_ITERS) >= o.max_iters) return status = ST_FAILED;
  if (grad_converged(E)) return status = ST_CONVERGED;
  const int n = E.sc->U;
  const int cap = o.mem + 1;
  const Layout& L = *E.L;
  const Arr grad = E.arr(L.grad), tmp = E.arr(L.tmp), dir = E.arr(L.dir), x = E.arr(L.x),
            cand = E.arr(L.cand), evg = E.arr(L.evgrad), hsy = E.arr(L.hsy);
  two_loop(E, grad, tmp);
  for (int k = 0; k < n; ++k) dir[k] = -tmp[k];
  double slope = vdot32(dir, grad, n);
  if (!(slope < 0.0)) {
    E.iv(IS_HCOUNT) = 0;
    E.iv(IS_HSTART) = 0;
    for (int k = 0; k < n; ++k) dir[k] = -grad[k];
    slope = vdot32(dir, grad, n);
  }
  double t = 1.0;
  bool accepted = false;
  const double fval = E.sv(SC_VALUE);
  for (int trial = 0; trial < o.max_line_search; ++trial) {
    for (int k = 0; k < n; ++k) cand[k] = x[k] + t * dir[k];
    if (all_finite(cand, n)) {
      double v;
      if (!obj_evaluate(E, cand, false, false, have_tau, &v)) return -1;
      if (isfinite(v) && v <= fval + o.armijo_c1 * t * slope && v < fval) {
        double v2;
        if (!obj_evaluate(E, cand, true, false, have_tau, &v2)) return -1;
        int h0 = E.iv(IS_HSTART), hc = E.iv(IS_HCOUNT);
        const int slot = (h0 + hc) % cap;
        const Arr sn = E.arr(L.hs + (long)slot * n), yn = E.arr(L.hy + (long)slot * n);
        for (int k = 0; k < n; ++k) {
          sn[k] = t * dir[k];
          yn[k] = evg[k] - grad[k];
        }
        const double sy = vdot32(sn, yn, n);
        if (sy > 1e-12) {
          hsy[slot] = sy;
          ++hc;
          if (hc > o.mem) {
            h0 = (h0 + 1) % cap;
            --hc;
          }
          E.iv(IS_HSTART) = h0;
          E.iv(IS_HCOUNT) = hc;
        }
        for (int k = 0; k < n; ++k) {
          x[k] = cand[k];
          grad[k] = evg[k];
        }
        E.sv(SC_VALUE) = v2;
        accepted = true;
        ++E.iv(IS_ACC);
        if (stagnation_update(E, fval, v2)) status = ST_CONVERGED;
        break;
      }
    }
    t *= o.backtrack_factor;
  }
  if (!accepted) status = ST_FAILED;
  finish_iteration(E);
  if (status == ST_RUNNING && E.iv(IS_ITERS) >= o.max_iters) status = ST_FAILED;
  return status;
}

__device__ __forceinline__ int solver_iterate(const Env& E, bool have_tau) {
  return E.sc->opt.kind == 1 ? lm_iterate(E, have_tau) : lbfgs_iterate(E, have_tau);
}

// ---------------------------------------------------------------------------
// stepper (stepper.cpp:14-147)
// ---------------------------------------------------------------------------
// fd_kinetic (stepper.cpp:14-22)
__device__ double fd_kinetic(const Env& E, const Arr& wp, const Arr& wn, double dt) {
  const DModel& m = *E.m;
  double ke = 0.0;
  for (int i = 0; i < m.N; ++i) {
    const M4 td = divs(sub(ldm(wn, i), ldm(wp, i)), dt);
    ke += 0.5 * ddot(mul(td, ldg4(m.S + 16 * i)), td);
  }
  return ke;
}
// gravity_potential (baseline.cpp:219-229) from world transforms
__device__ double gravity_potential(const Env& E, const Arr& w) {
  const DModel& m = *E.m;
  const double ghat[4] = {E.f->gravity[0], E.f->gravity[1], E.f->gravity[2], 0.0};
  const double e4[4] = {0.0, 0.0, 0.0, 1.0};
  double pe = 0.0;
  for (int i = 0; i < m.N; ++i) {
    double u[4], v[4];
    mul_vec4(ldg4(m.S + 16 * i), e4, u);
    mul_vec4(ldm(w, i), u, v);
    pe -= dot4(ghat, v);
  }
  return pe;
}
// kinetic_energy (baseline.cpp:208-217) with the velocity pass (baseline.cpp:20-54)
__device__ double kinetic_energy(const Env& E, const Arr& q, const Arr& qdot) {
  const DModel& m = *E.m;
  const Pass P = pass_at(E, 0);
  pass_make(E, q, P, false);
  const Arr tdot = E.arr(E.L->seeds);
  double ke = 0.0;
  for (int i = 0; i < m.N; ++i) {
    const int p = m.parent[i];
    const int off = m.dof_off[i];
    M4 ldot = m4_zero();
    for (int j = 0; j < m.dof_cnt[i]; ++j) addto(ldot, scale(qdot[off + j], ldm(P.d1, off + j)));
    const M4 ptd = (p >= 0) ? ldm(tdot, p) : m4_zero();
    const M4 td = add(mul(ptd, ldm(P.value, i)), mul(pworld(E, P, i), ldot));
    stm(tdot, i, td);
  }
  for (int i = 0; i < m.N; ++i) {
    const M4 td = ldm(tdot, i);
    ke += 0.5 * ddot(mul(td, ldg4(m.S + 16 * i)), td);
  }
  return ke;
}

// ---------------------------------------------------------------------------
// Newton-Euler baselines (baseline.cpp:56-206, simulate_baseline
// stepper.cpp:168-202): explicit integration of M(q) qdd = f(q, qd) - c(q, qd)
// with M = correlation_hess_ab(q, q) and the trace-form Coriolis vector.
// Workspace (per env, BaselineLayout offsets in Layout fields): pass 0 with
// d2, tdot / quad / seeds / cot / adj [N][16], mass [n][n], vectors.
// ---------------------------------------------------------------------------
enum { BL_OK = 0, BL_DIVERGED = 5, BL_SINGULAR = 6, BL_NONFINITE_CFG = 7 };

// velocity_pass (baseline.cpp:20-54) into tdot (and quad)
__device__ void bl_velocity_pass(const Env& E, const Pass& P, const Arr& qd, const Arr& tdot, const Arr* quad) {
  const DModel& m = *E.m;
  for (int i = 0; i < m.N; ++i) {
    const int p = m.parent[i];
    const int off = m.dof_off[i];
    const int dof = m.dof_cnt[i];
    M4 ldot = m4_zero();
    for (int j = 0; j < dof; ++j) addto(ldot, scale(qd[off + j], ldm(P.d1, off + j)));
    const M4 ptd = (p >= 0) ? ldm(tdot, p) : m4_zero();
    const M4 pw = pworld(E, P, i);
    const M4 V = ldm(P.value, i);
    stm(tdot, i, add(mul(ptd, V), mul(pw, ldot)));
    if (quad) {
      M4 lq = m4_zero();
      for (int l = 0; l < dof; ++l)
        for (int j = 0; j < dof; ++j) {
          const int a = j < l ? j : l, b = j < l ? l : j;  // d2_at(j, l), packed by the larger index
          addto(lq, scale(qd[off + j] * qd[off + l], ldm(P.d2, m.d2_off[i] + b * (b + 1) / 2 + a)));
        }
      const M4 pq = (p >= 0) ? ldm(*quad, p) : m4_zero();
      stm(*quad, i, add(add(mul(pq, V), mul(scale(2.0, ptd), ldot)), mul(pw, lq)));
    }
  }
}

struct BlArrs {
  Arr tdot, quad, cot, mass, cor, gf, rhs;
};

// acceleration (baseline.cpp:137-147): mass_and_coriolis, generalized_force, LLT
__device__ int bl_accel(const Env& E, const BlArrs& W, const Arr& q, const Arr& qd, const Arr& acc, double dt) {
  const DModel& m = *E.m;
  const DForces& f = *E.f;
  const int n = m.n, N = m.N;
  if (!all_finite(q, n)) return BL_NONFINITE_CFG;  // validate_configuration (model.cpp:114-123)
  const Pass P = pass_at(E, 0);
  pass_make(E, q, P, true, false);
  bl_velocity_pass(E, P, qd, W.tdot, &W.quad);
  correlation_hess_ab(E, P, P, W.mass);
  const Arr seeds = E.arr(E.L->seeds);
  for (int i = 0; i < N; ++i) stm(seeds, i, mul(ldm(W.quad, i), ldg4(m.S + 16 * i)));
  functional_grad(E, seeds, P, W.cor);
  // generalized_force (baseline.cpp:76-133)
  bool have = false;
  for (int i = 0; i < N; ++i) stm(W.cot, i, m4_zero());
  if (f.gravity_nonzero) {
    const double ghat[4] = {f.gravity[0], f.gravity[1], f.gravity[2], 0.0};
    const double e4[4] = {0.0, 0.0, 0.0, 1.0};
    for (int i = 0; i < N; ++i) {
      double u[4];
      mul_vec4(ldg4(m.S + 16 * i), e4, u);
      M4 g;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) g.a[r + 4 * c] = ghat[r] * u[c];
      stm(W.cot, i, add(ldm(W.cot, i), g));
    }
    have = true;
  }
  if (f.drag_d > 0.0) {
    const double sc = 2.0 * f.drag_d / dt;
    for (int i = 0; i < N; ++i)
      stm(W.cot, i, sub(ldm(W.cot, i), mul(scale(sc, ldm(W.tdot, i)), ldg4(m.S + 16 * i))));
    have = true;
  }
  if (f.has_contact && (f.d1 > 0.0 || f.d2 > 0.0)) {
    const double* nr = f.normal;
    double proj[9];  // I - n n^T, column-major
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int r = 0; r < 3; ++r) proj[r + 3 * c] = (r == c ? 1.0 : 0.0) - nr[r] * nr[c];
    for (int i = 0; i < N; ++i) {
      const M4 Wi = ldm(P.world, i);
      const M4 Ti = ldm(W.tdot, i);
      for (int sidx = m.sample_off[i]; sidx < m.sample_off[i + 1]; ++sidx) {
        const double ph[4] = {m.samples[3 * sidx], m.samples[3 * sidx + 1], m.samples[3 * sidx + 2], 1.0};
        double x[4];
        mul_vec4(Wi, ph, x);
        const double depth = f.plane_offset - dot3(nr, x);
        if (depth <= 0.0) continue;
        double fv[3];
        const double k1 = 2.0 * f.d1 * depth;
        for (int r = 0; r < 3; ++r) fv[r] = k1 * nr[r];
        if (f.d2 > 0.0) {
          double v[4], pv[3];
          mul_vec4(Ti, ph, v);
          for (int r = 0; r < 3; ++r) {
            double a = proj[r] * v[0];
            a = fma(proj[r + 3], v[1], a);
            pv[r] = fma(proj[r + 6], v[2], a);
          }
          const double k2 = 2.0 * f.d2 * depth * dot3(pv, pv);
          const double k3 = 2.0 * f.d2 * depth * depth / dt;
          for (int r = 0; r < 3; ++r) fv[r] = fv[r] + (k2 * nr[r] - k3 * pv[r]);
        }
        const double fh[4] = {fv[0], fv[1], fv[2], 0.0};
        M4 o;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int r = 0; r < 4; ++r) o.a[r + 4 * c] = fh[r] * ph[c];
        stm(W.cot, i, add(ldm(W.cot, i), o));
        have = true;
      }
    }
  }
  if (have) functional_grad(E, W.cot, P, W.gf);
  else
    for (int k = 0; k < n; ++k) W.gf[k] = 0.0;
  if (f.tau_len == n)
    for (int k = 0; k < n; ++k) W.gf[k] = W.gf[k] + f.tau[k];
  for (int k = 0; k < n; ++k) W.rhs[k] = W.gf[k] - W.cor[k];
  if (!llt_factor(W.mass, n)) return BL_SINGULAR;
  llt_solve(W.mass, n, W.rhs, acc);
  return BL_OK;
}

__device__ __forceinline__ bool bl_finite(const Arr& a, int n) { return all_finite(a, n); }

// simulate_baseline, one thread per trajectory
__global__ void __launch_bounds__(128) k_baseline(DModel m, DForces f, DSchedule sc, Layout L, double* ws, long B,
                                                  int scheme, const double* q0, const double* qd0, double* oq,
                                                  double* oe, int* nsamp, int* status) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B) return;
  Env E{&m, &f, &sc, &L, ws, nullptr, B, e};
  const int n = m.n, S = sc.total_steps;
  const double dt = sc.dt;
  const BlArrs W{E.arr(L.hw0), E.arr(L.hw1), E.arr(L.cot), E.arr(L.gn), E.arr(L.potgrad), E.arr(L.g),
                 E.arr(L.dd)};
  const Arr q = E.arr(L.x), qd = E.arr(L.grad), sq = E.arr(L.cand), sqd = E.arr(L.dir);
  const Arr a1 = E.arr(L.hs), a2 = E.arr(L.hs + n), a3 = E.arr(L.hs + 2 * n), a4 = E.arr(L.hs + 3 * n);
  const Arr s2q = E.arr(L.hy), s2qd = E.arr(L.hy + n), s3q = E.arr(L.hy + 2 * n), s3qd = E.arr(L.hy + 3 * n);
  for (int k = 0; k < n; ++k) {
    q[k] = q0[(long)e * n + k];
    qd[k] = qd0[(long)e * n + k];
  }
  const long S1 = S + 1;
  // the initial sample is logged unconditionally (q0 was validated by the
  // host), later ones with the inf substitution of stepper.cpp:193-198
  auto record = [&](int k) {
    double ke, pe;
    const bool qf = k == 0 || bl_finite(q, n), vf = k == 0 || bl_finite(qd, n);
    ke = (qf && vf) ? kinetic_energy(E, q, qd) : INFINITY;
    if (qf) {
      const Pass P = pass_at(E, 0);
      pass_make(E, q, P, false, false);
      pe = gravity_potential(E, P.world);
    } else {
      pe = INFINITY;
    }
    if (oq)
      for (int j = 0; j < n; ++j) oq[((long)e * S1 + k) * n + j] = q[j];
    if (oe) {
      oe[((long)e * S1 + k) * 2] = ke;
      oe[((long)e * S1 + k) * 2 + 1] = pe;
    }
  };
  record(0);
  int st = BL_OK, k = 0;
  const double h = 0.5 * dt, d6 = dt / 6.0;
  for (; k < S; ++k) {
    if (!bl_finite(q, n) || !bl_finite(qd, n)) {
      st = BL_DIVERGED;
      break;
    }
    int rc = bl_accel(E, W, q, qd, a1, dt);
    if (rc) { st = rc; break; }
    if (scheme == 0) {  // forward_euler
      for (int j = 0; j < n; ++j) {
        const double qn = q[j] + dt * qd[j];
        qd[j] = qd[j] + dt * a1[j];
        q[j] = qn;
      }
    } else if (scheme == 1) {  // semi_implicit
      for (int j = 0; j < n; ++j) {
        qd[j] = qd[j] + dt * a1[j];
        q[j] = q[j] + dt * qd[j];
      }
    } else if (scheme == 2) {  // rk2
      for (int j = 0; j < n; ++j) {
        sq[j] = q[j] + h * qd[j];
        sqd[j] = qd[j] + h * a1[j];
      }
      rc = bl_accel(E, W, sq, sqd, a2, dt);
      if (rc) { st = rc; break; }
      for (int j = 0; j < n; ++j) {
        q[j] = q[j] + dt * sqd[j];
        qd[j] = qd[j] + dt * a2[j];
      }
    } else if (scheme == 3) {  // rk3
      for (int j = 0; j < n; ++j) {
        s2q[j] = q[j] + h * qd[j];
        s2qd[j] = qd[j] + h * a1[j];
      }
      rc = bl_accel(E, W, s2q, s2qd, a2, dt);
      if (rc) { st = rc; break; }
      for (int j = 0; j < n; ++j) {
        s3q[j] = q[j] + dt * (2.0 * s2qd[j] - qd[j]);
        s3qd[j] = qd[j] + dt * (2.0 * a2[j] - a1[j]);
      }
      rc = bl_accel(E, W, s3q, s3qd, a3, dt);
      if (rc) { st = rc; break; }
      for (int j = 0; j < n; ++j) {
        const double qn = q[j] + d6 * ((qd[j] + 4.0 * s2qd[j]) + s3qd[j]);
        qd[j] = qd[j] + d6 * ((a1[j] + 4.0 * a2[j]) + a3[j]);
        q[j] = qn;
      }
    } else {  // rk4
      for (int j = 0; j < n; ++j) {
        s2q[j] = q[j] + h * qd[j];
        s2qd[j] = qd[j] + h * a1[j];
      }
      rc = bl_accel(E, W, s2q, s2qd, a2, dt);
      if (rc) { st = rc; break; }
      for (int j = 0; j < n; ++j) {
        s3q[j] = q[j] + h * s2qd[j];
        s3qd[j] = qd[j] + h * a2[j];
      }
      rc = bl_accel(E, W, s3q, s3qd, a3, dt);
      if (rc) { st = rc; break; }
      for (int j = 0; j < n; ++j) {  // s4 in (sq, sqd)
        sq[j] = q[j] + dt * s3qd[j];
        sqd[j] = qd[j] + dt * a3[j];
      }
      rc = bl_accel(E, W, sq, sqd, a4, dt);
      if (rc) { st = rc; break; }
      for (int j = 0; j < n; ++j) {
        const double qn = q[j] + d6 * (((qd[j] + 2.0 * s2qd[j]) + 2.0 * s3qd[j]) + sqd[j]);
        qd[j] = qd[j] + d6 * (((a1[j] + 2.0 * a2[j]) + 2.0 * a3[j]) + a4[j]);
        q[j] = qn;
      }
    }
    record(k + 1);
  }
  nsamp[e] = (st == BL_OK) ? S + 1 : k + 1;
  status[e] = st;
}

// bootstrap_history with refined_bootstrap (stepper.cpp:46-59): the history
// instant before the run start as the state reached from (q0, -qdot0) after
// 32 RK4 substeps of hs = span / 32 (baseline_step, baseline.cpp:152-206),
// one thread per trajectory; status BL_OK or the baseline_step failure
__global__ void __launch_bounds__(128) k_refined_bootstrap(DModel m, DForces f, DSchedule sc, Layout L, double* ws,
                                                           long B, const double* q0, const double* qd0, double hs,
                                                           double* hist0, int* status) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B) return;
  Env E{&m, &f, &sc, &L, ws, nullptr, B, e};
  const int n = m.n;
  const BlArrs W{E.arr(L.hw0), E.arr(L.hw1), E.arr(L.cot), E.arr(L.gn), E.arr(L.potgrad), E.arr(L.g),
                 E.arr(L.dd)};
  const Arr q = E.arr(L.x), qd = E.arr(L.grad), sq = E.arr(L.cand), sqd = E.arr(L.dir);
  const Arr a1 = E.arr(L.hs), a2 = E.arr(L.hs + n), a3 = E.arr(L.hs + 2 * n), a4 = E.arr(L.hs + 3 * n);
  const Arr s2q = E.arr(L.hy), s2qd = E.arr(L.hy + n), s3q = E.arr(L.hy + 2 * n), s3qd = E.arr(L.hy + 3 * n);
  for (int k = 0; k < n; ++k) {
    q[k] = q0[(long)e * n + k];
    qd[k] = -qd0[(long)e * n + k];
  }
  const double h = 0.5 * hs, d6 = hs / 6.0;
  int st = BL_OK;
  for (int k = 0; k < 32 && st == BL_OK; ++k) {
    int rc = bl_accel(E, W, q, qd, a1, hs);
    if (rc) { st = rc; break; }
    for (int j = 0; j < n; ++j) {
      s2q[j] = q[j] + h * qd[j];
      s2qd[j] = qd[j] + h * a1[j];
    }
    rc = bl_accel(E, W, s2q, s2qd, a2, hs);
    if (rc) { st = rc; break; }
    for (int j = 0; j < n; ++j) {
      s3q[j] = q[j] + h * s2qd[j];
      s3qd[j] = qd[j] + h * a2[j];
    }
    rc = bl_accel(E, W, s3q, s3qd, a3, hs);
    if (rc) { st = rc; break; }
    for (int j = 0; j < n; ++j) {
      sq[j] = q[j] + hs * s3qd[j];
      sqd[j] = qd[j] + hs * a3[j];
    }
    rc = bl_accel(E, W, sq, sqd, a4, hs);
    if (rc) { st = rc; break; }
    for (int j = 0; j < n; ++j) {
      const double qn = q[j] + d6 * (((qd[j] + 2.0 * s2qd[j]) + 2.0 * s3qd[j]) + sqd[j]);
      qd[j] = qd[j] + d6 * (((a1[j] + 2.0 * a2[j]) + 2.0 * a3[j]) + a4[j]);
      q[j] = qn;
    }
  }
  for (int k = 0; k < n; ++k) hist0[(long)e * n + k] = q[k];
  status[e] = st;
}


// ForceModel::tau_at (objective.hpp:28-58) into dst
__device__ void forces_tau_at(const Env& E, double t, const Arr& dst) {
  const DForces& f = *E.f;
  const int n = E.m->n;
  if (f.has_act && f.act_len == n) {
    for (int i = 0; i < n; ++i) {
      if (f.act_kind == 0) {
        dst[i] = f.act_amp[i];
      } else {
        const double ph = i < f.act_phase_len ? f.act_phase[i] : 0.0;
        double s, c;
        pbad_sincos(2.0 * 3.141592653589793 * f.act_freq * t + ph, &s, &c);
        dst[i] = f.act_amp[i] * s;
      }
    }
    return;
  }
  if (f.tau_len == n) {
    for (int i = 0; i < n; ++i) dst[i] = f.tau[i];
    return;
  }
  for (int i = 0; i < n; ++i) dst[i] = 0.0;
}

__device__ void record_sample(const Env& E, const Outputs& out, int k, const Arr& q, double ke, double pe) {
  const int n = E.m->n;
  if (out.q)
    for (int j = 0; j < n; ++j) out.q[out.qrow(E.e, k) * n + j] = q[j];
  if (out.energy) {
    out.energy[out.qrow(E.e, k) * 2] = ke;
    out.energy[out.qrow(E.e, k) * 2 + 1] = pe;
  }
  E.iv(IS_NSAMP) = k + 1;
}

// begin_step (stepper.cpp:83-115); returns 0 or a TR_* error
__device__ int begin_step(const Env& E) {
  const DSchedule& sc = *E.sc;
  const int n = E.m->n, u = sc.u;
  const Layout& L = *E.L;
  const double t0 = E.iv(IS_STEP) * sc.dt;
  for (int mm = 0; mm < u; ++mm) forces_tau_at(E, t0 + sc.times[2 + mm] * sc.dt, E.arr(L.tau + (long)mm * n));
  const double span = -sc.times[0];
  const Arr h0 = E.arr(L.hist0), h1 = E.arr(L.hist1), x = E.arr(L.x);
  for (int mm = 0; mm < u; ++mm) {
    const double tau_m = sc.times[2 + mm];
    for (int k = 0; k < n; ++k)
      x[mm * n + k] = sc.warm_start ? h1[k] + (tau_m / span) * (h1[k] - h0[k]) : h1[k];
  }
  if (!obj_init(E)) return TR_NONFINITE_CFG;
  return solver_init(E, true);
}

// finish_step (stepper.cpp:118-147); false when the fail limit is hit
__device__ bool finish_step(const Env& E, const Outputs& out) {
  const DSchedule& sc = *E.sc;
  const int n = E.m->n, u = sc.u;
  const Layout& L = *E.L;
  const int step = E.iv(IS_STEP);
  const bool converged = E.iv(IS_STATUS) == ST_CONVERGED;
  if (out.iterations) out.iterations[out.rrow(E.e, step)] = E.iv(IS_ITERS);
  if (out.converged) out.converged[out.rrow(E.e, step)] = converged;
  if (out.accepted) out.accepted[out.rrow(E.e, step)] = E.iv(IS_ACC);
  if (out.final_value) out.final_value[out.rrow(E.e, step)] = E.sv(SC_VALUE);
  if (out.final_grad_norm) out.final_grad_norm[out.rrow(E.e, step)] = infnorm(E.arr(L.grad), sc.U);
  E.iv(IS_NREP) = step + 1;
  int& fs = E.iv(IS_FAIL);
  fs = converged ? 0 : fs + 1;
  if (fs > sc.fail_limit) return false;
  const Arr h0 = E.arr(L.hist0), h1 = E.arr(L.hist1), x = E.arr(L.x);
  // new_hist0 = order==2 ? hist1 : x_{u-2};  new_hist1 = x_{u-1}
  for (int k = 0; k < n; ++k) {
    const double nh0 = (sc.order == 2) ? h1[k] : x[(u - 2) * n + k];
    h0[k] = nh0;
  }
  for (int k = 0; k < n; ++k) h1[k] = x[(u - 1) * n + k];
  // world_hist1 of the previous step is hw1 (forward_pass(hist1)); the new one goes to hw0
  const Arr wprev = E.arr(L.hw1), wnext = E.arr(L.hw0);
  forward_pass(E, h1, wnext);
  E.iv(IS_STEP) = step + 1;
  const double t = (step + 1) * sc.dt;
  record_sample(E, out, step + 1, h1, fd_kinetic(E, wprev, wnext, sc.dt), gravity_potential(E, wnext));
  (void)t;
  return true;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// init_pbad_run (stepper.cpp:62-80): q0, qdot0 device [B][n]
__global__ void __launch_bounds__(128) k_init(DModel m, DForces f, DSchedule sc, Layout L, double* ws,
                                              int* iws, long B, const double* q0, const double* qdot0,
                                              const double* hist0, Outputs out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B) return;
  Env E{&m, &f, &sc, &L, ws, iws, B, e};
  const int n = m.n;
  const Arr h0 = E.arr(L.hist0), h1 = E.arr(L.hist1), qd = E.arr(L.step);
  for (int k = 0; k < n; ++k) {
    h1[k] = q0[(long)e * n + k];
    qd[k] = qdot0[(long)e * n + k];
  }
  E.iv(IS_STEP) = 0;
  E.iv(IS_FAIL) = 0;
  E.iv(IS_NSAMP) = 0;
  E.iv(IS_NREP) = 0;
  if (!all_finite(h1, n)) {
    E.iv(IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  const double tl = sc.times[0] * sc.dt;
  if (hist0)  // refined_bootstrap (k_refined_bootstrap)
    for (int k = 0; k < n; ++k) h0[k] = hist0[(long)e * n + k];
  else
    for (int k = 0; k < n; ++k) h0[k] = h1[k] + tl * qd[k];
  const Arr w1 = E.arr(L.hw1);
  forward_pass(E, h1, w1);
  const double ke = kinetic_energy(E, h1, qd);
  record_sample(E, out, 0, h1, ke, gravity_potential(E, w1));
  E.iv(IS_RUN) = (sc.total_steps > 0) ? TR_RUNNING : TR_OK;
}

// One PBAD step (begin_step, iterate to completion, finish_step) per env.
__global__ void __launch_bounds__(128) k_step(DModel m, DForces f, DSchedule sc, Layout L, double* ws,
                                              int* iws, long B, Outputs out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B) return;
  Env E{&m, &f, &sc, &L, ws, iws, B, e};
  if (E.iv(IS_RUN) != TR_RUNNING) return;
  if (out.itv) E.itv = out.itv + out.rrow(e, E.iv(IS_STEP)) * out.itv_n;
  const int rc = begin_step(E);
  if (rc) {
    E.iv(IS_RUN) = rc;
    return;
  }
  int st;
  while ((st = solver_iterate(E, true)) == ST_RUNNING) {
  }
  if (st < 0) {
    E.iv(IS_RUN) = TR_NONFINITE_CFG;
    return;
  }
  if (!finish_step(E, out)) {
    E.iv(IS_RUN) = TR_FAIL_LIMIT;
    return;
  }
  if (E.iv(IS_STEP) >= sc.total_steps) E.iv(IS_RUN) = TR_OK;
}

// Batched StepObjective::evaluate.  hist [B][2][n], tau [B][u][n] or null,
// x [B][U]; outputs value [B], grad [B][U], gn [B][U][U] (column-major).
__global__ void __launch_bounds__(128) k_eval(DModel m, DForces f, DSchedule sc, Layout L, double* ws,
                                              int* iws, long B, const double* hist, const double* tau,
                                              const double* xin, int want_grad, int want_gn,
                                              double* value, double* grad, double* gn, int* err) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B) return;
  Env E{&m, &f, &sc, &L, ws, iws, B, e};
  const int n = m.n, U = sc.U;
  const Arr h0 = E.arr(L.hist0), h1 = E.arr(L.hist1), x = E.arr(L.x);
  for (int k = 0; k < n; ++k) {
    h0[k] = hist[(long)e * 2 * n + k];
    h1[k] = hist[(long)e * 2 * n + n + k];
  }
  for (int k = 0; k < U; ++k) x[k] = xin[(long)e * U + k];
  if (tau) {
    const Arr t = E.arr(L.tau);
    for (int k = 0; k < U; ++k) t[k] = tau[(long)e * U + k];
  }
  err[e] = 0;
  if (!obj_init(E)) {
    err[e] = TR_NONFINITE_CFG;
    return;
  }
  double v;
  if (!obj_evaluate(E, x, want_grad != 0, want_gn != 0, tau != nullptr, &v)) {
    err[e] = TR_NONFINITE_CFG;
    return;
  }
  value[e] = v;
  if (want_grad) {
    const Arr g = E.arr(L.evgrad);
    for (int k = 0; k < U; ++k) grad[(long)e * U + k] = g[k];
  }
  if (want_gn && gn) {
    const Arr G = E.arr(L.evgn);
    for (long k = 0; k < (long)U * U; ++k) gn[(long)e * U * U + k] = G[k];
  }
}

// Batched minimize() of step problems (optim.cpp:244-250).
__global__ void __launch_bounds__(128) k_minimize(DModel m, DForces f, DSchedule sc, Layout L, double* ws,
                                                  int* iws, long B, const double* hist, const double* tau,
                                                  const double* x0, double* xout, int* iters, int* conv,
                                                  double* fval, double* gnorm, int* err) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B) return;
  Env E{&m, &f, &sc, &L, ws, iws, B, e};
  const int n = m.n, U = sc.U;
  const Arr h0 = E.arr(L.hist0), h1 = E.arr(L.hist1), x = E.arr(L.x);
  for (int k = 0; k < n; ++k) {
    h0[k] = hist[(long)e * 2 * n + k];
    h1[k] = hist[(long)e * 2 * n + n + k];
  }
  for (int k = 0; k < U; ++k) x[k] = x0[(long)e * U + k];
  if (tau) {
    const Arr t = E.arr(L.tau);
    for (int k = 0; k < U; ++k) t[k] = tau[(long)e * U + k];
  }
  err[e] = 0;
  if (!obj_init(E)) {
    err[e] = TR_NONFINITE_CFG;
    return;
  }
  const int rc = solver_init(E, tau != nullptr);
  if (rc) {
    err[e] = rc;
    return;
  }
  int st;
  while ((st = solver_iterate(E, tau != nullptr)) == ST_RUNNING) {
  }
  if (st < 0) {
    err[e] = TR_NONFINITE_CFG;
    return;
  }
  for (int k = 0; k < U; ++k) xout[(long)e * U + k] = x[k];
  iters[e] = E.iv(IS_ITERS);
  conv[e] = E.iv(IS_STATUS) == ST_CONVERGED;
  fval[e] = E.sv(SC_VALUE);
  gnorm[e] = infnorm(E.arr(L.grad), U);
}

}  // namespace pbad_gpu

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
#include "pbad_launch.h"

namespace pbad_gpu {

// one thread per environment: blocks of 32 until the batch fills every SM
// with 128-thread blocks (a 4096 batch would otherwise occupy 32 SMs)
static inline int block_for(long B) { return B >= 148L * 128 ? 128 : 32; }
static inline unsigned grid_for(long B) { return (unsigned)((B + block_for(B) - 1) / block_for(B)); }

cudaError_t launch_init(const KernelArgs& a, const double* q0, const double* qdot0, const double* hist0,
                        const Outputs& out, cudaStream_t s) {
  k_init<<<grid_for(a.B), block_for(a.B), 0, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, q0, qdot0, hist0, out);
  return cudaGetLastError();
}
cudaError_t launch_step(const KernelArgs& a, const Outputs& out, cudaStream_t s) {
  k_step<<<grid_for(a.B), block_for(a.B), 0, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, out);
  return cudaGetLastError();
}
// Batched correlation derivatives (adjoint.cpp:113-192: correlation_and_grad,
// hessian_bb, hessian_ab) of I(qa, qb) with the (weighted) body integrals in
// m.S / m.weighted_mass; ConfigPass::make does not validate, so neither does
// this (non-finite inputs propagate).  Outputs per env, Hessians column-major.
__global__ void __launch_bounds__(128) k_correlation(DModel m, Layout L, double* ws, long B, const double* qa,
                                                     const double* qb, double* value, double* grad, double* hbb,
                                                     double* hab) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B) return;
  Env E{&m, nullptr, nullptr, &L, ws, nullptr, B, e};
  const int n = m.n;
  const Arr qA{const_cast<double*>(qa) + (long)e * n, 1}, qB{const_cast<double*>(qb) + (long)e * n, 1};
  const Pass pa = pass_at(E, 0), pb = pass_at(E, 1);
  pass_make(E, qA, pa, false, false);
  pass_make(E, qB, pb, hbb != nullptr, false);
  if (value) value[e] = correlation_value(E, pa.world, pb.world);
  if (grad || hbb) {
    const Arr seeds = E.arr(L.seeds);
    for (int i = 0; i < m.N; ++i) stm(seeds, i, mul(ldm(pa.world, i), ldg4(m.S + 16 * i)));
    if (grad) functional_grad(E, seeds, pb, Arr{grad + (long)e * n, 1});
    if (hbb) functional_hess(E, seeds, pb, Arr{hbb + (long)e * n * n, 1});
  }
  if (hab) correlation_hess_ab(E, pa, pb, Arr{hab + (long)e * n * n, 1});
}

cudaError_t launch_correlation(const DModel& m, const Layout& L, double* ws, long B, const double* qa,
                               const double* qb, double* value, double* grad, double* hbb, double* hab,
                               cudaStream_t s) {
  k_correlation<<<grid_for(B), block_for(B), 0, s>>>(m, L, ws, B, qa, qb, value, grad, hbb, hab);
  return cudaGetLastError();
}
cudaError_t launch_refined_bootstrap(const KernelArgs& a, const Layout& L, double* ws, long B, const double* q0,
                                     const double* qd0, double hs, double* hist0, int* status, cudaStream_t s) {
  k_refined_bootstrap<<<(unsigned)((B + 31) / 32), 32, 0, s>>>(a.m, a.f, a.sc, L, ws, B, q0, qd0, hs, hist0, status);
  return cudaGetLastError();
}
cudaError_t launch_baseline(const KernelArgs& a, const Layout& L, double* ws, long B, int scheme, const double* q0,
                            const double* qd0, double* oq, double* oe, int* nsamp, int* status, cudaStream_t s) {
  k_baseline<<<(unsigned)((B + 31) / 32), 32, 0, s>>>(a.m, a.f, a.sc, L, ws, B, scheme, q0, qd0, oq, oe, nsamp,
                                                      status);
  return cudaGetLastError();
}

cudaError_t launch_eval(const KernelArgs& a, const double* hist, const double* tau, const double* x,
                        int want_grad, int want_gn, double* value, double* grad, double* gn, int* err,
                        cudaStream_t s) {
  k_eval<<<grid_for(a.B), block_for(a.B), 0, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, hist, tau, x, want_grad,
                                       want_gn, value, grad, gn, err);
  return cudaGetLastError();
}
cudaError_t launch_minimize(const KernelArgs& a, const double* hist, const double* tau, const double* x0,
                            double* xout, int* iters, int* conv, double* fval, double* gnorm, int* err,
                            cudaStream_t s) {
  k_minimize<<<grid_for(a.B), block_for(a.B), 0, s>>>(a.m, a.f, a.sc, a.L, a.ws, a.iws, a.B, hist, tau, x0, xout, iters,
                                           conv, fval, gnorm, err);
  return cudaGetLastError();
}

}  // namespace pbad_gpu
