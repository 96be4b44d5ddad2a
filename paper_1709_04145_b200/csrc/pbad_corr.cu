// pbad_corr.cu -- the correlation / functional derivative suite for large
// trees: one CTA per request with the reference's per-link work items spread
// over its threads (parallel_correlation_suite, adjoint.cpp:241-336), and
// the standalone batched linear functional f(q) = sum_i ddot(C_i, T^i(q))
// with its gradient and exact Hessian (functional_value / functional_grad /
// functional_hess, adjoint.cpp:43-101).
//
// The reference's suite runs one work item per (link, quantity) on a worker
// pool; an item replays the serial subtree accumulation of its own link, so
// its adjoint equals the serial backward pass's bit for bit (the operations
// on adj[k], k in subtree(i), are the same sequence in both).  Here the
// backward passes run once (adj: functional_grad's, acc: correlation_hess_ab's
// subtree correlation) and every item reads them:
//   phase 1  joint jets, thread per link (kinematics.cpp:89-169)
//   phase 2  world transforms along the tree (ConfigPass::make), levers
//   phase 3  seeds C_i = T_a^i S_i and the value slots ddot(C_i, T_b^i)
//   phase 4  the ordered value reduction and the two backward passes
//   phase 5  per-link items: grad_b entries, hess_bb own block + ancestor
//            walk, hess_ab own block + ancestor walks (thread per item)
// Every output entry has exactly one contribution, written as the
// reference's `0 + h`; the suite assigns grad_b (adjoint.cpp:285-288) where
// functional_grad accumulates (0 + h), which only differs in the sign of a
// zero.  Operation sequences follow the numeric contract (pbad_math.cuh).
#include <cuda_runtime.h>

#include "pbad_joint.cuh"
#include "pbad_kernels.cuh"
#include "pbad_launch.h"
#include "pbad_math.cuh"

namespace pbad_gpu {
namespace corr {

__device__ __forceinline__ M4 ld(const double* p) {
  M4 m;
#pragma unroll
  for (int k = 0; k < 16; ++k) m.a[k] = p[k];
  return m;
}
__device__ __forceinline__ void st(double* p, const M4& m) {
#pragma unroll
  for (int k = 0; k < 16; ++k) p[k] = m.a[k];
}

// One request per CTA.  mode 0: parallel_correlation_suite (qa, qb, S);
// mode 1: functional value / grad / hess of seeds_in at qb.
__global__ void __launch_bounds__(256) k_suite(DModel m, SuiteLayout L, double* ws, const double* qa,
                                               const double* qb, const double* seeds_in, int mode, double* value,
                                               double* grad, double* hbb, double* hab) {
  const long e = blockIdx.x;
  const int N = m.N, n = m.n, T = blockDim.x, tid = threadIdx.x;
  double* w = ws + e * L.total;
  double *va = w + L.va, *wa = w + L.wa, *d1a = w + L.d1a, *la = w + L.la;
  double *vb = w + L.vb, *wb = w + L.wb, *pwb = w + L.pwb, *d1b = w + L.d1b, *lb = w + L.lb, *d2b = w + L.d2b;
  double *seeds = w + L.seeds, *adj = w + L.adj, *acc = w + L.acc, *slot = w + L.vslot;
  const bool want_ab = mode == 0 && hab != nullptr;
  const bool want_a = mode == 0;
  double* H = hbb ? hbb + e * (long)n * n : nullptr;
  double* HA = want_ab ? hab + e * (long)n * n : nullptr;
  // phase 1: jets of both configurations; zeroed outputs and accumulators
  for (int i = tid; i < N; i += T) {
    const int off = m.dof_off[i], dof = m.dof_cnt[i];
    const M4 offm = ld(m.offset + 16 * i);
    double q[6];
    M4 v, d1[6], d2[21];
    for (int j = 0; j < dof; ++j) q[j] = qb[e * n + off + j];
    joint_jet(m.kind[i], m.axis + 3 * i, offm, q, &v, d1, d2, H != nullptr);
    st(vb + 16 * i, v);
    for (int j = 0; j < dof; ++j) st(d1b + 16 * (off + j), d1[j]);
    if (H)
      for (int j = 0; j < dof * (dof + 1) / 2; ++j) st(d2b + 16 * (m.d2_off[i] + j), d2[j]);
    if (want_a) {
      for (int j = 0; j < dof; ++j) q[j] = qa[e * n + off + j];
      joint_jet(m.kind[i], m.axis + 3 * i, offm, q, &v, d1, d2, false);
      st(va + 16 * i, v);
      for (int j = 0; j < dof; ++j) st(d1a + 16 * (off + j), d1[j]);
    }
    st(adj + 16 * i, m4_zero());
    st(acc + 16 * i, m4_zero());
  }
  if (H)
    for (long k = tid; k < (long)n * n; k += T) H[k] = 0.0;
  if (HA)
    for (long k = tid; k < (long)n * n; k += T) HA[k] = 0.0;
  __syncthreads();
  // phase 2: world transforms root to leaves (ConfigPass::make, adjoint.cpp:9-27),
  // one serial sweep per configuration (warp 0 lane 0: qb, warp 1 lane 0: qa)
  if (tid == 0 || (want_a && tid == 32)) {
    const double* vv = tid == 0 ? vb : va;
    double* ww = tid == 0 ? wb : wa;
    for (int i = 0; i < N; ++i) {
      const int p = m.parent[i];
      const M4 pw = (p >= 0) ? ld(ww + 16 * p) : m4_identity();
      if (tid == 0) st(pwb + 16 * i, pw);
      st(ww + 16 * i, mul(pw, ld(vv + 16 * i)));
    }
  }
  __syncthreads();
  for (int t = tid; t < 2 * n; t += T) {  // levers parent_world * d1 of both configurations
    const int k = t % n;
    const bool a = t >= n;
    if (a && !want_a) continue;
    int lo = 0, hi = N - 1;  // the link of dof k: the last link whose dof offset is <= k
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (m.dof_off[mid] <= k) lo = mid;
      else hi = mid - 1;
    }
    const int i = lo;
    const int p = m.parent[i];
    const double* ww = a ? wa : wb;
    const M4 pw = (p >= 0) ? ld(ww + 16 * p) : m4_identity();
    st((a ? la : lb) + 16 * k, mul(pw, ld((a ? d1a : d1b) + 16 * k)));
  }
  // phase 3: seeds and value slots
  for (int i = tid; i < N; i += T) {
    const M4 c = mode == 0 ? mul(ld(wa + 16 * i), ld(m.S + 16 * i)) : ld(seeds_in + (e * N + i) * 16);
    st(seeds + 16 * i, c);
    slot[i] = ddot(c, ld(wb + 16 * i));
  }
  __syncthreads();
  // phase 4: the value in link order; the adjoint (functional_grad's
  // backward pass) and the subtree correlation acc (correlation_hess_ab's)
  if (tid == 0 && value) {
    double v = 0.0;
    for (int i = 0; i < N; ++i) v += slot[i];
    value[e] = mode == 0 ? v - m.weighted_mass : v;
  }
  if (tid == 32) {
    for (int i = N - 1; i >= 0; --i) {
      const M4 a = add(ld(adj + 16 * i), ld(seeds + 16 * i));
      st(adj + 16 * i, a);
      const int p = m.parent[i];
      if (p >= 0) st(adj + 16 * p, add(ld(adj + 16 * p), mul_bt(a, ld(vb + 16 * i))));
    }
  }
  if (tid == 64 && want_ab) {
    for (int i = N - 1; i >= 0; --i) {
      const M4 ai = add(ld(acc + 16 * i), ld(m.S + 16 * i));
      st(acc + 16 * i, ai);
      const int p = m.parent[i];
      if (p >= 0) st(acc + 16 * p, add(ld(acc + 16 * p), mul_bt(mul(ld(vb + 16 * i), ai), ld(va + 16 * i))));
    }
  }
  __syncthreads();
  // phase 5: per-link items (kind 0 grad, 1 hess_bb, 2 hess_ab), heaviest
  // (deepest links) first
  for (int t = tid; t < 3 * N; t += T) {
    const int i = N - 1 - t / 3, kind = t % 3;
    const int off = m.dof_off[i], dof = m.dof_cnt[i];
    const M4 a = ld(adj + 16 * i);
    if (kind == 0) {
      if (grad)
        for (int j = 0; j < dof; ++j) {
          const double g = ddot(ld(lb + 16 * (off + j)), a);
          grad[e * n + off + j] = mode == 0 ? g : 0.0 + g;
        }
    } else if (kind == 1) {
      if (!H) continue;
      const M4 pw = ld(pwb + 16 * i);
      for (int l = 0; l < dof; ++l)
        for (int j = 0; j <= l; ++j) {
          const double h = ddot(mul(pw, ld(d2b + 16 * (m.d2_off[i] + l * (l + 1) / 2 + j))), a);
          H[(off + j) + (long)n * (off + l)] = 0.0 + h;
          if (j != l) H[(off + l) + (long)n * (off + j)] = 0.0 + h;
        }
      M4 walk[6];
      for (int j = 0; j < dof; ++j) walk[j] = mul_bt(a, ld(d1b + 16 * (off + j)));
      for (int l = m.parent[i]; l >= 0; l = m.parent[l]) {
        const int offl = m.dof_off[l];
        for (int k = 0; k < m.dof_cnt[l]; ++k) {
          const M4 lev = ld(lb + 16 * (offl + k));
          for (int j = 0; j < dof; ++j) {
            const double h = ddot(lev, walk[j]);
            H[(offl + k) + (long)n * (off + j)] = 0.0 + h;
            H[(off + j) + (long)n * (offl + k)] = 0.0 + h;
          }
        }
        const M4 vl = ld(vb + 16 * l);
        for (int j = 0; j < dof; ++j) walk[j] = mul_bt(walk[j], vl);
      }
    } else {
      if (!HA) continue;
      const M4 ai = ld(acc + 16 * i);
      for (int j = 0; j < dof; ++j) {
        const M4 ua = ld(la + 16 * (off + j));
        for (int k = 0; k < dof; ++k)
          HA[(off + j) + (long)n * (off + k)] = 0.0 + trace(mul(mul_at(ua, ld(lb + 16 * (off + k))), ai));
      }
      M4 fwd = mul(ld(vb + 16 * i), ai);
      M4 bwd = mul_bt(ai, ld(va + 16 * i));
      for (int l = m.parent[i]; l >= 0; l = m.parent[l]) {
        const int offl = m.dof_off[l];
        for (int j = 0; j < dof; ++j) {
          const M4 ua = ld(la + 16 * (off + j));
          const M4 vbl = ld(lb + 16 * (off + j));
          for (int k = 0; k < m.dof_cnt[l]; ++k) {
            HA[(off + j) + (long)n * (offl + k)] = 0.0 + trace(mul(mul_at(ua, ld(lb + 16 * (offl + k))), fwd));
            HA[(offl + k) + (long)n * (off + j)] =
                0.0 + trace(mul(mul(transpose(ld(la + 16 * (offl + k))), vbl), bwd));
          }
        }
        fwd = mul(ld(vb + 16 * l), fwd);
        bwd = mul_bt(bwd, ld(va + 16 * l));
      }
    }
  }
}

}  // namespace corr

SuiteLayout suite_layout(int N, int n, int n_d2) {
  SuiteLayout L{};
  long o = 0;
  auto take = [&](long cnt) {
    const long at = o;
    o += cnt;
    return at;
  };
  L.va = take(16L * N);
  L.wa = take(16L * N);
  L.d1a = take(16L * n);
  L.la = take(16L * n);
  L.vb = take(16L * N);
  L.wb = take(16L * N);
  L.pwb = take(16L * N);
  L.d1b = take(16L * n);
  L.lb = take(16L * n);
  L.d2b = take(16L * n_d2);
  L.seeds = take(16L * N);
  L.adj = take(16L * N);
  L.acc = take(16L * N);
  L.vslot = take(N);
  L.total = o;
  return L;
}

cudaError_t launch_suite(const DModel& m, const SuiteLayout& L, double* ws, long B, const double* qa, const double* qb,
                         const double* seeds, int mode, double* value, double* grad, double* hbb, double* hab,
                         cudaStream_t s) {
  corr::k_suite<<<(unsigned)B, 256, 0, s>>>(m, L, ws, qa, qb, seeds, mode, value, grad, hbb, hab);
  return cudaGetLastError();
}

}  // namespace pbad_gpu
