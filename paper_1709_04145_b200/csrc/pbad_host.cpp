// pbad_host.cpp -- C ABI (include/pbad_gpu.h) of the B200 PBAD hot path.
//
// Host-side parts of the reference that run once per model / run:
// build_model + body_integral (model.cpp:9-123), build_scheme
// (collocation.cpp:26-95), and the batch_simulate driver (stepper.cpp:204-270)
// that here launches one stepping kernel per PBAD step for the whole batch.
// Compiled with -ffp-contract=off so the host constants match the kernels'
// numeric contract.
#include "pbad_gpu.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <type_traits>
#include <vector>

#include "pbad_launch.h"
#include "pbad_math.cuh"

using namespace pbad_gpu;

namespace {

thread_local std::string g_last_error;

int32_t fail(int32_t code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) return fail(PBAD_E_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

int kind_dofs(int kind) { return kind == PBAD_HINGE ? 1 : kind == PBAD_BALL ? 3 : kind == PBAD_FREE ? 6 : 0; }

}  // namespace

struct pbad_gpu_model {
  int N = 0, n = 0, n_d2 = 0;
  std::vector<int> parent, kind, dof_off, dof_cnt, d2_off, sample_off;
  std::vector<double> axis, offset, S, mass, samples;
  double weighted_mass = 0.0;
};

extern "C" {

int32_t pbad_gpu_abi_version(void) { return PBAD_GPU_ABI_VERSION; }

int32_t pbad_gpu_device_count(void) {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess ? n : 0;
}
const char* pbad_gpu_last_error(void) { return g_last_error.c_str(); }
const char* pbad_gpu_error_string(int32_t code) {
  switch (code) {
    case PBAD_OK: return "ok";
    case PBAD_E_MODEL: return "model error";
    case PBAD_E_ARGUMENT: return "invalid argument";
    case PBAD_E_CUDA: return "CUDA error";
    case PBAD_E_UNSUPPORTED: return "unsupported by the GPU path";
    case PBAD_E_RUNTIME: return "runtime error";
  }
  return "unknown";
}

void pbad_gpu_default_optimizer(pbad_optimizer_config* c) {
  c->kind = PBAD_LM;
  c->max_iters = 512;
  c->grad_tol = 1e-8;
  c->grad_rtol = 0.0;
  c->ftol = 1e-14;
  c->lbfgs_memory = 8;
  c->lm_lambda0 = 1e-3;
  c->lm_lambda_factor = 10.0;
  c->lm_lambda_max = 1e12;
  c->armijo_c1 = 1e-4;
  c->backtrack_factor = 0.5;
  c->max_line_search = 40;
}

void pbad_gpu_default_sim(pbad_sim_desc* s) {
  std::memset(s, 0, sizeof *s);
  s->dt = 0.01;
  s->duration = 1.0;
  s->order = 2;
  s->objective = PBAD_ENERGY_FORM;
  pbad_gpu_default_optimizer(&s->opt);
  s->consecutive_fail_limit = 25;
  s->warm_start = 1;
}

// body_integral, model.cpp:35-60
int32_t pbad_gpu_body_integral(const pbad_link_spec* L, double* S, double* mass_out) {
  double Sm[16] = {0};
  double mass = 0.0;
  if (L->geom_kind == PBAD_GEOM_BOX) {
    const double* sz = L->box_size;
    const double m = L->box_density * ((sz[0] * sz[1]) * sz[2]);
    const double* c = L->box_center;
    const double k12 = 1.0 / 12.0;
    const double dg[3] = {(sz[0] * sz[0]) * k12, (sz[1] * sz[1]) * k12, (sz[2] * sz[2]) * k12};
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) {
        const double delta = (i == j) ? dg[i] : 0.0 * k12;
        Sm[i + 4 * j] = m * ((c[i] * c[j]) + delta);
      }
    for (int i = 0; i < 3; ++i) Sm[i + 12] = m * c[i];
    for (int j = 0; j < 3; ++j) Sm[3 + 4 * j] = m * c[j];
    Sm[15] = m;
    mass = m;
  } else {
    for (int p = 0; p < L->n_points; ++p) {
      const double pm = L->point_mass[p];
      const double h[4] = {L->point_pos[3 * p], L->point_pos[3 * p + 1], L->point_pos[3 * p + 2], 1.0};
      double mh[4];
      for (int r = 0; r < 4; ++r) mh[r] = pm * h[r];
      for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) Sm[i + 4 * j] = Sm[i + 4 * j] + mh[i] * h[j];
      mass += pm;
    }
  }
  std::memcpy(S, Sm, sizeof Sm);
  *mass_out = mass;
  return PBAD_OK;
}

int32_t pbad_gpu_rotation_vector_matrix(const double theta[3], double R[9]) {
  const M3 r = rotation_vector_matrix(theta[0], theta[1], theta[2]);
  std::memcpy(R, r.a, sizeof r.a);
  return PBAD_OK;
}

// rotation_vector_from_matrix, scene.cpp:66-86 (principal branch of the log
// map; the inverse of pbad_gpu_rotation_vector_matrix).  R column-major.
int32_t pbad_gpu_rotation_vector_from_matrix(const double R[9], double theta[3]) {
  auto at = [&](int r, int c) { return R[r + 3 * c]; };
  const double tr = (at(0, 0) + at(1, 1)) + at(2, 2);
  const double c = std::min(std::max(0.5 * (tr - 1.0), -1.0), 1.0);
  const double angle = std::acos(c);
  const double sv[3] = {at(2, 1) - at(1, 2), at(0, 2) - at(2, 0), at(1, 0) - at(0, 1)};
  if (angle < 1e-9) {
    for (int i = 0; i < 3; ++i) theta[i] = 0.5 * sv[i];
    return PBAD_OK;
  }
  if (angle > 3.141592653589793 - 1e-6) {
    // near pi: axis from the dominant column of R + I, sign from sv
    double m[9];
    for (int k = 0; k < 9; ++k) m[k] = R[k];
    for (int i = 0; i < 3; ++i) m[i + 3 * i] = m[i + 3 * i] + 1.0;
    int col = 0;
    double best = 0.0;
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int i = 0; i < 3; ++i) acc = std::fma(m[i + 3 * j], m[i + 3 * j], acc);
      const double nj = std::sqrt(acc);
      if (j == 0 || nj > best) { best = nj; col = j; }
    }
    const double* a = m + 3 * col;
    double n2 = a[0] * a[0];
    n2 = std::fma(a[1], a[1], n2);
    n2 = std::fma(a[2], a[2], n2);
    const double n = std::sqrt(n2);
    double axis[3] = {a[0] / n, a[1] / n, a[2] / n};
    double d = sv[0] * axis[0];
    d = std::fma(sv[1], axis[1], d);
    d = std::fma(sv[2], axis[2], d);
    if (d < 0.0)
      for (int i = 0; i < 3; ++i) axis[i] = -axis[i];
    for (int i = 0; i < 3; ++i) theta[i] = angle * axis[i];
    return PBAD_OK;
  }
  double sn, cs;
  pbad_sincos(angle, &sn, &cs);
  const double k = angle * (0.5 / sn);
  for (int i = 0; i < 3; ++i) theta[i] = k * sv[i];
  return PBAD_OK;
}

// build_model, model.cpp:62-112
int32_t pbad_gpu_model_create(const pbad_link_spec* links, int32_t N, pbad_gpu_model** out) {
  *out = nullptr;
  auto m = new pbad_gpu_model();
  m->N = N;
  for (int i = 0; i < N; ++i) {
    const pbad_link_spec& L = links[i];
    if (L.parent >= 0 && L.parent >= i) {
      delete m;
      return fail(PBAD_E_MODEL, "link %d: parent index must be smaller than own index", i);
    }
    if (L.parent < -1) {
      delete m;
      return fail(PBAD_E_MODEL, "link %d: negative parent index", i);
    }
    if (L.joint_kind < 0 || L.joint_kind > 2) {
      delete m;
      return fail(PBAD_E_MODEL, "link %d: unknown joint kind", i);
    }
    double ax[3] = {L.axis[0], L.axis[1], L.axis[2]};
    if (L.joint_kind == PBAD_HINGE) {
      const double nn = std::sqrt(dot3(ax, ax));
      if (std::fabs(nn - 1.0) > 1e-12) {
        if (nn < 1e-12) {
          delete m;
          return fail(PBAD_E_MODEL, "link %d: zero-norm hinge axis", i);
        }
        for (double& v : ax) v = v / nn;
      }
    }
    // check_offset, model.cpp:9-21
    {
      const double* off = L.offset;
      double mx = 0.0;
      for (int j = 0; j < 3; ++j)
        for (int a = 0; a < 3; ++a) {
          double acc = off[4 * a] * off[4 * j];
          acc = std::fma(off[1 + 4 * a], off[1 + 4 * j], acc);
          acc = std::fma(off[2 + 4 * a], off[2 + 4 * j], acc);
          const double d = std::fabs(acc - ((a == j) ? 1.0 : 0.0));
          if ((a == 0 && j == 0) || d > mx) mx = d;
        }
      if (mx > 1e-10) {
        delete m;
        return fail(PBAD_E_MODEL, "link %d: joint offset rotation block is not orthonormal", i);
      }
      if (off[3] != 0.0 || off[7] != 0.0 || off[11] != 0.0 || off[15] != 1.0) {
        delete m;
        return fail(PBAD_E_MODEL, "link %d: joint offset bottom row must be (0,0,0,1)", i);
      }
    }
    m->sample_off.push_back((int)(m->samples.size() / 3));
    if (L.geom_kind == PBAD_GEOM_BOX) {
      if (L.box_density <= 0.0) {
        delete m;
        return fail(PBAD_E_MODEL, "link %d: non-positive density", i);
      }
      if (std::fmin(std::fmin(L.box_size[0], L.box_size[1]), L.box_size[2]) <= 0.0) {
        delete m;
        return fail(PBAD_E_MODEL, "link %d: non-positive box extent", i);
      }
      if (L.n_samples > 0) {
        m->samples.insert(m->samples.end(), L.samples, L.samples + 3 * L.n_samples);
      } else {
        const double h[3] = {0.5 * L.box_size[0], 0.5 * L.box_size[1], 0.5 * L.box_size[2]};
        for (int sx = -1; sx <= 1; sx += 2)
          for (int sy = -1; sy <= 1; sy += 2)
            for (int sz = -1; sz <= 1; sz += 2) {
              m->samples.push_back(L.box_center[0] + (double)sx * h[0]);
              m->samples.push_back(L.box_center[1] + (double)sy * h[1]);
              m->samples.push_back(L.box_center[2] + (double)sz * h[2]);
            }
      }
    } else {
      for (int p = 0; p < L.n_points; ++p)
        if (L.point_mass[p] <= 0.0) {
          delete m;
          return fail(PBAD_E_MODEL, "link %d: non-positive point mass", i);
        }
      if (L.n_samples > 0) m->samples.insert(m->samples.end(), L.samples, L.samples + 3 * L.n_samples);
      else if (L.n_points > 0) m->samples.insert(m->samples.end(), L.point_pos, L.point_pos + 3 * L.n_points);
    }
    double S[16], mass;
    pbad_gpu_body_integral(&L, S, &mass);
    m->parent.push_back(L.parent);
    m->kind.push_back(L.joint_kind);
    m->axis.insert(m->axis.end(), ax, ax + 3);
    m->offset.insert(m->offset.end(), L.offset, L.offset + 16);
    m->S.insert(m->S.end(), S, S + 16);
    m->mass.push_back(mass);
    const int dof = kind_dofs(L.joint_kind);
    m->dof_off.push_back(m->n);
    m->dof_cnt.push_back(dof);
    m->d2_off.push_back(m->n_d2);
    m->n += dof;
    m->n_d2 += dof * (dof + 1) / 2;
  }
  m->sample_off.push_back((int)(m->samples.size() / 3));
  // WeightedBody::make with unit weights, adjoint.cpp:29-41
  double wm = 0.0;
  for (int i = 0; i < N; ++i) wm += 1.0 * m->mass[i];
  m->weighted_mass = wm;
  *out = m;
  return PBAD_OK;
}

void pbad_gpu_model_destroy(pbad_gpu_model* m) { delete m; }
int32_t pbad_gpu_model_dofs(const pbad_gpu_model* m) { return m->n; }
int32_t pbad_gpu_model_links(const pbad_gpu_model* m) { return m->N; }

int32_t pbad_gpu_model_info(const pbad_gpu_model* m, double* S, double* mass, int32_t* dof_offset,
                            double* axis, int32_t* sample_count) {
  for (int i = 0; i < m->N; ++i) {
    if (S) std::memcpy(S + 16 * i, &m->S[16 * i], 16 * sizeof(double));
    if (mass) mass[i] = m->mass[i];
    if (dof_offset) dof_offset[i] = m->dof_off[i];
    if (axis) std::memcpy(axis + 3 * i, &m->axis[3 * i], 3 * sizeof(double));
    if (sample_count) sample_count[i] = m->sample_off[i + 1] - m->sample_off[i];
  }
  return PBAD_OK;
}

// validate_configuration, model.cpp:114-123
int32_t pbad_gpu_validate_configuration(const pbad_gpu_model* m, const double* q, int32_t len) {
  if (len != m->n)
    return fail(PBAD_E_MODEL, "configuration length %d does not match model DOF count %d", len, m->n);
  for (int k = 0; k < len; ++k)
    if (!std::isfinite(q[k])) return fail(PBAD_E_MODEL, "configuration contains a non-finite entry");
  return PBAD_OK;
}

}  // extern "C"

namespace {

// FullPivLU(A).inverse() with the eigen_lite definition.
bool fullpiv_inverse(const double* A_in, int k, double* inv) {
  std::vector<double> A(A_in, A_in + k * k), X(k * k, 0.0);
  std::vector<int> colperm(k);
  for (int i = 0; i < k; ++i) {
    X[i + k * i] = 1.0;
    colperm[i] = i;
  }
  auto AA = [&](int r, int c) -> double& { return A[r + k * c]; };
  auto XX = [&](int r, int c) -> double& { return X[r + k * c]; };
  for (int s = 0; s < k; ++s) {
    int pr = s, pc = s;
    double best = -1.0;
    for (int c = s; c < k; ++c)
      for (int r = s; r < k; ++r)
        if (std::fabs(AA(r, c)) > best) {
          best = std::fabs(AA(r, c));
          pr = r;
          pc = c;
        }
    if (!(best > 0.0)) return false;
    if (pr != s)
      for (int c = 0; c < k; ++c) {
        std::swap(AA(s, c), AA(pr, c));
        std::swap(XX(s, c), XX(pr, c));
      }
    if (pc != s) {
      for (int r = 0; r < k; ++r) std::swap(AA(r, s), AA(r, pc));
      std::swap(colperm[s], colperm[pc]);
    }
    const double piv = AA(s, s);
    for (int c = 0; c < k; ++c) {
      AA(s, c) = AA(s, c) / piv;
      XX(s, c) = XX(s, c) / piv;
    }
    for (int r = 0; r < k; ++r) {
      if (r == s) continue;
      const double f = AA(r, s);
      for (int c = 0; c < k; ++c) {
        AA(r, c) = std::fma(-f, AA(s, c), AA(r, c));
        XX(r, c) = std::fma(-f, XX(s, c), XX(r, c));
      }
    }
  }
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < k; ++c) inv[colperm[r] + k * c] = XX(r, c);
  return true;
}

struct Scheme {
  int order = 2;
  double alphas[8] = {0};
  double times[9] = {0};
  double H[81] = {0};
  double H2[81] = {0};
};

// legendre_points + build_scheme, collocation.cpp:26-95
int32_t build_scheme(int order, double dt, Scheme* s) {
  if (order < 2) return fail(PBAD_E_ARGUMENT, "collocation order must be >= 2");
  if (order > 7) return fail(PBAD_E_UNSUPPORTED, "collocation order above 7 is not supported");
  if (dt <= 0.0) return fail(PBAD_E_ARGUMENT, "dt must be positive");
  *s = Scheme();
  s->order = order;
  const int nr = order - 2;
  for (int i = 0; i < nr; ++i) {
    double sn, cs;
    pbad_sincos(3.141592653589793 * (i + 0.75) / (nr + 0.5), &sn, &cs);
    double x = -cs;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x, pv, dv;
      if (nr == 0) {
        pv = 1.0;
        dv = 0.0;
      } else {
        for (int k = 2; k <= nr; ++k) {
          const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        dv = nr * (x * p1 - p0) / (x * x - 1.0);
        pv = p1;
      }
      const double dx = pv / dv;
      x -= dx;
      if (std::fabs(dx) < 1e-14) break;
    }
    s->alphas[i] = 0.5 * (x + 1.0);
  }
  s->alphas[nr] = 1.0;
  const int k = order + 1;
  if (order == 2) {
    s->times[0] = -1.0;
    s->times[1] = 0.0;
  } else {
    s->times[0] = s->alphas[order - 3] - 1.0;
    s->times[1] = 0.0;
  }
  for (int i = 0; i < order - 1; ++i) s->times[2 + i] = s->alphas[i];
  double V[81];
  for (int j = 0; j < k; ++j) {
    double pw = 1.0;
    for (int p = 0; p < k; ++p) {
      V[p + k * j] = pw;
      pw *= s->times[j];
    }
  }
  if (!fullpiv_inverse(V, k, s->H))
    return fail(PBAD_E_RUNTIME, "collocation times produced a singular Vandermonde system");
  double mono2[81] = {0};
  for (int j = 0; j < k; ++j)
    for (int p = 2; p < k; ++p) mono2[p + k * j] = p * (p - 1) * std::pow(s->times[j], p - 2);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) {
      double acc = s->H[i] * mono2[k * j];
      for (int q = 1; q < k; ++q) acc = std::fma(s->H[i + k * q], mono2[q + k * j], acc);
      s->H2[i + k * j] = acc;
    }
  return PBAD_OK;
}

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) return nullptr;
  return static_cast<T*>(p);
}

template <class T>
bool dupload(T** dst, const std::vector<T>& v) {
  *dst = dalloc<T>(v.size());
  if (!*dst) return false;
  if (!v.empty() && cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
    return false;
  return true;
}

}  // namespace

extern "C" int32_t pbad_gpu_build_scheme(int32_t order, double dt, double* alphas, double* times, double* H,
                                         double* H2) {
  Scheme s;
  const int32_t rc = build_scheme(order, dt, &s);
  if (rc) return rc;
  const int k = order + 1;
  if (alphas) std::memcpy(alphas, s.alphas, sizeof(double) * (order - 1));
  if (times) std::memcpy(times, s.times, sizeof(double) * k);
  if (H) std::memcpy(H, s.H, sizeof(double) * k * k);
  if (H2) std::memcpy(H2, s.H2, sizeof(double) * k * k);
  return PBAD_OK;
}

struct pbad_gpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  pbad_gpu_model model;
  KernelArgs ka{};
  ChainArgs ca{};
  bool chain = false;      // rollouts use the quad chain kernels
  bool chain4 = false;     // ... in their warp-synchronous v4 form (pbad_chain4.cu)
  bool chain5 = false;     // ... or warp per environment, v5 (pbad_chain5.cu)
  bool chain6 = false;     // ... or two lanes per row, v6 (pbad_chain6.cu)
  bool chain7 = false;     // ... or 16 lanes per environment, link-parallel terms, v7 (pbad_chain7.cu)
  int chain4_pat = 0;      // v4 link-pattern instantiation
  long chain4_recw = 0;    // v4 record doubles per warp
  long v1_per_env = 0;     // general-kernel workspace size (allocated lazily)
  long chain_per_env = 0;
  bool tree = false;       // rollouts use the warp-per-env Newton kernel (pbad_tree.cu)
  TreeDesc td{};
  double* tws = nullptr;   // tree-path per-env workspace (GN, history transforms)
  int* tsync = nullptr;    // tree / residual multi-step launches: task counter + per-env step flags
  long launches = 0;       // step kernels launched by advance_steps (pbad_gpu_kernel_launches)
  bool resid = false;      // rollouts use the CTA-per-env residual-form kernel (pbad_resid.cu)
  ResidDesc rd{};
  double* rws = nullptr;
  std::vector<void*> owned;  // device allocations freed at destroy
  long max_batch = 0;
  long B = 0;  // current batch
  int total_steps = 0;
  int steps_done = 0;
  // device outputs for the current batch
  Outputs dout{};
  long out_q_cap = 0, out_r_cap = 0;  // allocated sample / report slots
  double* d_itv = nullptr;             // per_iteration_values slots (on request)
  bool refined = false;                // refined_bootstrap (stepper.cpp:46-59)
  double boot_hs = 0.0;                // its RK4 substep span / 32
  double* d_boot_ws = nullptr;         // bootstrap workspace, hist0 [B][n], status [B]
  double* d_boot_h0 = nullptr;
  int* d_boot_st = nullptr;
  long boot_cap = 0;
  long itv_cap = 0;
  int max_iters = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_work = nullptr;       // orders the ctx stream after a caller's stream
  cudaStream_t work_stream = nullptr;  // stream of the last begin/advance
  double device_ms = 0.0;
  double* d_q0 = nullptr;
  double* d_qd0 = nullptr;
  double* d_in = nullptr;  // eval/minimize staging
  long in_cap = 0;
  ~pbad_gpu_ctx() {
    if (device >= 0) cudaSetDevice(device);
    for (void* p : owned) cudaFree(p);
    if (dout.q) cudaFree(dout.q);
    if (dout.energy) cudaFree(dout.energy);
    if (dout.iterations) cudaFree(dout.iterations);
    if (dout.converged) cudaFree(dout.converged);
    if (dout.accepted) cudaFree(dout.accepted);
    if (dout.final_value) cudaFree(dout.final_value);
    if (dout.final_grad_norm) cudaFree(dout.final_grad_norm);
    if (d_in) cudaFree(d_in);
    if (d_itv) cudaFree(d_itv);
    if (d_boot_ws) cudaFree(d_boot_ws);
    if (d_boot_h0) cudaFree(d_boot_h0);
    if (d_boot_st) cudaFree(d_boot_st);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev_work) cudaEventDestroy(ev_work);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

Layout make_layout(const pbad_gpu_model& m, int order, int objective, int opt_kind, int mem, long* total) {
  Layout L{};
  const long N = m.N, n = m.n, n_d2 = m.n_d2;
  const long u = order - 1, U = n * u;
  const bool lm = opt_kind == PBAD_LM;
  const bool resid = objective == PBAD_RESIDUAL_FORM;
  long o = 0;
  auto take = [&](long cnt) {
    const long at = o;
    o += cnt;
    return at;
  };
  L.hist0 = take(n);
  L.hist1 = take(n);
  L.x = take(U);
  L.grad = take(U);
  L.cand = take(U);
  L.dir = take(U);
  L.tmp = take(U);
  L.step = take(U > n ? U : n);
  L.evgrad = take(U);
  L.hs = take(lm ? 0 : (mem + 1) * U);
  L.hy = take(lm ? 0 : (mem + 1) * U);
  L.hsy = take(mem + 1);
  L.alpha = take(mem + 1);
  L.tau = take(U);
  L.hw0 = take(N * 16);
  L.hw1 = take(N * 16);
  L.gn = take(lm ? U * U : 0);
  L.damped = take(lm ? U * U : 0);
  L.evgn = take(lm ? U * U : 0);
  L.p_value = 0;
  L.p_d1 = N * 16;
  L.p_world = L.p_d1 + n * 16;
  L.p_lever = L.p_world + N * 16;
  L.p_d2 = L.p_lever + n * 16;
  L.pass_stride = L.p_d2 + (resid ? n_d2 * 16 : 0);
  L.pass = take(u * L.pass_stride);
  L.seeds = take(N * 16);
  L.cot = take(N * 16);
  L.adj = take(N * 16);
  const bool need_nn = lm || resid;
  L.potgrad = take(n);
  L.potgn = take(need_nn ? n * n : 0);
  L.pothess = take(resid ? n * n : 0);
  L.ab = take(need_nn ? n * n : 0);
  L.fh = take(resid ? n * n : 0);
  L.resid = take(resid ? U : 0);
  L.J = take(resid ? U * U : 0);
  L.g = take(n);
  L.jx = take(3 * n);
  L.dd = take(n);
  L.jr = take(3 * n);
  L.tmp3 = take(3 * n);
  L.scal = take(SC_COUNT);
  L.total = o;
  *total = o;
  return L;
}

ChainLayout make_chain_layout(const pbad_gpu_model& m, int mem, long B, long rec_w, long* total) {
  // per-warp blocks of 8 environments (pbad_chain.cu): link arrays
  // [warp][N][32 lanes x 4], vectors [warp][n4][32 lanes]; v4 (rec_w > 0):
  // per-warp link records [warp][rec_w] and history rotations [warp][N][8][6]
  // instead of the link arrays
  ChainLayout L{};
  const long N = m.N, n4 = (m.n + 3) / 4, nw = (B + 7) / 8;
  // vectors: the v3/v4 quad layout or the v6 8-lane layout, whichever is larger
  const long link = rec_w > 0 ? 0 : nw * N * 128, vec = std::max(std::max(nw * n4 * 32, chain6_vector_doubles(B, m.n)), chain7_vector_doubles(B, m.n));
  long o = 0;
  auto take = [&](long cnt) {
    const long at = o;
    o += (cnt + 31) / 32 * 32;  // 256-byte aligned regions (TMA sources)
    return at;
  };
  if (rec_w > 0) {
    L.rec_w = rec_w;
    L.rec = take(nw * rec_w);
    L.hist = take(nw * N * chain4_hist_doubles());
  }
  L.tk = take(link);
  L.tk1 = take(link);
  L.seed = take(link);
  L.lev = take(link);
  L.lmat = take(link);
  L.vstride = vec;
  L.h0 = take(vec);
  L.h1 = take(vec);
  L.x = take(vec);
  L.g = take(vec);
  L.cand = take(vec);
  L.dir = take(vec);
  L.q = take(vec);
  L.evg = take(vec);
  L.tau = take(vec);
  L.hs = take((mem + 1) * vec);
  L.hy = take((mem + 1) * vec);
  L.hsy = take((mem + 1) * B);
  L.histc = take(B);
  L.total = o;
  *total = o;
  return L;
}

// v4 additionally needs every joint axis-aligned with an identity offset
// rotation (link classes 1..3) and its shared-memory footprint to fit.
bool chain4_eligible(const std::vector<int>& ck, int N, int mem) {
  if (std::getenv("PBAD_GPU_CHAIN_V3")) return false;
  if (mem > chain4_max_memory()) return false;
  for (int i = 0; i < N; ++i)
    if ((ck[i] & 3) == 0) return false;
  return chain4_smem_bytes(N) <= 227 * 1024;
}

// The quad chain kernels cover serial hinge chains, energy form, L-BFGS,
// gravity / constant or sinusoidal actuation (no drag or contact).
bool chain_eligible(const pbad_gpu_model& m, const pbad_forces* f, const pbad_sim_desc* sim) {
  if (std::getenv("PBAD_GPU_FORCE_GENERAL")) return false;
  if (sim->objective != PBAD_ENERGY_FORM || sim->order != 2 || sim->opt.kind != PBAD_LBFGS) return false;
  if (sim->opt.lbfgs_memory < 0 || sim->opt.lbfgs_memory > chain_max_memory()) return false;
  if (m.N > chain_max_links()) return false;
  if (f->drag_d > 0.0) return false;
  if (f->has_contact && (f->contact_d1 > 0.0 || f->contact_d2 > 0.0)) return false;
  for (int i = 0; i < m.N; ++i) {
    if (m.kind[i] != PBAD_HINGE) return false;
    if (m.parent[i] != i - 1) return false;
  }
  return true;
}

// The tree kernel covers any tree with the energy form, LM (Newton) or
// L-BFGS: gravity, drag, ground contact, constant or sinusoidal actuation
// (serial hinge chains with L-BFGS go to the chain kernels first).
bool tree_eligible(const pbad_gpu_model& m, const pbad_forces* f, const pbad_sim_desc* sim) {
  if (std::getenv("PBAD_GPU_FORCE_GENERAL")) return false;
  if (sim->objective != PBAD_ENERGY_FORM || sim->order != 2) return false;
  if (sim->opt.kind == PBAD_LBFGS && (sim->opt.lbfgs_memory < 0 || sim->opt.lbfgs_memory > 64)) return false;
  if (!tree_eligible_sizes(m.N, m.n)) return false;
  if (m.sample_off[m.N] > 1024) return false;
  for (int i = 0; i < m.N; ++i)
    if (m.dof_cnt[i] > 6) return false;
  return true;
}

// The residual-form kernel covers hinge trees with the residual objective and
// LM (the high-order collocation Newton path), gravity / drag / actuation /
// contact.
bool resid_eligible(const pbad_gpu_model& m, const pbad_forces* f, const pbad_sim_desc* sim) {
  if (std::getenv("PBAD_GPU_FORCE_GENERAL")) return false;
  if (sim->objective != PBAD_RESIDUAL_FORM || sim->opt.kind != PBAD_LM) return false;
  if (sim->order < 2 || sim->order - 1 > 8) return false;
  // contact: the per-sample terms of potential_terms (objective.cpp:74-126)
  // with a cotangent every instant (gravity or drag present, so have_cot is
  // constant) and a bounded sample count (the per-sample Jacobian buffer)
  if (f->has_contact && (f->contact_d1 > 0.0 || f->contact_d2 > 0.0)) {
    const bool grav = f->gravity[0] != 0.0 || f->gravity[1] != 0.0 || f->gravity[2] != 0.0;
    if (!grav && !(f->drag_d > 0.0)) return false;
    if (m.sample_off[m.N] > 1024) return false;
  }
  for (int i = 0; i < m.N; ++i)
    if (m.kind[i] != PBAD_HINGE) return false;
  return resid_eligible_sizes(m.N, sim->order - 1);
}

// ... and the energy form with LM on hinge trees the warp-per-environment tree
// kernel cannot hold (n > 96 or its shared-memory footprint): the same CTA per
// environment, u = 1 (pbad_resid.cu "energy form")
bool resid_energy_eligible(const pbad_gpu_model& m, const pbad_forces* f, const pbad_sim_desc* sim) {
  if (std::getenv("PBAD_GPU_FORCE_GENERAL")) return false;
  if (sim->objective != PBAD_ENERGY_FORM || sim->order != 2 || sim->opt.kind != PBAD_LM) return false;
  if (f->drag_d > 0.0) return false;
  if (f->has_contact && (f->contact_d1 > 0.0 || f->contact_d2 > 0.0)) return false;
  for (int i = 0; i < m.N; ++i)
    if (m.kind[i] != PBAD_HINGE) return false;
  return resid_eligible_sizes(m.N, 1);
}

// Host-side structure of the tree kernel: depth levels, children in
// descending index (the reference's accumulation order, adjoint.cpp:54-62),
// ancestor table and the GN task list (adjoint.cpp:132-176 loop nest).
struct TreeHost {
  std::vector<int> lvl_start, lvl_links, ch_start, ch_list, task_start, tasks, anc, depth, pk, dof_link;
  int D = 0;
};

TreeHost make_tree_host(const pbad_gpu_model& m) {
  TreeHost h;
  const int N = m.N, n = m.n;
  h.depth.assign(N, 0);
  for (int i = 0; i < N; ++i) h.depth[i] = m.parent[i] >= 0 ? h.depth[m.parent[i]] + 1 : 0;
  for (int i = 0; i < N; ++i) h.D = std::max(h.D, h.depth[i]);
  const int D = h.D;
  h.lvl_start.assign(D + 2, 0);
  for (int d = 0; d <= D; ++d) {
    h.lvl_start[d] = (int)h.lvl_links.size();
    for (int i = 0; i < N; ++i)
      if (h.depth[i] == d) h.lvl_links.push_back(i);
  }
  h.lvl_start[D + 1] = (int)h.lvl_links.size();
  h.ch_start.assign(N + 1, 0);
  for (int p = 0; p < N; ++p) {
    h.ch_start[p] = (int)h.ch_list.size();
    for (int c = N - 1; c > p; --c)
      if (m.parent[c] == p) h.ch_list.push_back(c);
  }
  h.ch_start[N] = (int)h.ch_list.size();
  h.anc.assign((size_t)N * (D + 1), -1);
  for (int i = 0; i < N; ++i) {
    int l = i;
    for (int s = 0; s <= D && l >= 0; ++s, l = m.parent[l]) h.anc[(size_t)i * (D + 1) + s] = l;
  }
  h.task_start.assign(D + 2, 0);
  for (int s = 0; s <= D; ++s) {
    h.task_start[s] = (int)h.tasks.size();
    for (int i = 0; i < N; ++i) {
      if (h.depth[i] < s) continue;
      const int l = h.anc[(size_t)i * (D + 1) + s];
      for (int j = 0; j < m.dof_cnt[i]; ++j)
        for (int k = (s == 0 ? j : 0); k < m.dof_cnt[l]; ++k) h.tasks.push_back(i | (l << 8) | (j << 16) | (k << 20));
    }
  }
  h.task_start[D + 1] = (int)h.tasks.size();
  for (int col = 0; col < n; ++col)
    for (int row = col; row < n; ++row) h.pk.push_back(row | (col << 16));
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < m.dof_cnt[i]; ++j) h.dof_link.push_back(i);
  return h;
}

bool ensure_v1(pbad_gpu_ctx* c) {
  if (c->ka.ws) return true;
  double* ws = dalloc<double>((size_t)c->v1_per_env * c->max_batch);
  int* iws = dalloc<int>((size_t)IS_COUNT * c->max_batch);
  if (!ws || !iws) {
    cudaFree(ws);
    cudaFree(iws);
    return false;
  }
  c->owned.push_back(ws);
  c->owned.push_back(iws);
  c->ka.ws = ws;
  c->ka.iws = iws;
  return true;
}

// Device outputs for B environments and a window of W steps: W + 1 sample
// slots and W report slots per environment (W = S: the whole trajectory).
int32_t ensure_outputs(pbad_gpu_ctx* c, long B, long W, bool want_itv = false) {
  const long n = c->model.n;
  const long need_q = B * (W + 1), need_r = B * W;
  const long mi = std::max(1, c->max_iters);
  if (want_itv && c->itv_cap < need_r * mi) {
    cudaFree(c->d_itv);
    c->d_itv = dalloc<double>(need_r * mi);
    if (!c->d_itv) {
      c->itv_cap = 0;
      return fail(PBAD_E_CUDA, "cudaMalloc of per_iteration_values failed (B=%ld, window %ld steps)", B, W);
    }
    c->itv_cap = need_r * mi;
  }
  c->dout.itv = want_itv ? c->d_itv : nullptr;
  c->dout.itv_n = mi;
  if (c->out_q_cap < need_q || c->out_r_cap < need_r) {
    cudaFree(c->dout.q);
    cudaFree(c->dout.energy);
    cudaFree(c->dout.iterations);
    cudaFree(c->dout.converged);
    cudaFree(c->dout.accepted);
    cudaFree(c->dout.final_value);
    cudaFree(c->dout.final_grad_norm);
    double* itv = c->dout.itv;
    c->dout = Outputs{};
    c->dout.itv = itv;
    c->dout.itv_n = mi;
    c->out_q_cap = c->out_r_cap = 0;
    c->dout.q = dalloc<double>(need_q * n);
    c->dout.energy = dalloc<double>(need_q * 2);
    c->dout.iterations = dalloc<int>(need_r);
    c->dout.converged = dalloc<int>(need_r);
    c->dout.accepted = dalloc<int>(need_r);
    c->dout.final_value = dalloc<double>(need_r);
    c->dout.final_grad_norm = dalloc<double>(need_r);
    if (!c->dout.q || !c->dout.energy || !c->dout.iterations || !c->dout.converged || !c->dout.accepted ||
        !c->dout.final_value || !c->dout.final_grad_norm)
      return fail(PBAD_E_CUDA, "cudaMalloc of rollout outputs failed (B=%ld, window %ld steps)", B, W);
    c->out_q_cap = need_q;
    c->out_r_cap = need_r;
  }
  c->dout.qs = W + 1;
  c->dout.rs = W;
  c->dout.qbase = 0;
  c->dout.rbase = 0;
  return PBAD_OK;
}

// Steps per output window of a rollout: the whole trajectory when its
// samples fit the budget (PBAD_TRAJ_WINDOW_MB, default 2048 MB of device
// memory), else the largest window that does; windows are drained to the
// host between launches so a rollout's device footprint does not grow with S.
long window_steps(const pbad_gpu_ctx* c, long B, bool want_itv) {
  const long S = c->total_steps, n = c->model.n;
  double mb = 2048.0;
  if (const char* e = std::getenv("PBAD_TRAJ_WINDOW_MB")) mb = std::atof(e);
  const double per_step = (double)B * (8.0 * (n + 2) + 4.0 * 3 + 16.0 + (want_itv ? 8.0 * std::max(1, c->max_iters) : 0.0));
  long W = (long)(mb * 1048576.0 / per_step) - 1;
  return std::max(1L, std::min(S, W));
}

cudaStream_t pick(pbad_gpu_ctx* c, void* s) { return s ? static_cast<cudaStream_t>(s) : c->stream; }

}  // namespace

extern "C" {

int32_t pbad_gpu_create(const pbad_gpu_model* model, const pbad_forces* f, const pbad_sim_desc* sim,
                        int32_t device, int32_t max_batch, pbad_gpu_ctx** out) {
  *out = nullptr;
  if (!model || !f || !sim) return fail(PBAD_E_ARGUMENT, "null argument");
  if (max_batch < 1) return fail(PBAD_E_ARGUMENT, "max_batch must be >= 1");
  // lbfgs_memory <= 0: the reference pushes and immediately pops every pair
  // (optim.cpp:183-186), i.e. steepest descent -- the same as memory 0
  pbad_sim_desc sim_eff = *sim;
  sim_eff.opt.lbfgs_memory = std::max(0, sim->opt.lbfgs_memory);
  sim = &sim_eff;
  if (sim->dt <= 0.0 || sim->duration <= 0.0) return fail(PBAD_E_MODEL, "dt and duration must be positive");
  // init_pbad_run's build_scheme (stepper.cpp:70) runs before the first
  // StepObjective (objective.cpp:167-168) checks the energy form's order
  Scheme scheme;
  int32_t rc = build_scheme(sim->order, sim->dt, &scheme);
  if (rc) return rc;
  if (sim->objective == PBAD_ENERGY_FORM && sim->order != 2)
    return fail(PBAD_E_MODEL, "the energy objective is only defined for order 2");

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(PBAD_E_CUDA, "no CUDA device available (the PBAD GPU path has no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(PBAD_E_CUDA, "device %d out of range (%d devices)", device, ndev);
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(PBAD_E_CUDA, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor);

  auto c = new pbad_gpu_ctx();
  c->device = device;
  c->model = *model;
  c->max_batch = max_batch;
  const pbad_gpu_model& m = c->model;
  c->total_steps = (int)std::ceil(sim->duration / sim->dt - 1e-9);
  c->max_iters = sim->opt.max_iters;
  c->refined = sim->refined_bootstrap != 0;
  {
    const double t_local_dt = scheme.times[0] * sim->dt;  // stepper.cpp:72, 46-59
    const double span = -t_local_dt;
    c->boot_hs = span / 32;
  }

  auto up_i = [&](const std::vector<int>& v) -> const int* {
    int* d = nullptr;
    if (!dupload(&d, v)) return nullptr;
    c->owned.push_back(d);
    return d;
  };
  auto up_d = [&](const std::vector<double>& v) -> const double* {
    double* d = nullptr;
    if (!dupload(&d, v)) return nullptr;
    c->owned.push_back(d);
    return d;
  };
  DModel dm{};
  dm.N = m.N;
  dm.n = m.n;
  dm.n_d2 = m.n_d2;
  dm.parent = up_i(m.parent);
  dm.kind = up_i(m.kind);
  dm.dof_off = up_i(m.dof_off);
  dm.dof_cnt = up_i(m.dof_cnt);
  dm.d2_off = up_i(m.d2_off);
  dm.axis = up_d(m.axis);
  dm.offset = up_d(m.offset);
  dm.S = up_d(m.S);
  dm.mass = up_d(m.mass);
  dm.sample_off = up_i(m.sample_off);
  dm.samples = up_d(m.samples);
  dm.weighted_mass = m.weighted_mass;
  {
    // chain-kernel link classes (exact structure tests, see pbad_chain.cu)
    std::vector<int> jk(m.N, 0), sk(m.N, 1);
    for (int i = 0; i < m.N; ++i) {
      const double* o = &m.offset[16 * i];
      const bool rot_identity = o[0] == 1.0 && o[1] == 0.0 && o[2] == 0.0 && o[4] == 0.0 && o[5] == 1.0 &&
                                o[6] == 0.0 && o[8] == 0.0 && o[9] == 0.0 && o[10] == 1.0;
      const double* a = &m.axis[3 * i];
      if (m.kind[i] == PBAD_HINGE && rot_identity) {
        if (a[0] == 1.0 && a[1] == 0.0 && a[2] == 0.0) jk[i] = 1;
        if (a[0] == 0.0 && a[1] == 1.0 && a[2] == 0.0) jk[i] = 2;
        if (a[0] == 0.0 && a[1] == 0.0 && a[2] == 1.0) jk[i] = 3;
      }
      bool zero = true;
      for (int k = 0; k < 16; ++k) zero = zero && m.S[16 * i + k] == 0.0;
      sk[i] = zero ? 0 : 1;
    }
    if (std::getenv("PBAD_GPU_NO_SPECIALIZE")) {
      std::fill(jk.begin(), jk.end(), 0);
      std::fill(sk.begin(), sk.end(), 1);
    }
    dm.jkind = up_i(jk);
    dm.skind = up_i(sk);
    std::vector<double> rec(20 * (size_t)m.N, 0.0);
    std::vector<int> ck(m.N);
    for (int i = 0; i < m.N; ++i) {
      for (int k = 0; k < 16; ++k) rec[20 * i + k] = m.S[16 * i + k];
      for (int k = 0; k < 3; ++k) rec[20 * i + 16 + k] = m.offset[16 * i + 12 + k];
      ck[i] = jk[i] | (sk[i] << 2);
    }
    dm.crec = up_d(rec);
    dm.ckind = up_i(ck);
    std::vector<int> roff(m.N + 1, 0);
    for (int i = 0; i < m.N; ++i) roff[i + 1] = roff[i] + (int)chain4_record_doubles(sk[i] != 0);
    dm.croff = up_i(roff);
    c->chain4 = chain4_eligible(ck, m.N, sim->opt.lbfgs_memory);
    c->chain4_pat = chain4_pattern(ck.data(), m.N);
    // v5 (warp per environment) while the batch fits one wave of resident
    // blocks, else v6 (two lanes per row); PBAD_GPU_CHAIN_V5 / _V6 / _V4 force one
    const int waves = chain5_waves(m.N, m.n, sim->opt.lbfgs_memory, max_batch, c->chain4_pat, device);
    c->chain5 = c->chain4 && !std::getenv("PBAD_GPU_CHAIN_V4") && !std::getenv("PBAD_GPU_CHAIN_V6") &&
                !std::getenv("PBAD_GPU_CHAIN_V7") &&
                (std::getenv("PBAD_GPU_CHAIN_V5") ? waves > 0 : waves == 1);
    c->chain4_recw = roff[m.N];
  }

  DForces df{};
  for (int k = 0; k < 3; ++k) df.gravity[k] = f->gravity[k];
  df.gravity_nonzero = !(std::fabs(f->gravity[0]) <= 1e-12 && std::fabs(f->gravity[1]) <= 1e-12 &&
                         std::fabs(f->gravity[2]) <= 1e-12);
  df.drag_d = f->drag_d;
  df.has_contact = f->has_contact;
  for (int k = 0; k < 3; ++k) df.normal[k] = f->plane_normal[k];
  df.plane_offset = f->plane_offset;
  df.d1 = f->contact_d1;
  df.d2 = f->contact_d2;
  df.tau_len = f->tau_len;
  df.tau = f->tau_len > 0 ? up_d(std::vector<double>(f->tau, f->tau + f->tau_len)) : nullptr;
  df.has_act = f->has_actuation;
  df.act_kind = f->act_kind;
  df.act_len = f->act_len;
  df.act_amp = f->act_len > 0 ? up_d(std::vector<double>(f->act_amplitude, f->act_amplitude + f->act_len)) : nullptr;
  df.act_freq = f->act_frequency_hz;
  df.act_phase_len = f->act_phase_len;
  df.act_phase = f->act_phase_len > 0 ? up_d(std::vector<double>(f->act_phase, f->act_phase + f->act_phase_len))
                                      : nullptr;

  DSchedule ds{};
  ds.dt = sim->dt;
  ds.order = sim->order;
  ds.objective = sim->objective;
  ds.u = sim->order - 1;
  ds.U = m.n * ds.u;
  ds.K1 = sim->order + 1;
  ds.fail_limit = sim->consecutive_fail_limit;
  ds.warm_start = sim->warm_start;
  ds.total_steps = c->total_steps;
  std::memcpy(ds.times, scheme.times, sizeof scheme.times);
  std::memcpy(ds.H2, scheme.H2, sizeof scheme.H2);
  ds.opt.kind = sim->opt.kind;
  ds.opt.max_iters = sim->opt.max_iters;
  ds.opt.mem = sim->opt.lbfgs_memory;
  ds.opt.max_line_search = sim->opt.max_line_search;
  ds.opt.grad_tol = sim->opt.grad_tol;
  ds.opt.grad_rtol = sim->opt.grad_rtol;
  ds.opt.ftol = sim->opt.ftol;
  ds.opt.lm_lambda0 = sim->opt.lm_lambda0;
  ds.opt.lm_lambda_factor = sim->opt.lm_lambda_factor;
  ds.opt.lm_lambda_max = sim->opt.lm_lambda_max;
  ds.opt.armijo_c1 = sim->opt.armijo_c1;
  ds.opt.backtrack_factor = sim->opt.backtrack_factor;

  long per_env = 0;
  const Layout L = make_layout(m, sim->order, sim->objective, sim->opt.kind,
                               sim->opt.lbfgs_memory > 0 ? sim->opt.lbfgs_memory : 1, &per_env);
  c->v1_per_env = per_env;
  c->ka = KernelArgs{dm, df, ds, L, nullptr, nullptr, max_batch};
  c->chain = chain_eligible(m, f, sim);
  c->chain4 = c->chain4 && c->chain;
  c->chain5 = c->chain5 && c->chain4;
  // beyond one v5 wave: v6 (two lanes per row) unless PBAD_GPU_CHAIN_V4
  c->chain6 = c->chain4 && !c->chain5 && !std::getenv("PBAD_GPU_CHAIN_V4") &&
              chain6_fits(m.N, sim->opt.lbfgs_memory);
  // v7 (16 lanes per environment, link-parallel energy terms) only on request
  // (PBAD_GPU_CHAIN_V7): it is bit-exact but measured slower than v6 on C3
  // (DESIGN.md 3).  It takes a massive link's row-3 energy term as S(3,3)
  // exactly, which needs S(3,3) != 0 (pbad_chain7.cu)
  if (c->chain6 && std::getenv("PBAD_GPU_CHAIN_V7") && chain7_fits(m.N, sim->opt.lbfgs_memory, c->chain4_pat)) {
    bool s33 = true;
    for (int i = 0; i < m.N; ++i) {
      bool massive = false;
      for (int k = 0; k < 16; ++k) massive = massive || m.S[16 * i + k] != 0.0;
      if (massive && m.S[16 * i + 15] == 0.0) s33 = false;
    }
    c->chain7 = s33;
    c->chain6 = !s33;
  }
  // PBAD_GPU_RESID_ENERGY: energy-form LM on the CTA kernel even where the
  // tree kernel fits (tests compare the two)
  c->tree = !c->chain && tree_eligible(m, f, sim) &&
            !(std::getenv("PBAD_GPU_RESID_ENERGY") && resid_energy_eligible(m, f, sim));
  if (c->tree) {
    const TreeHost th = make_tree_host(m);
    TreeDesc& td = c->td;
    td.N = m.N;
    td.n = m.n;
    td.D = th.D;
    td.np = m.n * (m.n + 1) / 2;
    td.n_tasks = (int)th.tasks.size();
    td.lvl_start = up_i(th.lvl_start);
    td.lvl_links = up_i(th.lvl_links);
    td.ch_start = up_i(th.ch_start);
    td.ch_list = th.ch_list.empty() ? up_i(std::vector<int>(1, 0)) : up_i(th.ch_list);
    td.task_start = up_i(th.task_start);
    td.tasks = up_i(th.tasks);
    td.anc = up_i(th.anc);
    td.depth = up_i(th.depth);
    td.pk = up_i(th.pk);
    td.dof_link = up_i(th.dof_link);
    const long np2 = (td.np + 3) & ~3L, N16 = 16L * m.N;
    td.o_hw0 = np2;
    td.o_hw1 = np2 + N16;
    td.o_t0 = np2 + 2 * N16;
    td.o_t1 = np2 + 3 * N16;
    td.o_gs = np2 + 4 * N16;
    td.pot = (f->drag_d > 0.0 || (f->has_contact && (f->contact_d1 > 0.0 || f->contact_d2 > 0.0))) ? 1 : 0;
    td.ns = (f->has_contact && (f->contact_d1 > 0.0 || f->contact_d2 > 0.0)) ? m.sample_off[m.N] : 0;
    td.o_abl = td.o_gs + 4 * 18L * m.N;
    td.o_abu = td.o_abl + (td.pot ? np2 : 0);
    td.o_cs = td.o_abu + (td.pot ? np2 : 0);
    td.lb = sim->opt.kind == PBAD_LBFGS ? 1 : 0;
    const long cap = td.lb ? sim->opt.lbfgs_memory + 1 : 0;
    td.o_hs = td.o_cs + 4L * m.n * td.ns;
    td.o_hy = td.o_hs + ((cap * m.n + 1) & ~1L);
    td.o_hsy = td.o_hy + ((cap * m.n + 1) & ~1L);
    td.o_alpha = td.o_hsy + ((cap + 1) & ~1L);
    td.gstride = td.o_alpha + ((cap + 1) & ~1L);
    td.smem_doubles = (int)(tree_smem_bytes(td) / sizeof(double));
    if (tree_smem_bytes(td) > 200 * 1024) c->tree = false;
  }
  if (!dm.parent || !dm.S) {
    delete c;
    return fail(PBAD_E_CUDA, "cudaMalloc of the model failed");
  }
  if (c->chain) {
    long tot = 0;
    const long rec_w = c->chain4 ? c->chain4_recw : 0;
    const ChainLayout CL = make_chain_layout(m, sim->opt.lbfgs_memory, max_batch, rec_w, &tot);
    double* cw = dalloc<double>((size_t)tot);
    int* ci = dalloc<int>((size_t)IS_COUNT * max_batch);
    if (!cw || !ci) {
      cudaFree(cw);
      cudaFree(ci);
      delete c;
      return fail(PBAD_E_CUDA, "cudaMalloc failed (chain workspace %.1f MB)", tot * 8.0 / 1e6);
    }
    c->owned.push_back(cw);
    c->owned.push_back(ci);
    c->chain_per_env = tot / max_batch;
    c->ca = ChainArgs{dm, df, ds, CL, cw, ci, max_batch};
  } else if (!ensure_v1(c)) {
    delete c;
    return fail(PBAD_E_CUDA, "cudaMalloc failed (workspace %.1f MB)", per_env * 8.0 * max_batch / 1e6);
  }
  c->resid = !c->chain && !c->tree && (resid_eligible(m, f, sim) || resid_energy_eligible(m, f, sim));
  if (c->resid) {
    const TreeHost th = make_tree_host(m);
    ResidDesc& rd = c->rd;
    const long N = m.N, n = m.n, u = sim->order - 1, U = n * u;
    rd.N = m.N;
    rd.n = m.n;
    rd.u = (int)u;
    rd.U = (int)U;
    rd.D = th.D;
    const bool contact = f->has_contact && (f->contact_d1 > 0.0 || f->contact_d2 > 0.0);
    bool chain = !contact;  // contact terms run on the tree walks (pot.hess before functional_hess)
    for (int i = 0; i < m.N; ++i) chain = chain && m.parent[i] == i - 1;
    rd.chain = chain;
    rd.ns = contact ? m.sample_off[m.N] : 0;
    rd.lvl_start = up_i(th.lvl_start);
    rd.lvl_links = up_i(th.lvl_links);
    rd.ch_start = up_i(th.ch_start);
    rd.ch_list = th.ch_list.empty() ? up_i(std::vector<int>(1, 0)) : up_i(th.ch_list);
    std::vector<int> wo(m.N);
    for (int i = 0; i < m.N; ++i) wo[i] = i;
    std::stable_sort(wo.begin(), wo.end(), [&](int a, int b) { return th.depth[a] > th.depth[b]; });
    rd.walk_order = up_i(wo);
    rd.pstride = 80 * N;
    long o = 0;
    auto take = [&](long cnt) {
      const long at = o;
      o += (cnt + 1) & ~1L;
      return at;
    };
    rd.oJ = take(U * U);
    rd.oGN = take(U * U);
    rd.oDM = take(U * U);
    const bool energy = sim->objective == PBAD_ENERGY_FORM;  // no functional_hess blocks
    rd.oFH = take(energy ? 0 : u * n * n);
    rd.oPH = take(energy ? 0 : u * n * n);
    rd.oPass = take(u * rd.pstride);
    rd.oHW0 = take(16 * N);
    rd.oHW1 = take(16 * N);
    rd.oHA = take(u * u * 4 * 16 * N);
    rd.oFA = take(2 * u * 2 * 16 * N);
    rd.oSeeds = take(u * 16 * N);
    rd.oCot = take((f->drag_d > 0.0 || rd.ns ? u : 1) * 16 * N);  // per-instant cotangents with drag / contact
    rd.oCJ = take(u * rd.ns * (3 * n + 10));  // contact: per (instant, sample) hxx, active flag, 3 x n Jacobian
    rd.oX = take(U);
    rd.oGrad = take(U);
    rd.oCand = take(std::max(U, 2 * n));
    rd.oRes = take(U);
    rd.oPg = take(U);
    rd.oTau = take(U);
    rd.oStep = take(U);
    rd.gstride = (o + 31) & ~31L;
    if (!ensure_v1(c)) {
      delete c;
      return fail(PBAD_E_CUDA, "cudaMalloc failed (workspace %.1f MB)", per_env * 8.0 * max_batch / 1e6);
    }
    c->rws = dalloc<double>((size_t)rd.gstride * max_batch);
    if (!c->rws) {
      delete c;
      return fail(PBAD_E_CUDA, "cudaMalloc failed (residual workspace %.1f MB)", rd.gstride * 8.0 * max_batch / 1e6);
    }
    c->owned.push_back(c->rws);
    double* ts = dalloc<double>((size_t)(max_batch + 2) / 2 + 1);
    if (!ts) {
      delete c;
      return fail(PBAD_E_CUDA, "cudaMalloc failed (residual step flags)");
    }
    c->owned.push_back(ts);
    c->tsync = reinterpret_cast<int*>(ts);
  }
  if (c->tree) {
    c->tws = dalloc<double>((size_t)c->td.gstride * max_batch);
    if (!c->tws) {
      delete c;
      return fail(PBAD_E_CUDA, "cudaMalloc failed (tree workspace %.1f MB)", c->td.gstride * 8.0 * max_batch / 1e6);
    }
    c->owned.push_back(c->tws);
    double* ts = dalloc<double>((size_t)(max_batch + 2) / 2 + 1);
    if (!ts) {
      delete c;
      return fail(PBAD_E_CUDA, "cudaMalloc failed (tree step flags)");
    }
    c->owned.push_back(ts);
    c->tsync = reinterpret_cast<int*>(ts);
  }
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_work, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return fail(PBAD_E_CUDA, "stream/event creation failed");
  }
  *out = c;
  return PBAD_OK;
}

void pbad_gpu_destroy(pbad_gpu_ctx* c) { delete c; }
int32_t pbad_gpu_total_steps(const pbad_gpu_ctx* c) { return c->total_steps; }
int64_t pbad_gpu_kernel_launches(const pbad_gpu_ctx* c) { return c->launches; }
int32_t pbad_gpu_path(const pbad_gpu_ctx* c) {
  return c->chain5 ? PBAD_PATH_CHAIN5
         : c->chain6 ? PBAD_PATH_CHAIN6
         : c->chain7 ? PBAD_PATH_CHAIN7
         : c->chain4 ? PBAD_PATH_CHAIN4
         : c->chain ? PBAD_PATH_CHAIN
         : c->tree  ? PBAD_PATH_TREE
         : c->resid ? PBAD_PATH_RESID
                    : PBAD_PATH_GENERAL;
}
const double* pbad_gpu_state_device(const pbad_gpu_ctx* c) {
  // chain path: quad-interleaved [n/4][B][4]; general path: [n][B]
  return c->chain ? c->ca.cw + c->ca.L.h1 : c->ka.ws + c->ka.L.hist1 * c->ka.B;
}

}  // extern "C"

namespace {

// simulate_baseline's general-kernel workspace layout (velocity pass, mass
// matrix, stage states), shared by pbad_gpu_simulate_baseline and the
// refined bootstrap
Layout baseline_layout(const pbad_gpu_model& m) {
  const long N = m.N, n = m.n;
  Layout L{};
  long o = 0;
  auto take = [&](long cnt) {
    const long at = o;
    o += cnt;
    return at;
  };
  L.p_value = 0;
  L.p_d1 = N * 16;
  L.p_world = L.p_d1 + n * 16;
  L.p_lever = L.p_world + N * 16;
  L.p_d2 = L.p_lever + n * 16;
  L.pass_stride = L.p_d2 + (long)m.n_d2 * 16;
  L.pass = take(L.pass_stride);
  L.seeds = take(N * 16);
  L.adj = take(N * 16);
  L.cot = take(N * 16);
  L.hw0 = take(N * 16);  // tdot
  L.hw1 = take(N * 16);  // quad
  L.gn = take(n * n);    // mass matrix / its factor
  L.x = take(n);
  L.grad = take(n);
  L.cand = take(n);
  L.dir = take(n);
  L.potgrad = take(n);   // Coriolis
  L.g = take(n);         // generalized force
  L.dd = take(n);        // right-hand side
  L.hs = take(4 * n);    // stage accelerations
  L.hy = take(4 * n);    // stage states
  L.total = o;
  return L;
}

// bootstrap_history's refined path (stepper.cpp:46-59) for the batch:
// hist0 into c->d_boot_h0, baseline_step failures into c->d_boot_st
int32_t refined_bootstrap(pbad_gpu_ctx* c, long B, const double* d_q0, const double* d_qdot0, cudaStream_t s) {
  const Layout L = baseline_layout(c->model);
  if (c->boot_cap < B) {
    cudaFree(c->d_boot_ws);
    cudaFree(c->d_boot_h0);
    cudaFree(c->d_boot_st);
    c->boot_cap = 0;
    c->d_boot_ws = dalloc<double>((size_t)L.total * B);
    c->d_boot_h0 = dalloc<double>((size_t)B * c->model.n);
    c->d_boot_st = dalloc<int>(B);
    if (!c->d_boot_ws || !c->d_boot_h0 || !c->d_boot_st)
      return fail(PBAD_E_CUDA, "cudaMalloc of the refined-bootstrap workspace failed (B=%ld)", B);
    c->boot_cap = B;
  }
  CUDA_TRY(launch_refined_bootstrap(c->ka, L, c->d_boot_ws, B, d_q0, d_qdot0, c->boot_hs, c->d_boot_h0,
                                    c->d_boot_st, s));
  return PBAD_OK;
}

// a failed bootstrap throws inside init_pbad_run, before sample 0 is recorded
__global__ void k_boot_status(const int* st, int* iws, long B) {
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B || st[e] == 0) return;
  int& run = iws[(long)IS_RUN * B + e];
  if (run == PBAD_TRAJ_NONFINITE_CFG && iws[(long)IS_NSAMP * B + e] == 0) return;  // q0 itself non-finite
  run = st[e] == 6 ? PBAD_TRAJ_BOOTSTRAP_SINGULAR : PBAD_TRAJ_NONFINITE_CFG;  // BL_SINGULAR / BL_NONFINITE_CFG
  iws[(long)IS_NSAMP * B + e] = 0;
  iws[(long)IS_NREP * B + e] = 0;
}

int32_t begin_batch(pbad_gpu_ctx* c, int32_t B, long W, const double* d_q0, const double* d_qdot0, cudaStream_t s,
                    bool want_itv = false) {
  if (B < 1 || B > c->max_batch) return fail(PBAD_E_ARGUMENT, "batch %d outside [1, %ld]", B, c->max_batch);
  CUDA_TRY(cudaSetDevice(c->device));
  int32_t rc = ensure_outputs(c, B, W, want_itv);
  if (rc) return rc;
  c->B = B;
  c->ka.B = B;
  c->ca.B = B;
  c->steps_done = 0;
  c->device_ms = 0.0;
  c->work_stream = s;
  const double* h0 = nullptr;
  if (c->refined) {
    rc = refined_bootstrap(c, B, d_q0, d_qdot0, s);
    if (rc) return rc;
    h0 = c->d_boot_h0;
  }
  if (c->chain) CUDA_TRY(launch_chain_init(c->ca, d_q0, d_qdot0, h0, c->dout, s));
  else CUDA_TRY(launch_init(c->ka, d_q0, d_qdot0, h0, c->dout, s));
  if (c->refined) {
    k_boot_status<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(c->d_boot_st, c->chain ? c->ca.ci : c->ka.iws, B);
    CUDA_TRY(cudaGetLastError());
  }
  return PBAD_OK;
}

int32_t advance_steps(pbad_gpu_ctx* c, long n_steps, cudaStream_t s) {
  c->work_stream = s;
  if (c->chain6) {
    const long k = std::min(n_steps, (long)c->total_steps - c->steps_done);
    if (k > 0) CUDA_TRY(launch_chain6_steps(c->ca, c->chain4_pat, c->dout, (int)k, s, &c->launches));
    if (k > 0) c->steps_done += k;
    return PBAD_OK;
  }
  if (c->resid) {
    // one persistent launch per window (pbad_resid.cu k_resid_steps)
    const long k = std::min(n_steps, (long)c->total_steps - c->steps_done);
    if (k > 0) CUDA_TRY(launch_resid_steps(c->ka, c->rd, c->rws, c->dout, (int)k, c->tsync, s, &c->launches));
    if (k > 0) c->steps_done += k;
    return PBAD_OK;
  }
  if (c->tree && !c->td.lb) {
    // the tree family runs a window's steps in one persistent launch (pbad_tree.cu)
    const long k = std::min(n_steps, (long)c->total_steps - c->steps_done);
    if (k > 0) CUDA_TRY(launch_tree_steps(c->ka, c->td, c->tws, c->dout, (int)k, c->tsync, s, &c->launches));
    if (k > 0) c->steps_done += k;
    return PBAD_OK;
  }
  for (long k = 0; k < n_steps && c->steps_done < c->total_steps; ++k, ++c->steps_done, ++c->launches)
    CUDA_TRY(c->chain5  ? launch_chain5_step(c->ca, c->chain4_pat, c->chain4_recw / 8, c->dout, s)
             : c->chain7 ? launch_chain7_step(c->ca, c->chain4_pat, c->dout, s)
             : c->chain4 ? launch_chain4_step(c->ca, c->chain4_pat, c->dout, s)
             : c->chain ? launch_chain_step(c->ca, c->dout, s)
             : c->tree  ? launch_tree_step(c->ka, c->td, c->tws, c->dout, s)
             : c->resid ? launch_resid_step(c->ka, c->rd, c->rws, c->dout, s)
                        : launch_step(c->ka, c->dout, s));
  return PBAD_OK;
}

// the ctx stream waits for the caller's stream of the last begin/advance
int32_t join_work(pbad_gpu_ctx* c) {
  if (c->work_stream && c->work_stream != c->stream) {
    CUDA_TRY(cudaEventRecord(c->ev_work, c->work_stream));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_work, 0));
  }
  return PBAD_OK;
}

// Copies samples [s_lo, s_hi] and reports [r_lo, r_hi) held in the current
// output window to the host buffers of `o`, whose environment 0 is this
// context's environment env0 (sharded rollouts), on the ctx stream.
int32_t drain_window(pbad_gpu_ctx* c, const pbad_rollout_out* o, long env0, long s_lo, long s_hi, long r_lo,
                     long r_hi) {
  const long B = c->B, S = c->total_steps, n = c->model.n;
  const Outputs& d = c->dout;
  const cudaStream_t st = c->stream;
  if (s_hi >= s_lo) {
    const long cnt = s_hi - s_lo + 1;
    if (o->q)
      CUDA_TRY(cudaMemcpy2DAsync(o->q + (env0 * (S + 1) + s_lo) * n, sizeof(double) * (S + 1) * n,
                                 d.q + (s_lo - d.qbase) * n, sizeof(double) * d.qs * n, sizeof(double) * cnt * n, B,
                                 cudaMemcpyDeviceToHost, st));
    if (o->energy)
      CUDA_TRY(cudaMemcpy2DAsync(o->energy + (env0 * (S + 1) + s_lo) * 2, sizeof(double) * (S + 1) * 2,
                                 d.energy + (s_lo - d.qbase) * 2, sizeof(double) * d.qs * 2, sizeof(double) * cnt * 2,
                                 B, cudaMemcpyDeviceToHost, st));
  }
  if (r_hi > r_lo) {
    const long cnt = r_hi - r_lo;
    auto rep = [&](auto* host, auto* dev) -> cudaError_t {
      using T = std::remove_pointer_t<decltype(dev)>;
      if (!host) return cudaSuccess;
      return cudaMemcpy2DAsync(host + env0 * S + r_lo, sizeof(T) * S, dev + (r_lo - d.rbase), sizeof(T) * d.rs,
                               sizeof(T) * cnt, B, cudaMemcpyDeviceToHost, st);
    };
    CUDA_TRY(rep(o->iterations, d.iterations));
    CUDA_TRY(rep(o->converged, d.converged));
    CUDA_TRY(rep(o->accepted, d.accepted));
    CUDA_TRY(rep(o->final_value, d.final_value));
    CUDA_TRY(rep(o->final_grad_norm, d.final_grad_norm));
    if (o->iteration_values && d.itv) {
      const long mi = d.itv_n;
      CUDA_TRY(cudaMemcpy2DAsync(o->iteration_values + (env0 * S + r_lo) * mi, sizeof(double) * S * mi,
                                 d.itv + (r_lo - d.rbase) * mi, sizeof(double) * d.rs * mi,
                                 sizeof(double) * cnt * mi, B, cudaMemcpyDeviceToHost, st));
    }
  }
  return PBAD_OK;
}

// per-environment status words (n_samples, status, fail streak, reports)
int32_t drain_status(pbad_gpu_ctx* c, const pbad_rollout_out* o, long env0) {
  const long B = c->B;
  const int* iws = c->chain ? c->ca.ci : c->ka.iws;
  const cudaStream_t st = c->stream;
  if (o->n_samples)
    CUDA_TRY(cudaMemcpyAsync(o->n_samples + env0, iws + (long)IS_NSAMP * B, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  if (o->status)
    CUDA_TRY(cudaMemcpyAsync(o->status + env0, iws + (long)IS_RUN * B, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  if (o->fail_streak)
    CUDA_TRY(cudaMemcpyAsync(o->fail_streak + env0, iws + (long)IS_FAIL * B, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  if (o->n_reports)
    CUDA_TRY(cudaMemcpyAsync(o->n_reports + env0, iws + (long)IS_NREP * B, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  return PBAD_OK;
}

// One context's share of a (possibly sharded) rollout, advanced window by
// window so several devices step concurrently.
struct RolloutJob {
  pbad_gpu_ctx* c;
  long env0, B, W, ws;
};

int32_t job_start(RolloutJob& j, const double* q0, const double* qdot0, bool want_itv) {
  pbad_gpu_ctx* c = j.c;
  const long n = c->model.n;
  CUDA_TRY(cudaSetDevice(c->device));
  if (!c->d_q0) {
    c->d_q0 = dalloc<double>((size_t)c->max_batch * n);
    c->d_qd0 = dalloc<double>((size_t)c->max_batch * n);
    if (!c->d_q0 || !c->d_qd0) return fail(PBAD_E_CUDA, "cudaMalloc of q0 staging failed");
    c->owned.push_back(c->d_q0);
    c->owned.push_back(c->d_qd0);
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_q0, q0 + j.env0 * n, sizeof(double) * j.B * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_qd0, qdot0 + j.env0 * n, sizeof(double) * j.B * n, cudaMemcpyHostToDevice, c->stream));
  int32_t rc = begin_batch(c, (int32_t)j.B, j.W, c->d_q0, c->d_qd0, c->stream, want_itv);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
  j.ws = 0;
  return PBAD_OK;
}

// launches the next window's steps; returns 1 while windows remain
int32_t job_advance(RolloutJob& j) {
  pbad_gpu_ctx* c = j.c;
  if (j.ws >= c->total_steps) return 0;
  CUDA_TRY(cudaSetDevice(c->device));
  c->dout.qbase = j.ws;
  c->dout.rbase = j.ws;
  const long w = std::min(j.W, (long)c->total_steps - j.ws);
  const int32_t rc = advance_steps(c, w, c->stream);
  if (rc) return rc;
  if (j.ws + w >= c->total_steps) CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
  return 1;
}

int32_t job_drain(RolloutJob& j, const pbad_rollout_out* o) {
  pbad_gpu_ctx* c = j.c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long w = std::min(j.W, (long)c->total_steps - j.ws);
  // the window's samples: its own steps' samples, plus sample 0 in window 0
  const int32_t rc = drain_window(c, o, j.env0, j.ws == 0 ? 0 : j.ws + 1, j.ws + w, j.ws, j.ws + w);
  j.ws += w;
  return rc;
}

int32_t job_finish(RolloutJob& j, const pbad_rollout_out* o) {
  pbad_gpu_ctx* c = j.c;
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->total_steps == 0) {
    const int32_t rc = drain_window(c, o, j.env0, 0, 0, 0, 0);
    if (rc) return rc;
  }
  return drain_status(c, o, j.env0);
}

int32_t job_wait(RolloutJob& j, float* ms) {
  pbad_gpu_ctx* c = j.c;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  float t = 0.f;
  if (c->total_steps > 0) CUDA_TRY(cudaEventElapsedTime(&t, c->ev0, c->ev1));
  c->device_ms = t;
  *ms = t;
  return PBAD_OK;
}

int32_t run_jobs(std::vector<RolloutJob>& jobs, const double* q0, const double* qdot0, pbad_rollout_out* out) {
  for (auto& j : jobs) {
    const int32_t rc = job_start(j, q0, qdot0, out->iteration_values != nullptr);
    if (rc) return rc;
  }
  // window by window: every device's steps are queued before the drains, so
  // devices overlap even when a drain into pageable memory blocks the host
  for (;;) {
    bool more = false;
    std::vector<char> launched(jobs.size(), 0);
    for (size_t i = 0; i < jobs.size(); ++i) {
      const int32_t rc = job_advance(jobs[i]);
      if (rc < 0) return rc;
      launched[i] = (char)rc;
      more = more || rc;
    }
    if (!more) break;
    for (size_t i = 0; i < jobs.size(); ++i)
      if (launched[i]) {
        const int32_t rc = job_drain(jobs[i], out);
        if (rc) return rc;
      }
  }
  float worst = 0.f;
  for (auto& j : jobs) {
    const int32_t rc = job_finish(j, out);
    if (rc) return rc;
  }
  for (auto& j : jobs) {
    float ms = 0.f;
    const int32_t rc = job_wait(j, &ms);
    if (rc) return rc;
    worst = std::max(worst, ms);
  }
  if (out->device_ms) out->device_ms[0] = worst;
  return PBAD_OK;
}

__global__ void k_gather_final(const double* q, long qs, long qbase, const int* nsamp, long B, int n, double* dst) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * n) return;
  const long e = t / n, k = t - e * n;
  const long s = (long)nsamp[e] - 1;
  dst[t] = q[(e * qs + (s - qbase)) * n + k];
}

}  // namespace

extern "C" {

int32_t pbad_gpu_begin(pbad_gpu_ctx* c, int32_t B, const double* d_q0, const double* d_qdot0, void* stream) {
  return begin_batch(c, B, c->total_steps, d_q0, d_qdot0, pick(c, stream));
}

int32_t pbad_gpu_advance(pbad_gpu_ctx* c, int32_t n_steps, void* stream) {
  CUDA_TRY(cudaSetDevice(c->device));
  return advance_steps(c, n_steps, pick(c, stream));
}

int32_t pbad_gpu_sync_outputs(pbad_gpu_ctx* c, pbad_rollout_out* o) {
  CUDA_TRY(cudaSetDevice(c->device));
  int32_t rc = join_work(c);
  if (rc) return rc;
  rc = drain_window(c, o, 0, 0, c->total_steps, 0, c->total_steps);
  if (rc) return rc;
  rc = drain_status(c, o, 0);
  if (rc) return rc;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (o->device_ms) o->device_ms[0] = (float)c->device_ms;
  return PBAD_OK;
}

int32_t pbad_gpu_final_state(pbad_gpu_ctx* c, double* d_dst, void* stream) {
  if (!c->B) return fail(PBAD_E_ARGUMENT, "no batch has been started on this context");
  if (c->dout.qbase != 0 || c->dout.qs != c->total_steps + 1)
    return fail(PBAD_E_ARGUMENT, "final_state needs the whole-trajectory output geometry (pbad_gpu_begin)");
  CUDA_TRY(cudaSetDevice(c->device));
  const cudaStream_t s = pick(c, stream);
  const int* iws = c->chain ? c->ca.ci : c->ka.iws;
  const long tot = c->B * (long)c->model.n;
  k_gather_final<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(c->dout.q, c->dout.qs, c->dout.qbase,
                                                               iws + (long)IS_NSAMP * c->B, c->B, c->model.n, d_dst);
  CUDA_TRY(cudaGetLastError());
  return PBAD_OK;
}

int32_t pbad_gpu_rollout(pbad_gpu_ctx* c, int32_t B, const double* q0, const double* qdot0,
                         pbad_rollout_out* out) {
  if (B < 1 || B > c->max_batch) return fail(PBAD_E_ARGUMENT, "batch %d outside [1, %ld]", B, c->max_batch);
  std::vector<RolloutJob> jobs{RolloutJob{c, 0, B, window_steps(c, B, out->iteration_values != nullptr), 0}};
  return run_jobs(jobs, q0, qdot0, out);
}

int32_t pbad_gpu_rollout_sharded(pbad_gpu_ctx* const* ctxs, int32_t n_ctx, int32_t B, const double* q0,
                                 const double* qdot0, pbad_rollout_out* out) {
  if (!ctxs || n_ctx < 1) return fail(PBAD_E_ARGUMENT, "need at least one context");
  if (B < n_ctx) return fail(PBAD_E_ARGUMENT, "batch %d smaller than the context count %d", B, n_ctx);
  std::vector<RolloutJob> jobs;
  for (int i = 0; i < n_ctx; ++i) {
    pbad_gpu_ctx* c = ctxs[i];
    if (!c) return fail(PBAD_E_ARGUMENT, "context %d is null", i);
    for (int k = 0; k < i; ++k)
      if (ctxs[k] == c) return fail(PBAD_E_ARGUMENT, "context %d appears twice (one context per shard)", i);
    if (c->model.n != ctxs[0]->model.n || c->total_steps != ctxs[0]->total_steps)
      return fail(PBAD_E_ARGUMENT, "contexts differ in DOF count or step count");
    const long lo = (long)B * i / n_ctx, hi = (long)B * (i + 1) / n_ctx;
    if (hi - lo > c->max_batch)
      return fail(PBAD_E_ARGUMENT, "shard %d has %ld environments, context max_batch is %ld", i, hi - lo, c->max_batch);
    jobs.push_back(RolloutJob{c, lo, hi - lo, window_steps(c, hi - lo, out->iteration_values != nullptr), 0});
  }
  return run_jobs(jobs, q0, qdot0, out);
}

static int32_t stage_inputs(pbad_gpu_ctx* c, int32_t B, const double* history, const double* tau,
                            const double* x, double** dh, double** dt, double** dx, long extra) {
  const long n = c->model.n, U = c->ka.sc.U;
  const long need = B * (2 * n + U + U) + extra;
  if (c->in_cap < need) {
    cudaFree(c->d_in);
    c->d_in = dalloc<double>(need);
    if (!c->d_in) return fail(PBAD_E_CUDA, "cudaMalloc of eval staging failed");
    c->in_cap = need;
  }
  *dh = c->d_in;
  *dt = tau ? c->d_in + B * 2 * n : nullptr;
  *dx = c->d_in + B * (2 * n + U);
  CUDA_TRY(cudaMemcpy(*dh, history, sizeof(double) * B * 2 * n, cudaMemcpyHostToDevice));
  if (tau) CUDA_TRY(cudaMemcpy(*dt, tau, sizeof(double) * B * U, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(*dx, x, sizeof(double) * B * U, cudaMemcpyHostToDevice));
  return PBAD_OK;
}

int32_t pbad_gpu_eval(pbad_gpu_ctx* c, int32_t B, const double* history, const double* tau, const double* x,
                      int32_t want_grad, int32_t want_gn, double* value, double* grad, double* gn) {
  if (B < 1 || B > c->max_batch) return fail(PBAD_E_ARGUMENT, "batch %d outside [1, %ld]", B, c->max_batch);
  if (want_gn && c->ka.sc.opt.kind != PBAD_LM)
    return fail(PBAD_E_ARGUMENT, "GN output needs a context created with the LM optimizer (workspace)");
  CUDA_TRY(cudaSetDevice(c->device));
  if (!ensure_v1(c)) return fail(PBAD_E_CUDA, "cudaMalloc of the evaluation workspace failed");
  const long U = c->ka.sc.U;
  double *dh, *dt, *dx;
  int32_t rc = stage_inputs(c, B, history, tau, x, &dh, &dt, &dx, 0);
  if (rc) return rc;
  double* dval = dalloc<double>(B);
  double* dgrad = dalloc<double>((size_t)B * U);
  double* dgn = want_gn ? dalloc<double>((size_t)B * U * U) : nullptr;
  int* derr = dalloc<int>(B);
  KernelArgs ka = c->ka;
  ka.B = B;
  cudaError_t e = launch_eval(ka, dh, dt, dx, want_grad, want_gn, dval, dgrad, dgn, derr, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  std::vector<int> err(B);
  if (e == cudaSuccess) e = cudaMemcpy(err.data(), derr, sizeof(int) * B, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && value) e = cudaMemcpy(value, dval, sizeof(double) * B, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && want_grad && grad) e = cudaMemcpy(grad, dgrad, sizeof(double) * B * U, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && want_gn && gn) e = cudaMemcpy(gn, dgn, sizeof(double) * B * U * U, cudaMemcpyDeviceToHost);
  cudaFree(dval);
  cudaFree(dgrad);
  if (dgn) cudaFree(dgn);
  cudaFree(derr);
  if (e != cudaSuccess) return fail(PBAD_E_CUDA, "eval: %s", cudaGetErrorString(e));
  for (int b = 0; b < B; ++b)
    if (err[b]) return fail(PBAD_E_MODEL, "configuration contains a non-finite entry (env %d)", b);
  return PBAD_OK;
}

// simulate_baseline (stepper.cpp:168-202): explicit Newton-Euler schemes for
// B trajectories of the context's model/forces with its dt and duration
int32_t pbad_gpu_simulate_baseline(pbad_gpu_ctx* c, int32_t scheme, int32_t B, const double* q0,
                                   const double* qdot0, double* q_out, double* energy, int32_t* n_samples,
                                   int32_t* status) {
  if (B < 1) return fail(PBAD_E_ARGUMENT, "batch %d must be >= 1", B);
  if (scheme < 0 || scheme > 4) return fail(PBAD_E_ARGUMENT, "unknown baseline scheme %d", scheme);
  if (!q0 || !qdot0 || !n_samples || !status) return fail(PBAD_E_ARGUMENT, "q0, qdot0, n_samples, status required");
  const pbad_gpu_model& m = c->model;
  const long n = m.n;
  for (long k = 0; k < (long)B * n; ++k)
    if (!std::isfinite(q0[k])) return fail(PBAD_E_MODEL, "configuration contains a non-finite entry");
  CUDA_TRY(cudaSetDevice(c->device));
  const long S = c->ka.sc.total_steps;
  const Layout L = baseline_layout(m);
  double* ws = dalloc<double>((size_t)L.total * B);
  double* dq = dalloc<double>((size_t)2 * B * n);
  double* doq = q_out ? dalloc<double>((size_t)B * (S + 1) * n) : nullptr;
  double* doe = energy ? dalloc<double>((size_t)B * (S + 1) * 2) : nullptr;
  int* dns = dalloc<int>(B);
  int* dst = dalloc<int>(B);
  cudaError_t e = (ws && dq && dns && dst && (!q_out || doq) && (!energy || doe)) ? cudaSuccess
                                                                                   : cudaErrorMemoryAllocation;
  if (e == cudaSuccess) e = cudaMemcpy(dq, q0, sizeof(double) * B * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dq + (size_t)B * n, qdot0, sizeof(double) * B * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = launch_baseline(c->ka, L, ws, B, scheme, dq, dq + (size_t)B * n, doq, doe, dns, dst, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && doq) e = cudaMemcpy(q_out, doq, sizeof(double) * B * (S + 1) * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && doe) e = cudaMemcpy(energy, doe, sizeof(double) * B * (S + 1) * 2, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(n_samples, dns, sizeof(int) * B, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(status, dst, sizeof(int) * B, cudaMemcpyDeviceToHost);
  for (void* p : {(void*)ws, (void*)dq, (void*)doq, (void*)doe, (void*)dns, (void*)dst})
    if (p) cudaFree(p);
  if (e != cudaSuccess) return fail(PBAD_E_CUDA, "simulate_baseline: %s", cudaGetErrorString(e));
  return PBAD_OK;
}

// correlation_and_grad / hessian_bb / hessian_ab (adjoint.cpp:178-192) for a
// batch of (qa, qb) pairs; WeightedBody::make (adjoint.cpp:29-41) on the host
int32_t pbad_gpu_correlation(pbad_gpu_ctx* c, int32_t B, const double* qa, const double* qb,
                             const double* weight_per_body, double* value, double* grad_b, double* hess_bb,
                             double* hess_ab) {
  if (B < 1) return fail(PBAD_E_ARGUMENT, "batch %d must be >= 1", B);
  if (!qa || !qb) return fail(PBAD_E_ARGUMENT, "qa and qb are required");
  CUDA_TRY(cudaSetDevice(c->device));
  const pbad_gpu_model& m = c->model;
  const long N = m.N, n = m.n;
  DModel dm = c->ka.m;
  double* dS = nullptr;
  if (weight_per_body) {
    std::vector<double> wS(16 * N);
    double wm = 0.0;
    for (long i = 0; i < N; ++i) {
      const double w = weight_per_body[i];
      for (int k = 0; k < 16; ++k) wS[16 * i + k] = w * m.S[16 * i + k];
      wm += w * m.mass[i];
    }
    dS = dalloc<double>(16 * N);
    if (!dS) return fail(PBAD_E_CUDA, "cudaMalloc of the weighted body integrals failed");
    CUDA_TRY(cudaMemcpy(dS, wS.data(), sizeof(double) * 16 * N, cudaMemcpyHostToDevice));
    dm.S = dS;
    dm.weighted_mass = wm;
  }
  Layout L{};
  L.p_value = 0;
  L.p_d1 = N * 16;
  L.p_world = L.p_d1 + n * 16;
  L.p_lever = L.p_world + N * 16;
  L.p_d2 = L.p_lever + n * 16;
  L.pass_stride = L.p_d2 + (long)m.n_d2 * 16;
  L.pass = 0;
  L.seeds = 2 * L.pass_stride;
  L.adj = L.seeds + N * 16;
  L.total = L.adj + N * 16;
  double* ws = dalloc<double>((size_t)L.total * B);
  double* dq = dalloc<double>((size_t)2 * B * n);
  double* dv = value ? dalloc<double>(B) : nullptr;
  double* dg = grad_b ? dalloc<double>((size_t)B * n) : nullptr;
  double* dbb = hess_bb ? dalloc<double>((size_t)B * n * n) : nullptr;
  double* dab = hess_ab ? dalloc<double>((size_t)B * n * n) : nullptr;
  cudaError_t e = (ws && dq && (!value || dv) && (!grad_b || dg) && (!hess_bb || dbb) && (!hess_ab || dab))
                      ? cudaSuccess : cudaErrorMemoryAllocation;
  if (e == cudaSuccess) e = cudaMemcpy(dq, qa, sizeof(double) * B * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dq + (size_t)B * n, qb, sizeof(double) * B * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_correlation(dm, L, ws, B, dq, dq + (size_t)B * n, dv, dg, dbb, dab, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && dv) e = cudaMemcpy(value, dv, sizeof(double) * B, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && dg) e = cudaMemcpy(grad_b, dg, sizeof(double) * B * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && dbb) e = cudaMemcpy(hess_bb, dbb, sizeof(double) * B * n * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && dab) e = cudaMemcpy(hess_ab, dab, sizeof(double) * B * n * n, cudaMemcpyDeviceToHost);
  for (void* p : {(void*)dS, (void*)ws, (void*)dq, (void*)dv, (void*)dg, (void*)dbb, (void*)dab})
    if (p) cudaFree(p);
  if (e != cudaSuccess) return fail(PBAD_E_CUDA, "correlation: %s", cudaGetErrorString(e));
  return PBAD_OK;
}

// One CTA per request (pbad_corr.cu): mode 0 parallel_correlation_suite,
// mode 1 the linear functional of caller seeds.
static int32_t run_suite(pbad_gpu_ctx* c, int32_t B, int mode, const double* qa, const double* qb,
                         const double* seeds, const double* weight_per_body, double* value, double* grad,
                         double* hess_bb, double* hess_ab) {
  if (B < 1) return fail(PBAD_E_ARGUMENT, "batch %d must be >= 1", B);
  if (!qb || (mode == 0 && !qa) || (mode == 1 && !seeds)) return fail(PBAD_E_ARGUMENT, "missing input array");
  CUDA_TRY(cudaSetDevice(c->device));
  const pbad_gpu_model& m = c->model;
  const long N = m.N, n = m.n;
  DModel dm = c->ka.m;
  std::vector<void*> tmp;
  auto dev = [&](size_t cnt) {
    double* p = dalloc<double>(cnt);
    tmp.push_back(p);
    return p;
  };
  auto release = [&]() {
    for (void* p : tmp)
      if (p) cudaFree(p);
  };
  cudaError_t e = cudaSuccess;
  if (mode == 0 && weight_per_body) {  // WeightedBody::make (adjoint.cpp:29-41)
    std::vector<double> wS(16 * N);
    double wm = 0.0;
    for (long i = 0; i < N; ++i) {
      const double w = weight_per_body[i];
      for (int k = 0; k < 16; ++k) wS[16 * i + k] = w * m.S[16 * i + k];
      wm += w * m.mass[i];
    }
    double* dS = dev(16 * N);
    if (dS) e = cudaMemcpy(dS, wS.data(), sizeof(double) * 16 * N, cudaMemcpyHostToDevice);
    dm.S = dS;
    dm.weighted_mass = wm;
  }
  const SuiteLayout L = suite_layout(m.N, m.n, m.n_d2);
  double* ws = dev((size_t)L.total * B);
  double* dqa = mode == 0 ? dev((size_t)B * n) : nullptr;
  double* dqb = dev((size_t)B * n);
  double* dseeds = mode == 1 ? dev((size_t)B * N * 16) : nullptr;
  double* dv = value ? dev(B) : nullptr;
  double* dg = grad ? dev((size_t)B * n) : nullptr;
  double* dbb = hess_bb ? dev((size_t)B * n * n) : nullptr;
  double* dab = (mode == 0 && hess_ab) ? dev((size_t)B * n * n) : nullptr;
  for (void* p : tmp)
    if (!p) e = cudaErrorMemoryAllocation;
  if (e == cudaSuccess && dqa) e = cudaMemcpy(dqa, qa, sizeof(double) * B * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dqb, qb, sizeof(double) * B * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && dseeds) e = cudaMemcpy(dseeds, seeds, sizeof(double) * B * N * 16, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_suite(dm, L, ws, B, dqa, dqb, dseeds, mode, dv, dg, dbb, dab, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && dv) e = cudaMemcpy(value, dv, sizeof(double) * B, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && dg) e = cudaMemcpy(grad, dg, sizeof(double) * B * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && dbb) e = cudaMemcpy(hess_bb, dbb, sizeof(double) * B * n * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && dab) e = cudaMemcpy(hess_ab, dab, sizeof(double) * B * n * n, cudaMemcpyDeviceToHost);
  release();
  if (e != cudaSuccess) return fail(PBAD_E_CUDA, "correlation suite: %s", cudaGetErrorString(e));
  return PBAD_OK;
}

int32_t pbad_gpu_correlation_suite(pbad_gpu_ctx* c, int32_t B, const double* qa, const double* qb,
                                   const double* weight_per_body, double* value, double* grad_b, double* hess_bb,
                                   double* hess_ab) {
  return run_suite(c, B, 0, qa, qb, nullptr, weight_per_body, value, grad_b, hess_bb, hess_ab);
}

int32_t pbad_gpu_functional(pbad_gpu_ctx* c, int32_t B, const double* q, const double* seeds, double* value,
                            double* grad, double* hess) {
  return run_suite(c, B, 1, nullptr, q, seeds, nullptr, value, grad, hess, nullptr);
}

int32_t pbad_gpu_minimize(pbad_gpu_ctx* c, int32_t B, const double* history, const double* tau,
                          const double* x0, double* x_out, int32_t* iterations, int32_t* converged,
                          double* final_value, double* final_grad_norm) {
  if (B < 1 || B > c->max_batch) return fail(PBAD_E_ARGUMENT, "batch %d outside [1, %ld]", B, c->max_batch);
  CUDA_TRY(cudaSetDevice(c->device));
  if (!ensure_v1(c)) return fail(PBAD_E_CUDA, "cudaMalloc of the evaluation workspace failed");
  const long U = c->ka.sc.U;
  double *dh, *dt, *dx;
  int32_t rc = stage_inputs(c, B, history, tau, x0, &dh, &dt, &dx, 0);
  if (rc) return rc;
  double* dxo = dalloc<double>((size_t)B * U);
  int* dit = dalloc<int>(B);
  int* dcv = dalloc<int>(B);
  double* dfv = dalloc<double>(B);
  double* dgn = dalloc<double>(B);
  int* derr = dalloc<int>(B);
  KernelArgs ka = c->ka;
  ka.B = B;
  cudaError_t e = launch_minimize(ka, dh, dt, dx, dxo, dit, dcv, dfv, dgn, derr, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  std::vector<int> err(B);
  if (e == cudaSuccess) e = cudaMemcpy(err.data(), derr, sizeof(int) * B, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && x_out) e = cudaMemcpy(x_out, dxo, sizeof(double) * B * U, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && iterations) e = cudaMemcpy(iterations, dit, sizeof(int) * B, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && converged) e = cudaMemcpy(converged, dcv, sizeof(int) * B, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && final_value) e = cudaMemcpy(final_value, dfv, sizeof(double) * B, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && final_grad_norm) e = cudaMemcpy(final_grad_norm, dgn, sizeof(double) * B, cudaMemcpyDeviceToHost);
  cudaFree(dxo);
  cudaFree(dit);
  cudaFree(dcv);
  cudaFree(dfv);
  cudaFree(dgn);
  cudaFree(derr);
  if (e != cudaSuccess) return fail(PBAD_E_CUDA, "minimize: %s", cudaGetErrorString(e));
  for (int b = 0; b < B; ++b) {
    if (err[b] == 2) return fail(PBAD_E_ARGUMENT, "objective is non-finite at the initial point");
    if (err[b]) return fail(PBAD_E_MODEL, "configuration contains a non-finite entry");
  }
  return PBAD_OK;
}

}  // extern "C"
