/*
 * pbad_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference PBAD hot path
 * (/root/reference/proj/src/{model,kinematics,adjoint,collocation,objective,
 * optim,stepper,baseline}.cpp).  It is the checker the CUDA path is compared
 * against; nothing in the product links or calls it.  Each function cites the
 * reference lines it follows and keeps the reference's evaluation order
 * (full 4x4 matrices, same loops), with Eigen's unspecified rounding orders
 * fixed by pbo_math.h.  Build: oracle/Makefile (-ffp-contract=off).
 */
#include "pbad_oracle.h"

#include <float.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include "pbo_math.h"

#define PBO_ERRLEN 256

/* ------------------------------------------------------------------ */
/* error plumbing: reference exceptions become (code, message)         */
/* ------------------------------------------------------------------ */
typedef struct {
  int failed;
  char msg[PBO_ERRLEN];
} pbo_err;

static void err_set(pbo_err* e, const char* fmt, ...) {
  if (e->failed) return;
  e->failed = 1;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(e->msg, sizeof e->msg, fmt, ap);
  va_end(ap);
}

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) {
    fprintf(stderr, "pbad_oracle: out of memory\n");
    abort();
  }
  return p;
}

void pbo_sincos(double x, double* s, double* c) { pbm_sincos(x, s, c); }

/* ------------------------------------------------------------------ */
/* model (model.hpp:24-88, model.cpp:9-123)                            */
/* ------------------------------------------------------------------ */
struct pbo_model {
  int N, n, n_d2;
  int* parent;
  int* kind;
  int* dof_off;
  int* dof_cnt;
  int* d2_off;
  double* axis;     /* [N][3] normalised */
  pbo_m4* offset;   /* [N] */
  pbo_m4* S;        /* [N] */
  double* mass;     /* [N] */
  int* sample_off;  /* [N+1] */
  double* samples;  /* [total][3] */
};

static int kind_dofs(int kind) {
  switch (kind) {
    case PBO_HINGE: return 1;
    case PBO_BALL: return 3;
    case PBO_FREE: return 6;
  }
  return 0;
}

/* body_integral, model.cpp:35-60 */
void pbo_body_integral(const pbo_link_spec* link, double* S_out, double* mass_out) {
  pbo_m4 S = m4_zero();
  double mass = 0.0;
  if (link->geom_kind == PBO_BOX) {
    const double* sz = link->box_size;
    const double m = link->box_density * ((sz[0] * sz[1]) * sz[2]);
    const double* c = link->box_center;
    const double k12 = 1.0 / 12.0;
    const double dg[3] = {(sz[0] * sz[0]) * k12, (sz[1] * sz[1]) * k12,
                          (sz[2] * sz[2]) * k12};
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) {
        const double delta = (i == j) ? dg[i] : 0.0 * k12;
        M4E(S, i, j) = m * ((c[i] * c[j]) + delta);
      }
    for (int i = 0; i < 3; ++i) M4E(S, i, 3) = m * c[i];
    for (int j = 0; j < 3; ++j) M4E(S, 3, j) = m * c[j];
    M4E(S, 3, 3) = m;
    mass = m;
  } else {
    for (int p = 0; p < link->n_points; ++p) {
      const double pm = link->point_mass[p];
      const double h[4] = {link->point_pos[3 * p], link->point_pos[3 * p + 1],
                           link->point_pos[3 * p + 2], 1.0};
      double mh[4];
      for (int r = 0; r < 4; ++r) mh[r] = pm * h[r];
      for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) M4E(S, i, j) = M4E(S, i, j) + mh[i] * h[j];
      mass += pm;
    }
  }
  memcpy(S_out, S.a, sizeof S.a);
  *mass_out = mass;
}

/* check_offset, model.cpp:9-21 */
static void check_offset(const double* off, int i, pbo_err* e) {
  pbo_m3 r, rtr;
  for (int c = 0; c < 3; ++c)
    for (int k = 0; k < 3; ++k) M3E(r, k, c) = off[k + 4 * c];
  for (int j = 0; j < 3; ++j)
    for (int a = 0; a < 3; ++a) {
      double acc = M3E(r, 0, a) * M3E(r, 0, j);
      acc = fma(M3E(r, 1, a), M3E(r, 1, j), acc);
      acc = fma(M3E(r, 2, a), M3E(r, 2, j), acc);
      M3E(rtr, a, j) = acc;
    }
  double mx = 0.0;
  for (int k = 0; k < 9; ++k) {
    const double d = fabs(rtr.a[k] - ((k % 4 == 0) ? 1.0 : 0.0));
    if (k == 0 || d > mx) mx = d;
  }
  if (mx > 1e-10) {
    err_set(e, "link %d: joint offset rotation block is not orthonormal", i);
    return;
  }
  if (off[3] != 0.0 || off[7] != 0.0 || off[11] != 0.0 || off[15] != 1.0)
    err_set(e, "link %d: joint offset bottom row must be (0,0,0,1)", i);
}

void pbo_model_free(pbo_model* m) {
  if (!m) return;
  free(m->parent); free(m->kind); free(m->dof_off); free(m->dof_cnt); free(m->d2_off);
  free(m->axis); free(m->offset); free(m->S); free(m->mass); free(m->sample_off);
  free(m->samples);
  free(m);
}

/* build_model, model.cpp:62-112 */
int pbo_model_create(const pbo_link_spec* links, int32_t N, pbo_model** out, char* err,
                     int32_t errlen) {
  pbo_err e = {0};
  pbo_model* m = (pbo_model*)xcalloc(1, sizeof *m);
  m->N = N;
  m->parent = (int*)xcalloc(N, sizeof(int));
  m->kind = (int*)xcalloc(N, sizeof(int));
  m->dof_off = (int*)xcalloc(N, sizeof(int));
  m->dof_cnt = (int*)xcalloc(N, sizeof(int));
  m->d2_off = (int*)xcalloc(N, sizeof(int));
  m->axis = (double*)xcalloc(3 * (size_t)N, sizeof(double));
  m->offset = (pbo_m4*)xcalloc(N, sizeof(pbo_m4));
  m->S = (pbo_m4*)xcalloc(N, sizeof(pbo_m4));
  m->mass = (double*)xcalloc(N, sizeof(double));
  m->sample_off = (int*)xcalloc(N + 1, sizeof(int));
  int total_samples = 0;
  for (int i = 0; i < N; ++i) {
    const pbo_link_spec* L = &links[i];
    if (L->n_samples > 0) total_samples += L->n_samples;
    else if (L->geom_kind == PBO_BOX) total_samples += 8;
    else total_samples += L->n_points;
  }
  m->samples = (double*)xcalloc(3 * (size_t)total_samples, sizeof(double));
  int sp = 0;
  for (int i = 0; i < N && !e.failed; ++i) {
    const pbo_link_spec* L = &links[i];
    if (L->parent >= 0 && L->parent >= i) {
      err_set(&e, "link %d: parent index must be smaller than own index", i);
      break;
    }
    if (L->parent < -1) {
      err_set(&e, "link %d: negative parent index", i);
      break;
    }
    m->parent[i] = L->parent;
    m->kind[i] = L->joint_kind;
    double ax[3] = {L->axis[0], L->axis[1], L->axis[2]};
    if (L->joint_kind == PBO_HINGE) {
      const double nn = sqrt(vfix_dot(ax, ax, 3));
      if (fabs(nn - 1.0) > 1e-12) {
        if (nn < 1e-12) {
          err_set(&e, "link %d: zero-norm hinge axis", i);
          break;
        }
        for (int k = 0; k < 3; ++k) ax[k] = ax[k] / nn;
      }
    }
    memcpy(&m->axis[3 * i], ax, sizeof ax);
    check_offset(L->offset, i, &e);
    if (e.failed) break;
    memcpy(m->offset[i].a, L->offset, sizeof(double) * 16);
    m->sample_off[i] = sp;
    if (L->geom_kind == PBO_BOX) {
      if (L->box_density <= 0.0) {
        err_set(&e, "link %d: non-positive density", i);
        break;
      }
      const double mn = fmin(fmin(L->box_size[0], L->box_size[1]), L->box_size[2]);
      if (mn <= 0.0) {
        err_set(&e, "link %d: non-positive box extent", i);
        break;
      }
      if (L->n_samples > 0) {
        memcpy(&m->samples[3 * sp], L->samples, sizeof(double) * 3 * L->n_samples);
        sp += L->n_samples;
      } else {
        /* box_corners, model.cpp:23-31 */
        const double h[3] = {0.5 * L->box_size[0], 0.5 * L->box_size[1],
                             0.5 * L->box_size[2]};
        for (int sx = -1; sx <= 1; sx += 2)
          for (int sy = -1; sy <= 1; sy += 2)
            for (int sz = -1; sz <= 1; sz += 2) {
              m->samples[3 * sp + 0] = L->box_center[0] + (double)sx * h[0];
              m->samples[3 * sp + 1] = L->box_center[1] + (double)sy * h[1];
              m->samples[3 * sp + 2] = L->box_center[2] + (double)sz * h[2];
              ++sp;
            }
      }
    } else {
      for (int p = 0; p < L->n_points; ++p)
        if (L->point_mass[p] <= 0.0) {
          err_set(&e, "link %d: non-positive point mass", i);
          break;
        }
      if (e.failed) break;
      if (L->n_samples > 0) {
        memcpy(&m->samples[3 * sp], L->samples, sizeof(double) * 3 * L->n_samples);
        sp += L->n_samples;
      } else {
        memcpy(&m->samples[3 * sp], L->point_pos, sizeof(double) * 3 * L->n_points);
        sp += L->n_points;
      }
    }
    double S[16], mass;
    pbo_body_integral(L, S, &mass);
    memcpy(m->S[i].a, S, sizeof S);
    m->mass[i] = mass;
    m->dof_off[i] = m->n;
    m->dof_cnt[i] = kind_dofs(L->joint_kind);
    m->d2_off[i] = m->n_d2;
    m->n += m->dof_cnt[i];
    m->n_d2 += m->dof_cnt[i] * (m->dof_cnt[i] + 1) / 2;
  }
  m->sample_off[N] = sp;
  if (e.failed) {
    if (err && errlen > 0) snprintf(err, errlen, "%s", e.msg);
    pbo_model_free(m);
    *out = NULL;
    return -1;
  }
  *out = m;
  return 0;
}

int32_t pbo_model_dofs(const pbo_model* m) { return m->n; }
int32_t pbo_model_links(const pbo_model* m) { return m->N; }

void pbo_model_info(const pbo_model* m, double* S, double* mass, int32_t* dof_offset,
                    double* axis, int32_t* sample_count) {
  for (int i = 0; i < m->N; ++i) {
    if (S) memcpy(&S[16 * i], m->S[i].a, sizeof(double) * 16);
    if (mass) mass[i] = m->mass[i];
    if (dof_offset) dof_offset[i] = m->dof_off[i];
    if (axis) memcpy(&axis[3 * i], &m->axis[3 * i], sizeof(double) * 3);
    if (sample_count) sample_count[i] = m->sample_off[i + 1] - m->sample_off[i];
  }
}

int32_t pbo_model_samples(const pbo_model* m, int32_t link, double* out) {
  const int k = m->sample_off[link + 1] - m->sample_off[link];
  if (out) memcpy(out, &m->samples[3 * m->sample_off[link]], sizeof(double) * 3 * k);
  return k;
}

/* validate_configuration, model.cpp:114-123 */
static int validate_configuration(const pbo_model* m, const double* q, int len,
                                  pbo_err* e) {
  if (len != m->n) {
    err_set(e, "configuration length %d does not match model DOF count %d", len, m->n);
    return -1;
  }
  if (!vdyn_allfinite(q, len)) {
    err_set(e, "configuration contains a non-finite entry");
    return -1;
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* kinematics (kinematics.cpp:16-192)                                  */
/* ------------------------------------------------------------------ */
typedef struct {
  double A, B, f1, f2, g1, g2;
} rot_coeffs;

/* rotation_coeffs, kinematics.cpp:20-45 */
static rot_coeffs rotation_coeffs(double n) {
  rot_coeffs c;
  const double n2 = n * n;
  if (n < 1e-4) {
    const double n4 = n2 * n2;
    c.A = 1.0 - n2 / 6.0 + n4 / 120.0;
    c.B = 0.5 - n2 / 24.0 + n4 / 720.0;
    c.f1 = -1.0 / 3.0 + n2 / 30.0 - n4 / 840.0;
    c.f2 = -1.0 / 12.0 + n2 / 180.0 - n4 / 6720.0;
    c.g1 = 1.0 / 15.0 - n2 / 210.0 + n4 / 7560.0;
    c.g2 = 1.0 / 90.0 - n2 / 1680.0 + n4 / 75600.0;
  } else {
    double s, co;
    pbm_sincos(n, &s, &co);
    const double n3 = n2 * n, n4 = n2 * n2;
    c.A = s / n;
    c.B = (1.0 - co) / n2;
    c.f1 = (n * co - s) / n3;
    c.f2 = (n * s + 2.0 * co - 2.0) / n4;
    c.g1 = (-n2 * s - 3.0 * n * co + 3.0 * s) / (n4 * n);
    c.g2 = (n2 * co - 5.0 * n * s - 8.0 * co + 8.0) / (n4 * n2);
  }
  return c;
}

static double vec3_norm(const double t[3]) { return sqrt(vfix_dot(t, t, 3)); }

/* rotation_vector_jet, kinematics.cpp:49-87 */
static void rotation_vector_jet(const double theta[3], pbo_m3* R, pbo_m3 dR[3],
                                pbo_m3 d2R[3][3]) {
  const double n = vec3_norm(theta);
  const rot_coeffs c = rotation_coeffs(n);
  const pbo_m3 K = m3_skew(theta);
  const pbo_m3 K2 = m3_mul(&K, &K);
  pbo_m3 Kb[3];
  for (int j = 0; j < 3; ++j) {
    const double u[3] = {j == 0 ? 1.0 : 0.0, j == 1 ? 1.0 : 0.0, j == 2 ? 1.0 : 0.0};
    Kb[j] = m3_skew(u);
  }
  {
    const pbo_m3 I = m3_identity();
    const pbo_m3 aK = m3_scale(c.A, &K);
    const pbo_m3 bK2 = m3_scale(c.B, &K2);
    const pbo_m3 t = m3_add(&I, &aK);
    *R = m3_add(&t, &bK2);
  }
  pbo_m3 KbK_sym[3];
  for (int j = 0; j < 3; ++j) {
    const pbo_m3 p1 = m3_mul(&Kb[j], &K);
    const pbo_m3 p2 = m3_mul(&K, &Kb[j]);
    KbK_sym[j] = m3_add(&p1, &p2);
    const pbo_m3 t1 = m3_scale(c.f1 * theta[j], &K);
    const pbo_m3 t2 = m3_scale(c.A, &Kb[j]);
    const pbo_m3 t3 = m3_scale(c.f2 * theta[j], &K2);
    const pbo_m3 t4 = m3_scale(c.B, &KbK_sym[j]);
    pbo_m3 s = m3_add(&t1, &t2);
    s = m3_add(&s, &t3);
    dR[j] = m3_add(&s, &t4);
  }
  for (int j = 0; j < 3; ++j) {
    for (int l = j; l < 3; ++l) {
      const double tjl = theta[j] * theta[l];
      const double djl = (j == l) ? 1.0 : 0.0;
      const pbo_m3 a1 = m3_scale(c.f1 * djl + c.g1 * tjl, &K);
      const pbo_m3 u1 = m3_scale(theta[j], &Kb[l]);
      const pbo_m3 u2 = m3_scale(theta[l], &Kb[j]);
      const pbo_m3 u12 = m3_add(&u1, &u2);
      const pbo_m3 a2 = m3_scale(c.f1, &u12);
      const pbo_m3 a3 = m3_scale(c.f2 * djl + c.g2 * tjl, &K2);
      const pbo_m3 v1 = m3_scale(theta[j], &KbK_sym[l]);
      const pbo_m3 v2 = m3_scale(theta[l], &KbK_sym[j]);
      const pbo_m3 v12 = m3_add(&v1, &v2);
      const pbo_m3 a4 = m3_scale(c.f2, &v12);
      const pbo_m3 w1 = m3_mul(&Kb[j], &Kb[l]);
      const pbo_m3 w2 = m3_mul(&Kb[l], &Kb[j]);
      const pbo_m3 w12 = m3_add(&w1, &w2);
      const pbo_m3 a5 = m3_scale(c.B, &w12);
      pbo_m3 mm = m3_add(&a1, &a2);
      mm = m3_add(&mm, &a3);
      mm = m3_add(&mm, &a4);
      mm = m3_add(&mm, &a5);
      d2R[j][l] = mm;
      d2R[l][j] = mm;
    }
  }
}

/* rotation_vector_matrix, kinematics.cpp:91-96 */
static pbo_m3 rotation_vector_matrix(const double theta[3]) {
  const double n = vec3_norm(theta);
  const rot_coeffs c = rotation_coeffs(n);
  const pbo_m3 K = m3_skew(theta);
  const pbo_m3 K2 = m3_mul(&K, &K);
  const pbo_m3 I = m3_identity();
  const pbo_m3 aK = m3_scale(c.A, &K);
  const pbo_m3 bK2 = m3_scale(c.B, &K2);
  const pbo_m3 t = m3_add(&I, &aK);
  return m3_add(&t, &bK2);
}

void pbo_rotation_vector_matrix(const double theta[3], double R[9]) {
  const pbo_m3 r = rotation_vector_matrix(theta);
  memcpy(R, r.a, sizeof r.a);
}

static pbo_m4 motion_rot(const pbo_m3* R) {
  pbo_m4 m = m4_identity();
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) M4E(m, i, c) = M3E(*R, i, c);
  return m;
}

/* joint_transform, kinematics.cpp:98-117 */
static pbo_m4 joint_transform(int kind, const double* axis, const pbo_m4* offset,
                              const double* q) {
  pbo_m4 motion = m4_identity();
  switch (kind) {
    case PBO_HINGE: {
      const double th[3] = {axis[0] * q[0], axis[1] * q[0], axis[2] * q[0]};
      const pbo_m3 R = rotation_vector_matrix(th);
      motion = motion_rot(&R);
      break;
    }
    case PBO_BALL: {
      const pbo_m3 R = rotation_vector_matrix(q);
      motion = motion_rot(&R);
      break;
    }
    default: {
      const pbo_m3 R = rotation_vector_matrix(q + 3);
      motion = motion_rot(&R);
      for (int k = 0; k < 3; ++k) M4E(motion, k, 3) = q[k];
      break;
    }
  }
  return m4_mul(offset, &motion);
}

/* joint_jet, kinematics.cpp:119-169. d1[dof], d2[dof(dof+1)/2] */
static void joint_jet(int kind, const double* axis, const pbo_m4* offset, const double* q,
                      pbo_m4* value, pbo_m4* d1, pbo_m4* d2) {
  switch (kind) {
    case PBO_HINGE: {
      const pbo_m3 Ka = m3_skew(axis);
      const double th[3] = {axis[0] * q[0], axis[1] * q[0], axis[2] * q[0]};
      const pbo_m3 R = rotation_vector_matrix(th);
      const pbo_m4 motion = motion_rot(&R);
      *value = m4_mul(offset, &motion);
      const pbo_m3 KaR = m3_mul(&Ka, &R);
      const pbo_m4 e1 = m4_embed_rotation(&KaR);
      d1[0] = m4_mul(offset, &e1);
      const pbo_m3 KaKa = m3_mul(&Ka, &Ka);
      const pbo_m3 KaKaR = m3_mul(&KaKa, &R);
      const pbo_m4 e2 = m4_embed_rotation(&KaKaR);
      d2[0] = m4_mul(offset, &e2);
      break;
    }
    case PBO_BALL: {
      pbo_m3 R, dR[3], d2R[3][3];
      rotation_vector_jet(q, &R, dR, d2R);
      const pbo_m4 motion = motion_rot(&R);
      *value = m4_mul(offset, &motion);
      for (int j = 0; j < 3; ++j) {
        const pbo_m4 e = m4_embed_rotation(&dR[j]);
        d1[j] = m4_mul(offset, &e);
      }
      int idx = 0;
      for (int l = 0; l < 3; ++l)
        for (int j = 0; j <= l; ++j) {
          const pbo_m4 e = m4_embed_rotation(&d2R[j][l]);
          d2[idx++] = m4_mul(offset, &e);
        }
      break;
    }
    default: {
      pbo_m3 R, dR[3], d2R[3][3];
      rotation_vector_jet(q + 3, &R, dR, d2R);
      pbo_m4 motion = motion_rot(&R);
      for (int k = 0; k < 3; ++k) M4E(motion, k, 3) = q[k];
      *value = m4_mul(offset, &motion);
      for (int j = 0; j < 3; ++j) {
        pbo_m4 dt = m4_zero();
        M4E(dt, j, 3) = 1.0;
        d1[j] = m4_mul(offset, &dt);
        const pbo_m4 e = m4_embed_rotation(&dR[j]);
        d1[3 + j] = m4_mul(offset, &e);
      }
      for (int k = 0; k < 21; ++k) d2[k] = m4_zero();
      int idx = 0;
      for (int l = 0; l < 6; ++l)
        for (int j = 0; j <= l; ++j, ++idx)
          if (j >= 3 && l >= 3) {
            const pbo_m4 e = m4_embed_rotation(&d2R[j - 3][l - 3]);
            d2[idx] = m4_mul(offset, &e);
          }
      break;
    }
  }
}

int pbo_joint_jet(int32_t kind, const double axis[3], const double offset[16],
                  const double* q, double value[16], double* d1, double* d2) {
  pbo_m4 off, v, D1[6], D2[21];
  memcpy(off.a, offset, sizeof off.a);
  joint_jet(kind, axis, &off, q, &v, D1, D2);
  const int dof = kind_dofs(kind);
  memcpy(value, v.a, sizeof v.a);
  if (d1)
    for (int j = 0; j < dof; ++j) memcpy(&d1[16 * j], D1[j].a, sizeof(double) * 16);
  if (d2)
    for (int j = 0; j < dof * (dof + 1) / 2; ++j)
      memcpy(&d2[16 * j], D2[j].a, sizeof(double) * 16);
  return 0;
}

int pbo_joint_transform(int32_t kind, const double axis[3], const double offset[16],
                        const double* q, double value[16]) {
  pbo_m4 off;
  memcpy(off.a, offset, sizeof off.a);
  const pbo_m4 v = joint_transform(kind, axis, &off, q);
  memcpy(value, v.a, sizeof v.a);
  return 0;
}

/* forward_pass, kinematics.cpp:171-181 */
static int forward_pass(const pbo_model* m, const double* q, pbo_m4* world, pbo_err* e) {
  if (validate_configuration(m, q, m->n, e)) return -1;
  for (int i = 0; i < m->N; ++i) {
    const pbo_m4 local =
        joint_transform(m->kind[i], &m->axis[3 * i], &m->offset[i], q + m->dof_off[i]);
    const int p = m->parent[i];
    world[i] = (p >= 0) ? m4_mul(&world[p], &local) : local;
  }
  return 0;
}

int pbo_forward_pass(const pbo_model* m, const double* q, double* world) {
  pbo_err e = {0};
  pbo_m4* w = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  const int rc = forward_pass(m, q, w, &e);
  if (!rc) memcpy(world, w, sizeof(pbo_m4) * m->N);
  free(w);
  return rc;
}

/* ------------------------------------------------------------------ */
/* adjoint (adjoint.cpp:9-176)                                         */
/* ------------------------------------------------------------------ */
typedef struct {
  pbo_m4* value;  /* [N]  jets[i].value */
  pbo_m4* d1;     /* [n]  jets[i].d1[j] at dof_off[i]+j */
  pbo_m4* d2;     /* [n_d2] */
  pbo_m4* world;  /* [N] */
  pbo_m4* pworld; /* [N] parent_world */
  pbo_m4* lever;  /* [n] */
} pbo_pass;

static void pass_alloc(const pbo_model* m, pbo_pass* p) {
  p->value = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  p->d1 = (pbo_m4*)xcalloc(m->n, sizeof(pbo_m4));
  p->d2 = (pbo_m4*)xcalloc(m->n_d2, sizeof(pbo_m4));
  p->world = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  p->pworld = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  p->lever = (pbo_m4*)xcalloc(m->n, sizeof(pbo_m4));
}
static void pass_free(pbo_pass* p) {
  free(p->value); free(p->d1); free(p->d2); free(p->world); free(p->pworld); free(p->lever);
  memset(p, 0, sizeof *p);
}

/* ConfigPass::make, adjoint.cpp:9-27 (all_joint_jets validates q) */
static int pass_make(const pbo_model* m, const double* q, pbo_pass* p, pbo_err* e) {
  if (validate_configuration(m, q, m->n, e)) return -1;
  for (int i = 0; i < m->N; ++i) {
    pbo_m4 d2[21];
    pbo_m4 d1[6];
    joint_jet(m->kind[i], &m->axis[3 * i], &m->offset[i], q + m->dof_off[i], &p->value[i],
              d1, d2);
    const int dof = m->dof_cnt[i];
    for (int j = 0; j < dof; ++j) p->d1[m->dof_off[i] + j] = d1[j];
    for (int j = 0; j < dof * (dof + 1) / 2; ++j) p->d2[m->d2_off[i] + j] = d2[j];
  }
  for (int i = 0; i < m->N; ++i) {
    const int par = m->parent[i];
    p->pworld[i] = (par >= 0) ? p->world[par] : m4_identity();
    p->world[i] = m4_mul(&p->pworld[i], &p->value[i]);
    for (int j = 0; j < m->dof_cnt[i]; ++j)
      p->lever[m->dof_off[i] + j] = m4_mul(&p->pworld[i], &p->d1[m->dof_off[i] + j]);
  }
  return 0;
}

static const pbo_m4* d2_at(const pbo_model* m, const pbo_pass* p, int i, int j, int l) {
  if (j > l) {
    const int t = j;
    j = l;
    l = t;
  }
  return &p->d2[m->d2_off[i] + l * (l + 1) / 2 + j];
}

/* WeightedBody::make, adjoint.cpp:29-41 */
typedef struct {
  pbo_m4* S;
  double weighted_mass;
} pbo_wb;

static void wb_make(const pbo_model* m, const double* w, pbo_wb* wb) {
  wb->S = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  wb->weighted_mass = 0.0;
  for (int i = 0; i < m->N; ++i) {
    const double wi = w ? w[i] : 1.0;
    wb->S[i] = m4_scale(wi, &m->S[i]);
    wb->weighted_mass += wi * m->mass[i];
  }
}

/* functional_value, adjoint.cpp:43-47 */
static double functional_value(const pbo_model* m, const pbo_m4* seeds, const pbo_pass* p) {
  double v = 0.0;
  for (int i = 0; i < m->N; ++i) v += m4_ddot(&seeds[i], &p->world[i]);
  return v;
}

/* functional_grad, adjoint.cpp:49-64 */
static void functional_grad(const pbo_model* m, const pbo_m4* seeds, const pbo_pass* p,
                            double* grad) {
  const int N = m->N;
  for (int k = 0; k < m->n; ++k) grad[k] = 0.0;
  pbo_m4* adj = (pbo_m4*)xcalloc(N, sizeof(pbo_m4));
  for (int i = N - 1; i >= 0; --i) {
    m4_addto(&adj[i], &seeds[i]);
    const int off = m->dof_off[i];
    for (int j = 0; j < m->dof_cnt[i]; ++j)
      grad[off + j] += m4_ddot(&p->lever[off + j], &adj[i]);
    const int par = m->parent[i];
    if (par >= 0) {
      const pbo_m4 t = m4_mul_bt(&adj[i], &p->value[i]);
      m4_addto(&adj[par], &t);
    }
  }
  free(adj);
}

/* functional_hess, adjoint.cpp:66-101 (hess col-major n x n) */
static void functional_hess(const pbo_model* m, const pbo_m4* seeds, const pbo_pass* p,
                            double* hess) {
  const int N = m->N, n = m->n;
  for (int k = 0; k < n * n; ++k) hess[k] = 0.0;
  pbo_m4* adj = (pbo_m4*)xcalloc(N, sizeof(pbo_m4));
  pbo_m4 walk[6];
#define H(r, c) hess[(r) + (size_t)n * (c)]
  for (int i = N - 1; i >= 0; --i) {
    m4_addto(&adj[i], &seeds[i]);
    const int off = m->dof_off[i];
    const int dof = m->dof_cnt[i];
    for (int l = 0; l < dof; ++l)
      for (int j = 0; j <= l; ++j) {
        const pbo_m4 pd = m4_mul(&p->pworld[i], d2_at(m, p, i, j, l));
        const double h = m4_ddot(&pd, &adj[i]);
        H(off + j, off + l) += h;
        if (j != l) H(off + l, off + j) += h;
      }
    for (int j = 0; j < dof; ++j) walk[j] = m4_mul_bt(&adj[i], &p->d1[off + j]);
    for (int l = m->parent[i]; l >= 0; l = m->parent[l]) {
      const int offl = m->dof_off[l];
      for (int k = 0; k < m->dof_cnt[l]; ++k)
        for (int j = 0; j < dof; ++j) {
          const double h = m4_ddot(&p->lever[offl + k], &walk[j]);
          H(offl + k, off + j) += h;
          H(off + j, offl + k) += h;
        }
      for (int j = 0; j < dof; ++j) walk[j] = m4_mul_bt(&walk[j], &p->value[l]);
    }
    const int par = m->parent[i];
    if (par >= 0) {
      const pbo_m4 t = m4_mul_bt(&adj[i], &p->value[i]);
      m4_addto(&adj[par], &t);
    }
  }
#undef H
  free(adj);
}

/* correlation_value, adjoint.cpp:113-120 */
static double correlation_value(const pbo_model* m, const pbo_wb* wb, const pbo_pass* pa,
                                const pbo_pass* pb) {
  double value = 0.0;
  for (int i = 0; i < m->N; ++i) {
    const pbo_m4 ts = m4_mul(&pa->world[i], &wb->S[i]);
    value += m4_ddot(&ts, &pb->world[i]);
  }
  return value - wb->weighted_mass;
}

/* correlation_seeds, adjoint.cpp:105-109 */
static void correlation_seeds(const pbo_model* m, const pbo_wb* wb, const pbo_pass* pa,
                              pbo_m4* seeds) {
  for (int i = 0; i < m->N; ++i) seeds[i] = m4_mul(&pa->world[i], &wb->S[i]);
}

/* trace(A^T * B * C) with the shim's left-to-right evaluation */
static double trace3_at(const pbo_m4* A, const pbo_m4* B, const pbo_m4* C) {
  const pbo_m4 t = m4_mul_at(A, B);
  const pbo_m4 u = m4_mul(&t, C);
  return m4_trace(&u);
}

/* correlation_hess_ab, adjoint.cpp:132-176 */
static void correlation_hess_ab(const pbo_model* m, const pbo_wb* wb, const pbo_pass* pa,
                                const pbo_pass* pb, double* hess) {
  const int N = m->N, n = m->n;
  for (int k = 0; k < n * n; ++k) hess[k] = 0.0;
  pbo_m4* acc = (pbo_m4*)xcalloc(N, sizeof(pbo_m4));
#define H(r, c) hess[(r) + (size_t)n * (c)]
  for (int i = N - 1; i >= 0; --i) {
    m4_addto(&acc[i], &wb->S[i]);
    const int off = m->dof_off[i];
    const int dof = m->dof_cnt[i];
    for (int j = 0; j < dof; ++j)
      for (int k = 0; k < dof; ++k)
        H(off + j, off + k) += trace3_at(&pa->lever[off + j], &pb->lever[off + k], &acc[i]);
    pbo_m4 fwd = m4_mul(&pb->value[i], &acc[i]);
    pbo_m4 bwd = m4_mul_bt(&acc[i], &pa->value[i]);
    for (int l = m->parent[i]; l >= 0; l = m->parent[l]) {
      const int offl = m->dof_off[l];
      for (int j = 0; j < dof; ++j) {
        const pbo_m4* ua = &pa->lever[off + j]; /* used transposed */
        const pbo_m4* vb = &pb->lever[off + j];
        for (int k = 0; k < m->dof_cnt[l]; ++k) {
          H(off + j, offl + k) += trace3_at(ua, &pb->lever[offl + k], &fwd);
          const pbo_m4 lat = m4_transpose(&pa->lever[offl + k]);
          const pbo_m4 t = m4_mul(&lat, vb);
          const pbo_m4 u = m4_mul(&t, &bwd);
          H(offl + k, off + j) += m4_trace(&u);
        }
      }
      fwd = m4_mul(&pb->value[l], &fwd);
      bwd = m4_mul_bt(&bwd, &pa->value[l]);
    }
    const int par = m->parent[i];
    if (par >= 0) {
      const pbo_m4 t = m4_mul(&pb->value[i], &acc[i]);
      const pbo_m4 u = m4_mul_bt(&t, &pa->value[i]);
      m4_addto(&acc[par], &u);
    }
  }
#undef H
  free(acc);
}

int pbo_correlation(const pbo_model* m, const double* qa, const double* qb,
                    const double* weights, double* value, double* grad_b, double* hess_bb,
                    double* hess_ab) {
  pbo_err e = {0};
  pbo_pass pa, pb;
  pass_alloc(m, &pa);
  pass_alloc(m, &pb);
  pbo_wb wb;
  wb_make(m, weights, &wb);
  int rc = pass_make(m, qa, &pa, &e);
  if (!rc) rc = pass_make(m, qb, &pb, &e);
  if (!rc) {
    if (value) *value = correlation_value(m, &wb, &pa, &pb);
    pbo_m4* seeds = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
    correlation_seeds(m, &wb, &pa, seeds);
    if (grad_b) functional_grad(m, seeds, &pb, grad_b);
    if (hess_bb) functional_hess(m, seeds, &pb, hess_bb);
    if (hess_ab) correlation_hess_ab(m, &wb, &pa, &pb, hess_ab);
    free(seeds);
  }
  free(wb.S);
  pass_free(&pa);
  pass_free(&pb);
  return rc;
}

int pbo_functional(const pbo_model* m, const double* seeds_in, const double* q,
                   double* value, double* grad, double* hess) {
  pbo_err e = {0};
  pbo_pass p;
  pass_alloc(m, &p);
  int rc = pass_make(m, q, &p, &e);
  if (!rc) {
    pbo_m4* seeds = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
    memcpy(seeds, seeds_in, sizeof(pbo_m4) * m->N);
    if (value) *value = functional_value(m, seeds, &p);
    if (grad) functional_grad(m, seeds, &p, grad);
    if (hess) functional_hess(m, seeds, &p, hess);
    free(seeds);
  }
  pass_free(&p);
  return rc;
}

/* ------------------------------------------------------------------ */
/* collocation (collocation.cpp:12-95)                                 */
/* ------------------------------------------------------------------ */
static void legendre_eval(int n, double x, double* pv, double* dv) {
  double p0 = 1.0, p1 = x;
  if (n == 0) {
    *pv = 1.0;
    *dv = 0.0;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  const double d = n * (x * p1 - p0) / (x * x - 1.0);
  *pv = p1;
  *dv = d;
}

int pbo_legendre_points(int32_t order, double* out) {
  if (order < 2) return -1;
  const int n = order - 2;
  for (int i = 0; i < n; ++i) {
    double x = -pbm_cos(3.141592653589793 * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p, d;
      legendre_eval(n, x, &p, &d);
      const double dx = p / d;
      x -= dx;
      if (fabs(dx) < 1e-14) break;
    }
    out[i] = 0.5 * (x + 1.0);
  }
  out[n] = 1.0;
  return 0;
}

/*
 * FullPivLU(A).inverse() -- the eigen_lite definition: Gauss-Jordan on
 * [A | I] with complete pivoting (largest |a| of the trailing block, first
 * in column-major scan order on ties), row/column swaps, then undo the
 * column permutation on the rows of the inverse.
 */
static int fullpiv_inverse(const double* A_in, int k, double* inv) {
  double* A = (double*)xcalloc((size_t)k * k, sizeof(double));
  double* X = (double*)xcalloc((size_t)k * k, sizeof(double));
  int* colperm = (int*)xcalloc(k, sizeof(int));
  memcpy(A, A_in, sizeof(double) * k * k);
  for (int i = 0; i < k; ++i) {
    X[i + k * i] = 1.0;
    colperm[i] = i;
  }
#define AA(r, c) A[(r) + (size_t)k * (c)]
#define XX(r, c) X[(r) + (size_t)k * (c)]
  int ok = 1;
  for (int s = 0; s < k; ++s) {
    int pr = s, pc = s;
    double best = -1.0;
    for (int c = s; c < k; ++c)
      for (int r = s; r < k; ++r)
        if (fabs(AA(r, c)) > best) {
          best = fabs(AA(r, c));
          pr = r;
          pc = c;
        }
    if (!(best > 0.0)) {
      ok = 0;
      break;
    }
    if (pr != s) {
      for (int c = 0; c < k; ++c) {
        double t = AA(s, c); AA(s, c) = AA(pr, c); AA(pr, c) = t;
        t = XX(s, c); XX(s, c) = XX(pr, c); XX(pr, c) = t;
      }
    }
    if (pc != s) {
      for (int r = 0; r < k; ++r) {
        const double t = AA(r, s); AA(r, s) = AA(r, pc); AA(r, pc) = t;
      }
      const int t = colperm[s]; colperm[s] = colperm[pc]; colperm[pc] = t;
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
        AA(r, c) = fma(-f, AA(s, c), AA(r, c));
        XX(r, c) = fma(-f, XX(s, c), XX(r, c));
      }
    }
  }
  if (ok) {
    /* A P = ... => inverse rows permuted by colperm */
    for (int r = 0; r < k; ++r)
      for (int c = 0; c < k; ++c) inv[colperm[r] + (size_t)k * c] = XX(r, c);
  }
#undef AA
#undef XX
  free(A);
  free(X);
  free(colperm);
  return ok ? 0 : -1;
}

typedef struct {
  int order;
  double alphas[8];
  double times[9];
  double H[81];
  double H2[81];
} pbo_scheme;

/* build_scheme, collocation.cpp:53-95 */
static int build_scheme(int order, double dt, pbo_scheme* s, pbo_err* e) {
  if (order < 2) {
    err_set(e, "collocation order must be >= 2");
    return -1;
  }
  if (order > 7) {
    err_set(e, "collocation order above 7 is not supported by the oracle");
    return -1;
  }
  if (dt <= 0.0) {
    err_set(e, "dt must be positive");
    return -1;
  }
  memset(s, 0, sizeof *s);
  s->order = order;
  pbo_legendre_points(order, s->alphas);
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
  if (fullpiv_inverse(V, k, s->H)) {
    err_set(e, "collocation times produced a singular Vandermonde system");
    return -1;
  }
  double mono2[81];
  for (int q = 0; q < k * k; ++q) mono2[q] = 0.0;
  for (int j = 0; j < k; ++j)
    for (int p = 2; p < k; ++p) mono2[p + k * j] = p * (p - 1) * pow(s->times[j], p - 2);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) {
      double acc = s->H[i] * mono2[k * j];
      for (int q = 1; q < k; ++q) acc = fma(s->H[i + k * q], mono2[q + k * j], acc);
      s->H2[i + k * j] = acc;
    }
  return 0;
}

int pbo_build_scheme(int32_t order, double dt, double* alphas, double* times, double* H,
                     double* H2) {
  pbo_err e = {0};
  pbo_scheme s;
  if (build_scheme(order, dt, &s, &e)) return -1;
  const int k = order + 1;
  if (alphas) memcpy(alphas, s.alphas, sizeof(double) * (order - 1));
  if (times) memcpy(times, s.times, sizeof(double) * k);
  if (H) memcpy(H, s.H, sizeof(double) * k * k);
  if (H2) memcpy(H2, s.H2, sizeof(double) * k * k);
  return 0;
}

/* ------------------------------------------------------------------ */
/* potentials (objective.cpp:25-138)                                   */
/* ------------------------------------------------------------------ */
typedef struct {
  double value;
  double* grad; /* [n] */
  double* gn;   /* [n*n] or NULL */
  double* hess; /* [n*n] or NULL */
} pbo_pot;

/* Eigen isZero(): all |x| <= 1e-12 */
static int vec3_is_zero(const double* g) {
  return fabs(g[0]) <= 1e-12 && fabs(g[1]) <= 1e-12 && fabs(g[2]) <= 1e-12;
}

static void m4_mul_vec(const pbo_m4* A, const double* x, double* y) {
  for (int i = 0; i < 4; ++i) {
    double acc = M4E(*A, i, 0) * x[0];
    acc = fma(M4E(*A, i, 1), x[1], acc);
    acc = fma(M4E(*A, i, 2), x[2], acc);
    acc = fma(M4E(*A, i, 3), x[3], acc);
    y[i] = acc;
  }
}

/* potential_terms, objective.cpp:25-138 */
static void potential_terms(const pbo_model* m, const pbo_forces* f, const pbo_pass* pn,
                            const pbo_m4* world_prev, double dt, int want_grad,
                            int want_gn, int want_hess, const double* hess_ab_next,
                            pbo_pot* out) {
  const int N = m->N, n = m->n;
  out->value = 0.0;
  for (int k = 0; k < n; ++k) out->grad[k] = 0.0;
  if (want_gn)
    for (size_t k = 0; k < (size_t)n * n; ++k) out->gn[k] = 0.0;
  if (want_hess)
    for (size_t k = 0; k < (size_t)n * n; ++k) out->hess[k] = 0.0;

  const int needs_ab = (want_gn || want_hess) && f->drag_d > 0.0;
  double* ab_local = NULL;
  const double* ab = hess_ab_next;
  if (needs_ab && ab == NULL) {
    pbo_wb wb;
    wb_make(m, NULL, &wb);
    ab_local = (double*)xcalloc((size_t)n * n, sizeof(double));
    correlation_hess_ab(m, &wb, pn, pn, ab_local);
    free(wb.S);
    ab = ab_local;
  }
  pbo_m4* cot = (pbo_m4*)xcalloc(N, sizeof(pbo_m4));
  int have_cot = 0;

  if (!vec3_is_zero(f->gravity)) {
    const double ghat[4] = {f->gravity[0], f->gravity[1], f->gravity[2], 0.0};
    const double e4[4] = {0.0, 0.0, 0.0, 1.0};
    for (int i = 0; i < N; ++i) {
      double u[4];
      m4_mul_vec(&m->S[i], e4, u);
      pbo_m4 c;
      for (int s = 0; s < 4; ++s)
        for (int r = 0; r < 4; ++r) M4E(c, r, s) = (-ghat[r]) * u[s];
      out->value += m4_ddot(&c, &pn->world[i]);
      m4_addto(&cot[i], &c);
    }
    have_cot = 1;
  }

  if (f->drag_d > 0.0) {
    const double scale = f->drag_d / (dt * dt);
    for (int i = 0; i < N; ++i) {
      const pbo_m4 diff = m4_sub(&pn->world[i], &world_prev[i]);
      const pbo_m4 diff_s = m4_mul(&diff, &m->S[i]);
      out->value += scale * m4_ddot(&diff_s, &diff);
      const pbo_m4 t = m4_scale(2.0 * scale, &diff_s);
      m4_addto(&cot[i], &t);
    }
    have_cot = 1;
    const double s2 = 2.0 * scale;
    if (want_gn)
      for (size_t k = 0; k < (size_t)n * n; ++k) out->gn[k] = out->gn[k] + s2 * ab[k];
    if (want_hess)
      for (size_t k = 0; k < (size_t)n * n; ++k) out->hess[k] = out->hess[k] + s2 * ab[k];
  }

  if (f->has_contact && (f->contact_d1 > 0.0 || f->contact_d2 > 0.0)) {
    const double* nrm = f->plane_normal;
    const double d1c = f->contact_d1, d2c = f->contact_d2;
    double proj[9];
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) proj[r + 3 * c] = ((r == c) ? 1.0 : 0.0) - nrm[r] * nrm[c];
    const int need_jx = want_gn || want_hess;
    double* jx = need_jx ? (double*)xcalloc(3 * (size_t)n, sizeof(double)) : NULL;
    double* dd = need_jx ? (double*)xcalloc(n, sizeof(double)) : NULL;
    double* jr = need_jx ? (double*)xcalloc(3 * (size_t)n, sizeof(double)) : NULL;
    double* tmp = need_jx ? (double*)xcalloc(3 * (size_t)n, sizeof(double)) : NULL;
    for (int i = 0; i < N; ++i) {
      for (int sidx = m->sample_off[i]; sidx < m->sample_off[i + 1]; ++sidx) {
        const double ph[4] = {m->samples[3 * sidx], m->samples[3 * sidx + 1],
                              m->samples[3 * sidx + 2], 1.0};
        double x4[4], xp4[4];
        m4_mul_vec(&pn->world[i], ph, x4);
        const double depth = f->plane_offset - vfix_dot(nrm, x4, 3);
        if (depth <= 0.0) continue;
        m4_mul_vec(&world_prev[i], ph, xp4);
        double v[3], pv[3];
        for (int k = 0; k < 3; ++k) v[k] = (x4[k] - xp4[k]) / dt;
        for (int r = 0; r < 3; ++r) {
          double acc = proj[r] * v[0];
          acc = fma(proj[r + 3], v[1], acc);
          acc = fma(proj[r + 6], v[2], acc);
          pv[r] = acc;
        }
        const double pv2 = vfix_dot(pv, pv, 3);
        out->value += d1c * depth * depth + d2c * depth * depth * pv2;
        const double a = -2.0 * d1c * depth - 2.0 * d2c * depth * pv2;
        const double b = 2.0 * d2c * depth * depth / dt;
        double dq[4];
        for (int k = 0; k < 3; ++k) dq[k] = a * nrm[k] + b * pv[k];
        dq[3] = 0.0;
        pbo_m4 oc;
        for (int s = 0; s < 4; ++s)
          for (int r = 0; r < 4; ++r) M4E(oc, r, s) = dq[r] * ph[s];
        m4_addto(&cot[i], &oc);
        have_cot = 1;

        if (need_jx) {
          for (int k = 0; k < 3 * n; ++k) jx[k] = 0.0;
          double y[4] = {ph[0], ph[1], ph[2], ph[3]};
          for (int l = i; l >= 0; l = m->parent[l]) {
            const int off = m->dof_off[l];
            for (int j = 0; j < m->dof_cnt[l]; ++j) {
              double t4[4];
              m4_mul_vec(&pn->lever[off + j], y, t4);
              for (int r = 0; r < 3; ++r) jx[r + 3 * (off + j)] = t4[r];
            }
            double y2[4];
            m4_mul_vec(&pn->value[l], y, y2);
            memcpy(y, y2, sizeof y);
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
                out->gn[aa + (size_t)n * bb] = out->gn[aa + (size_t)n * bb] + (c2 * dd[aa]) * dd[bb];
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
                for (int r = 0; r < 3; ++r)
                  jr[r + 3 * k] = pv[r] * dd[k] + ddt * tmp[r + 3 * k];
              const double c3 = 2.0 * d2c;
              for (int bb = 0; bb < n; ++bb)
                for (int aa = 0; aa < n; ++aa) {
                  double acc = (c3 * jr[3 * aa]) * jr[3 * bb];
                  acc = fma(c3 * jr[1 + 3 * aa], jr[1 + 3 * bb], acc);
                  acc = fma(c3 * jr[2 + 3 * aa], jr[2 + 3 * bb], acc);
                  out->gn[aa + (size_t)n * bb] = out->gn[aa + (size_t)n * bb] + acc;
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
            /* (jx^T * hxx) * jx */
            for (int k = 0; k < n; ++k)
              for (int c = 0; c < 3; ++c) {
                double acc = jx[3 * k] * hxx[3 * c];
                acc = fma(jx[1 + 3 * k], hxx[1 + 3 * c], acc);
                acc = fma(jx[2 + 3 * k], hxx[2 + 3 * c], acc);
                tmp[k + (size_t)n * c] = acc; /* n x 3 col-major */
              }
            for (int bb = 0; bb < n; ++bb)
              for (int aa = 0; aa < n; ++aa) {
                double acc = tmp[aa] * jx[3 * bb];
                acc = fma(tmp[aa + (size_t)n], jx[1 + 3 * bb], acc);
                acc = fma(tmp[aa + 2 * (size_t)n], jx[2 + 3 * bb], acc);
                out->hess[aa + (size_t)n * bb] = out->hess[aa + (size_t)n * bb] + acc;
              }
          }
        }
      }
    }
    free(jx);
    free(dd);
    free(jr);
    free(tmp);
  }

  if (have_cot) {
    if (want_grad) functional_grad(m, cot, pn, out->grad);
    if (want_hess) {
      double* fh = (double*)xcalloc((size_t)n * n, sizeof(double));
      functional_hess(m, cot, pn, fh);
      for (size_t k = 0; k < (size_t)n * n; ++k) out->hess[k] = out->hess[k] + fh[k];
      free(fh);
    }
  }
  free(cot);
  free(ab_local);
}

int pbo_eval_potentials(const pbo_model* m, const pbo_forces* f, const double* q_next,
                        const double* q_prev, double dt, int32_t want_gn,
                        int32_t want_hess, double* value, double* grad, double* gn,
                        double* hess) {
  pbo_err e = {0};
  if (validate_configuration(m, q_next, m->n, &e)) return -1;
  if (validate_configuration(m, q_prev, m->n, &e)) return -1;
  pbo_pass pn;
  pass_alloc(m, &pn);
  pass_make(m, q_next, &pn, &e);
  pbo_m4* wp = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  forward_pass(m, q_prev, wp, &e);
  const int n = m->n;
  pbo_pot pot;
  pot.grad = (double*)xcalloc(n, sizeof(double));
  pot.gn = want_gn ? (double*)xcalloc((size_t)n * n, sizeof(double)) : NULL;
  pot.hess = want_hess ? (double*)xcalloc((size_t)n * n, sizeof(double)) : NULL;
  potential_terms(m, f, &pn, wp, dt, 1, want_gn, want_hess, NULL, &pot);
  if (value) *value = pot.value;
  if (grad) memcpy(grad, pot.grad, sizeof(double) * n);
  if (gn && want_gn) memcpy(gn, pot.gn, sizeof(double) * n * n);
  if (hess && want_hess) memcpy(hess, pot.hess, sizeof(double) * n * n);
  free(pot.grad);
  free(pot.gn);
  free(pot.hess);
  free(wp);
  pass_free(&pn);
  return 0;
}

/* ------------------------------------------------------------------ */
/* StepObjective (objective.cpp:155-343)                               */
/* ------------------------------------------------------------------ */
typedef struct {
  const pbo_model* m;
  const pbo_forces* f;
  const pbo_scheme* scheme;
  double dt;
  int kind;
  double* hist0; /* [n] */
  double* hist1; /* [n] */
  double* tau;   /* [u][n] tau_at_instants */
  int tau_count;
  /* Cache */
  pbo_wb wb;
  pbo_pass hp[2];
  double hist_const;
} pbo_objective;

typedef struct {
  double value;
  double* grad; /* [dim] */
  double* gn;   /* [dim*dim] or NULL */
  int has_gn;
} pbo_eval;

static int obj_dim(const pbo_objective* o) { return o->m->n * (o->scheme->order - 1); }

/* StepObjective ctor, objective.cpp:162-185 */
static int obj_init(pbo_objective* o, const pbo_model* m, const pbo_forces* f,
                    const pbo_scheme* scheme, double dt, int kind, const double* h0,
                    const double* h1, const double* tau_instants, int tau_count,
                    pbo_err* e) {
  memset(o, 0, sizeof *o);
  o->m = m;
  o->f = f;
  o->scheme = scheme;
  o->dt = dt;
  o->kind = kind;
  const int n = m->n;
  if (kind == PBO_ENERGY && scheme->order != 2) {
    err_set(e, "the energy objective is only defined for order 2");
    return -1;
  }
  if (dt <= 0.0) {
    err_set(e, "step problem dt must be positive");
    return -1;
  }
  if (validate_configuration(m, h0, n, e)) return -1;
  if (validate_configuration(m, h1, n, e)) return -1;
  o->hist0 = (double*)xcalloc(n, sizeof(double));
  o->hist1 = (double*)xcalloc(n, sizeof(double));
  memcpy(o->hist0, h0, sizeof(double) * n);
  memcpy(o->hist1, h1, sizeof(double) * n);
  o->tau_count = tau_instants ? tau_count : 0;
  if (o->tau_count) {
    o->tau = (double*)xcalloc((size_t)n * tau_count, sizeof(double));
    memcpy(o->tau, tau_instants, sizeof(double) * n * tau_count);
  }
  wb_make(m, NULL, &o->wb);
  pass_alloc(m, &o->hp[0]);
  pass_alloc(m, &o->hp[1]);
  pass_make(m, h0, &o->hp[0], e);
  pass_make(m, h1, &o->hp[1], e);
  if (kind == PBO_ENERGY) {
    const pbo_pass* prev2 = &o->hp[0];
    const pbo_pass* prev1 = &o->hp[1];
    o->hist_const = 4.0 * correlation_value(m, &o->wb, prev1, prev1) +
                    correlation_value(m, &o->wb, prev2, prev2) -
                    4.0 * correlation_value(m, &o->wb, prev1, prev2);
  }
  return 0;
}

static void obj_free(pbo_objective* o) {
  free(o->hist0);
  free(o->hist1);
  free(o->tau);
  free(o->wb.S);
  pass_free(&o->hp[0]);
  pass_free(&o->hp[1]);
}

/* actuation_at, objective.cpp:195-204 (tau written into out) */
static void actuation_at(const pbo_objective* o, int instant, double* out) {
  const int n = o->m->n;
  if (instant < o->tau_count) {
    memcpy(out, o->tau + (size_t)instant * n, sizeof(double) * n);
    return;
  }
  if (o->f->tau_len == n) {
    memcpy(out, o->f->tau, sizeof(double) * n);
    return;
  }
  for (int k = 0; k < n; ++k) out[k] = 0.0;
}

/* diagnostic: number of StepObjective evaluations (value or evaluate) */
static long long g_eval_count = 0;
long long pbo_eval_counter(int reset) {
  const long long v = g_eval_count;
  if (reset) g_eval_count = 0;
  return v;
}

/* StepObjective::evaluate_impl, objective.cpp:206-334 */
static int obj_evaluate(const pbo_objective* o, const double* x, int want_grad, int want_gn,
                        pbo_eval* out, pbo_err* e) {
  const pbo_model* m = o->m;
  const pbo_scheme* sc = o->scheme;
  const int N = m->N, n = m->n;
  const double dt = o->dt;
  const double inv_dt2 = 1.0 / (dt * dt);
  out->has_gn = 0;
  __atomic_add_fetch(&g_eval_count, 1, __ATOMIC_RELAXED);

  if (o->kind == PBO_ENERGY) {
    pbo_pass pass;
    pass_alloc(m, &pass);
    if (pass_make(m, x, &pass, e)) {
      pass_free(&pass);
      return -1;
    }
    const pbo_wb* wb = &o->wb;
    const pbo_pass* prev2 = &o->hp[0];
    const pbo_pass* prev1 = &o->hp[1];
    const double inertial =
        0.5 * inv_dt2 *
        (correlation_value(m, wb, &pass, &pass) -
         4.0 * correlation_value(m, wb, prev1, &pass) +
         2.0 * correlation_value(m, wb, prev2, &pass) + o->hist_const);
    double* ab = NULL;
    if (want_gn) {
      ab = (double*)xcalloc((size_t)n * n, sizeof(double));
      correlation_hess_ab(m, wb, &pass, &pass, ab);
    }
    pbo_pot pot;
    pot.grad = (double*)xcalloc(n, sizeof(double));
    pot.gn = want_gn ? (double*)xcalloc((size_t)n * n, sizeof(double)) : NULL;
    pot.hess = NULL;
    potential_terms(m, o->f, &pass, prev1->world, dt, want_grad, want_gn, 0, ab, &pot);
    double* tau = (double*)xcalloc(n, sizeof(double));
    actuation_at(o, 0, tau);
    out->value = inertial + pot.value - vdyn_dot(tau, x, n);
    if (want_grad) {
      pbo_m4* seeds = (pbo_m4*)xcalloc(N, sizeof(pbo_m4));
      for (int i = 0; i < N; ++i) {
        const pbo_m4 t2 = m4_scale(2.0, &prev1->world[i]);
        pbo_m4 d = m4_sub(&pass.world[i], &t2);
        d = m4_add(&d, &prev2->world[i]);
        d = m4_scale(inv_dt2, &d);
        seeds[i] = m4_mul(&d, &wb->S[i]);
      }
      double* g = (double*)xcalloc(n, sizeof(double));
      functional_grad(m, seeds, &pass, g);
      for (int k = 0; k < n; ++k) out->grad[k] = (g[k] + pot.grad[k]) - tau[k];
      free(g);
      free(seeds);
    }
    if (want_gn) {
      double* gn = (double*)xcalloc((size_t)n * n, sizeof(double));
      for (size_t k = 0; k < (size_t)n * n; ++k) gn[k] = inv_dt2 * ab[k] + pot.gn[k];
      for (int c = 0; c < n; ++c)
        for (int r = 0; r < n; ++r)
          out->gn[r + (size_t)n * c] = 0.5 * (gn[r + (size_t)n * c] + gn[c + (size_t)n * r]);
      out->has_gn = 1;
      free(gn);
    }
    free(tau);
    free(pot.grad);
    free(pot.gn);
    free(ab);
    pass_free(&pass);
    return 0;
  }

  /* --- residual form, objective.cpp:258-334 --- */
  const int u = sc->order - 1;
  const int U = n * u;
  const int K1 = sc->order + 1;
  pbo_pass* up = (pbo_pass*)xcalloc(u, sizeof(pbo_pass));
  const pbo_pass** window = (const pbo_pass**)xcalloc(K1, sizeof(pbo_pass*));
  window[0] = &o->hp[0];
  window[1] = &o->hp[1];
  int rc = 0;
  for (int mm = 0; mm < u; ++mm) {
    pass_alloc(m, &up[mm]);
    if (!rc && pass_make(m, x + (size_t)mm * n, &up[mm], e)) rc = -1;
    window[2 + mm] = &up[mm];
  }
  if (rc) {
    for (int mm = 0; mm < u; ++mm) pass_free(&up[mm]);
    free(up);
    free(window);
    return -1;
  }
  double* resid = (double*)xcalloc((size_t)U, sizeof(double));
  double* jac = want_grad ? (double*)xcalloc((size_t)U * U, sizeof(double)) : NULL;
  double* ab_mm = (double*)xcalloc((size_t)n * n, sizeof(double));
  double* fh = (double*)xcalloc((size_t)n * n, sizeof(double));
  double* tau = (double*)xcalloc(n, sizeof(double));
  pbo_m4* seeds = (pbo_m4*)xcalloc(N, sizeof(pbo_m4));
  pbo_pot pot;
  pot.grad = (double*)xcalloc(n, sizeof(double));
  pot.gn = NULL;
  pot.hess = want_grad ? (double*)xcalloc((size_t)n * n, sizeof(double)) : NULL;
#define J(r, c) jac[(r) + (size_t)U * (c)]
  for (int mm = 0; mm < u; ++mm) {
    const pbo_pass* pass_m = window[2 + mm];
    const double* stencil = &sc->H2[K1 * (2 + mm)]; /* H2.col(2+m) */
    for (int i = 0; i < N; ++i) {
      pbo_m4 acc = m4_zero();
      for (int j = 0; j < K1; ++j) {
        const pbo_m4 t = m4_scale(stencil[j], &window[j]->world[i]);
        m4_addto(&acc, &t);
      }
      const pbo_m4 sa = m4_scale(inv_dt2, &acc);
      seeds[i] = m4_mul(&sa, &o->wb.S[i]);
    }
    double* g = resid + (size_t)mm * n;
    functional_grad(m, seeds, pass_m, g);
    if (want_grad) correlation_hess_ab(m, &o->wb, pass_m, pass_m, ab_mm);
    const double t_local = sc->times[2 + mm];
    potential_terms(m, o->f, pass_m, o->hp[1].world, t_local * dt, 1, 0, want_grad,
                    want_grad ? ab_mm : NULL, &pot);
    actuation_at(o, mm, tau);
    for (int k = 0; k < n; ++k) g[k] = g[k] + (pot.grad[k] - tau[k]);
    if (want_grad) {
      functional_hess(m, seeds, pass_m, fh);
      const double cm = inv_dt2 * stencil[2 + mm];
      for (int c = 0; c < n; ++c)
        for (int r = 0; r < n; ++r)
          J(mm * n + r, mm * n + c) =
              (fh[r + (size_t)n * c] + cm * ab_mm[c + (size_t)n * r]) + pot.hess[r + (size_t)n * c];
      for (int l = 0; l < u; ++l) {
        if (l == mm) continue;
        correlation_hess_ab(m, &o->wb, window[2 + l], pass_m, fh);
        const double cl = inv_dt2 * stencil[2 + l];
        for (int c = 0; c < n; ++c)
          for (int r = 0; r < n; ++r) J(mm * n + r, l * n + c) = cl * fh[c + (size_t)n * r];
      }
    }
  }
  out->value = 0.0;
  for (int mm = 0; mm < u; ++mm) out->value += vdyn_sqnorm(resid + (size_t)mm * n, n);
  if (want_grad) {
    /* grad = (2 J^T) g */
    for (int a = 0; a < U; ++a) {
      double acc = (2.0 * J(0, a)) * resid[0];
      for (int k = 1; k < U; ++k) acc = fma(2.0 * J(k, a), resid[k], acc);
      out->grad[a] = acc;
    }
    if (want_gn) {
      double* gn = (double*)xcalloc((size_t)U * U, sizeof(double));
      for (int b = 0; b < U; ++b)
        for (int a = 0; a < U; ++a) {
          double acc = (2.0 * J(0, a)) * J(0, b);
          for (int k = 1; k < U; ++k) acc = fma(2.0 * J(k, a), J(k, b), acc);
          gn[a + (size_t)U * b] = acc;
        }
      for (int c = 0; c < U; ++c)
        for (int r = 0; r < U; ++r)
          out->gn[r + (size_t)U * c] = 0.5 * (gn[r + (size_t)U * c] + gn[c + (size_t)U * r]);
      out->has_gn = 1;
      free(gn);
    }
  }
#undef J
  free(pot.grad);
  free(pot.hess);
  free(seeds);
  free(tau);
  free(fh);
  free(ab_mm);
  free(jac);
  free(resid);
  for (int mm = 0; mm < u; ++mm) pass_free(&up[mm]);
  free(up);
  free(window);
  return 0;
}

int pbo_step_eval(const pbo_model* m, const pbo_forces* f, int32_t order, double dt,
                  int32_t objective, const double* history, const double* tau_instants,
                  const double* x, int32_t want_grad, int32_t want_gn, double* value,
                  double* grad, double* gn) {
  pbo_err e = {0};
  pbo_scheme sc;
  if (build_scheme(order, dt, &sc, &e)) return -1;
  pbo_objective o;
  const int n = m->n;
  if (obj_init(&o, m, f, &sc, dt, objective, history, history + n, tau_instants,
               order - 1, &e)) {
    obj_free(&o);
    return -1;
  }
  const int dim = obj_dim(&o);
  pbo_eval ev;
  ev.grad = (double*)xcalloc(dim, sizeof(double));
  ev.gn = want_gn ? (double*)xcalloc((size_t)dim * dim, sizeof(double)) : NULL;
  const int rc = obj_evaluate(&o, x, want_grad, want_gn, &ev, &e);
  if (!rc) {
    if (value) *value = ev.value;
    if (grad && want_grad) memcpy(grad, ev.grad, sizeof(double) * dim);
    if (gn && want_gn && ev.has_gn) memcpy(gn, ev.gn, sizeof(double) * dim * dim);
  }
  free(ev.grad);
  free(ev.gn);
  obj_free(&o);
  return rc;
}

/* ------------------------------------------------------------------ */
/* optim (optim.cpp:11-250)                                            */
/* ------------------------------------------------------------------ */

/* spd_solve = LLT, optim.cpp:11-15; eigen_lite LLT definition:
 * right-looking column Cholesky, fma updates in ascending k, fails on a
 * pivot <= 0 (NaN passes, as in Eigen); forward substitution ascending,
 * backward substitution column-oriented (descending). */
static int llt_factor(double* A, int n) {
#define AA(r, c) A[(r) + (size_t)n * (c)]
  for (int k = 0; k < n; ++k) {
    const double x = AA(k, k);
    if (x <= 0.0) return -1;
    const double d = sqrt(x);
    AA(k, k) = d;
    for (int i = k + 1; i < n; ++i) AA(i, k) = AA(i, k) / d;
    for (int j = k + 1; j < n; ++j) {
      const double ljk = AA(j, k);
      for (int i = j; i < n; ++i) AA(i, j) = fma(-AA(i, k), ljk, AA(i, j));
    }
  }
  return 0;
}
#define AA_L(L, n, r, c) (L)[(r) + (size_t)(n) * (c)]
static void llt_solve(const double* L, int n, const double* b, double* x) {
  for (int i = 0; i < n; ++i) x[i] = b[i];
  for (int j = 0; j < n; ++j) {
    x[j] = x[j] / AA_L(L, n, j, j);
    for (int i = j + 1; i < n; ++i) x[i] = fma(-AA_L(L, n, i, j), x[j], x[i]);
  }
  for (int j = n - 1; j >= 0; --j) {
    x[j] = x[j] / AA_L(L, n, j, j);
    for (int i = 0; i < j; ++i) x[i] = fma(-AA_L(L, n, j, i), x[j], x[i]);
  }
}
#undef AA

int pbo_spd_solve(const double* A, const double* b, int32_t n, double* x) {
  double* L = (double*)xcalloc((size_t)n * n, sizeof(double));
  memcpy(L, A, sizeof(double) * n * n);
  int rc = llt_factor(L, n);
  if (!rc) llt_solve(L, n, b, x);
  free(L);
  return rc ? 1 : 0;
}

void pbo_default_optimizer(pbo_optimizer_config* c) {
  c->kind = PBO_LM;
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

void pbo_default_sim(pbo_sim_config* s) {
  memset(s, 0, sizeof *s);
  s->dt = 0.01;
  s->duration = 1.0;
  s->order = 2;
  s->objective = PBO_ENERGY;
  pbo_default_optimizer(&s->opt);
  s->consecutive_fail_limit = 25;
  s->refined_bootstrap = 0;
  s->warm_start = 1;
}

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_FAILED = 2 };

typedef struct {
  pbo_optimizer_config cfg;
  int dim;
  double* x;
  double value;
  double* grad;
  double grad0_norm;
  int status;
  int iterations;
  int stagnant;
  int accepted;
  double* values; /* [max_iters] */
  /* LM */
  double* gn;
  double lambda;
  /* LBFGS ring (deque) */
  int hcount, hstart;
  double* hs; /* [mem][dim] */
  double* hy;
  double* hsy;
  /* scratch */
  double *dir, *cand, *tmp, *alpha, *damped, *step;
  pbo_eval ev;
} pbo_solver;

static double scaled_tol(const pbo_solver* s) {
  return s->cfg.grad_tol * fmax(1.0, vdyn_infnorm(s->x, s->dim));
}
/* SolverBase::grad_converged, optim.cpp:47-52 */
static int grad_converged(const pbo_solver* s) {
  const double g = vdyn_infnorm(s->grad, s->dim);
  if (g <= scaled_tol(s)) return 1;
  if (s->cfg.grad_rtol > 0.0 && g <= s->cfg.grad_rtol * s->grad0_norm) return 1;
  return 0;
}
/* SolverBase::stagnation_update, optim.cpp:55-62 */
static int stagnation_update(pbo_solver* s, double old_value, double new_value) {
  if (old_value - new_value <= s->cfg.ftol * fmax(1.0, fabs(old_value))) ++s->stagnant;
  else s->stagnant = 0;
  return s->stagnant >= 2;
}
static void finish_iteration(pbo_solver* s) {
  if (s->iterations < s->cfg.max_iters) s->values[s->iterations] = s->value;
  ++s->iterations;
}

static void solver_free(pbo_solver* s) {
  free(s->x); free(s->grad); free(s->values); free(s->gn); free(s->hs); free(s->hy);
  free(s->hsy); free(s->dir); free(s->cand); free(s->tmp); free(s->alpha);
  free(s->damped); free(s->step); free(s->ev.grad); free(s->ev.gn);
}

/* make_solver + LmSolver/LbfgsSolver ctors, optim.cpp:82-93,143-150,236-242 */
static int solver_init(pbo_solver* s, const pbo_optimizer_config* cfg, const double* x0,
                       const pbo_objective* o, pbo_err* e) {
  memset(s, 0, sizeof *s);
  s->cfg = *cfg;
  const int dim = obj_dim(o);
  s->dim = dim;
  s->x = (double*)xcalloc(dim, sizeof(double));
  memcpy(s->x, x0, sizeof(double) * dim);
  s->grad = (double*)xcalloc(dim, sizeof(double));
  s->values = (double*)xcalloc(cfg->max_iters > 0 ? cfg->max_iters : 1, sizeof(double));
  s->dir = (double*)xcalloc(dim, sizeof(double));
  s->cand = (double*)xcalloc(dim, sizeof(double));
  s->tmp = (double*)xcalloc(dim, sizeof(double));
  s->step = (double*)xcalloc(dim, sizeof(double));
  s->ev.grad = (double*)xcalloc(dim, sizeof(double));
  const int lm = cfg->kind == PBO_LM;
  if (lm) {
    s->ev.gn = (double*)xcalloc((size_t)dim * dim, sizeof(double));
    s->gn = (double*)xcalloc((size_t)dim * dim, sizeof(double));
    s->damped = (double*)xcalloc((size_t)dim * dim, sizeof(double));
    s->lambda = cfg->lm_lambda0;
  } else {
    const int mem = cfg->lbfgs_memory > 0 ? cfg->lbfgs_memory : 1;
    s->hs = (double*)xcalloc((size_t)(mem + 1) * dim, sizeof(double));
    s->hy = (double*)xcalloc((size_t)(mem + 1) * dim, sizeof(double));
    s->hsy = (double*)xcalloc(mem + 1, sizeof(double));
    s->alpha = (double*)xcalloc(mem + 1, sizeof(double));
  }
  if (obj_evaluate(o, s->x, 1, lm, &s->ev, e)) return -1;
  if (!isfinite(s->ev.value)) {
    err_set(e, "objective is non-finite at the initial point");
    return -1;
  }
  s->value = s->ev.value;
  memcpy(s->grad, s->ev.grad, sizeof(double) * dim);
  if (lm) {
    if (!s->ev.has_gn) {
      err_set(e, "LM requires an objective with a Gauss-Newton matrix");
      return -1;
    }
    memcpy(s->gn, s->ev.gn, sizeof(double) * dim * dim);
  }
  s->grad0_norm = vdyn_infnorm(s->grad, dim);
  return 0;
}

/* LmSolver::iterate, optim.cpp:95-134 */
static int lm_iterate(pbo_solver* s, const pbo_objective* o, pbo_err* e) {
  if (s->status != ST_RUNNING) return s->status;
  if (s->iterations >= s->cfg.max_iters) return s->status = ST_FAILED;
  if (grad_converged(s)) return s->status = ST_CONVERGED;
  const int n = s->dim;
  memcpy(s->damped, s->gn, sizeof(double) * n * n);
  for (int k = 0; k < n; ++k) s->damped[k + (size_t)n * k] += s->lambda;
  for (int k = 0; k < n; ++k) s->tmp[k] = -s->grad[k];
  int accepted = 0;
  const int ok = llt_factor(s->damped, n) == 0;
  if (ok) llt_solve(s->damped, n, s->tmp, s->step);
  if (ok && vdyn_allfinite(s->step, n)) {
    for (int k = 0; k < n; ++k) s->cand[k] = s->x[k] + s->step[k];
    if (obj_evaluate(o, s->cand, 0, 0, &s->ev, e)) return -1;
    const double trial_value = s->ev.value;
    if (isfinite(trial_value) && trial_value < s->value) {
      const double old_value = s->value;
      memcpy(s->x, s->cand, sizeof(double) * n);
      if (obj_evaluate(o, s->x, 1, 1, &s->ev, e)) return -1;
      s->value = s->ev.value;
      memcpy(s->grad, s->ev.grad, sizeof(double) * n);
      memcpy(s->gn, s->ev.gn, sizeof(double) * n * n);
      s->lambda = fmax(s->lambda / s->cfg.lm_lambda_factor, 1e-12);
      accepted = 1;
      ++s->accepted;
      if (stagnation_update(s, old_value, s->value)) s->status = ST_CONVERGED;
    }
  }
  if (!accepted) {
    s->lambda *= s->cfg.lm_lambda_factor;
    if (s->lambda > s->cfg.lm_lambda_max) s->status = ST_FAILED;
  }
  finish_iteration(s);
  if (s->status == ST_RUNNING && s->iterations >= s->cfg.max_iters) s->status = ST_FAILED;
  return s->status;
}

/* ring helpers: deque index i (0 = oldest) */
static double* hist_s(pbo_solver* s, int i) {
  const int cap = s->cfg.lbfgs_memory + 1;
  return s->hs + (size_t)((s->hstart + i) % cap) * s->dim;
}
static double* hist_y(pbo_solver* s, int i) {
  const int cap = s->cfg.lbfgs_memory + 1;
  return s->hy + (size_t)((s->hstart + i) % cap) * s->dim;
}
static double* hist_sy(pbo_solver* s, int i) {
  const int cap = s->cfg.lbfgs_memory + 1;
  return &s->hsy[(s->hstart + i) % cap];
}

/* LbfgsSolver::two_loop, optim.cpp:213-229: q = H g, written to out */
static void two_loop(pbo_solver* s, const double* g, double* q) {
  const int n = s->dim;
  memcpy(q, g, sizeof(double) * n);
  const int H = s->hcount;
  for (int i = H - 1; i >= 0; --i) {
    const double* si = hist_s(s, i);
    const double* yi = hist_y(s, i);
    s->alpha[i] = vdyn_dot(si, q, n) / *hist_sy(s, i);
    for (int k = 0; k < n; ++k) q[k] = q[k] - s->alpha[i] * yi[k];
  }
  if (H > 0) {
    const double* yl = hist_y(s, H - 1);
    const double sc = *hist_sy(s, H - 1) / vdyn_sqnorm(yl, n);
    for (int k = 0; k < n; ++k) q[k] = q[k] * sc;
  }
  for (int i = 0; i < H; ++i) {
    const double* si = hist_s(s, i);
    const double* yi = hist_y(s, i);
    const double beta = vdyn_dot(yi, q, n) / *hist_sy(s, i);
    const double c = s->alpha[i] - beta;
    for (int k = 0; k < n; ++k) q[k] = q[k] + c * si[k];
  }
}

/* LbfgsSolver::iterate, optim.cpp:152-205 */
static int lbfgs_iterate(pbo_solver* s, const pbo_objective* o, pbo_err* e) {
  if (s->status != ST_RUNNING) return s->status;
  if (s->iterations >= s->cfg.max_iters) return s->status = ST_FAILED;
  if (grad_converged(s)) return s->status = ST_CONVERGED;
  const int n = s->dim;
  two_loop(s, s->grad, s->tmp);
  for (int k = 0; k < n; ++k) s->dir[k] = -s->tmp[k];
  double slope = vdyn_dot(s->dir, s->grad, n);
  if (!(slope < 0.0)) {
    s->hcount = 0;
    s->hstart = 0;
    for (int k = 0; k < n; ++k) s->dir[k] = -s->grad[k];
    slope = vdyn_dot(s->dir, s->grad, n);
  }
  double t = 1.0;
  int accepted = 0;
  for (int trial = 0; trial < s->cfg.max_line_search; ++trial) {
    for (int k = 0; k < n; ++k) s->cand[k] = s->x[k] + t * s->dir[k];
    if (vdyn_allfinite(s->cand, n)) {
      if (obj_evaluate(o, s->cand, 0, 0, &s->ev, e)) return -1;
      const double v = s->ev.value;
      if (isfinite(v) && v <= s->value + s->cfg.armijo_c1 * t * slope && v < s->value) {
        if (obj_evaluate(o, s->cand, 1, 0, &s->ev, e)) return -1;
        /* s = t*dir, y = g+ - g, pushed iff s.y > 1e-12 */
        const int cap = s->cfg.lbfgs_memory + 1;
        double* sn = s->hs + (size_t)((s->hstart + s->hcount) % cap) * n;
        double* yn = s->hy + (size_t)((s->hstart + s->hcount) % cap) * n;
        for (int k = 0; k < n; ++k) {
          sn[k] = t * s->dir[k];
          yn[k] = s->ev.grad[k] - s->grad[k];
        }
        const double sy = vdyn_dot(sn, yn, n);
        if (sy > 1e-12) {
          s->hsy[(s->hstart + s->hcount) % cap] = sy;
          ++s->hcount;
          if (s->hcount > s->cfg.lbfgs_memory) {
            s->hstart = (s->hstart + 1) % cap;
            --s->hcount;
          }
        }
        const double old_value = s->value;
        memcpy(s->x, s->cand, sizeof(double) * n);
        s->value = s->ev.value;
        memcpy(s->grad, s->ev.grad, sizeof(double) * n);
        accepted = 1;
        ++s->accepted;
        if (stagnation_update(s, old_value, s->value)) s->status = ST_CONVERGED;
        break;
      }
    }
    t *= s->cfg.backtrack_factor;
  }
  if (!accepted) s->status = ST_FAILED;
  finish_iteration(s);
  if (s->status == ST_RUNNING && s->iterations >= s->cfg.max_iters) s->status = ST_FAILED;
  return s->status;
}

static int solver_iterate(pbo_solver* s, const pbo_objective* o, pbo_err* e) {
  return s->cfg.kind == PBO_LM ? lm_iterate(s, o, e) : lbfgs_iterate(s, o, e);
}

int pbo_step_minimize(const pbo_model* m, const pbo_forces* f, int32_t order, double dt,
                      int32_t objective, const double* history,
                      const double* tau_instants, const double* x0,
                      const pbo_optimizer_config* cfg, double* x_out,
                      int32_t* iterations, int32_t* converged, double* final_value,
                      double* final_grad_norm, double* per_iter_values) {
  pbo_err e = {0};
  pbo_scheme sc;
  if (build_scheme(order, dt, &sc, &e)) return -1;
  pbo_objective o;
  int rc = obj_init(&o, m, f, &sc, dt, objective, history, history + m->n, tau_instants,
                    order - 1, &e);
  pbo_solver s;
  memset(&s, 0, sizeof s);
  if (!rc) rc = solver_init(&s, cfg, x0, &o, &e);
  while (!rc) {
    const int st = solver_iterate(&s, &o, &e);
    if (st < 0) rc = -1;
    else if (st != ST_RUNNING) break;
  }
  if (!rc) {
    memcpy(x_out, s.x, sizeof(double) * s.dim);
    if (iterations) *iterations = s.iterations;
    if (converged) *converged = s.status == ST_CONVERGED;
    if (final_value) *final_value = s.value;
    if (final_grad_norm) *final_grad_norm = vdyn_infnorm(s.grad, s.dim);
    if (per_iter_values)
      memcpy(per_iter_values, s.values,
             sizeof(double) * (s.iterations < cfg->max_iters ? s.iterations : cfg->max_iters));
  }
  solver_free(&s);
  obj_free(&o);
  return rc;
}

/* ------------------------------------------------------------------ */
/* energy audit (baseline.cpp:20-54,208-229; stepper.cpp:14-22)        */
/* ------------------------------------------------------------------ */
static void velocity_tdot(const pbo_model* m, const pbo_pass* p, const double* qdot,
                          pbo_m4* tdot) {
  for (int i = 0; i < m->N; ++i) {
    const int par = m->parent[i];
    const int off = m->dof_off[i];
    pbo_m4 ldot = m4_zero();
    for (int j = 0; j < m->dof_cnt[i]; ++j) {
      const pbo_m4 t = m4_scale(qdot[off + j], &p->d1[off + j]);
      m4_addto(&ldot, &t);
    }
    const pbo_m4 ptd = (par >= 0) ? tdot[par] : m4_zero();
    const pbo_m4 a = m4_mul(&ptd, &p->value[i]);
    const pbo_m4 b = m4_mul(&p->pworld[i], &ldot);
    tdot[i] = m4_add(&a, &b);
  }
}

static int kinetic_energy(const pbo_model* m, const double* q, const double* qdot,
                          double* ke, pbo_err* e) {
  pbo_pass p;
  pass_alloc(m, &p);
  if (pass_make(m, q, &p, e)) {
    pass_free(&p);
    return -1;
  }
  pbo_m4* tdot = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  velocity_tdot(m, &p, qdot, tdot);
  double k = 0.0;
  for (int i = 0; i < m->N; ++i) {
    const pbo_m4 ts = m4_mul(&tdot[i], &m->S[i]);
    k += 0.5 * m4_ddot(&ts, &tdot[i]);
  }
  *ke = k;
  free(tdot);
  pass_free(&p);
  return 0;
}

static double gravity_potential_w(const pbo_model* m, const double g[3], const pbo_m4* world) {
  const double ghat[4] = {g[0], g[1], g[2], 0.0};
  const double e4[4] = {0.0, 0.0, 0.0, 1.0};
  double pe = 0.0;
  for (int i = 0; i < m->N; ++i) {
    double u[4], w[4];
    m4_mul_vec(&m->S[i], e4, u);
    m4_mul_vec(&world[i], u, w);
    pe -= vfix_dot(ghat, w, 4);
  }
  return pe;
}

int pbo_kinetic_energy(const pbo_model* m, const double* q, const double* qdot, double* ke) {
  pbo_err e = {0};
  return kinetic_energy(m, q, qdot, ke, &e);
}

int pbo_gravity_potential(const pbo_model* m, const double g[3], const double* q,
                          double* pe) {
  pbo_err e = {0};
  pbo_m4* w = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  const int rc = forward_pass(m, q, w, &e);
  if (!rc) *pe = gravity_potential_w(m, g, w);
  free(w);
  return rc;
}

/* fd_kinetic, stepper.cpp:14-22 */
static double fd_kinetic(const pbo_model* m, const pbo_m4* wp, const pbo_m4* wn, double dt) {
  double ke = 0.0;
  for (int i = 0; i < m->N; ++i) {
    const pbo_m4 d = m4_sub(&wn[i], &wp[i]);
    const pbo_m4 tdot = m4_div(&d, dt);
    const pbo_m4 ts = m4_mul(&tdot, &m->S[i]);
    ke += 0.5 * m4_ddot(&ts, &tdot);
  }
  return ke;
}

/* ------------------------------------------------------------------ */
/* stepper (stepper.cpp:24-166)                                        */
/* ------------------------------------------------------------------ */
/* ForceModel::tau_at / ActuationSpec::tau_at, objective.hpp:28-58 */
static void forces_tau_at(const pbo_forces* f, double t, int dofs, double* out) {
  if (f->has_actuation && f->act_len == dofs) {
    if (f->act_kind == 0) {
      memcpy(out, f->act_amplitude, sizeof(double) * dofs);
      return;
    }
    for (int i = 0; i < dofs; ++i) {
      const double ph = i < f->act_phase_len ? f->act_phase[i] : 0.0;
      out[i] = f->act_amplitude[i] *
               pbm_sin(2.0 * 3.141592653589793 * f->act_frequency_hz * t + ph);
    }
    return;
  }
  if (f->tau_len == dofs) {
    memcpy(out, f->tau, sizeof(double) * dofs);
    return;
  }
  for (int i = 0; i < dofs; ++i) out[i] = 0.0;
}

typedef struct {
  pbo_scheme scheme;
  double* hist0;
  double* hist1;
  pbo_m4* world_hist1;
  pbo_m4* world_next;
  int step, total_steps, fail_streak;
  pbo_trajectory* traj;
  /* per-step */
  double* x0;
  double* tau;
  pbo_objective obj;
  pbo_solver solver;
  int live;
} pbo_run;

static void record_sample(pbo_run* r, int n, double t, const double* q, double ke,
                          double pe) {
  pbo_trajectory* T = r->traj;
  const int k = T->n_samples;
  if (k > T->capacity_steps) return;
  if (T->times) T->times[k] = t;
  if (T->q) memcpy(&T->q[(size_t)k * n], q, sizeof(double) * n);
  if (T->energy) {
    T->energy[2 * k] = ke;
    T->energy[2 * k + 1] = pe;
  }
  T->n_samples = k + 1;
}

/* init_pbad_run, stepper.cpp:62-80 */
static int init_run(pbo_run* r, const pbo_model* m, const pbo_forces* f,
                    const pbo_sim_config* sim, pbo_err* e) {
  const int n = m->n;
  if (validate_configuration(m, sim->q0, n, e)) return -1;
  if (!sim->qdot0) {
    err_set(e, "initial velocity length does not match model DOF count");
    return -1;
  }
  if (sim->dt <= 0.0 || sim->duration <= 0.0) {
    err_set(e, "dt and duration must be positive");
    return -1;
  }
  if (build_scheme(sim->order, sim->dt, &r->scheme, e)) return -1;
  if (sim->refined_bootstrap) {
    err_set(e, "refined_bootstrap (RK4 baseline) is outside the oracle's scope");
    return -1;
  }
  r->hist0 = (double*)xcalloc(n, sizeof(double));
  r->hist1 = (double*)xcalloc(n, sizeof(double));
  r->world_hist1 = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  r->world_next = (pbo_m4*)xcalloc(m->N, sizeof(pbo_m4));
  const double tl = r->scheme.times[0] * sim->dt;
  for (int k = 0; k < n; ++k) r->hist0[k] = sim->q0[k] + tl * sim->qdot0[k];
  memcpy(r->hist1, sim->q0, sizeof(double) * n);
  forward_pass(m, r->hist1, r->world_hist1, e);
  r->total_steps = (int)ceil(sim->duration / sim->dt - 1e-9);
  double ke;
  if (kinetic_energy(m, sim->q0, sim->qdot0, &ke, e)) return -1;
  record_sample(r, n, 0.0, sim->q0, ke, gravity_potential_w(m, f->gravity, r->world_hist1));
  return 0;
}

static void end_step_scratch(pbo_run* r) {
  if (r->live) {
    solver_free(&r->solver);
    obj_free(&r->obj);
    memset(&r->solver, 0, sizeof r->solver);
    memset(&r->obj, 0, sizeof r->obj);
    r->live = 0;
  }
}

/* begin_step, stepper.cpp:83-115 */
static int begin_step(pbo_run* r, const pbo_model* m, const pbo_forces* f,
                      const pbo_sim_config* sim, pbo_err* e) {
  const int n = m->n;
  const double t0 = r->step * sim->dt;
  const int u = r->scheme.order - 1;
  free(r->tau);
  free(r->x0);
  r->tau = (double*)xcalloc((size_t)n * u, sizeof(double));
  r->x0 = (double*)xcalloc((size_t)n * u, sizeof(double));
  for (int mm = 0; mm < u; ++mm) {
    const double t = t0 + r->scheme.times[2 + mm] * sim->dt;
    forces_tau_at(f, t, n, r->tau + (size_t)mm * n);
  }
  const double span = -r->scheme.times[0];
  for (int mm = 0; mm < u; ++mm) {
    const double tau_m = r->scheme.times[2 + mm];
    double* xm = r->x0 + (size_t)mm * n;
    for (int k = 0; k < n; ++k)
      xm[k] = sim->warm_start ? r->hist1[k] + (tau_m / span) * (r->hist1[k] - r->hist0[k])
                              : r->hist1[k];
  }
  memset(&r->solver, 0, sizeof r->solver);
  memset(&r->obj, 0, sizeof r->obj);
  r->live = 1;
  if (obj_init(&r->obj, m, f, &r->scheme, sim->dt, sim->objective, r->hist0, r->hist1,
               r->tau, u, e))
    return -1;
  if (solver_init(&r->solver, &sim->opt, r->x0, &r->obj, e)) return -1;
  return 0;
}

/* finish_step, stepper.cpp:118-147. Returns 0 ok, 1 fail-limit reached. */
static int finish_step(pbo_run* r, const pbo_model* m, const pbo_forces* f,
                       const pbo_sim_config* sim, pbo_err* e) {
  const int n = m->n;
  pbo_solver* s = &r->solver;
  pbo_trajectory* T = r->traj;
  const int converged = s->status == ST_CONVERGED;
  if (r->step < T->capacity_steps) {
    if (T->iterations) T->iterations[r->step] = s->iterations;
    if (T->converged) T->converged[r->step] = converged;
    if (T->accepted) T->accepted[r->step] = s->accepted;
    if (T->final_value) T->final_value[r->step] = s->value;
    if (T->final_grad_norm) T->final_grad_norm[r->step] = vdyn_infnorm(s->grad, s->dim);
  }
  r->fail_streak = converged ? 0 : r->fail_streak + 1;
  if (r->fail_streak > sim->consecutive_fail_limit) return 1;
  const int u = r->scheme.order - 1;
  double* nh0 = (double*)xcalloc(n, sizeof(double));
  double* nh1 = (double*)xcalloc(n, sizeof(double));
  memcpy(nh0, (sim->order == 2) ? r->hist1 : s->x + (size_t)(u - 2) * n, sizeof(double) * n);
  memcpy(nh1, s->x + (size_t)(u - 1) * n, sizeof(double) * n);
  forward_pass(m, nh1, r->world_next, e);
  ++r->step;
  const double t = r->step * sim->dt;
  record_sample(r, n, t, nh1, fd_kinetic(m, r->world_hist1, r->world_next, sim->dt),
                gravity_potential_w(m, f->gravity, r->world_next));
  memcpy(r->hist0, nh0, sizeof(double) * n);
  memcpy(r->hist1, nh1, sizeof(double) * n);
  memcpy(r->world_hist1, r->world_next, sizeof(pbo_m4) * m->N);
  free(nh0);
  free(nh1);
  end_step_scratch(r);
  return 0;
}

static void run_free(pbo_run* r) {
  end_step_scratch(r);
  free(r->hist0);
  free(r->hist1);
  free(r->world_hist1);
  free(r->world_next);
  free(r->x0);
  free(r->tau);
}

/* simulate, stepper.cpp:151-166 */
int pbo_simulate(const pbo_model* m, const pbo_forces* f, const pbo_sim_config* sim,
                 pbo_trajectory* out) {
  pbo_err e = {0};
  pbo_run r;
  memset(&r, 0, sizeof r);
  r.traj = out;
  out->n_samples = 0;
  out->has_error = 0;
  out->error[0] = 0;
  int rc = init_run(&r, m, f, sim, &e);
  while (!rc && r.step < r.total_steps) {
    if (begin_step(&r, m, f, sim, &e)) {
      rc = -1;
      break;
    }
    int st;
    while ((st = solver_iterate(&r.solver, &r.obj, &e)) == ST_RUNNING) {
    }
    if (st < 0) {
      rc = -1;
      break;
    }
    const int fr = finish_step(&r, m, f, sim, &e);
    if (fr == 1) {
      char buf[64];
      snprintf(buf, sizeof buf, "%f", r.step * sim->dt);
      err_set(&e, "optimizer failed %d consecutive steps around t=%s", r.fail_streak, buf);
      rc = -1;
    }
  }
  if (rc) {
    out->has_error = 1;
    snprintf(out->error, sizeof out->error, "%s", e.msg);
  }
  run_free(&r);
  return rc;
}

typedef struct {
  const pbo_model* m;
  const pbo_forces* f;
  const pbo_sim_config* sims;
  pbo_trajectory* outs;
  int count;
  int next;
  pthread_mutex_t mu;
} batch_ctx;

static void* batch_worker(void* arg) {
  batch_ctx* b = (batch_ctx*)arg;
  for (;;) {
    pthread_mutex_lock(&b->mu);
    const int t = b->next++;
    pthread_mutex_unlock(&b->mu);
    if (t >= b->count) break;
    pbo_simulate(b->m, b->f, &b->sims[t], &b->outs[t]);
  }
  return NULL;
}

/* batch_simulate, stepper.cpp:204-270: per-trajectory results equal
 * simulate(); an error is recorded per trajectory and never aborts. */
int pbo_batch_simulate(const pbo_model* m, const pbo_forces* f, const pbo_sim_config* sims,
                       int32_t count, int32_t workers, pbo_trajectory* outs) {
  if (workers < 1) return -1;
  batch_ctx b;
  b.m = m;
  b.f = f;
  b.sims = sims;
  b.outs = outs;
  b.count = count;
  b.next = 0;
  pthread_mutex_init(&b.mu, NULL);
  const int nt = workers < count ? workers : (count > 0 ? count : 1);
  pthread_t* th = (pthread_t*)xcalloc(nt, sizeof(pthread_t));
  for (int w = 1; w < nt; ++w) pthread_create(&th[w], NULL, batch_worker, &b);
  batch_worker(&b);
  for (int w = 1; w < nt; ++w) pthread_join(th[w], NULL);
  free(th);
  pthread_mutex_destroy(&b.mu);
  return 0;
}
