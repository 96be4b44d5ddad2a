/*
 * pbo_math.h -- TEST INFRASTRUCTURE ONLY (the CPU oracle).
 *
 * Canonical FP64 arithmetic shared by the oracle restatement (pbad_oracle.c)
 * and the eigen_lite shim that the reference sources are compiled against
 * (oracle/eigen_lite).  Eigen does not specify the order in which products
 * and reductions round; this file fixes one, so that the reference build,
 * the oracle and the CUDA kernels are bit-comparable:
 *
 *   product    C(i,j) = a(i,0)*b(0,j), then acc = fma(a(i,k), b(k,j), acc)
 *              for k = 1..K-1 (inner index ascending)
 *   ddot       A.cwiseProduct(B).sum() (math_types.hpp:33-35): per-row
 *              fma chains over the columns, combined ((r0+r1)+r2)+r3
 *   trace      ((m00 + m11) + m22) + m33
 *   fixed dot  Vec3/Vec4 dot/squaredNorm: fma chain, index ascending
 *   VecX dot   32 interleaved fma partial sums (i mod 32), then a
 *              pairwise tree (p += p+16, p += p+8, ... )
 *   sin/cos    pbo_sincos below (portable: rint + fma + IEEE ops only),
 *              because glibc and CUDA libdevice disagree in the last ulp
 *   all other  element-wise IEEE operations, in C++ evaluation order
 *
 * Compile with -ffp-contract=off (no implicit contraction).
 */
#ifndef PBO_MATH_H
#define PBO_MATH_H

#include <math.h>
#include <string.h>

typedef struct { double a[16]; } pbo_m4; /* column-major: a[r + 4*c] */
typedef struct { double a[9]; } pbo_m3;  /* column-major: a[r + 3*c] */

#define M4E(M, r, c) ((M).a[(r) + 4 * (c)])
#define M3E(M, r, c) ((M).a[(r) + 3 * (c)])

static inline pbo_m4 m4_zero(void) { pbo_m4 m; memset(&m, 0, sizeof m); return m; }
static inline pbo_m4 m4_identity(void) {
  pbo_m4 m = m4_zero();
  m.a[0] = m.a[5] = m.a[10] = m.a[15] = 1.0;
  return m;
}
static inline pbo_m3 m3_zero(void) { pbo_m3 m; memset(&m, 0, sizeof m); return m; }
static inline pbo_m3 m3_identity(void) {
  pbo_m3 m = m3_zero();
  m.a[0] = m.a[4] = m.a[8] = 1.0;
  return m;
}

/* C = A * B */
static inline pbo_m4 m4_mul(const pbo_m4* A, const pbo_m4* B) {
  pbo_m4 C;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) {
      double acc = M4E(*A, i, 0) * M4E(*B, 0, j);
      acc = fma(M4E(*A, i, 1), M4E(*B, 1, j), acc);
      acc = fma(M4E(*A, i, 2), M4E(*B, 2, j), acc);
      acc = fma(M4E(*A, i, 3), M4E(*B, 3, j), acc);
      M4E(C, i, j) = acc;
    }
  return C;
}
/* C = A * B^T */
static inline pbo_m4 m4_mul_bt(const pbo_m4* A, const pbo_m4* B) {
  pbo_m4 C;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) {
      double acc = M4E(*A, i, 0) * M4E(*B, j, 0);
      acc = fma(M4E(*A, i, 1), M4E(*B, j, 1), acc);
      acc = fma(M4E(*A, i, 2), M4E(*B, j, 2), acc);
      acc = fma(M4E(*A, i, 3), M4E(*B, j, 3), acc);
      M4E(C, i, j) = acc;
    }
  return C;
}
/* C = A^T * B */
static inline pbo_m4 m4_mul_at(const pbo_m4* A, const pbo_m4* B) {
  pbo_m4 C;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) {
      double acc = M4E(*A, 0, i) * M4E(*B, 0, j);
      acc = fma(M4E(*A, 1, i), M4E(*B, 1, j), acc);
      acc = fma(M4E(*A, 2, i), M4E(*B, 2, j), acc);
      acc = fma(M4E(*A, 3, i), M4E(*B, 3, j), acc);
      M4E(C, i, j) = acc;
    }
  return C;
}
static inline pbo_m4 m4_transpose(const pbo_m4* A) {
  pbo_m4 C;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) M4E(C, i, j) = M4E(*A, j, i);
  return C;
}
static inline pbo_m4 m4_add(const pbo_m4* A, const pbo_m4* B) {
  pbo_m4 C;
  for (int e = 0; e < 16; ++e) C.a[e] = A->a[e] + B->a[e];
  return C;
}
static inline pbo_m4 m4_sub(const pbo_m4* A, const pbo_m4* B) {
  pbo_m4 C;
  for (int e = 0; e < 16; ++e) C.a[e] = A->a[e] - B->a[e];
  return C;
}
static inline pbo_m4 m4_scale(double s, const pbo_m4* A) {
  pbo_m4 C;
  for (int e = 0; e < 16; ++e) C.a[e] = s * A->a[e];
  return C;
}
static inline pbo_m4 m4_div(const pbo_m4* A, double s) {
  pbo_m4 C;
  for (int e = 0; e < 16; ++e) C.a[e] = A->a[e] / s;
  return C;
}
static inline void m4_addto(pbo_m4* A, const pbo_m4* B) {
  for (int e = 0; e < 16; ++e) A->a[e] = A->a[e] + B->a[e];
}
/* ddot(A, B) = A.cwiseProduct(B).sum(), math_types.hpp:33-35 */
static inline double m4_ddot(const pbo_m4* A, const pbo_m4* B) {
  double rs[4];
  for (int r = 0; r < 4; ++r) {
    double acc = M4E(*A, r, 0) * M4E(*B, r, 0);
    acc = fma(M4E(*A, r, 1), M4E(*B, r, 1), acc);
    acc = fma(M4E(*A, r, 2), M4E(*B, r, 2), acc);
    acc = fma(M4E(*A, r, 3), M4E(*B, r, 3), acc);
    rs[r] = acc;
  }
  return ((rs[0] + rs[1]) + rs[2]) + rs[3];
}
static inline double m4_trace(const pbo_m4* A) {
  return ((A->a[0] + A->a[5]) + A->a[10]) + A->a[15];
}

static inline pbo_m3 m3_mul(const pbo_m3* A, const pbo_m3* B) {
  pbo_m3 C;
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {
      double acc = M3E(*A, i, 0) * M3E(*B, 0, j);
      acc = fma(M3E(*A, i, 1), M3E(*B, 1, j), acc);
      acc = fma(M3E(*A, i, 2), M3E(*B, 2, j), acc);
      M3E(C, i, j) = acc;
    }
  return C;
}
static inline pbo_m3 m3_add(const pbo_m3* A, const pbo_m3* B) {
  pbo_m3 C;
  for (int e = 0; e < 9; ++e) C.a[e] = A->a[e] + B->a[e];
  return C;
}
static inline pbo_m3 m3_scale(double s, const pbo_m3* A) {
  pbo_m3 C;
  for (int e = 0; e < 9; ++e) C.a[e] = s * A->a[e];
  return C;
}
/* skew(v), math_types.hpp:16-22 */
static inline pbo_m3 m3_skew(const double v[3]) {
  pbo_m3 m;
  M3E(m, 0, 0) = 0.0;   M3E(m, 0, 1) = -v[2]; M3E(m, 0, 2) = v[1];
  M3E(m, 1, 0) = v[2];  M3E(m, 1, 1) = 0.0;   M3E(m, 1, 2) = -v[0];
  M3E(m, 2, 0) = -v[1]; M3E(m, 2, 1) = v[0];  M3E(m, 2, 2) = 0.0;
  return m;
}
/* embed_rotation(r), math_types.hpp:26-30 */
static inline pbo_m4 m4_embed_rotation(const pbo_m3* r) {
  pbo_m4 m = m4_zero();
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) M4E(m, i, c) = M3E(*r, i, c);
  return m;
}

/* fixed-size dot (Vec3 / Vec4): fma chain */
static inline double vfix_dot(const double* a, const double* b, int n) {
  double acc = a[0] * b[0];
  for (int i = 1; i < n; ++i) acc = fma(a[i], b[i], acc);
  return acc;
}

/* VecX dot: 32 interleaved partials + pairwise tree */
static inline double vdyn_dot(const double* a, const double* b, int n) {
  double p[32];
  for (int k = 0; k < 32; ++k) p[k] = 0.0;
  for (int i = 0; i < n; ++i) p[i & 31] = fma(a[i], b[i], p[i & 31]);
  for (int s = 16; s >= 1; s >>= 1)
    for (int k = 0; k < s; ++k) p[k] = p[k] + p[k + s];
  return p[0];
}
static inline double vdyn_sqnorm(const double* a, int n) { return vdyn_dot(a, a, n); }
/* lpNorm<Infinity>: max |a_i| (fmax ignores NaN, like the CUDA kernels) */
static inline double vdyn_infnorm(const double* a, int n) {
  double m = 0.0;
  for (int i = 0; i < n; ++i) m = fmax(m, fabs(a[i]));
  return m;
}
static inline int vdyn_allfinite(const double* a, int n) {
  for (int i = 0; i < n; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

/*
 * Portable sin/cos: x = k*pi/2 + r (fma Cody-Waite, two-term pi/2),
 * fdlibm minimax kernels on |r| <= pi/4 evaluated with fma Horner.
 * Only rint/fma/+,-,*,/ and fmod are used, all IEEE-exact on x86-64 and
 * sm_100a, so the CUDA kernels reproduce it bit for bit.
 */
static inline void pbm_sincos(double x, double* s_out, double* c_out) {
  if (!isfinite(x)) {
    *s_out = x - x;
    *c_out = x - x;
    return;
  }
  if (fabs(x) > 1.0e9) x = fmod(x, 6.283185307179586);
  const double k = rint(x * 0.6366197723675814);
  double r = fma(-k, 1.5707963267948966, x);
  r = fma(-k, 6.123233995736766e-17, r);
  const double z = r * r;
  double ps = fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08);
  ps = fma(z, ps, 2.75573137070700676789e-06);
  ps = fma(z, ps, -1.98412698298579493134e-04);
  ps = fma(z, ps, 8.33333333332248946124e-03);
  ps = fma(z, ps, -1.66666666666666324348e-01);
  const double sr = fma(r * z, ps, r);
  double pc = fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09);
  pc = fma(z, pc, -2.75573143513906633035e-07);
  pc = fma(z, pc, 2.48015872894767294178e-05);
  pc = fma(z, pc, -1.38888888888741095749e-03);
  pc = fma(z, pc, 4.16666666666666019037e-02);
  const double cr = fma(z * z, pc, 1.0 - 0.5 * z);
  const double kq = k - 4.0 * floor(k * 0.25);
  const int q = (int)kq;
  switch (q) {
    case 0: *s_out = sr; *c_out = cr; break;
    case 1: *s_out = cr; *c_out = -sr; break;
    case 2: *s_out = -sr; *c_out = -cr; break;
    default: *s_out = -cr; *c_out = sr; break;
  }
}
static inline double pbm_sin(double x) { double s, c; pbm_sincos(x, &s, &c); return s; }
static inline double pbm_cos(double x) { double s, c; pbm_sincos(x, &s, &c); return c; }

#endif
