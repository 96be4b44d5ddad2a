// pbad_math.cuh -- FP64 device math for the PBAD kernels (sm_100a).
//
// The kernels reproduce the reference's arithmetic bit for bit.  The
// reference is written against Eigen, which leaves product / reduction
// rounding order unspecified; this project fixes it (DESIGN.md "numeric
// contract") and compiles everything with --fmad=false so the only fused
// multiply-adds are the explicit fma() calls below:
//   product  C(i,j) = a(i,0)*b(0,j); acc = fma(a(i,k), b(k,j), acc), k ascending
//   ddot     per-row fma chains over the columns, ((r0+r1)+r2)+r3
//            (math_types.hpp:33-35)
//   trace    ((m00 + m11) + m22) + m33
//   Vec3/4   dot = fma chain;  VecX dot = 32 interleaved partials + tree
//   sin/cos  pbad_sincos (rint + fma Cody-Waite + fdlibm kernels)
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define PBAD_HD __host__ __device__ __forceinline__
#else
#define PBAD_HD inline
#endif

namespace pbad_gpu {

struct M4 {
  double a[16];  // column-major a[r + 4c]
};
struct M3 {
  double a[9];
};

PBAD_HD M4 m4_zero() {
  M4 m;
#pragma unroll
  for (int e = 0; e < 16; ++e) m.a[e] = 0.0;
  return m;
}
PBAD_HD M4 m4_identity() {
  M4 m = m4_zero();
  m.a[0] = m.a[5] = m.a[10] = m.a[15] = 1.0;
  return m;
}
PBAD_HD M3 m3_zero() {
  M3 m;
#pragma unroll
  for (int e = 0; e < 9; ++e) m.a[e] = 0.0;
  return m;
}
PBAD_HD M3 m3_identity() {
  M3 m = m3_zero();
  m.a[0] = m.a[4] = m.a[8] = 1.0;
  return m;
}

PBAD_HD M4 mul(const M4& A, const M4& B) {
  M4 C;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double acc = A.a[i] * B.a[4 * j];
      acc = fma(A.a[i + 4], B.a[1 + 4 * j], acc);
      acc = fma(A.a[i + 8], B.a[2 + 4 * j], acc);
      acc = fma(A.a[i + 12], B.a[3 + 4 * j], acc);
      C.a[i + 4 * j] = acc;
    }
  return C;
}
// A * B^T
PBAD_HD M4 mul_bt(const M4& A, const M4& B) {
  M4 C;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double acc = A.a[i] * B.a[j];
      acc = fma(A.a[i + 4], B.a[j + 4], acc);
      acc = fma(A.a[i + 8], B.a[j + 8], acc);
      acc = fma(A.a[i + 12], B.a[j + 12], acc);
      C.a[i + 4 * j] = acc;
    }
  return C;
}
// A^T * B
PBAD_HD M4 mul_at(const M4& A, const M4& B) {
  M4 C;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double acc = A.a[4 * i] * B.a[4 * j];
      acc = fma(A.a[1 + 4 * i], B.a[1 + 4 * j], acc);
      acc = fma(A.a[2 + 4 * i], B.a[2 + 4 * j], acc);
      acc = fma(A.a[3 + 4 * i], B.a[3 + 4 * j], acc);
      C.a[i + 4 * j] = acc;
    }
  return C;
}
PBAD_HD M4 transpose(const M4& A) {
  M4 C;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) C.a[i + 4 * j] = A.a[j + 4 * i];
  return C;
}
PBAD_HD M4 add(const M4& A, const M4& B) {
  M4 C;
#pragma unroll
  for (int e = 0; e < 16; ++e) C.a[e] = A.a[e] + B.a[e];
  return C;
}
PBAD_HD M4 sub(const M4& A, const M4& B) {
  M4 C;
#pragma unroll
  for (int e = 0; e < 16; ++e) C.a[e] = A.a[e] - B.a[e];
  return C;
}
PBAD_HD M4 scale(double s, const M4& A) {
  M4 C;
#pragma unroll
  for (int e = 0; e < 16; ++e) C.a[e] = s * A.a[e];
  return C;
}
PBAD_HD M4 divs(const M4& A, double s) {
  M4 C;
#pragma unroll
  for (int e = 0; e < 16; ++e) C.a[e] = A.a[e] / s;
  return C;
}
PBAD_HD void addto(M4& A, const M4& B) {
#pragma unroll
  for (int e = 0; e < 16; ++e) A.a[e] = A.a[e] + B.a[e];
}
// one row of ddot: fma chain over the 4 columns
PBAD_HD double ddot_row(const double* a, const double* b) {
  double acc = a[0] * b[0];
  acc = fma(a[1], b[1], acc);
  acc = fma(a[2], b[2], acc);
  return fma(a[3], b[3], acc);
}
PBAD_HD double ddot(const M4& A, const M4& B) {
  double rs[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    double acc = A.a[r] * B.a[r];
    acc = fma(A.a[r + 4], B.a[r + 4], acc);
    acc = fma(A.a[r + 8], B.a[r + 8], acc);
    acc = fma(A.a[r + 12], B.a[r + 12], acc);
    rs[r] = acc;
  }
  return ((rs[0] + rs[1]) + rs[2]) + rs[3];
}
PBAD_HD double trace(const M4& A) { return ((A.a[0] + A.a[5]) + A.a[10]) + A.a[15]; }

PBAD_HD M3 mul3(const M3& A, const M3& B) {
  M3 C;
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double acc = A.a[i] * B.a[3 * j];
      acc = fma(A.a[i + 3], B.a[1 + 3 * j], acc);
      acc = fma(A.a[i + 6], B.a[2 + 3 * j], acc);
      C.a[i + 3 * j] = acc;
    }
  return C;
}
PBAD_HD M3 add3(const M3& A, const M3& B) {
  M3 C;
#pragma unroll
  for (int e = 0; e < 9; ++e) C.a[e] = A.a[e] + B.a[e];
  return C;
}
PBAD_HD M3 scale3(double s, const M3& A) {
  M3 C;
#pragma unroll
  for (int e = 0; e < 9; ++e) C.a[e] = s * A.a[e];
  return C;
}
PBAD_HD M3 skew(double x, double y, double z) {
  M3 m;
  m.a[0] = 0.0; m.a[3] = -z;  m.a[6] = y;
  m.a[1] = z;   m.a[4] = 0.0; m.a[7] = -x;
  m.a[2] = -y;  m.a[5] = x;   m.a[8] = 0.0;
  return m;
}
PBAD_HD M4 embed_rotation(const M3& r) {
  M4 m = m4_zero();
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < 3; ++i) m.a[i + 4 * c] = r.a[i + 3 * c];
  return m;
}
PBAD_HD M4 motion_rot(const M3& R) {
  M4 m = m4_identity();
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < 3; ++i) m.a[i + 4 * c] = R.a[i + 3 * c];
  return m;
}
PBAD_HD void mul_vec4(const M4& A, const double* x, double* y) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double acc = A.a[i] * x[0];
    acc = fma(A.a[i + 4], x[1], acc);
    acc = fma(A.a[i + 8], x[2], acc);
    acc = fma(A.a[i + 12], x[3], acc);
    y[i] = acc;
  }
}
PBAD_HD double dot3(const double* a, const double* b) {
  double acc = a[0] * b[0];
  acc = fma(a[1], b[1], acc);
  return fma(a[2], b[2], acc);
}
PBAD_HD double dot4(const double* a, const double* b) {
  double acc = a[0] * b[0];
  acc = fma(a[1], b[1], acc);
  acc = fma(a[2], b[2], acc);
  return fma(a[3], b[3], acc);
}

// Portable sin/cos: identical on host and device.
PBAD_HD void pbad_sincos(double x, double* s_out, double* c_out) {
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
  if (q == 0) {
    *s_out = sr;
    *c_out = cr;
  } else if (q == 1) {
    *s_out = cr;
    *c_out = -sr;
  } else if (q == 2) {
    *s_out = -sr;
    *c_out = -cr;
  } else {
    *s_out = -cr;
    *c_out = sr;
  }
}

struct RotCoeffs {
  double A, B, f1, f2, g1, g2;
};

// rotation_coeffs, kinematics.cpp:20-45
PBAD_HD RotCoeffs rotation_coeffs(double n) {
  RotCoeffs c;
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
    pbad_sincos(n, &s, &co);
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

// rotation_vector_matrix, kinematics.cpp:91-96
PBAD_HD M3 rotation_vector_matrix(double tx, double ty, double tz) {
  const double th[3] = {tx, ty, tz};
  const double n = sqrt(dot3(th, th));
  const RotCoeffs c = rotation_coeffs(n);
  const M3 K = skew(tx, ty, tz);
  const M3 K2 = mul3(K, K);
  const M3 aK = scale3(c.A, K);
  const M3 bK2 = scale3(c.B, K2);
  const M3 t = add3(m3_identity(), aK);
  return add3(t, bK2);
}

// rotation_vector_jet, kinematics.cpp:49-87
PBAD_HD void rotation_vector_jet(const double* theta, M3* R, M3* dR, M3 (*d2R)[3],
                                 bool want_d2) {
  const double n = sqrt(dot3(theta, theta));
  const RotCoeffs c = rotation_coeffs(n);
  const M3 K = skew(theta[0], theta[1], theta[2]);
  const M3 K2 = mul3(K, K);
  M3 Kb[3];
  Kb[0] = skew(1.0, 0.0, 0.0);
  Kb[1] = skew(0.0, 1.0, 0.0);
  Kb[2] = skew(0.0, 0.0, 1.0);
  {
    const M3 aK = scale3(c.A, K);
    const M3 bK2 = scale3(c.B, K2);
    const M3 t = add3(m3_identity(), aK);
    *R = add3(t, bK2);
  }
  M3 KbK[3];
  for (int j = 0; j < 3; ++j) {
    KbK[j] = add3(mul3(Kb[j], K), mul3(K, Kb[j]));
    M3 s = add3(scale3(c.f1 * theta[j], K), scale3(c.A, Kb[j]));
    s = add3(s, scale3(c.f2 * theta[j], K2));
    dR[j] = add3(s, scale3(c.B, KbK[j]));
  }
  if (!want_d2) return;
  for (int j = 0; j < 3; ++j)
    for (int l = j; l < 3; ++l) {
      const double tjl = theta[j] * theta[l];
      const double djl = (j == l) ? 1.0 : 0.0;
      const M3 a1 = scale3(c.f1 * djl + c.g1 * tjl, K);
      const M3 a2 = scale3(c.f1, add3(scale3(theta[j], Kb[l]), scale3(theta[l], Kb[j])));
      const M3 a3 = scale3(c.f2 * djl + c.g2 * tjl, K2);
      const M3 a4 = scale3(c.f2, add3(scale3(theta[j], KbK[l]), scale3(theta[l], KbK[j])));
      const M3 a5 = scale3(c.B, add3(mul3(Kb[j], Kb[l]), mul3(Kb[l], Kb[j])));
      M3 mm = add3(a1, a2);
      mm = add3(mm, a3);
      mm = add3(mm, a4);
      mm = add3(mm, a5);
      d2R[j][l] = mm;
      d2R[l][j] = mm;
    }
}

// VecX dot with 32 interleaved partials + pairwise tree (numeric contract)
template <class ArrA, class ArrB>
PBAD_HD double vdot32(const ArrA& a, const ArrB& b, int n) {
  double p[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) p[k] = 0.0;
  for (int i = 0; i < n; ++i) p[i & 31] = fma(a[i], b[i], p[i & 31]);
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1)
#pragma unroll
    for (int k = 0; k < s; ++k) p[k] = p[k] + p[k + s];
  return p[0];
}

}  // namespace pbad_gpu
