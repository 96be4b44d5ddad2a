// pbad_joint.cuh -- joint jets (kinematics.cpp:89-169) shared by the general
// (thread-per-env) and tree (warp-per-env) kernels.  Same operation sequence
// as the reference under the numeric contract (pbad_math.cuh).
#pragma once

#include "pbad_math.cuh"

namespace pbad_gpu {

// ---------------------------------------------------------------------------
// kinematics (kinematics.cpp:98-169)
// ---------------------------------------------------------------------------
static __device__ void joint_jet(int kind, const double* axis, const M4& off, const double* q, M4* value,
                          M4* d1, M4* d2, bool want_d2) {
  if (kind == 0) {
    const M3 Ka = skew(axis[0], axis[1], axis[2]);
    const M3 R = rotation_vector_matrix(axis[0] * q[0], axis[1] * q[0], axis[2] * q[0]);
    *value = mul(off, motion_rot(R));
    d1[0] = mul(off, embed_rotation(mul3(Ka, R)));
    if (want_d2) d2[0] = mul(off, embed_rotation(mul3(mul3(Ka, Ka), R)));
  } else if (kind == 1) {
    M3 R, dR[3], d2R[3][3];
    rotation_vector_jet(q, &R, dR, d2R, want_d2);
    *value = mul(off, motion_rot(R));
    for (int j = 0; j < 3; ++j) d1[j] = mul(off, embed_rotation(dR[j]));
    if (want_d2) {
      int idx = 0;
      for (int l = 0; l < 3; ++l)
        for (int j = 0; j <= l; ++j) d2[idx++] = mul(off, embed_rotation(d2R[j][l]));
    }
  } else {
    M3 R, dR[3], d2R[3][3];
    rotation_vector_jet(q + 3, &R, dR, d2R, want_d2);
    M4 motion = motion_rot(R);
    motion.a[12] = q[0];
    motion.a[13] = q[1];
    motion.a[14] = q[2];
    *value = mul(off, motion);
    for (int j = 0; j < 3; ++j) {
      M4 dt = m4_zero();
      dt.a[j + 12] = 1.0;
      d1[j] = mul(off, dt);
      d1[3 + j] = mul(off, embed_rotation(dR[j]));
    }
    if (want_d2) {
      int idx = 0;
      for (int l = 0; l < 6; ++l)
        for (int j = 0; j <= l; ++j, ++idx)
          d2[idx] = (j >= 3 && l >= 3) ? mul(off, embed_rotation(d2R[j - 3][l - 3])) : m4_zero();
    }
  }
}

// joint_transform (kinematics.cpp:98-117)
static __device__ M4 joint_transform(int kind, const double* axis, const M4& off, const double* q) {
  M4 motion;
  if (kind == 0) {
    motion = motion_rot(rotation_vector_matrix(axis[0] * q[0], axis[1] * q[0], axis[2] * q[0]));
  } else if (kind == 1) {
    motion = motion_rot(rotation_vector_matrix(q[0], q[1], q[2]));
  } else {
    motion = motion_rot(rotation_vector_matrix(q[3], q[4], q[5]));
    motion.a[12] = q[0];
    motion.a[13] = q[1];
    motion.a[14] = q[2];
  }
  return mul(off, motion);
}

}  // namespace pbad_gpu
