// hs_numpy_order.cuh -- FP64 helpers that round exactly like the reference's
// numpy expressions (shared by K1/K7 and the densification kernels).  Include
// only from translation units compiled with -fmad=false where bit-exactness is
// wanted.
#pragma once
#include <cmath>

namespace hs {

// sigmoid, geometry.py:349-352: x >= 0 ? 1 / (1 + exp(-x)) : exp(x) / (1 + exp(x)).
// Both branches need exp(-|x|) once: computed branch-free with one exp and one
// division, bit for bit the reference's value (same operations, same rounding).
__device__ __forceinline__ double sigmoid_ref(double x) {
  const double e = exp(-fabs(x));
  return (x >= 0.0 ? 1.0 : e) / (1.0 + e);
}

// quat_to_rot, geometry.py:27-49 (normalises its input again, as the reference
// calls it on the already-normalised quaternion, rasterizer.py:174-176).
__device__ __forceinline__ void quat_to_rot_ref(const double q_in[4], double R[9]) {
  double ss = 0.0;
  for (int k = 0; k < 4; ++k) ss += q_in[k] * q_in[k];
  const double n = sqrt(ss);
  const double w = q_in[0] / n, x = q_in[1] / n, y = q_in[2] / n, z = q_in[3] / n;
  R[0] = 1 - 2 * (y * y + z * z);
  R[1] = 2 * (x * y - w * z);
  R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);
  R[4] = 1 - 2 * (x * x + z * z);
  R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);
  R[7] = 2 * (y * z + w * x);
  R[8] = 1 - 2 * (x * x + y * y);
}

// einsum("nab,nb->na"): numpy pairs the 3-term reduction as (x0 + x2) + x1.
__device__ __forceinline__ void matvec_einsum(const double M[9], const double v[3], double out[3]) {
  for (int a = 0; a < 3; ++a) {
    const double x0 = M[3 * a] * v[0], x1 = M[3 * a + 1] * v[1], x2 = M[3 * a + 2] * v[2];
    out[a] = (x0 + x2) + x1;
  }
}

// (N,3) @ (3,3)^T through OpenBLAS: fma(v2, M[a,2], fma(v1, M[a,1], v0 * M[a,0])).
__device__ __forceinline__ void matvec_blas(const double M[9], const double v[3], double out[3]) {
  for (int a = 0; a < 3; ++a)
    out[a] = fma(v[2], M[3 * a + 2], fma(v[1], M[3 * a + 1], v[0] * M[3 * a]));
}

}  // namespace hs
