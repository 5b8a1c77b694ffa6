// hs_adam.cu -- the optimizer step after K7: per-group Adam on every scene
// parameter in one launch (trainer.py:139-226).
//
// Groups (trainer.py:81-82): mu, log_scale, rotation, sh_dc, sh_rest, normal,
// opacity_a, opacity_b, each with its own learning rate and step count.  The
// launch walks six segments of work units:
//   mu, log_scale, rotation   one element per unit
//   sh_coeffs                 one element per unit; coefficient 0 is sh_dc,
//                             the rest sh_rest (different lr / bias correction)
//   normal                    one row (3 elements) per unit: Adam on the row,
//                             then renormalise it if any of its updates is
//                             non-zero (trainer.py:214-221)
//   opacity a + b             one primitive per unit, both halves, then the
//                             'full'-kernel tie raw_opacity_b = raw_opacity_a
//                             (trainer.py:222-224)
// A frozen group (inactive mode or lr 0, trainer.py:195-200) is skipped
// entirely: parameters and moments untouched.  The update follows the
// reference's numpy statement order (m *= b1; m += (1-b1) g; v *= b2;
// v += (1-b2) g g; m/(1-b1^t); v/(1-b2^t); lr m_hat / (sqrt(v_hat) + eps)) in
// the storage precision, and this file is compiled with -fmad=false, so a
// float64 scene steps bit-identically to the reference.  HBM-bound: 28 B per
// float32 element (param, m, v, grad in; param, m, v out).
#include <cmath>
#include <cstdint>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

constexpr double kAdamBeta1 = 0.9;    // trainer.py:23
constexpr double kAdamBeta2 = 0.999;  // trainer.py:24
constexpr double kAdamEps = 1e-15;    // trainer.py:25

// Per-group constants in the arithmetic type.  float64 keeps the reference's
// divisions (bit-identical steps); float32 multiplies by the bias-correction
// reciprocals and uses the fast divide (within float32 rounding either way).
template <typename T>
struct GroupK {
  T lr, bc1, bc2;  // T = float: bc1 / bc2 hold 1/(1-b1^t), 1/(1-b2^t)
  bool on;
};

template <typename T>
__device__ __forceinline__ GroupK<T> group_k(const AdamSeg& sg, int j) {
  if constexpr (sizeof(T) == 8)
    return {sg.lr[j], sg.bc1[j], sg.bc2[j], sg.active[j] != 0};
  else
    return {(float)sg.lr[j], (float)(1.0 / sg.bc1[j]), (float)(1.0 / sg.bc2[j]),
            sg.active[j] != 0};
}

// One element; returns the update (trainer.py:202-213).
template <typename T>
__device__ __forceinline__ T adam_elem(T& p, T& m, T& v, T g, const GroupK<T>& k) {
  const T b1 = (T)kAdamBeta1, b2 = (T)kAdamBeta2;
  const T omb1 = (T)(1.0 - kAdamBeta1), omb2 = (T)(1.0 - kAdamBeta2), eps = (T)kAdamEps;
  T mm = m * b1;
  mm = mm + omb1 * g;
  T vv = v * b2;
  vv = vv + omb2 * g * g;
  m = mm;
  v = vv;
  T upd;
  if constexpr (sizeof(T) == 8) {
    const T m_hat = mm / k.bc1;
    const T v_hat = vv / k.bc2;
    upd = k.lr * m_hat / (sqrt(v_hat) + eps);
  } else {
    const T m_hat = mm * k.bc1;
    const T v_hat = vv * k.bc2;
    upd = __fdividef(k.lr * m_hat, sqrtf(v_hat) + eps);
  }
  p = p - upd;
  return upd;
}

template <typename T> struct AdamVec;
template <> struct AdamVec<float> { using type = float4; };
template <> struct AdamVec<double> { using type = double2; };

// Elementwise segments (plain, sh) in 16-B vector units of kV elements.
template <typename T, bool SH>
__device__ void adam_vector_seg(const AdamSeg& sg, int64_t first, int64_t stride) {
  using V = typename AdamVec<T>::type;
  constexpr int kV = 16 / sizeof(T);
  const GroupK<T> k0 = group_k<T>(sg, 0);
  const GroupK<T> k1 = SH ? group_k<T>(sg, 1) : k0;
  const uint32_t row = 3u * (uint32_t)sg.K;  // sh: elements per primitive
  V* P = static_cast<V*>(sg.param[0]);
  V* M = static_cast<V*>(sg.m[0]);
  V* Vv = static_cast<V*>(sg.v[0]);
  const V* G = static_cast<const V*>(sg.grad[0]);
  for (int64_t u = first; u < sg.units; u += stride) {
    V p = P[u], m = M[u], v = Vv[u];
    const V g = G[u];
    T* pe = reinterpret_cast<T*>(&p);
    T* me = reinterpret_cast<T*>(&m);
    T* ve = reinterpret_cast<T*>(&v);
    const T* ge = reinterpret_cast<const T*>(&g);
    uint32_t pos = SH ? (uint32_t)((u * kV) % row) : 0u;
#pragma unroll
    for (int e = 0; e < kV; ++e) {
      // sh: coefficient 0 (a primitive's first 3 elements) is sh_dc, the rest sh_rest
      const bool dc = !SH || pos < 3u;
      const GroupK<T>& k = dc ? k0 : k1;
      if (k.on) adam_elem<T>(pe[e], me[e], ve[e], ge[e], k);
      if (SH && ++pos == row) pos = 0u;
    }
    P[u] = p;
    M[u] = m;
    Vv[u] = v;
  }
}

template <typename T>
__device__ void adam_scalar_seg(const AdamSeg& sg, int64_t first, int64_t stride, int tie) {
  T* p0 = static_cast<T*>(sg.param[0]);
  T* m0 = static_cast<T*>(sg.m[0]);
  T* v0 = static_cast<T*>(sg.v[0]);
  const T* g0 = static_cast<const T*>(sg.grad[0]);
  const GroupK<T> k0 = group_k<T>(sg, 0), k1 = group_k<T>(sg, 1);
  const uint32_t row = 3u * (uint32_t)sg.K;
  for (int64_t i = first; i < sg.units; i += stride) {
    switch (sg.kind) {
      case kAdamPlain:
        adam_elem<T>(p0[i], m0[i], v0[i], g0[i], k0);
        break;
      case kAdamSh: {
        const GroupK<T>& k = (uint32_t)(i % row) < 3u ? k0 : k1;
        if (k.on) adam_elem<T>(p0[i], m0[i], v0[i], g0[i], k);
        break;
      }
      case kAdamNormal: {
        T q[3], upd[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          q[c] = p0[3 * i + c];
          T m = m0[3 * i + c], v = v0[3 * i + c];
          upd[c] = adam_elem<T>(q[c], m, v, g0[3 * i + c], k0);
          m0[3 * i + c] = m;
          v0[3 * i + c] = v;
        }
        // renormalise rows the update moved (trainer.py:214-221)
        if (upd[0] != T(0) || upd[1] != T(0) || upd[2] != T(0)) {
          T nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);  // np.linalg.norm
          if (nrm == T(0)) nrm = T(1);
#pragma unroll
          for (int c = 0; c < 3; ++c) q[c] = q[c] / nrm;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) p0[3 * i + c] = q[c];
        break;
      }
      case kAdamOpacity: {
        T* p1 = static_cast<T*>(sg.param[1]);
        if (k0.on) adam_elem<T>(p0[i], m0[i], v0[i], g0[i], k0);
        if (k1.on)
          adam_elem<T>(p1[i], static_cast<T*>(sg.m[1])[i], static_cast<T*>(sg.v[1])[i],
                       static_cast<const T*>(sg.grad[1])[i], k1);
        if (tie) p1[i] = p0[i];  // trainer.py:222-224
        break;
      }
    }
  }
}

// Each CTA works on one segment (CTAs apportioned by units on the host), so
// the kind branch is uniform and there is no per-unit segment search.
template <typename T>
__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a) {
  int s = 0;
  while ((int)blockIdx.x >= a.cta_start[s + 1]) ++s;
  const AdamSeg& sg = a.seg[s];
  const int64_t first = (int64_t)(blockIdx.x - a.cta_start[s]) * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)(a.cta_start[s + 1] - a.cta_start[s]) * blockDim.x;
  if (sg.vec) {
    if (sg.kind == kAdamSh)
      adam_vector_seg<T, true>(sg, first, stride);
    else
      adam_vector_seg<T, false>(sg, first, stride);
  } else {
    adam_scalar_seg<T>(sg, first, stride, a.tie_opacities);
  }
}

cudaError_t launch_adam(AdamArgs a, int dtype, cudaStream_t stream) {
  int64_t total = 0;
  for (int s = 0; s < a.nseg; ++s) total += a.seg[s].units;
  if (total == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // ~8 resident CTAs of 256 per SM, split over the segments by their units
  const int64_t budget = (int64_t)sms * 8;
  int c = 0;
  for (int s = 0; s < a.nseg; ++s) {
    const int64_t want = (a.seg[s].units + 255) / 256;
    int64_t share = (budget * a.seg[s].units + total - 1) / total;
    if (share < 1) share = 1;
    a.cta_start[s] = c;
    c += (int)(want < share ? want : share);
  }
  a.cta_start[a.nseg] = c;
  if (dtype == 0)
    adam_kernel<float><<<c, 256, 0, stream>>>(a);
  else
    adam_kernel<double><<<c, 256, 0, stream>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hs
