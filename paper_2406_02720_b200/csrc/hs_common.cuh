// hs_common.cuh -- shared constants, the per-splat record layout and the FP32
// half-Gaussian weight primitives used by every kernel of the rasterizer.
#pragma once

#include <atomic>
#include <mutex>
#include <cstdint>
#include <cuda_runtime.h>

namespace hs {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) per kernel and device, raised
// whenever a launch needs more than was set before (the attribute is per-device
// state and a launch above it fails; never lowered, so concurrent callers with
// different sizes stay valid).
template <auto Kernel>
inline cudaError_t set_dynamic_smem(int bytes) {
  static std::mutex mu;
  static int set_bytes[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64)
    return cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  std::lock_guard<std::mutex> lock(mu);
  if (set_bytes[dev] >= bytes && set_bytes[dev] > 0) return cudaSuccess;
  e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) set_bytes[dev] = bytes;
  return e;
}


constexpr int kTile = 16;              // rasterizer.py:35
constexpr double kRadiusSigmas = 3.5;  // rasterizer.py:39
constexpr double kLowpass = 0.3;       // geometry.py:20 LOWPASS_DILATION
constexpr double kCondLimit = 1e8;     // geometry.py:24 FRAME_COND_LIMIT
constexpr double kNormalEps = 1e-6;    // kernels.py:25 NORMAL_EPS
constexpr float kTerminationT = 1e-4f; // _blend_cy.pyx:16
constexpr float kWeightClamp = 0.99f;  // _blend_cy.pyx:17
constexpr float kInvSqrtPi = 0.5641895835477563f;  // _blend_cy.pyx:18
constexpr float kLog2e = 1.4426950408889634f;

// Per-splat record: 64 bytes, one per primitive (indexed by original index).
// Slots 0..12 are the reference's `packed` columns rounded to float32
// (layout of _blend_py.py:9-15; mu_hat keeps its rounding residual in R_MU_LO so
// pixel offsets are exact to ~3e-8 px even at 4K); slots 13..15 carry the blend
// mode and the pair-row bookkeeping the backward needs.
enum RecordSlot {
  R_MUX = 0, R_MUY, R_CA, R_CB, R_CC, R_ZA, R_ZB, R_C1, R_C2,
  R_RED, R_GREEN, R_BLUE, R_DEPTH,
  R_FLAGS,       // u32: mode (bits 0-1) | steep (bit 2) | may-clamp (bit 3) | bad frame (bit 4)
                 //      | no strip windows (bit 5) | spans_x << 6
  R_ROW_ORIGIN,  // i32: pair_base - ty0*spans_x - tx0; pair (tx,ty) -> row origin + ty*spans_x + tx
  R_MU_LO        // half2: (mux - (float)mux, muy - (float)muy)
};
constexpr int kRecordFloats = 16;

// "Steep" splats: erf argument z = za*dx + zb*dy with |za|,|zb| so large (the
// splitting plane nearly contains the ray, |n_ray.z| small) that FP32 cannot
// resolve z near the plane.  Their z is evaluated in FP64 from this side record;
// the flag also rides in bit 31 of the sort value so the blend's staging lane
// knows to fetch it.  Criterion: (|za| + |zb|) * reach > kSteepLimit, reach =
// radius + 24 px bounds |dx|,|dy| inside any covered tile, so non-steep splats
// keep |z| rounding error below ~6e-8 * 256 = 1.5e-5 (a weight error below
// 0.56 * 1.5e-5 = 9e-6).  About 10% of the c3 pairs are steep.
//
// The side record holds the erf argument in a cancellation-free form.  With K
// the larger of |za|, |zb| and r = (smaller / larger) coefficient:
//   y-form (|zb| >= |za|):  z = zb * ((py - muy) + r (px - mux))
//   x-form (|za| >  |zb|):  z = za * ((px - mux) + r (py - muy))
// A lane evaluates the bracket at its column and first row in FP64, splits it
// into float hi + lo, and steps down its rows in FP32 with one FMA per pixel
// (exact product + single rounding), so z keeps ~1e-7 relative accuracy on the
// packed FP32 path (steep_setup / steep_z in hs_blend.cu).
struct __align__(16) SteepRec {
  double mux, muy;
  double r;        // smaller / larger erf coefficient, |r| <= 1
  float K;         // the larger coefficient (zb in the y-form, za in the x-form)
  uint32_t xform;  // 1: x-form
};
__host__ __device__ __forceinline__ SteepRec make_steep(double mux, double muy, double za,
                                                        double zb) {
  SteepRec s;
  s.mux = mux;
  s.muy = muy;
  s.xform = fabs(za) > fabs(zb) ? 1u : 0u;
  s.r = s.xform ? zb / za : za / zb;
  s.K = (float)(s.xform ? za : zb);
  return s;
}
constexpr double kSteepLimit = 256.0;
constexpr uint32_t kSteepBit = 0x80000000u;
constexpr uint32_t kIndexMask = 0x7fffffffu;

// Internal generation-order pair rows: the reference's 12 columns
// (_blend_py.py:16-18) plus column 12 = sum over pixels of d_z * z, which gives
// d(loss)/d(1/(sqrt2 |n3|)) without the cancellation of za*d_za + zb*d_zb.
constexpr int kRowFloats = 16;
constexpr int kColSumDzZ = 12;

constexpr uint32_t kFlagSteep = 4u;
constexpr uint32_t kFlagClamp = 8u;
// the whitening fell back to the identity (rasterizer.py:233-234, 246-247); K7
// replays K1's decision from this bit instead of re-deciding it
constexpr uint32_t kFlagBad = 16u;
// Large splats (3.5-sigma radius above kWinMaxRadius px).  Their conic is stored
// in a cancellation-free form: slot R_CA = a, R_CB = r = b / a, R_CC = D =
// c - b^2 / a (all from FP64), so the exponent a dx^2 + 2b dx dy + c dy^2 is
// evaluated as a (dx + r dy)^2 + D dy^2, a sum of two non-negative terms.  With the
// plain (a, b, c) in FP32, the terms of a long, thin splat far from its centre
// reach ~a r^2 and cancel; their rounding grew the blend's error past 1e-4.  These
// splats take the blend's generic path and no strip windows (whose FP32 box bound
// has the same cancellation); conic_abc() gives back (a, b, c).
constexpr uint32_t kFlagNoWin = 32u;
constexpr double kWinMaxRadius = 256.0;
__host__ __device__ __forceinline__ void conic_abc(float a, float s1, float s2, uint32_t flags,
                                                   float& b, float& c) {
  if (flags & kFlagNoWin) {
    b = s1 * a;
    c = fmaf(a * s1, s1, s2);
  } else {
    b = s1;
    c = s2;
  }
}
constexpr int kFlagSpanShift = 6;
// Splats whose weight can never reach the 0.99 clamp (c1 + |c2| bounds
// (c1 + c2 E) g; 0.989 leaves room for FP32 rounding) skip the clamp and the
// backward's gating test.
__host__ __device__ __forceinline__ bool may_clamp(double c1, double c2) {
  return c1 + fabs(c2) > 0.989;
}
__host__ __device__ __forceinline__ uint32_t pack_flags(int mode, bool steep, bool clamp,
                                                        int spans_x, bool bad = false,
                                                        bool nowin = false) {
  return (uint32_t)mode | (steep ? kFlagSteep : 0u) | (clamp ? kFlagClamp : 0u) |
         (bad ? kFlagBad : 0u) | (nowin ? kFlagNoWin : 0u) |
         ((uint32_t)spans_x << kFlagSpanShift);
}
__host__ __device__ __forceinline__ bool is_steep(double za, double zb, double reach) {
  return (fabs(za) + fabs(zb)) * reach > kSteepLimit;
}

// Blend modes (_blend_py.py:13-14).
constexpr int kModeErf = 0;
constexpr int kModeSign = 1;
constexpr int kModePlain = 2;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Branch-free FP32 erf: erf(z) = sign(z) * (1 - 2^Q(|z|)), Q(x) = x*R(x) with
// R a degree-5 minimax fit of log2(erfc(x))/x on [0, 3.92] (erfc(3.92) is
// below half an ulp of 1.0f).  Max abs error 3.3e-7 including FP32 rounding
// (tools/fit_erf32.py); it enters a pixel as c2*g*error <= 1.7e-7 per splat,
// far inside the 1e-4 image tolerance.  The sign is applied last, so
// erf(-z) == -erf(z) bit for bit, the property _blend_cy.pyx:40-63 /
// kernels.py:136-147 rely on.  One MUFU.EX2, six FMA-pipe ops and no divergent
// branches (the reference's 3-way piecewise polynomial would serialise warps
// whose pixels straddle the branches).
__device__ __forceinline__ float erf32(float z) {
  const float a = fminf(fabsf(z), 3.92f);
  float r = 1.420475164e-04f;
  r = fmaf(r, a, -3.664300777e-03f);
  r = fmaf(r, a, 3.089622408e-02f);
  r = fmaf(r, a, -1.496994644e-01f);
  r = fmaf(r, a, -9.181654453e-01f);
  r = fmaf(r, a, -1.627925038e+00f);
  r = r * a;
  return copysignf(1.0f - ex2_approx(r), z);
}

// _blend_cy.pyx:66-71
__device__ __forceinline__ float sign32(float x) {
  return x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f);
}

}  // namespace hs

// Process-wide launch counter (reported by bench.py as gpu_launches).
namespace hs {
void note_launch(int n = 1);
}
