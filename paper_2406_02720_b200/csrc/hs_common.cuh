// hs_common.cuh -- shared constants, the per-splat record layout and the FP32
// half-Gaussian weight primitives used by every kernel of the rasterizer.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hs {

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
// (layout of _blend_py.py:9-15); slots 13..15 carry the blend mode and the
// pair-row bookkeeping the backward needs.
enum RecordSlot {
  R_MUX = 0, R_MUY, R_CA, R_CB, R_CC, R_ZA, R_ZB, R_C1, R_C2,
  R_RED, R_GREEN, R_BLUE, R_DEPTH,
  R_MODE_SPANX,  // u32: mode (bits 0-1) | spans_x << 2
  R_PAIR_BASE,   // u32: first generation-order pair index of this splat
  R_TXY          // u32: tx0 | ty0 << 16 (tile rect origin)
};
constexpr int kRecordFloats = 16;

// Blend modes (_blend_py.py:13-14).
constexpr int kModeErf = 0;
constexpr int kModeSign = 1;
constexpr int kModePlain = 2;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Branch-free FP32 erf: erf(z) = sign(z) * (1 - 2^Q(|z|)), Q(x) = x*R(x) with
// R a degree-8 minimax fit of log2(erfc(x))/x on [0, 3.92] (erfc(3.92) is
// below half an ulp of 1.0f).  Max abs error 8.4e-8 including FP32 rounding
// (tools/fit_erf32.py).  The sign is applied last, so erf(-z) == -erf(z)
// bit for bit, the property _blend_cy.pyx:40-63 / kernels.py:136-147 rely on.
// One MUFU.EX2 and no divergent branches (the reference's 3-way piecewise
// polynomial would serialise warps whose pixels straddle the branches).
__device__ __forceinline__ float erf32(float z) {
  const float a = fminf(fabsf(z), 3.92f);
  float r = 1.160483589e-05f;
  r = fmaf(r, a, -1.529645961e-04f);
  r = fmaf(r, a, 8.482352714e-04f);
  r = fmaf(r, a, -2.274787286e-03f);
  r = fmaf(r, a, 8.480722317e-05f);
  r = fmaf(r, a, 2.772447467e-02f);
  r = fmaf(r, a, -1.483079046e-01f);
  r = fmaf(r, a, -9.184429049e-01f);
  r = fmaf(r, a, -1.627907276e+00f);
  r = r * a;
  return copysignf(1.0f - ex2_approx(r), z);
}

// _blend_cy.pyx:66-71
__device__ __forceinline__ float sign32(float x) {
  return x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f);
}

__host__ __device__ __forceinline__ uint32_t pack_mode_spanx(int mode, int spans_x) {
  return (uint32_t)mode | ((uint32_t)spans_x << 2);
}

}  // namespace hs

// Process-wide launch counter (reported by bench.py as gpu_launches).
namespace hs {
void note_launch(int n = 1);
}
