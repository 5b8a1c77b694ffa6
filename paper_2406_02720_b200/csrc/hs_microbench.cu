// hs_microbench.cu -- FP32 FMA and MUFU.EX2 throughput probes.  MEASURED_PEAKS.json
// carries only HBM and bf16 tensor peaks; the blend kernels are FP32/SFU bound, so
// bench.py measures these denominators on the box it runs on.
#include <cstdint>

#include "../../include/halfsplat_b200.h"
#include "hs_common.cuh"

namespace hs {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) fma_probe_kernel(float* out, int iters, float m, float a) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], m, a);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

__device__ __forceinline__ float2 ffma2_probe(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n"
      " mov.b64 rc, {%6,%7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0,%1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// packed FP32 (FFMA2, sm_100): 2 FMAs per lane per instruction
__global__ void __launch_bounds__(256) fma2_probe_kernel(float* out, int iters, float m, float a) {
  float2 x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  const float2 mm = make_float2(m, m), aa = make_float2(a, a);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = ffma2_probe(x[c], mm, aa);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c].x + x[c].y;
  if (s == 12345.678f) out[0] = s;
}

__global__ void __launch_bounds__(256) ex2_probe_kernel(float* out, int iters) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = -(threadIdx.x * 1e-3f + c);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = -ex2_approx(x[c]);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678f) out[0] = s;
}

// The blend kernels' erf32 (hs_common.cuh) on the hardware's MUFU.EX2, so its
// accuracy bound is checked on the device rather than on an exact-exp2 emulation.
__global__ void erf32_probe_kernel(const float* __restrict__ z, float* __restrict__ out,
                                   int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = erf32(z[i]);
}

}  // namespace hs

extern "C" int hs_probe_erf32(const float* z, float* out, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!z || !out))) return HS_ERR_INVALID_ARG;
  if (n == 0) return HS_OK;
  const int threads = 256;
  const int blocks = (int)((n + threads - 1) / threads < 4096 ? (n + threads - 1) / threads : 4096);
  hs::erf32_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(z, out, n);
  hs::note_launch();
  return cudaGetLastError() == cudaSuccess ? HS_OK : HS_ERR_CUDA;
}

static double g_fma2_tflops = 0.0;
extern "C" double hs_last_fma2_tflops(void) { return g_fma2_tflops; }

extern "C" int hs_measure_fp32_peaks(double* fma_tflops, double* ex2_gops) {
  using namespace hs;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HS_ERR_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  if (cudaMalloc(&out, 16) != cudaSuccess) return HS_ERR_CUDA;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float best_fma = 1e30f, best_ex2 = 1e30f, best_fma2 = 1e30f, ms = 0.f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    fma_probe_kernel<<<blocks, threads>>>(out, iters, 0.9999f, 1e-3f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_fma) best_fma = ms;
    cudaEventRecord(a);
    fma2_probe_kernel<<<blocks, threads>>>(out, iters, 0.9999f, 1e-3f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_fma2) best_fma2 = ms;
    cudaEventRecord(a);
    ex2_probe_kernel<<<blocks, threads>>>(out, iters / 4);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_ex2) best_ex2 = ms;
  }
  note_launch(15);
  const double n = (double)blocks * threads * kChains;
  if (fma_tflops) *fma_tflops = 2.0 * n * iters / (best_fma * 1e-3) / 1e12;
  if (ex2_gops) *ex2_gops = n * (iters / 4) / (best_ex2 * 1e-3) / 1e9;
  g_fma2_tflops = 4.0 * n * iters / (best_fma2 * 1e-3) / 1e12;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? HS_OK : HS_ERR_CUDA;
}
