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

}  // namespace hs

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
  float best_fma = 1e30f, best_ex2 = 1e30f, ms = 0.f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    fma_probe_kernel<<<blocks, threads>>>(out, iters, 0.9999f, 1e-3f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_fma) best_fma = ms;
    cudaEventRecord(a);
    ex2_probe_kernel<<<blocks, threads>>>(out, iters / 4);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_ex2) best_ex2 = ms;
  }
  note_launch(10);
  const double n = (double)blocks * threads * kChains;
  if (fma_tflops) *fma_tflops = 2.0 * n * iters / (best_fma * 1e-3) / 1e12;
  if (ex2_gops) *ex2_gops = n * (iters / 4) / (best_ex2 * 1e-3) / 1e9;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? HS_OK : HS_ERR_CUDA;
}
