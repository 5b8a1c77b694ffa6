// hs_loss.cu -- the training loss between K5 and K6: (1 - lambda) L1 +
// lambda (1 - SSIM) of the rendered image against the target, and its exact
// gradient, which is the cotangent d_color that K6 consumes
// (loss.py:48-106; lambda = 0.2 at trainer.py:40).
//
// SSIM is the reference's: 11-tap Gaussian window (sigma 1.5) applied
// separably with zero padding, C1 = 0.01^2, C2 = 0.03^2, mean over pixels and
// channels (loss.py:13-79).  Two tiled kernels, one CTA per 32x16 output tile
// and group of up to 4 channels (so the interleaved HWC images are read once):
//   L1 (loss_stats_kernel): stage the tile's 42x26 halo of both images in
//      shared memory, per channel filter x, y, x^2, y^2, xy (vertical then
//      horizontal, register-blocked; as
//      correlate1d axis 0 then axis 1), and per pixel form the SSIM map and
//      the three adjoint maps of ssim_with_grad (d_m1 - 2 m1 d_s1 - m2 d_s12,
//      d_s1, d_s12); per-CTA partial sums of |x - y| and of the SSIM map.
//   L2 (loss_grad_kernel): filter the adjoint maps the same way (the window is
//      symmetric, so the blur is self-adjoint), combine with the pixel values
//      and the L1 term into d_color; CTA 0 also reduces the partials into the
//      loss (and the MSE of metrics.psnr) in a fixed order: deterministic.
// Arithmetic is FP64 on the FP32 images (their squares and products are exact
// in FP64); the window taps are summed in scipy's symmetric order, centre
// first, then the outer pairs inwards, with FMA contraction and one division
// per pixel, so loss and gradient agree with the reference's float64 to a few
// ulp.  The adjoint maps live in the workspace planar, (C, H, W).
#include <cmath>
#include <cstdint>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

constexpr int kWinR = 5;                   // (SSIM_WINDOW - 1) / 2, loss.py:13
constexpr int kLTX = 32, kLTY = 16;        // output tile
constexpr int kLHX = kLTX + 2 * kWinR;     // 42: halo width
constexpr int kLHY = kLTY + 2 * kWinR;     // 26: halo height
constexpr int kLossThreads = 256;  // = kLTX * kLTY / kHOut: one thread per pixel pair
constexpr double kSsimC1 = 0.01 * 0.01;  // loss.py:15
constexpr double kSsimC2 = 0.03 * 0.03;  // loss.py:16

// scipy's correlate1d with a symmetric kernel: centre tap, then the pairs
// (i-5, i+5), (i-4, i+4), ... each summed before scaling.  `w` is the window
// in the kernel's parameter space (LossArgs::win).
template <typename F>
__device__ __forceinline__ double win_sum(const double* w, F at) {
  double s = at(0) * w[kWinR];
#pragma unroll
  for (int j = kWinR; j >= 1; --j) s += (at(-j) + at(j)) * w[kWinR - j];
  return s;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kLossThreads / 32; ++w) s += red[w];
  return s;
}

__device__ __forceinline__ int cta_linear() {
  return (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
}

// NOUT consecutive window sums from NOUT + 10 consecutive values in registers
// (register blocking: each staged value is read from shared memory once per
// thread instead of once per tap).
template <int NOUT>
__device__ __forceinline__ void win_run(const double* v, const double* w, double* out) {
#pragma unroll
  for (int i = 0; i < NOUT; ++i)
    out[i] = win_sum(w, [&](int j) { return v[i + kWinR + j]; });
}

constexpr int kVRows = 2;                        // vertical outputs per thread
constexpr int kVItems = kLHX * (kLTY / kVRows);  // 336 column segments
constexpr int kHOut = 2;                         // horizontal outputs per thread
constexpr int kMaxCG = 4;                        // channels per CTA (grid.z groups beyond)
static_assert(kLossThreads * kHOut == kLTX * kLTY, "one thread per pixel pair");

// Vertical pass over NM maps: vs[m][r][q] = window sum over rows r .. r+10 of
// src(m, ., q), for the tile's kLTY output rows.
template <int NM, typename Src>
__device__ __forceinline__ void vertical_pass(const double* w, Src src,
                                              double (*vs)[kLTY][kLHX]) {
  for (int e = threadIdx.x; e < kVItems; e += kLossThreads) {
    const int g = e / kLHX, q = e - g * kLHX, r0 = g * kVRows;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      double v[kVRows + 2 * kWinR], o[kVRows];
#pragma unroll
      for (int i = 0; i < kVRows + 2 * kWinR; ++i) v[i] = src(m, r0 + i, q);
      win_run<kVRows>(v, w, o);
#pragma unroll
      for (int i = 0; i < kVRows; ++i) vs[m][r0 + i][q] = o[i];
    }
  }
}

// Horizontal window sums of one row of vs for outputs tx0 and tx0 + 1.
__device__ __forceinline__ void horizontal_pair(const double* w, const double* row, int tx0,
                                                double* out) {
  double v[kHOut + 2 * kWinR];
  const double2* p = reinterpret_cast<const double2*>(row + tx0);
#pragma unroll
  for (int i = 0; i < (kHOut + 2 * kWinR) / 2; ++i) {
    const double2 d = p[i];
    v[2 * i] = d.x;
    v[2 * i + 1] = d.y;
  }
  win_run<kHOut>(v, w, out);
}

// The images in their input type: float32 (the render's, hs_loss) or float64
// (a reference caller's host arrays, hs_loss_f64).
template <typename TI>
__device__ __forceinline__ const TI* image_x(const LossArgs& a);
template <>
__device__ __forceinline__ const float* image_x<float>(const LossArgs& a) { return a.x; }
template <>
__device__ __forceinline__ const double* image_x<double>(const LossArgs& a) { return a.x64; }
template <typename TI>
__device__ __forceinline__ const TI* image_y(const LossArgs& a);
template <>
__device__ __forceinline__ const float* image_y<float>(const LossArgs& a) { return a.y; }
template <>
__device__ __forceinline__ const double* image_y<double>(const LossArgs& a) { return a.y64; }

// Dynamic shared memory of L1: the interleaved halo rows of both images for the
// CTA's channel group, in the input type (converted to FP64 on use).
template <typename TI>
__host__ __device__ constexpr size_t loss_stats_smem(int cg) {
  return (size_t)2 * kLHY * kLHX * cg * sizeof(TI);
}

template <typename TI, bool SSIM, int CG>
__global__ void __launch_bounds__(kLossThreads, sizeof(TI) == 4 ? 3 : 2)
loss_stats_kernel(LossArgs a) {
  extern __shared__ __align__(16) unsigned char halo_raw[];
  TI* halo = reinterpret_cast<TI*>(halo_raw);  // x then y, [kLHY][kLHX * cg]
  __shared__ __align__(16) double vs[5][kLTY][kLHX];  // vertical sums of x, y, xx, yy, xy
  __shared__ double red[kLossThreads / 32];
  const int group = a.group0 + blockIdx.z;
  const int x0 = blockIdx.x * kLTX, y0 = blockIdx.y * kLTY, c0 = group * kMaxCG;
  const int tid = threadIdx.x;
  const int64_t W = a.width, H = a.height, C = a.channels;
  constexpr int cg = CG;  // channels of this CTA (a tail group has its own launch)
  constexpr int rowf = kLHX * cg;  // floats per staged halo row
  TI* xs = halo;
  TI* ys = halo + kLHY * rowf;
  const TI* ax = image_x<TI>(a);
  const TI* ay = image_y<TI>(a);
  double l1 = 0.0, ssum = 0.0, sq = 0.0;
  if (SSIM) {
    // the halo rows of all cg channels: contiguous runs of the HWC images
    for (int e = tid; e < kLHY * rowf; e += kLossThreads) {
      const int r = e / rowf, f = e - r * rowf, q = f / cg, cc = f - q * cg;
      const int gy = y0 - kWinR + r, gx = x0 - kWinR + q;
      const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
      const int64_t k = (gy * W + gx) * C + c0 + cc;
      xs[e] = in ? ax[k] : TI(0);  // mode="constant", cval 0 (loss.py:31-32)
      ys[e] = in ? ay[k] : TI(0);
    }
    __syncthreads();
  }
  const int ty = tid / (kLTX / kHOut), tx0 = (tid - ty * (kLTX / kHOut)) * kHOut;
  const int64_t gy = y0 + ty;
  for (int cc = 0; cc < cg; ++cc) {
    double f[5][kHOut];
    if (SSIM) {
      // x^2, y^2 and xy in FP64 (exact for FP32 inputs; numpy's products for
      // float64 ones, loss.py:62-64)
      vertical_pass<5>(a.win, [&](int m, int r, int q) {
        const double x = xs[r * rowf + q * cg + cc], y = ys[r * rowf + q * cg + cc];
        return m == 0 ? x : m == 1 ? y : m == 2 ? x * x : m == 3 ? y * y : x * y;
      }, vs);
      __syncthreads();
#pragma unroll
      for (int m = 0; m < 5; ++m) horizontal_pair(a.win, vs[m][ty], tx0, f[m]);
      __syncthreads();  // vs is rewritten by the next channel
    }
    const int c = c0 + cc;
#pragma unroll
    for (int i = 0; i < kHOut; ++i) {
      const int64_t gx = x0 + tx0 + i;
      if (gx >= W || gy >= H) continue;
      double x, y;
      if (SSIM) {  // the centre of the staged halo
        const int h = (ty + kWinR) * rowf + (tx0 + i + kWinR) * cg + cc;
        x = xs[h];
        y = ys[h];
      } else {
        const int64_t k = (gy * W + gx) * C + c;
        x = ax[k];
        y = ay[k];
      }
      l1 += fabs(x - y);
      sq += (x - y) * (x - y);  // metrics.psnr's MSE (metrics.py:13-22)
      if (!SSIM) continue;
      const int64_t kp = ((int64_t)c * H + gy) * W + gx;  // planar adjoint maps
      // ssim_with_grad, loss.py:60-73 (one division: 1/b1 and 1/b2 from 1/(b1 b2))
      const double m1 = f[0][i], m2 = f[1][i];
      const double s1 = f[2][i] - m1 * m1, s2 = f[3][i] - m2 * m2, s12 = f[4][i] - m1 * m2;
      const double a1 = 2.0 * m1 * m2 + kSsimC1, a2 = 2.0 * s12 + kSsimC2;
      const double b1 = m1 * m1 + m2 * m2 + kSsimC1, b2 = s1 + s2 + kSsimC2;
      const double r = 1.0 / (b1 * b2), rb1 = b2 * r, rb2 = b1 * r;
      const double smap = a1 * a2 * r;
      ssum += smap;
      const double d_m1 = 2.0 * a2 * r * (m2 - m1 * a1 * rb1) * a.inv_n;
      const double d_s1 = -smap * rb2 * a.inv_n;
      const double d_s12 = 2.0 * a1 * r * a.inv_n;
      a.adj_m[kp] = d_m1 - 2.0 * m1 * d_s1 - m2 * d_s12;  // loss.py:75
      a.adj_s1[kp] = d_s1;
      a.adj_s12[kp] = d_s12;
    }
  }
  l1 = block_sum(l1, red);
  ssum = block_sum(ssum, red);
  sq = block_sum(sq, red);
  if (tid == 0) {
    const int cta = (group * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    a.partial[3 * cta] = l1;
    a.partial[3 * cta + 1] = ssum;
    a.partial[3 * cta + 2] = sq;
  }
}

template <typename TI, bool SSIM>
__global__ void __launch_bounds__(kLossThreads) loss_grad_kernel(LossArgs a) {
  __shared__ __align__(16) double hs_[3][kLHY][kLHX];  // adjoint maps with halo
  __shared__ __align__(16) double vs[3][kLTY][kLHX];
  __shared__ double red[kLossThreads / 32];
  const int x0 = blockIdx.x * kLTX, y0 = blockIdx.y * kLTY, c0 = blockIdx.z * kMaxCG;
  const int tid = threadIdx.x;
  const int64_t W = a.width, H = a.height, C = a.channels;
  const int cg = (int)(C - c0 < kMaxCG ? C - c0 : kMaxCG);
  if (cta_linear() == 0) {
    // loss.py:95 and 102: fixed-order reduction of the L1 partials
    double l1 = 0.0, ss = 0.0, sq = 0.0;
    for (int i = tid; i < a.n_partials; i += kLossThreads) {
      l1 += a.partial[3 * i];
      ss += a.partial[3 * i + 1];
      sq += a.partial[3 * i + 2];
    }
    l1 = block_sum(l1, red) / a.n;
    ss = block_sum(ss, red) / a.n;
    sq = block_sum(sq, red) / a.n;
    if (tid == 0) {
      a.loss[0] = SSIM ? (1.0 - a.lambda) * l1 + a.lambda * (1.0 - ss) : l1;
      a.loss[1] = l1;
      a.loss[2] = SSIM ? ss : 0.0;
      a.loss[3] = sq;
    }
  }
  const double w_l1 = 1.0 - a.lambda;
  const int ty = tid / (kLTX / kHOut), tx0 = (tid - ty * (kLTX / kHOut)) * kHOut;
  const int64_t gy = y0 + ty;
  for (int cc = 0; cc < cg; ++cc) {
    const int c = c0 + cc;
    double f[3][kHOut];
    if (SSIM) {
      for (int e = tid; e < kLHY * kLHX; e += kLossThreads) {
        const int r = e / kLHX, q = e - r * kLHX;
        const int gyy = y0 - kWinR + r, gx = x0 - kWinR + q;
        const bool in = gx >= 0 && gx < W && gyy >= 0 && gyy < H;
        const int64_t k = ((int64_t)c * H + gyy) * W + gx;
        hs_[0][r][q] = in ? a.adj_m[k] : 0.0;
        hs_[1][r][q] = in ? a.adj_s1[k] : 0.0;
        hs_[2][r][q] = in ? a.adj_s12[k] : 0.0;
      }
      __syncthreads();
      vertical_pass<3>(a.win, [&](int m, int r, int q) { return hs_[m][r][q]; }, vs);
      __syncthreads();
#pragma unroll
      for (int m = 0; m < 3; ++m) horizontal_pair(a.win, vs[m][ty], tx0, f[m]);
      __syncthreads();  // hs_ and vs are rewritten by the next channel
    }
#pragma unroll
    for (int i = 0; i < kHOut; ++i) {
      const int64_t gx = x0 + tx0 + i;
      if (gx >= W || gy >= H) continue;
      const int64_t k = (gy * W + gx) * C + c;
      const double x = image_x<TI>(a)[k], y = image_y<TI>(a)[k];
      const double diff = x - y;
      const double sg = diff > 0.0 ? 1.0 : (diff < 0.0 ? -1.0 : (diff == 0.0 ? 0.0 : diff));
      double g = w_l1 * (sg * a.inv_n);  // loss.py:96-99
      if (SSIM) {
        const double s_grad = f[0][i] + 2.0 * x * f[1][i] + y * f[2][i];  // loss.py:74-78
        g = g - a.lambda * s_grad;                                       // loss.py:103
      }
      if (a.d_f32) a.d_f32[k] = (float)g;
      if (a.d_f64) a.d_f64[k] = g;
    }
  }
}

template <typename TI, int CG>
static cudaError_t launch_stats(const LossArgs& a, dim3 grid, cudaStream_t stream) {
  if (!a.ssim) {
    loss_stats_kernel<TI, false, CG><<<grid, kLossThreads, 0, stream>>>(a);
    return cudaGetLastError();
  }
  constexpr size_t smem = loss_stats_smem<TI>(CG);
  const cudaError_t attr = set_dynamic_smem<loss_stats_kernel<TI, true, CG>>((int)smem);
  if (attr != cudaSuccess) return attr;
  loss_stats_kernel<TI, true, CG><<<grid, kLossThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

template <typename TI>
static cudaError_t launch_loss_t(const LossArgs& a, cudaStream_t stream) {
  // channel groups of kMaxCG; a tail group of fewer channels gets its own launch
  const int full = a.channels / kMaxCG, tail = a.channels - full * kMaxCG;
  const unsigned gx = (unsigned)((a.width + kLTX - 1) / kLTX);
  const unsigned gy = (unsigned)((a.height + kLTY - 1) / kLTY);
  cudaError_t e = cudaSuccess;
  if (full > 0) e = launch_stats<TI, kMaxCG>(a, dim3(gx, gy, (unsigned)full), stream);
  if (e == cudaSuccess && tail > 0) {
    LossArgs t = a;
    t.group0 = full;
    const dim3 g(gx, gy, 1);
    e = tail == 1 ? launch_stats<TI, 1>(t, g, stream)
                  : tail == 2 ? launch_stats<TI, 2>(t, g, stream) : launch_stats<TI, 3>(t, g, stream);
  }
  if (e != cudaSuccess) return e;
  const dim3 grid(gx, gy, (unsigned)(full + (tail > 0)));
  if (a.ssim)
    loss_grad_kernel<TI, true><<<grid, kLossThreads, 0, stream>>>(a);
  else
    loss_grad_kernel<TI, false><<<grid, kLossThreads, 0, stream>>>(a);
  note_launch((full > 0) + (tail > 0) + 1);
  return cudaGetLastError();
}

cudaError_t launch_loss(const LossArgs& a, cudaStream_t stream) {
  return a.x64 ? launch_loss_t<double>(a, stream) : launch_loss_t<float>(a, stream);
}

int64_t loss_partials(int width, int height, int channels) {
  return (int64_t)((width + kLTX - 1) / kLTX) * ((height + kLTY - 1) / kLTY) *
         ((channels + kMaxCG - 1) / kMaxCG);
}

}  // namespace hs
