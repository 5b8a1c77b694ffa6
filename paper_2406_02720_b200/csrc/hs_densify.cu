// hs_densify.cu -- density control on the device: the screen-space gradient
// statistics, densify_and_prune and reset_opacity (trainer.py:229-350).
//
//   D0 stats_update      grad_sum += pos_grad_norm, mu_grad_sum += d_mu,
//                        count += touch_count (DensifyStats.update, 241-244)
//   D1 classify          per primitive: average gradient, both opacities, the
//                        largest scale -> prune / clone / split candidates
//                        (trainer.py:254-266); three exclusive scans (CUB) give
//                        every candidate its rank in index order
//   -- the host reads the totals, applies the max_primitives budget exactly as
//      the reference's two sequential loops do (268-288) and sizes the scene --
//   D2 emit              every primitive writes its own rows of the new scene
//                        at scan positions: survivors in index order, then the
//                        accepted clones (stepped down the accumulated mu
//                        gradient, 298-307), then split children of draw 1 and
//                        of draw 2 (mu from the parent Gaussian, log-scale
//                        shrunk, 308-320); Adam moments follow the survivors,
//                        new rows start at zero (AdamState.select /
//                        append_zeros, 334-335)
//   D3 reset_opacity     both logits clamped to logit(ceiling), opacity moments
//                        zeroed (343-350)
// FP64 in the reference's statement order (-fmad=false): with the reference's
// split offsets (rng.normal draws passed in) a float64 scene densifies
// bit-identically.  Without offsets, D2 draws its own standard normals
// (Philox4x32-10 + Box-Muller, keyed by seed, draw, split rank and axis).
#include <cmath>
#include <cstdint>

#include <cub/cub.cuh>

#include "hs_common.cuh"
#include "hs_internal.h"
#include "hs_numpy_order.cuh"

namespace hs {

template <typename T>
__global__ void __launch_bounds__(256) densify_stats_kernel(DensifyStatsArgs st, const T* pgn,
                                                            const T* d_mu, const int32_t* touch,
                                                            int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  st.grad_sum[i] += (double)pgn[i];
  for (int k = 0; k < 3; ++k) st.mu_grad_sum[3 * i + k] += (double)d_mu[3 * i + k];
  st.count[i] += touch[i];
}

// flags of D1
constexpr uint8_t kDPrune = 1, kDClone = 2, kDSplit = 4;

template <typename T>
__global__ void __launch_bounds__(256) densify_classify_kernel(
    DensifyStatsArgs st, const T* log_scale, const T* ra, const T* rb, int64_t n,
    DensifyParams p, uint8_t* flags, int32_t* f_surv, int32_t* f_clone, int32_t* f_split) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {  // the scans run over n + 1 entries so their last entry is the total
    f_surv[n] = f_clone[n] = f_split[n] = 0;
    return;
  }
  const int64_t c = st.count[i];
  const double avg = c > 0 ? st.grad_sum[i] / (double)(c > 1 ? c : 1) : 0.0;  // 255
  const double a1 = sigmoid_ref((double)ra[i]), a2 = sigmoid_ref((double)rb[i]);
  double max_scale = exp((double)log_scale[3 * i]);
  for (int k = 1; k < 3; ++k) max_scale = fmax(max_scale, exp((double)log_scale[3 * i + k]));
  const bool prune = (fmax(a1, a2) < p.prune_opacity_threshold) ||
                     (max_scale > p.prune_extent_factor * p.scene_extent);
  const double dense_limit = p.percent_dense * p.scene_extent;
  const bool hot = (avg >= p.densify_grad_threshold) && !prune;
  const bool clone = hot && (max_scale <= dense_limit);
  const bool split = hot && (max_scale > dense_limit);
  flags[i] = (prune ? kDPrune : 0) | (clone ? kDClone : 0) | (split ? kDSplit : 0);
  f_surv[i] = !prune && !split;
  f_clone[i] = clone;
  f_split[i] = split;
}

// Philox4x32-10 (Salmon et al., SC'11) and Box-Muller: a standard normal per
// (seed, draw, split rank, axis).
__device__ __forceinline__ uint4 philox(uint4 ctr, uint2 key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += 0x9E3779B9u;
    key.y += 0xBB67AE85u;
  }
  return ctr;
}

__device__ __forceinline__ double philox_normal(uint64_t seed, uint32_t draw, uint64_t rank,
                                                uint32_t axis) {
  const uint4 r = philox(make_uint4((uint32_t)rank, (uint32_t)(rank >> 32), draw, axis),
                         make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const double u1 = ((double)(((uint64_t)r.x << 21) ^ r.y) + 0.5) * 0x1p-53;  // (0, 1)
  const double u2 = ((double)(((uint64_t)r.z << 21) ^ r.w) + 0.5) * 0x1p-53;
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

template <typename T>
__global__ void __launch_bounds__(256) densify_emit_kernel(DensifyEmitArgs<T> a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const uint8_t f = a.flags[i];
  const int64_t srank = a.split_rank[i];
  const bool split_acc = (f & kDSplit) && srank < a.acc_split;
  const bool clone_acc = (f & kDClone) && a.clone_rank[i] < a.acc_clone;
  const int K3 = 3 * a.K;
  auto copy_row = [&](int64_t dst, int64_t src, bool with_moments) {
    for (int k = 0; k < 3; ++k) {
      a.out.mu[3 * dst + k] = a.in.mu[3 * src + k];
      a.out.ls[3 * dst + k] = a.in.ls[3 * src + k];
      a.out.nrm[3 * dst + k] = a.in.nrm[3 * src + k];
    }
    for (int k = 0; k < 4; ++k) a.out.rot[4 * dst + k] = a.in.rot[4 * src + k];
    for (int k = 0; k < K3; ++k) a.out.sh[K3 * dst + k] = a.in.sh[K3 * src + k];
    a.out.ra[dst] = a.in.ra[src];
    a.out.rb[dst] = a.in.rb[src];
    // Adam moments: the field order of hs_adam_state (mu, ls, rot, sh, nrm, ra, rb)
    const int64_t w[7] = {3, 3, 4, K3, 3, 1, 1};
    for (int fld = 0; fld < 7; ++fld) {
      if (!a.m_out[fld]) continue;
      T* mo = static_cast<T*>(a.m_out[fld]);
      T* vo = static_cast<T*>(a.v_out[fld]);
      const T* mi = static_cast<const T*>(a.m_in[fld]);
      const T* vi = static_cast<const T*>(a.v_in[fld]);
      for (int64_t k = 0; k < w[fld]; ++k) {
        mo[w[fld] * dst + k] = with_moments ? mi[w[fld] * src + k] : T(0);
        vo[w[fld] * dst + k] = with_moments ? vi[w[fld] * src + k] : T(0);
      }
    }
  };
  // survivors: not pruned and not an accepted split (over-budget splits stay, 284-286)
  if (!(f & kDPrune) && !split_acc) {
    const int64_t rejected_before = srank > a.acc_split ? srank - a.acc_split : 0;
    copy_row(a.surv_rank[i] + rejected_before, i, true);
  }
  if (clone_acc) {
    // copy shifted a small step down the accumulated position gradient (298-307)
    const int64_t dst = a.n_surv + a.clone_rank[i];
    copy_row(dst, i, false);
    const double g0 = a.mu_grad_sum[3 * i], g1 = a.mu_grad_sum[3 * i + 1],
                 g2 = a.mu_grad_sum[3 * i + 2];
    const double nrm = sqrt(g0 * g0 + g1 * g1 + g2 * g2);
    const double dn = nrm > 0 ? nrm : 1.0;
    const double dir[3] = {nrm > 0 ? g0 / dn : 0.0, nrm > 0 ? g1 / dn : 0.0,
                           nrm > 0 ? g2 / dn : 0.0};
    const double l0 = a.in.ls[3 * i], l1 = a.in.ls[3 * i + 1], l2 = a.in.ls[3 * i + 2];
    const double step = 0.1 * exp((l0 + l1 + l2) / 3.0);
    for (int k = 0; k < 3; ++k)
      a.out.mu[3 * dst + k] = (T)((double)a.in.mu[3 * i + k] - dir[k] * step);
  }
  if (split_acc) {
    // two children drawn from the parent Gaussian (308-320)
    double q[4], R[9];
    for (int k = 0; k < 4; ++k) q[k] = a.in.rot[4 * i + k];
    quat_to_rot_ref(q, R);
    double s[3];
    for (int k = 0; k < 3; ++k) s[k] = exp((double)a.in.ls[3 * i + k]);
    for (int d = 0; d < 2; ++d) {
      const int64_t dst = a.n_surv + a.acc_clone + d * a.acc_split + srank;
      copy_row(dst, i, false);
      double scaled[3], world[3];
      for (int k = 0; k < 3; ++k) {
        const double o = a.offsets ? a.offsets[(d * a.acc_split + srank) * 3 + k]
                                   : philox_normal(a.seed, (uint32_t)d, (uint64_t)srank, (uint32_t)k);
        scaled[k] = o * s[k];
      }
      matvec_einsum(R, scaled, world);
      for (int k = 0; k < 3; ++k) {
        a.out.mu[3 * dst + k] = (T)((double)a.in.mu[3 * i + k] + world[k]);
        a.out.ls[3 * dst + k] = (T)((double)a.in.ls[3 * i + k] - a.log_split_scale);
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) reset_opacity_kernel(T* ra, T* rb, void* ma, void* va,
                                                            void* mb, void* vb, int64_t n,
                                                            double cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // np.minimum(raw, cap): NaN propagates
  const double a = ra[i], b = rb[i];
  ra[i] = (T)(a != a ? a : fmin(a, cap));
  rb[i] = (T)(b != b ? b : fmin(b, cap));
  if (ma) {
    static_cast<T*>(ma)[i] = T(0);
    static_cast<T*>(va)[i] = T(0);
  }
  if (mb) {
    static_cast<T*>(mb)[i] = T(0);
    static_cast<T*>(vb)[i] = T(0);
  }
}

// ---------------------------------------------------------------------------
static unsigned blocks(int64_t n) { return (unsigned)((n + 255) / 256); }

cudaError_t launch_densify_stats(const DensifyStatsArgs& st, const void* pgn, const void* d_mu,
                                 const int32_t* touch, int64_t n, int dtype, cudaStream_t s) {
  if (dtype == 0)
    densify_stats_kernel<float><<<blocks(n), 256, 0, s>>>(st, (const float*)pgn,
                                                          (const float*)d_mu, touch, n);
  else
    densify_stats_kernel<double><<<blocks(n), 256, 0, s>>>(st, (const double*)pgn,
                                                           (const double*)d_mu, touch, n);
  note_launch();
  return cudaGetLastError();
}

size_t densify_scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                (int)(n + 1));
  return bytes;
}

cudaError_t launch_densify_classify(const DensifyStatsArgs& st, const void* log_scale,
                                    const void* ra, const void* rb, int64_t n, int dtype,
                                    const DensifyParams& p, DensifyBufs& b, cudaStream_t s) {
  if (dtype == 0)
    densify_classify_kernel<float><<<blocks(n + 1), 256, 0, s>>>(
        st, (const float*)log_scale, (const float*)ra, (const float*)rb, n, p, b.flags, b.f_surv,
        b.f_clone, b.f_split);
  else
    densify_classify_kernel<double><<<blocks(n + 1), 256, 0, s>>>(
        st, (const double*)log_scale, (const double*)ra, (const double*)rb, n, p, b.flags,
        b.f_surv, b.f_clone, b.f_split);
  note_launch();
  cudaError_t e = cudaGetLastError();
  int32_t* in[3] = {b.f_surv, b.f_clone, b.f_split};
  int32_t* out[3] = {b.surv_rank, b.clone_rank, b.split_rank};
  for (int k = 0; k < 3 && e == cudaSuccess; ++k) {
    size_t bytes = b.temp_bytes;
    e = cub::DeviceScan::ExclusiveSum(b.temp, bytes, in[k], out[k], (int)(n + 1), s);
    note_launch();
  }
  return e;
}

template <typename T>
cudaError_t launch_densify_emit_t(const DensifyEmitArgs<T>& a, cudaStream_t s) {
  densify_emit_kernel<T><<<blocks(a.n), 256, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}
template cudaError_t launch_densify_emit_t<float>(const DensifyEmitArgs<float>&, cudaStream_t);
template cudaError_t launch_densify_emit_t<double>(const DensifyEmitArgs<double>&, cudaStream_t);

cudaError_t launch_reset_opacity(void* ra, void* rb, void* ma, void* va, void* mb, void* vb,
                                 int64_t n, double cap, int dtype, cudaStream_t s) {
  if (dtype == 0)
    reset_opacity_kernel<float><<<blocks(n), 256, 0, s>>>((float*)ra, (float*)rb, ma, va, mb,
                                                          vb, n, cap);
  else
    reset_opacity_kernel<double><<<blocks(n), 256, 0, s>>>((double*)ra, (double*)rb, ma, va, mb,
                                                           vb, n, cap);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hs

namespace hs {
// opacity_disparity (trainer.py:353-358): mean |sigmoid(a) - sigmoid(b)|, one CUB
// reduction over a transform iterator (deterministic for a given size).
template <typename T>
struct AlphaGap {
  const T* ra;
  const T* rb;
  __device__ double operator()(int64_t i) const {
    return fabs(sigmoid_ref((double)ra[i]) - sigmoid_ref((double)rb[i]));
  }
};

template <typename T>
static cudaError_t disparity_t(const void* ra, const void* rb, int64_t n, double* out, void* temp,
                               size_t* temp_bytes, cudaStream_t s) {
  auto it = cub::TransformInputIterator<double, AlphaGap<T>, cub::CountingInputIterator<int64_t>>(
      cub::CountingInputIterator<int64_t>(0), AlphaGap<T>{(const T*)ra, (const T*)rb});
  return cub::DeviceReduce::Sum(temp, *temp_bytes, it, out, (int)n, s);
}

cudaError_t opacity_disparity_sum(const void* ra, const void* rb, int64_t n, int dtype,
                                  double* out, void* temp, size_t* temp_bytes, cudaStream_t s) {
  cudaError_t e = dtype == 0 ? disparity_t<float>(ra, rb, n, out, temp, temp_bytes, s)
                             : disparity_t<double>(ra, rb, n, out, temp, temp_bytes, s);
  if (temp) note_launch();
  return e;
}
}  // namespace hs
