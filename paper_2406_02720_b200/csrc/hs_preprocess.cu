// hs_preprocess.cu -- K1 (per-Gaussian preprocess) and K7 (per-Gaussian
// geometry backward), one thread per primitive, FP64 geometry.
//
// K1 is compiled with -fmad=false: every floating-point
// operation below rounds exactly where the reference's numpy expression rounds,
// and fma() appears only where numpy's own kernels fuse (the (N,3)@(3,3) and
// batched 3x3 matmuls go through OpenBLAS FMA chains; the einsum reductions do
// not).  With the same inputs this reproduces prepare()'s FP64 intermediates
// bit for bit except where libm/numpy `exp` differ by an ulp, which is what makes
// `valid`, `tile_rect`, `mode` and the sort order exact.
//
// K7 needs no such exactness (its outputs are gradients under a 1e-3 contract),
// so hs_geometry_bwd.cu compiles this same file with HS_GEOMETRY_BWD_TU defined
// and FMA contraction on; it replays K1's discrete decisions from the record
// flags (forward_state<..., kReplay>).
#include <cmath>
#include <cstdint>
#include <type_traits>

#include <cuda_fp16.h>

#include "hs_common.cuh"
#include "hs_internal.h"
#include "hs_numpy_order.cuh"

namespace hs {

// numpy float64 -> int64 cast of ceil/floor results (x86 cvttsd2si: values out
// of range and NaN become INT64_MIN, which the on-screen test then rejects).
__device__ __forceinline__ long long to_i64_numpy(double x) {
  if (!(x > -9.2233720368547758e18 && x < 9.2233720368547758e18)) return LLONG_MIN;
  return (long long)x;
}

template <typename T>
__device__ __forceinline__ double ld(const T* p, int64_t i) { return (double)p[i]; }

// 1 / (1 + e^-x) in FP32 (MUFU ex2 + rcp), saturating cleanly at both ends
__device__ __forceinline__ double sigmoid_f32(float x) {
  return (double)__frcp_rn(1.0f + exp2f(-1.4426950408889634f * x));
}

// Forward state of one primitive for one view: the subset of FrameGeometry
// (rasterizer.py:108-147) that K1 emits and K7 needs.  Recomputed by K7 rather
// than stored (about 1 KB per splat in the reference).
struct FwdState {
  double t[3];
  double qu[4], qnorm;
  double R[9], s[3], cov[9];
  double ccam[9], J[9], cray[9];
  double mux, muy;
  double a, b, c, det, radius;
  long long px0, px1, py0, py1;  // clipped pixel rect
  bool in_front, visible;
  double L[9];
  bool bad;
  double v00, v10, v11;
  double nnorm, nu[3];
  double hw[3], hc[3], hr[3];
  double y[3], ynorm;
  double nray[3];
  double a1, a2, c1, c2, za, zb;
  int mode;
  double vdir[3], vdist;
  double basis[16];
  double rgbu[3];
};

// eval_sh_basis, sh.py:32-61 (left-to-right evaluation of each product)
__device__ __forceinline__ void sh_basis(const double d[3], int deg, double* out) {
  const double SH_C0 = 0.28209479177387814, SH_C1 = 0.4886025119029199;
  const double x = d[0], y = d[1], z = d[2];
  out[0] = SH_C0;
  if (deg >= 1) {
    out[1] = -SH_C1 * y;
    out[2] = SH_C1 * z;
    out[3] = -SH_C1 * x;
  }
  if (deg >= 2) {
    const double xx = x * x, yy = y * y, zz = z * z;
    out[4] = 1.0925484305920792 * x * y;
    out[5] = -1.0925484305920792 * y * z;
    out[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
    out[7] = -1.0925484305920792 * x * z;
    out[8] = 0.5462742152960396 * (xx - yy);
    if (deg >= 3) {
      out[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
      out[10] = 2.890611442640554 * x * y * z;
      out[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
      out[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
      out[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
      out[14] = 1.445305721320277 * z * (xx - yy);
      out[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
    }
  }
}

// One primitive's R staged values from its dense shared-memory row (16-B loads for
// float rows: the row start is 16-B aligned when 3K is a multiple of 4).
template <int R, typename T, bool VEC = std::is_same<T, float>::value && R % 4 == 0>
__device__ __forceinline__ void load_row(const T* p, float (&out)[R]) {
  if constexpr (VEC) {
    const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
    for (int j = 0; j < R / 4; ++j) {
      const float4 v = q[j];
      out[4 * j] = v.x; out[4 * j + 1] = v.y; out[4 * j + 2] = v.z; out[4 * j + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) out[j] = (float)p[j];
  }
}

// K7's SH backward in FP32 (eval_sh_basis / eval_sh_basis_grad, sh.py:32-98):
// sh holds the primitive's (K,3) coefficients (a dense shared-memory row) and is
// overwritten with d_sh = basis (x) dpre; d_dir = sum_k (sum_ch sh[k,ch] dpre[ch])
// d basis_k / d dir.
// a + b rounded on its own (never contracted into an FMA with the product that
// made b): the multi-view K7's sums match K7's per-view accumulation bit for bit
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <int DEG, bool ACC = false, typename E>
__device__ __forceinline__ void sh_bwd_f32(const float d[3], const float dpre[3], E* sh,
                                           float d_dir[3], E* out = nullptr) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  const float x = d[0], y = d[1], z = d[2];
  float b[K];
  b[0] = 0.28209479177387814f;
  if (DEG >= 1) {
    b[1] = -0.4886025119029199f * y;
    b[2] = 0.4886025119029199f * z;
    b[3] = -0.4886025119029199f * x;
  }
  const float xx = x * x, yy = y * y, zz = z * z;
  if (DEG >= 2) {
    b[4] = 1.0925484305920792f * x * y;
    b[5] = -1.0925484305920792f * y * z;
    b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    b[7] = -1.0925484305920792f * x * z;
    b[8] = 0.5462742152960396f * (xx - yy);
  }
  if (DEG >= 3) {
    b[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    b[10] = 2.890611442640554f * x * y * z;
    b[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    b[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    b[14] = 1.445305721320277f * z * (xx - yy);
    b[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
  }
  float cf[3 * K];
  load_row<3 * K>(sh, cf);
  // ACC: the coefficients stay, d_sh adds into `out` (the multi-view K7)
  E* dst = ACC ? out : sh;
  float db[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    db[k] = cf[3 * k] * dpre[0] + cf[3 * k + 1] * dpre[1] + cf[3 * k + 2] * dpre[2];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      if constexpr (ACC) dst[3 * k + ch] = add_rn(dst[3 * k + ch], E(__fmul_rn(b[k], dpre[ch])));
      else dst[3 * k + ch] = E(b[k] * dpre[ch]);
    }
  }
  float gx = 0.f, gy = 0.f, gz = 0.f;
  if (DEG >= 1) {
    const float c1 = 0.4886025119029199f;
    gy -= c1 * db[1];
    gz += c1 * db[2];
    gx -= c1 * db[3];
  }
  if (DEG >= 2) {
    const float c0 = 1.0925484305920792f, c2 = 0.31539156525252005f, c4 = 0.5462742152960396f;
    gx += c0 * y * db[4];
    gy += c0 * x * db[4];
    gy -= c0 * z * db[5];
    gz -= c0 * y * db[5];
    gx += c2 * (-2.0f * x) * db[6];
    gy += c2 * (-2.0f * y) * db[6];
    gz += c2 * (4.0f * z) * db[6];
    gx -= c0 * z * db[7];
    gz -= c0 * x * db[7];
    gx += c4 * (2.0f * x) * db[8];
    gy += c4 * (-2.0f * y) * db[8];
  }
  if (DEG >= 3) {
    const float e0 = -0.5900435899266435f, e1 = 2.890611442640554f, e2 = -0.4570457994644658f,
                e3 = 0.3731763325901154f, e5 = 1.445305721320277f;
    gx += e0 * (6.0f * x * y) * db[9];
    gy += e0 * (3.0f * xx - 3.0f * yy) * db[9];
    gx += e1 * (y * z) * db[10];
    gy += e1 * (x * z) * db[10];
    gz += e1 * (x * y) * db[10];
    gx += e2 * (-2.0f * x * y) * db[11];
    gy += e2 * (4.0f * zz - xx - 3.0f * yy) * db[11];
    gz += e2 * (8.0f * y * z) * db[11];
    gx += e3 * (-6.0f * x * z) * db[12];
    gy += e3 * (-6.0f * y * z) * db[12];
    gz += e3 * (6.0f * zz - 3.0f * xx - 3.0f * yy) * db[12];
    gx += e2 * (4.0f * zz - 3.0f * xx - yy) * db[13];
    gy += e2 * (-2.0f * x * y) * db[13];
    gz += e2 * (8.0f * x * z) * db[13];
    gx += e5 * (2.0f * x * z) * db[14];
    gy += e5 * (-2.0f * y * z) * db[14];
    gz += e5 * (xx - yy) * db[14];
    gx += e0 * (3.0f * xx - 3.0f * yy) * db[15];
    gy += e0 * (-6.0f * x * y) * db[15];
  }
  d_dir[0] = gx;
  d_dir[1] = gy;
  d_dir[2] = gz;
}

// einsum("ab,nbc,dc->nad") / ("nab,nbc,ndc->nad"): sequential over b then c,
// each term ((A[a,b] * C[b,c]) * A[d,c]), accumulated from 0.
__device__ __forceinline__ void sandwich(const double A[9], const double C[9], double out[9]) {
  for (int a = 0; a < 3; ++a)
    for (int d = 0; d < 3; ++d) {
      double s = 0.0;
      for (int b = 0; b < 3; ++b)
        for (int c = 0; c < 3; ++c) s += A[3 * a + b] * C[3 * b + c] * A[3 * d + c];
      out[3 * a + d] = s;
    }
}

// K7's replay (no numpy-exact rounding needed): the same product as two 3x3
// multiplications, out = (A C) A^T, with C symmetric (6 unique outputs).
__device__ __forceinline__ void sandwich_fast(const double A[9], const double C[9],
                                              double out[9]) {
  double AC[9];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      AC[3 * a + c] = A[3 * a] * C[c] + A[3 * a + 1] * C[3 + c] + A[3 * a + 2] * C[6 + c];
  for (int a = 0; a < 3; ++a)
    for (int d = a; d < 3; ++d) {
      const double v = AC[3 * a] * A[3 * d] + AC[3 * a + 1] * A[3 * d + 1] +
                       AC[3 * a + 2] * A[3 * d + 2];
      out[3 * a + d] = v;
      out[3 * d + a] = v;
    }
}

// ---------------------------------------------------------------------------
// Shared-memory staging of one CTA's primitives.  The scene is array-of-structs
// per field ((N,3), (N,K,3), ...); a thread reading its own primitive would issue
// ~60 scalar loads with 12..192-byte strides.  Instead the CTA copies its NT
// primitives field by field with consecutive threads on consecutive elements
// (fully coalesced), and every thread reads its own from shared memory.  SH rows
// are padded to an odd stride (3K+1) so the per-thread reads are conflict-free.
// K7 reuses the same slots to stage its gradient outputs for coalesced stores.
template <typename T, int K, int NT>
struct Staged {
  // float scenes with whole 16-B SH rows (deg 1, 3) stage them dense (the global
  // layout, 16-B cp.async of one contiguous block) and read them back as 16-B
  // vectors; otherwise rows are padded to an odd stride so per-thread scalar reads
  // are conflict-free
  static constexpr bool DENSE = std::is_same<T, float>::value && (3 * K) % 4 == 0;
  static constexpr int SHS = DENSE ? 3 * K : 3 * K + 1;
  alignas(16) T mu[NT * 3];
  alignas(16) T ls[NT * 3];
  alignas(16) T rot[NT * 4];
  alignas(16) T nrm[NT * 3];
  alignas(16) T ra[NT];
  alignas(16) T rb[NT];
  alignas(16) T sh[NT * SHS];
  uint64_t bar;  // the bulk-copy path's transaction barrier
};

// One element global -> shared without a register round trip (LDGSTS), so a
// thread's whole share of the staging is in flight at once.
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(d), "l"(gmem), "n"(sizeof(T)));
}

// Bulk-copy staging (cp.async.bulk, the TMA engine's 1-D form): with dense SH rows
// every field of a CTA's primitives is ONE contiguous block in global memory and in
// shared memory, so one thread issues seven bulk copies that complete on a
// transaction-count mbarrier, instead of every thread issuing ~30 LDGSTS.  Needs
// 16-B aligned sources and block sizes that are multiples of 16 B (a full CTA of a
// torch-allocated scene); other CTAs take the LDGSTS path below.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
template <typename T>
__device__ __forceinline__ bool bulk_ok(const T* src, int64_t elems) {
  return ((uintptr_t)src & 15) == 0 && ((elems * (int64_t)sizeof(T)) & 15) == 0;
}

__device__ __forceinline__ void bulk_wait(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)) : "memory");
}

// Returns whether the CTA staged with bulk copies (uniform over the CTA).  With
// wait = false the caller completes the staging with stage_wait (then syncs).
template <typename T, int K, int NT>
__device__ __forceinline__ bool stage_in(Staged<T, K, NT>& s, const SceneArgs<T>& sc,
                                         int64_t base, int cnt, bool wait = true) {
  const int tid = threadIdx.x;
  if constexpr (Staged<T, K, NT>::DENSE) {
    constexpr int R = 3 * K;
    const bool bulk = bulk_ok(sc.mu + base * 3, cnt * 3) && bulk_ok(sc.ls + base * 3, cnt * 3) &&
                      bulk_ok(sc.nrm + base * 3, cnt * 3) && bulk_ok(sc.rot + base * 4, cnt * 4) &&
                      bulk_ok(sc.ra + base, cnt) && bulk_ok(sc.rb + base, cnt) &&
                      bulk_ok(sc.sh + base * R, (int64_t)cnt * R);  // uniform over the CTA
    if (bulk) {
      if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&s.bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        const unsigned b3 = cnt * 3 * sizeof(T), b1 = cnt * sizeof(T);
        const unsigned total = 3 * b3 + 4 * b1 + 2 * b1 + cnt * R * sizeof(T);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                     ::"r"(smem_u32(&s.bar)), "r"(total) : "memory");
        bulk_g2s(s.mu, sc.mu + base * 3, b3, &s.bar);
        bulk_g2s(s.ls, sc.ls + base * 3, b3, &s.bar);
        bulk_g2s(s.nrm, sc.nrm + base * 3, b3, &s.bar);
        bulk_g2s(s.rot, sc.rot + base * 4, 4 * b1, &s.bar);
        bulk_g2s(s.ra, sc.ra + base, b1, &s.bar);
        bulk_g2s(s.rb, sc.rb + base, b1, &s.bar);
        bulk_g2s(s.sh, sc.sh + base * R, cnt * R * sizeof(T), &s.bar);
      }
      // (the barrier's init is visible to the waiting threads after this sync)
      __syncthreads();
      if (wait) {
        bulk_wait(&s.bar);
        __syncthreads();
      }
      return true;
    }
  }
  for (int e = tid; e < cnt * 3; e += NT) {
    cp_async_elem(&s.mu[e], &sc.mu[base * 3 + e]);
    cp_async_elem(&s.ls[e], &sc.ls[base * 3 + e]);
    cp_async_elem(&s.nrm[e], &sc.nrm[base * 3 + e]);
  }
  for (int e = tid; e < cnt * 4; e += NT) cp_async_elem(&s.rot[e], &sc.rot[base * 4 + e]);
  for (int e = tid; e < cnt; e += NT) {
    cp_async_elem(&s.ra[e], &sc.ra[base + e]);
    cp_async_elem(&s.rb[e], &sc.rb[base + e]);
  }
  if constexpr (!Staged<T, K, NT>::DENSE) {
    constexpr int R = 3 * K;
    for (int e = tid; e < cnt * R; e += NT) {
      const int t = e / R, c = e - t * R;
      cp_async_elem(&s.sh[t * Staged<T, K, NT>::SHS + c], &sc.sh[base * R + e]);
    }
  } else {
    constexpr int R = 3 * K, kV = 16 / sizeof(T);
    const T* src = sc.sh + base * R;
    const int n = cnt * R;
    const int nv = ((uintptr_t)src & 15) ? 0 : n / kV;
    for (int v = tid; v < nv; v += NT) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(&s.sh[v * kV]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + v * kV));
    }
    for (int e = nv * kV + tid; e < n; e += NT) cp_async_elem(&s.sh[e], &src[e]);
  }
  asm volatile("cp.async.commit_group;\n" ::);
  if (wait) {
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
  }
  return false;
}

// Completes a stage_in(wait = false) of this thread's share (the caller syncs).
template <typename T, int K, int NT>
__device__ __forceinline__ void stage_wait(Staged<T, K, NT>& s, bool bulk) {
  if (bulk)
    bulk_wait(&s.bar);
  else
    asm volatile("cp.async.wait_all;\n" ::);
}

// One thread's view of its staged primitive (the inputs of forward_state).
template <typename T, int K, int NT>
struct StagedView {
  const Staged<T, K, NT>& s;
  int t;
  __device__ __forceinline__ double mu(int k) const { return (double)s.mu[3 * t + k]; }
  __device__ __forceinline__ double ls(int k) const { return (double)s.ls[3 * t + k]; }
  __device__ __forceinline__ double rot(int k) const { return (double)s.rot[4 * t + k]; }
  __device__ __forceinline__ double nrm(int k) const { return (double)s.nrm[3 * t + k]; }
  __device__ __forceinline__ double ra() const { return (double)s.ra[t]; }
  __device__ __forceinline__ double rb() const { return (double)s.rb[t]; }
  __device__ __forceinline__ double sh(int k, int ch) const {
    return (double)s.sh[t * Staged<T, K, NT>::SHS + 3 * k + ch];
  }
  // f(flat index 3k + ch, value) for every coefficient in index order: 16-B reads
  // of a dense row (a per-element read of a dense row would conflict 16 ways)
  template <typename F>
  __device__ __forceinline__ void for_each_sh(F&& f) const {
    const T* row = s.sh + t * Staged<T, K, NT>::SHS;
    if constexpr (Staged<T, K, NT>::DENSE) {
      const float4* q = reinterpret_cast<const float4*>(row);
#pragma unroll
      for (int j = 0; j < 3 * K / 4; ++j) {
        const float4 v = q[j];
        f(4 * j, (double)v.x);
        f(4 * j + 1, (double)v.y);
        f(4 * j + 2, (double)v.z);
        f(4 * j + 3, (double)v.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 3 * K; ++j) f(j, (double)row[j]);
    }
  }
};

// kReplay (K7): the primitive is known visible and K1's discrete decisions --
// the identity-whitening fallback and the blend mode -- are taken from its
// record flags, so a K7 build with different rounding cannot branch otherwise.
// The camera-independent part of the forward state (rasterizer.py:174-179, 241-244,
// 256-258): quaternion, rotation, scales, covariance, unit normal, cov . n, the two
// opacities.  A batch of views computes it once per primitive
// (preprocess_fwd_views_kernel); the arithmetic is the same either way.
template <bool kReplay = false, typename Src>
__device__ __forceinline__ void indep_state(const Src& src, FwdState& st) {
  // covariance build (rasterizer.py:174-179)
  double q[4];
  for (int k = 0; k < 4; ++k) q[k] = src.rot(k);
  {
    double ss = 0.0;
    for (int k = 0; k < 4; ++k) ss += q[k] * q[k];
    st.qnorm = sqrt(ss);
  }
  if constexpr (kReplay) {
    // K7: reciprocals instead of divisions; the rotation straight from the unit
    // quaternion (quat_to_rot's second normalisation is a no-op up to rounding)
    const double rq = 1.0 / st.qnorm;
    for (int k = 0; k < 4; ++k) st.qu[k] = q[k] * rq;
    const double w = st.qu[0], x = st.qu[1], y = st.qu[2], z = st.qu[3];
    st.R[0] = 1 - 2 * (y * y + z * z);
    st.R[1] = 2 * (x * y - w * z);
    st.R[2] = 2 * (x * z + w * y);
    st.R[3] = 2 * (x * y + w * z);
    st.R[4] = 1 - 2 * (x * x + z * z);
    st.R[5] = 2 * (y * z - w * x);
    st.R[6] = 2 * (x * z - w * y);
    st.R[7] = 2 * (y * z + w * x);
    st.R[8] = 1 - 2 * (x * x + y * y);
  } else {
    for (int k = 0; k < 4; ++k) st.qu[k] = q[k] / st.qnorm;
    quat_to_rot_ref(st.qu, st.R);
  }
  for (int k = 0; k < 3; ++k) st.s[k] = exp(src.ls(k));
  double M[9];
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) M[3 * r + k] = st.R[3 * r + k] * st.s[k];
  for (int a = 0; a < 3; ++a)
    for (int d = 0; d < 3; ++d)
      st.cov[3 * a + d] = fma(M[3 * a + 2], M[3 * d + 2],
                              fma(M[3 * a + 1], M[3 * d + 1], M[3 * a] * M[3 * d]));
  double nrm[3];
  for (int k = 0; k < 3; ++k) nrm[k] = src.nrm(k);
  st.nnorm = sqrt(nrm[0] * nrm[0] + nrm[1] * nrm[1] + nrm[2] * nrm[2]);
  if constexpr (kReplay) {
    const double rn = 1.0 / st.nnorm;
    for (int k = 0; k < 3; ++k) st.nu[k] = nrm[k] * rn;
  } else {
    for (int k = 0; k < 3; ++k) st.nu[k] = nrm[k] / st.nnorm;
  }
  matvec_einsum(st.cov, st.nu, st.hw);
  if constexpr (kReplay) {
    // K7 only needs alpha (1 - alpha) for the logits' gradients: FP32 is ample
    st.a1 = sigmoid_f32((float)src.ra());
    st.a2 = sigmoid_f32((float)src.rb());
  } else {
    st.a1 = sigmoid_ref(src.ra());
    st.a2 = sigmoid_ref(src.rb());
  }
}

// The per-view part: camera-space mean, projection, conic, radius, rect, whitening,
// ray-space normal, mode, erf coefficients, SH colour (rasterizer.py:170, 183-285).
// Needs indep_state's fields.
template <int DEG, bool kReplay = false, typename Src>
__device__ __forceinline__ void view_state(const Src& src, const CamArgs& cam, int kernel,
                                           FwdState& st, uint32_t flags = 0) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  // t_all = mu @ rot.T + translation (rasterizer.py:170)
  {
    const double mv[3] = {src.mu(0), src.mu(1), src.mu(2)};
    double tt[3];
    matvec_blas(cam.R, mv, tt);
    for (int a = 0; a < 3; ++a) st.t[a] = tt[a] + cam.tr[a];
  }
  st.in_front = st.t[2] > cam.near_clip;
  st.visible = false;
  if (!kReplay && !st.in_front) return;
  // cov_cam, Jacobian, ray covariance (rasterizer.py:183-185; geometry.py:189-207)
  if constexpr (kReplay) sandwich_fast(cam.R, st.cov, st.ccam);
  else sandwich(cam.R, st.cov, st.ccam);
  const double tx = st.t[0], ty = st.t[1], tz = st.t[2];
  const double invz = 1.0 / tz;
  const double ell = sqrt(tx * tx + ty * ty + tz * tz);
  st.J[0] = cam.fx * invz; st.J[1] = 0.0; st.J[2] = -cam.fx * tx * invz * invz;
  st.J[3] = 0.0; st.J[4] = cam.fy * invz; st.J[5] = -cam.fy * ty * invz * invz;
  if constexpr (kReplay) {
    const double rl = 1.0 / ell;
    st.J[6] = tx * rl; st.J[7] = ty * rl; st.J[8] = tz * rl;
    sandwich_fast(st.J, st.ccam, st.cray);
  } else {
    st.J[6] = tx / ell; st.J[7] = ty / ell; st.J[8] = tz / ell;
    sandwich(st.J, st.ccam, st.cray);
  }
  st.mux = cam.fx * tx * invz + cam.cx;  // rasterizer.py:188-191
  st.muy = cam.fy * ty * invz + cam.cy;
  // dilated conic, radius, pixel rect, on-screen test (rasterizer.py:194-210)
  st.a = st.cray[0] + kLowpass;
  st.b = st.cray[1];
  st.c = st.cray[4] + kLowpass;
  st.det = st.a * st.c - st.b * st.b;
  if (kReplay) {
    st.visible = true;  // K7 needs neither the radius nor the rect
  } else {
  const double mid = 0.5 * (st.a + st.c);
  const double lam = mid + sqrt(fmax(mid * mid - st.det, 0.0));
  st.radius = kRadiusSigmas * sqrt(fmax(lam, 0.0));
  long long x0 = to_i64_numpy(ceil(st.mux - st.radius - 0.5));
  long long x1 = to_i64_numpy(floor(st.mux + st.radius - 0.5));
  long long y0 = to_i64_numpy(ceil(st.muy - st.radius - 0.5));
  long long y1 = to_i64_numpy(floor(st.muy + st.radius - 0.5));
  const long long W1 = cam.width - 1, H1 = cam.height - 1;
  st.visible = ((x1 >= 0) && (x0 <= W1) && (y1 >= 0) && (y0 <= H1) && (x1 >= x0) &&
                           (y1 >= y0) && (st.det > 0.0));
  if (!st.visible) return;
  st.px0 = x0 < 0 ? 0 : (x0 > W1 ? W1 : x0);  // np.clip, rasterizer.py:225-228
  st.px1 = x1 < 0 ? 0 : (x1 > W1 ? W1 : x1);
  st.py0 = y0 < 0 ? 0 : (y0 > H1 ? H1 : y0);
  st.py1 = y1 < 0 ? 0 : (y1 > H1 ? H1 : y1);
  }
  // whitening: chol3_batch on the undilated ray covariance (geometry.py:126-160)
  {
    const double* A = st.cray;
    const double d0 = A[0];
    const double l00 = sqrt(fmax(d0, 0.0));
    const double l10 = A[3] / l00;
    const double l20 = A[6] / l00;
    const double d1 = A[4] - l10 * l10;
    const double l11 = sqrt(fmax(d1, 0.0));
    const double l21 = (A[7] - l20 * l10) / l11;
    const double d2 = A[8] - l20 * l20 - l21 * l21;
    const double l22 = sqrt(fmax(d2, 0.0));
    const double dmin = fmin(fmin(l00, l11), l22), dmax = fmax(fmax(l00, l11), l22);
    const bool finite = isfinite(l00) && isfinite(l11) && isfinite(l22);
    // numpy min/max propagate NaN; any NaN diag already fails `finite`.
    st.bad = kReplay ? (flags & kFlagBad) != 0
                     : (d0 <= 0.0) || (d1 <= 0.0) || (d2 <= 0.0) || !finite ||
                           (dmin * kCondLimit < dmax);
    for (int k = 0; k < 9; ++k) st.L[k] = 0.0;
    if (st.bad) {
      st.L[0] = st.L[4] = st.L[8] = 1.0;
    } else {
      st.L[0] = l00; st.L[3] = l10; st.L[4] = l11; st.L[6] = l20; st.L[7] = l21; st.L[8] = l22;
    }
  }
  st.v00 = 1.0 / st.L[0];  // rasterizer.py:236-238
  st.v11 = 1.0 / st.L[4];
  st.v10 = -st.L[3] * st.v00 * st.v11;
  // ray-space splitting normal (rasterizer.py:241-254); hw = cov nu from indep_state
  matvec_blas(cam.R, st.hw, st.hc);
  matvec_einsum(st.J, st.hc, st.hr);
  st.y[0] = st.hr[0] * st.v00;
  st.y[1] = (st.hr[1] - st.L[3] * st.y[0]) / st.L[4];
  st.y[2] = (st.hr[2] - st.L[6] * st.y[0] - st.L[7] * st.y[1]) / st.L[8];
  const double yn = sqrt(st.y[0] * st.y[0] + st.y[1] * st.y[1] + st.y[2] * st.y[2]);
  if (!kReplay) st.bad = st.bad || (yn < 1e-12) || !isfinite(yn);
  st.ynorm = st.bad ? 1.0 : yn;
  if (st.bad) {
    st.nray[0] = 0.0; st.nray[1] = 0.0; st.nray[2] = 1.0;
  } else if constexpr (kReplay) {
    const double ry = 1.0 / st.ynorm;
    for (int k = 0; k < 3; ++k) st.nray[k] = st.y[k] * ry;
  } else {
    for (int k = 0; k < 3; ++k) st.nray[k] = st.y[k] / st.ynorm;
  }
  // blend mode, erf coefficients (rasterizer.py:256-277; the opacities from indep_state)
  st.c1 = 0.5 * (st.a1 + st.a2);
  if (kernel == 1) {
    st.c2 = 0.0;
    st.mode = kModePlain;
  } else {
    st.c2 = 0.5 * (st.a1 - st.a2);
    st.mode = kReplay ? (int)(flags & 3u)
                      : st.bad ? kModePlain
                               : (fabs(st.nray[2]) < kNormalEps ? kModeSign : kModeErf);
  }
  st.za = 0.0;
  st.zb = 0.0;
  if (st.mode == kModeErf) {
    const double inv = 1.0 / (1.4142135623730951 * fabs(st.nray[2]));
    st.za = inv * (st.nray[0] * st.v00 + st.nray[1] * st.v10);
    st.zb = inv * (st.nray[1] * st.v11);
  } else if (st.mode == kModeSign) {
    st.za = st.nray[0] * st.v00 + st.nray[1] * st.v10;
    st.zb = st.nray[1] * st.v11;
  }
  // view-dependent colour (rasterizer.py:280-285)
  double vv[3] = {src.mu(0) - cam.center[0], src.mu(1) - cam.center[1],
                  src.mu(2) - cam.center[2]};
  st.vdist = sqrt(vv[0] * vv[0] + vv[1] * vv[1] + vv[2] * vv[2]);
  if constexpr (kReplay) {
    const double rv = 1.0 / st.vdist;
    for (int k = 0; k < 3; ++k) st.vdir[k] = vv[k] * rv;
  } else {
    for (int k = 0; k < 3; ++k) st.vdir[k] = vv[k] / st.vdist;
  }
  // K7 takes the colour clamp from the record (merge_rows_kernel) and evaluates
  // the basis in FP32 (sh_bwd_f32)
  if (!kReplay) {
    sh_basis(st.vdir, DEG, st.basis);
    // each channel sums basis[k] * sh[k, ch] over k in order (the coefficients are
    // read in index order; the three sums interleave but do not mix)
    double acc[3] = {0.0, 0.0, 0.0};
    src.for_each_sh([&](int j, double v) { acc[j % 3] += st.basis[j / 3] * v; });
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) st.rgbu[ch] = acc[ch] + 0.5;
  }
}

template <int DEG, bool kReplay = false, typename Src>
__device__ __forceinline__ void forward_state(const Src& src, const CamArgs& cam, int kernel,
                                              FwdState& st, uint32_t flags = 0) {
  indep_state<kReplay>(src, st);
  view_state<DEG, kReplay>(src, cam, kernel, st, flags);
}

#ifndef HS_GEOMETRY_BWD_TU
// K1's outputs for one primitive of one view: the 64-B record, side record, tile
// rect, pair count, depth-rank sort key and value, radius; culled: count 0, key ~0.
__device__ __forceinline__ void write_fwd_outputs(const FwdState& st, int64_t i,
                                                  const FwdOut& o) {
  float4* __restrict__ rec = o.rec;
  SteepRec* __restrict__ side = o.side;
  int4* __restrict__ rect = o.rect;
  int32_t* __restrict__ count = o.count;
  uint64_t* __restrict__ dkey = o.dkey;
  uint32_t* __restrict__ dval = o.dval;
  int32_t* __restrict__ radii = o.radii;
  uint32_t* __restrict__ depth_range = o.range;
  if (!st.visible) {
    dval[i] = (uint32_t)i;
    count[i] = 0;
    dkey[i] = ~0ull;
    if (radii) radii[i] = 0;
    return;
  }
  const int tx0 = (int)(st.px0 / kTile), tx1 = (int)(st.px1 / kTile);
  const int ty0 = (int)(st.py0 / kTile), ty1 = (int)(st.py1 / kTile);
  const int spans_x = tx1 - tx0 + 1, spans_y = ty1 - ty0 + 1;
  rect[i] = make_int4(tx0, tx1, ty0, ty1);
  count[i] = spans_x * spans_y;
  // positive depths order like their IEEE bit patterns; the stable radix sort
  // then breaks exact ties by primitive index, as np.lexsort does.
  dkey[i] = (uint64_t)__double_as_longlong(st.t[2]);
  if (depth_range) {
    // the visible depths' range of upper words, for the 24-bit rank sort: one
    // atomic pair per group of converged lanes
    const uint32_t hi = (uint32_t)((uint64_t)__double_as_longlong(st.t[2]) >> 32);
    const unsigned am = __activemask();
    const uint32_t mn = __reduce_min_sync(am, hi), mx = __reduce_max_sync(am, hi);
    if ((threadIdx.x & 31) == __ffs(am) - 1) {
      atomicMin(depth_range, mn);
      atomicMax(depth_range + 1, mx);
    }
  }
  if (radii) radii[i] = (int32_t)ceil(st.radius);
  const bool steep = st.mode != kModePlain && is_steep(st.za, st.zb, st.radius + 24.0);
  dval[i] = (uint32_t)i | (steep ? kSteepBit : 0u);
  if (steep) side[i] = make_steep(st.mux, st.muy, st.za, st.zb);
  const float mux = (float)st.mux, muy = (float)st.muy;
  const __half2 lo = __floats2half2_rn((float)(st.mux - (double)mux), (float)(st.muy - (double)muy));
  // conic = inverse of the dilated covariance [[a, b], [b, c]]; a large splat stores
  // (c/det, -b/c, 1/c) = (a_c, b_c / a_c, c_c - b_c^2 / a_c) instead (kFlagNoWin)
  const bool large = st.radius > kWinMaxRadius;
  float4 r0 = make_float4(mux, muy, (float)(st.c / st.det),
                          large ? (float)(-st.b / st.c) : (float)(-st.b / st.det));
  float4 r1 = make_float4(large ? (float)(1.0 / st.c) : (float)(st.a / st.det), (float)st.za,
                          (float)st.zb, (float)st.c1);
  float4 r2 = make_float4((float)st.c2, (float)fmax(st.rgbu[0], 0.0), (float)fmax(st.rgbu[1], 0.0),
                          (float)fmax(st.rgbu[2], 0.0));
  float4 r3 = make_float4((float)st.t[2], __uint_as_float(pack_flags(st.mode, steep, may_clamp(st.c1, st.c2), spans_x, st.bad, large)),
                          __uint_as_float(0u), __uint_as_float(*reinterpret_cast<const uint32_t*>(&lo)));
  float4* dst = rec + 4 * i;
  dst[0] = r0;
  dst[1] = r1;
  dst[2] = r2;
  dst[3] = r3;
}

// ---------------------------------------------------------------------------
// K1: preprocess forward.  Writes the 64-B record, tile rect, pair count and
// the depth-rank sort key of each primitive (culled: count 0, key ~0).
template <typename T, int DEG, int NT>
#ifndef HS_K1_MINB
#define HS_K1_MINB 5  // resident CTAs per SM to cap registers for (0: no cap): 96 registers,
                      // 20 warps/SM; 0.289 -> 0.274 ms with the ranks at c3
#endif
#if HS_K1_MINB > 0
#define HS_K1_BOUNDS __launch_bounds__(NT, HS_K1_MINB)
#else
#define HS_K1_BOUNDS __launch_bounds__(NT)
#endif
__global__ void HS_K1_BOUNDS preprocess_fwd_kernel(
    SceneArgs<T> sc, CamArgs cam, int kernel, int64_t n, float4* __restrict__ rec,
    SteepRec* __restrict__ side, int4* __restrict__ rect, int32_t* __restrict__ count,
    uint64_t* __restrict__ dkey, uint32_t* __restrict__ dval, int32_t* __restrict__ radii,
    uint32_t* __restrict__ depth_range) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  __shared__ Staged<T, K, NT> sm;
  const int64_t base = (int64_t)blockIdx.x * NT;
  const int cnt = (int)(n - base < NT ? n - base : NT);
  stage_in(sm, sc, base, cnt);
  const int t = threadIdx.x;
  if (t >= cnt) return;
  const int64_t i = base + t;
  FwdState st;
  forward_state<DEG>(StagedView<T, K, NT>{sm, t}, cam, kernel, st);
  write_fwd_outputs(st, i, FwdOut{rec, side, rect, count, dkey, dval, radii, depth_range});
}

// K1 for a batch of views of one scene (multiview.ViewBatch): a CTA stages its
// primitives once and computes their camera-independent state once (indep_state:
// quaternion, rotation, scales, covariance, unit normal, cov . n, opacities, ~30%
// of K1's FP64 work), keeps it in shared memory, then runs every view's projection
// (view_state) and writes each view's outputs.  Same arithmetic as K1, so the
// outputs are bit-identical.
template <typename T, int NT>
struct IndepStage {
  double cov[9][NT], hw[3][NT], a1[NT], a2[NT];
};
#ifndef HS_K1V_MINB
#define HS_K1V_MINB 4
#endif
template <typename T, int DEG, int NT>
__global__ void __launch_bounds__(NT, HS_K1V_MINB) preprocess_fwd_views_kernel(
    SceneArgs<T> sc, FwdViewsArgs va, int kernel, int64_t n) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  __shared__ Staged<T, K, NT> sm;
  __shared__ IndepStage<T, NT> ind;
  const int64_t base = (int64_t)blockIdx.x * NT;
  const int cnt = (int)(n - base < NT ? n - base : NT);
  stage_in(sm, sc, base, cnt);
  const int t = threadIdx.x;
  if (t >= cnt) return;
  const int64_t i = base + t;
  const StagedView<T, K, NT> src{sm, t};
  {
    FwdState st;
    indep_state(src, st);
#pragma unroll
    for (int k = 0; k < 9; ++k) ind.cov[k][t] = st.cov[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) ind.hw[k][t] = st.hw[k];
    ind.a1[t] = st.a1;
    ind.a2[t] = st.a2;
  }
  for (int v = 0; v < va.n_views; ++v) {
    FwdState st;
#pragma unroll
    for (int k = 0; k < 9; ++k) st.cov[k] = ind.cov[k][t];
#pragma unroll
    for (int k = 0; k < 3; ++k) st.hw[k] = ind.hw[k][t];
    st.a1 = ind.a1[t];
    st.a2 = ind.a2[t];
    view_state<DEG>(src, va.cam[v], kernel, st);
    write_fwd_outputs(st, i, va.out[v]);
  }
}

// ---------------------------------------------------------------------------
// ScreenSplat export (rasterizer.py:578-603): the FP64 projected quantities of
// every visible primitive (introspection only; reads the scene directly).
template <typename T, int K>
struct GlobalView {
  const SceneArgs<T>& sc;
  int64_t i;
  __device__ __forceinline__ double mu(int k) const { return (double)sc.mu[3 * i + k]; }
  __device__ __forceinline__ double ls(int k) const { return (double)sc.ls[3 * i + k]; }
  __device__ __forceinline__ double rot(int k) const { return (double)sc.rot[4 * i + k]; }
  __device__ __forceinline__ double nrm(int k) const { return (double)sc.nrm[3 * i + k]; }
  __device__ __forceinline__ double ra() const { return (double)sc.ra[i]; }
  __device__ __forceinline__ double rb() const { return (double)sc.rb[i]; }
  __device__ __forceinline__ double sh(int k, int ch) const {
    return (double)sc.sh[(i * K + k) * 3 + ch];
  }
  template <typename F>
  __device__ __forceinline__ void for_each_sh(F&& f) const {
#pragma unroll
    for (int j = 0; j < 3 * K; ++j) f(j, (double)sc.sh[i * K * 3 + j]);
  }
};

template <typename T, int DEG>
__global__ void __launch_bounds__(128) screen_splats_kernel(SceneArgs<T> sc, CamArgs cam,
                                                            int kernel, int64_t n,
                                                            double* __restrict__ out) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  FwdState st;
  forward_state<DEG>(GlobalView<T, K>{sc, i}, cam, kernel, st);
  double* o = out + 20 * i;
  if (!st.visible) {
    for (int k = 0; k < 20; ++k) o[k] = 0.0;
    return;
  }
  const double v[20] = {st.mux, st.muy, st.c / st.det, -st.b / st.det, st.a / st.det,
                        st.v00, st.v10, st.v11, st.nray[0], st.nray[1], st.nray[2],
                        st.a1, st.a2, fmax(st.rgbu[0], 0.0), fmax(st.rgbu[1], 0.0),
                        fmax(st.rgbu[2], 0.0), st.t[2], st.radius, st.za, st.zb};
  for (int k = 0; k < 20; ++k) o[k] = v[k];
}

template <typename T>
cudaError_t launch_screen_splats_t(const SceneArgs<T>& sc, const CamArgs& cam, int kernel,
                                   int64_t n, double* out, cudaStream_t stream) {
  const int64_t grid = (n + 127) / 128;
  switch (sc.deg) {
    case 0: screen_splats_kernel<T, 0><<<(unsigned)grid, 128, 0, stream>>>(sc, cam, kernel, n, out); break;
    case 1: screen_splats_kernel<T, 1><<<(unsigned)grid, 128, 0, stream>>>(sc, cam, kernel, n, out); break;
    case 2: screen_splats_kernel<T, 2><<<(unsigned)grid, 128, 0, stream>>>(sc, cam, kernel, n, out); break;
    case 3: screen_splats_kernel<T, 3><<<(unsigned)grid, 128, 0, stream>>>(sc, cam, kernel, n, out); break;
    default: return cudaErrorInvalidValue;
  }
  note_launch();
  return cudaGetLastError();
}
template cudaError_t launch_screen_splats_t<float>(const SceneArgs<float>&, const CamArgs&, int,
                                                   int64_t, double*, cudaStream_t);
template cudaError_t launch_screen_splats_t<double>(const SceneArgs<double>&, const CamArgs&, int,
                                                    int64_t, double*, cudaStream_t);

#endif  // !HS_GEOMETRY_BWD_TU

#ifdef HS_GEOMETRY_BWD_TU
// ---------------------------------------------------------------------------
// K7: merge the splat's pair rows (np.add.at, rasterizer.py:419-420) and chain
// them through the projection to the primitive parameters
// (_geometry_backward, rasterizer.py:424-575).  FP64 throughout.
// K7a: merge each visible splat's pair rows (np.add.at, rasterizer.py:419-420):
// the tiles of its rect in row-major (= sorted k) order, skipping pairs past
// the tile's last composited position (never written by K6).  A separate,
// register-light kernel so the dependent gathers are hidden by occupancy.
// G lanes per splat (a power of two <= 32): lane j of the group takes rows
// j, j + G, ... and the group's partial sums meet in a fixed xor-shuffle tree,
// so the result is deterministic (G = 1: plain row-order sums).  The launcher
// picks G from the frame's mean rows per primitive (HS_K7A_WIDE_ROWS).
template <int G>
__global__ void __launch_bounds__(256) merge_rows_kernel(
    int64_t n, int tiles_x, const float4* __restrict__ rec,
    const int32_t* __restrict__ row_origin, const int4* __restrict__ rect,
    const int32_t* __restrict__ count, const uint32_t* __restrict__ rank_of,
    const int32_t* __restrict__ last_rank, const float* __restrict__ rows,
    float4* __restrict__ merged, int64_t begin, int mark) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = begin + tid / G;
  const int sub = (int)(tid % G);
  // with G > 1 every lane stays to the shuffles (a group never straddles a warp)
  const int cnt = i < n ? count[i] : 0;
  // mark: rows for a multi-view K7 (hs_merge_rows): a splat this view culled gets an
  // explicit empty row (visibility .z = 0), the buffer outliving the frame's counts
  if (mark && cnt == 0 && i < n && sub == 0) {
    float4* dst = merged + 4 * i;
    dst[0] = dst[1] = dst[2] = dst[3] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (G == 1 && cnt == 0) return;
  // FP32 sums (in a fixed order, so still deterministic): 62 registers instead of 76
  // raise the occupancy this gather-bound kernel lives on (c4 0.232 -> 0.162 ms per
  // view, c5 K7a + K7 0.713 -> 0.504 ms); a splat's rows number a few to a few hundred,
  // far inside the gradients' 1e-3 contract (HS_K7A_ACC=double restores FP64)
#ifndef HS_K7A_ACC
#define HS_K7A_ACC float
#endif
  HS_K7A_ACC m[13];
#pragma unroll
  for (int k = 0; k < 13; ++k) m[k] = 0.0;
  int4 rc = make_int4(0, 0, 0, 0);
  int spans_x = 1, base = 0, r = 0;
  float4 r2 = make_float4(0.f, 0.f, 0.f, 0.f), r3 = r2;
  if (cnt > 0) {
    rc = rect[i];
    spans_x = rc.y - rc.x + 1;
    r2 = rec[4 * i + 2];
    r3 = rec[4 * i + 3];
    base = row_origin[i] + rc.z * spans_x + rc.x;
    r = (int)rank_of[i];
  }
  // row l of the splat is tile (rc.z + l / spans_x, rc.x + l % spans_x); the
  // lane walks l = sub, sub + G, ... keeping (lx, ly) incrementally
  int ly = sub / spans_x, lx = sub - ly * spans_x;
  auto next_tile_of = [&]() {
    const int tile = (rc.z + ly) * tiles_x + rc.x + lx;
    lx += G;
    while (lx >= spans_x) {
      lx -= spans_x;
      ++ly;
    }
    return tile;
  };
  auto load_row = [&](int l, float4 (&u)[4]) {
    const float4* row = reinterpret_cast<const float4*>(rows + (size_t)(base + l) * kRowFloats);
    u[0] = row[0]; u[1] = row[1]; u[2] = row[2]; u[3] = row[3];
  };
  auto add_row = [&](const float4 (&u)[4]) {
    m[0] += u[0].x; m[1] += u[0].y; m[2] += u[0].z; m[3] += u[0].w;
    m[4] += u[1].x; m[5] += u[1].y; m[6] += u[1].z; m[7] += u[1].w;
    m[8] += u[2].x; m[9] += u[2].y; m[10] += u[2].z; m[11] += u[2].w;
    m[12] += u[3].x;
  };
  // HS_K7A_ROWS rows in flight per step: the tiles' last ranks first, then the
  // gathers of the rows below them only (rows past a tile's last composited
  // rank were never written, and at c5 they are most of them), additions in
  // row order (the same sum).  With FP32 sums the occupancy carries the latency:
  // one row per step (c4 0.159 -> 0.145 ms per view; 3 or 4 rows are slower)
#ifndef HS_K7A_ROWS
#define HS_K7A_ROWS 1
#endif
  constexpr int U = HS_K7A_ROWS;
  int l = sub;
  for (; l + (U - 1) * G < cnt; l += U * G) {
    int lr[U];
    float4 u[U][4];
#pragma unroll
    for (int k = 0; k < U; ++k) lr[k] = last_rank[next_tile_of()];
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (r <= lr[k]) load_row(l + k * G, u[k]);
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (r <= lr[k]) add_row(u[k]);
  }
  for (; l < cnt; l += G) {
    const int tl = next_tile_of();
    if (r > last_rank[tl]) continue;
    float4 u[4];
    load_row(l, u);
    add_row(u);
  }
  if (G > 1) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
      for (int k = 0; k < 13; ++k) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o, G);
    if (sub != 0 || cnt == 0) return;
  }
  // colour clamp (rasterizer.py:544): the record holds max(rgb, 0), which is > 0
  // exactly when the unclamped FP64 colour is, so the gradient of a clamped
  // channel is dropped here and K7 does not re-evaluate the colour
  if (!(r2.y > 0.f)) m[9] = 0.0;
  if (!(r2.z > 0.f)) m[10] = 0.0;
  if (!(r2.w > 0.f)) m[11] = 0.0;
  float4* dst = merged + 4 * i;
  dst[0] = make_float4((float)m[0], (float)m[1], (float)m[2], (float)m[3]);
  dst[1] = make_float4((float)m[4], (float)m[5], (float)m[6], (float)m[7]);
  dst[2] = make_float4((float)m[8], (float)m[9], (float)m[10], (float)m[11]);
  // .y: K1's record flags for K7; .z: visible in this view (the multi-view K7)
  dst[3] = make_float4((float)m[12], r3.y, 1.f, 0.f);
}

// The multi-view K7's per-primitive gradient accumulators (the staged inputs stay
// untouched across the views).
template <typename T, int K, int NT>
struct AccStage {
  T mu[NT * 3], ls[NT * 3], nrm[NT * 3], rot[NT * 4], ra[NT], rb[NT], pgn[NT];
  T sh[NT * Staged<T, K, NT>::SHS];
};

// One primitive's geometry backward for one view.  ACC = false (K7): the gradients
// overwrite the thread's staged inputs (read before), visibility from count.  ACC =
// true (the multi-view K7): they add into `acc`, visibility from the row's marker.
template <typename T, int DEG, int NT, bool ACC = false>
__device__ __forceinline__ void preprocess_bwd_one(
    Staged<T, (DEG + 1) * (DEG + 1), NT>& sm, T* pgn_s, int32_t* touch_s, int t, int64_t i,
    const CamArgs& cam, int kernel, const int32_t* __restrict__ count,
    const float4* __restrict__ merged,
    AccStage<T, (DEG + 1) * (DEG + 1), NT>* acc = nullptr) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  using St = Staged<T, K, NT>;
#define K7_PUT(field, idx, val)                                        \
  do {                                                                 \
    if constexpr (ACC) acc->field[idx] = add_rn(acc->field[idx], T(val));      \
    else sm.field[idx] = T(val);                                               \
  } while (0)
  const int cnt = ACC ? 1 : count[i];
  if (cnt == 0) {
    for (int k = 0; k < 3; ++k) sm.mu[3 * t + k] = sm.ls[3 * t + k] = sm.nrm[3 * t + k] = T(0);
    for (int k = 0; k < 4; ++k) sm.rot[4 * t + k] = T(0);
    for (int k = 0; k < 3 * K; ++k) sm.sh[t * St::SHS + k] = T(0);
    sm.ra[t] = sm.rb[t] = T(0);
    pgn_s[t] = T(0);
    touch_s[t] = 0;
    return;
  }
  double m[13];
  uint32_t flags;
  {
    const float4* src = merged + 4 * i;
    const float4 u0 = src[0], u1 = src[1], u2 = src[2], u3 = src[3];
    m[0] = u0.x; m[1] = u0.y; m[2] = u0.z; m[3] = u0.w;
    m[4] = u1.x; m[5] = u1.y; m[6] = u1.z; m[7] = u1.w;
    m[8] = u2.x; m[9] = u2.y; m[10] = u2.z; m[11] = u2.w;
    m[12] = u3.x;
    flags = __float_as_uint(u3.y);
    if (ACC && u3.z == 0.f) return;  // culled in this view
  }
  FwdState st;
  forward_state<DEG, true>(StagedView<T, K, NT>{sm, t}, cam, kernel, st, flags);

  const double d_mux = m[0], d_muy = m[1];
  const double d_ca = m[2], d_cb = m[3], d_cc = m[4];
  const double d_za = m[5], d_zb = m[6], d_c1 = m[7], d_c2 = m[8];
  const double d_rgb[3] = {m[9], m[10], m[11]};

  // opacities (rasterizer.py:446-450)
  {
    const double d_a1 = 0.5 * (d_c1 + d_c2), d_a2 = 0.5 * (d_c1 - d_c2);
    K7_PUT(ra, t, d_a1 * st.a1 * (1.0 - st.a1));
    K7_PUT(rb, t, d_a2 * st.a2 * (1.0 - st.a2));
  }
  // erf coefficients -> n_ray and whitening (rasterizer.py:452-466)
  const bool mode0 = st.mode == kModeErf;
  const double n1 = st.nray[0], n2 = st.nray[1], n3 = st.nray[2];
  const double inv = mode0 ? 1.0 / (1.4142135623730951 * fabs(n3)) : 0.0;
  const double d_za0 = mode0 ? d_za : 0.0, d_zb0 = mode0 ? d_zb : 0.0;
  // d_inv = d_za*(n1 v00 + n2 v10) + d_zb*(n2 v11) (rasterizer.py:459) equals
  // (sum_px d_z * z) / inv; the blend accumulates that sum directly (column 12),
  // which stays accurate when za*dx and zb*dy nearly cancel (|n3| -> 0).
  const double d_inv = mode0 ? m[kColSumDzZ] * (1.4142135623730951 * fabs(n3)) : 0.0;
  double d_nray[3];
  d_nray[0] = d_za0 * inv * st.v00;
  d_nray[1] = d_za0 * inv * st.v10 + d_zb0 * inv * st.v11;
  {
    const double sg = n3 > 0.0 ? 1.0 : (n3 < 0.0 ? -1.0 : 0.0);
    // 1 / (sqrt2 n3^2) = sqrt2 * inv^2
    d_nray[2] = mode0 ? -d_inv * sg * (1.4142135623730951 * inv * inv) : 0.0;
  }
  const double d_v00 = d_za0 * inv * n1, d_v10 = d_za0 * inv * n2, d_v11 = d_zb0 * inv * n2;
  // n_ray = y/|y| (rasterizer.py:469)
  double d_y[3];
  {
    const double dot = d_nray[0] * n1 + d_nray[1] * n2 + d_nray[2] * n3;
    const double rn = 1.0 / st.ynorm;
    for (int k = 0; k < 3; ++k) d_y[k] = (d_nray[k] - dot * st.nray[k]) * rn;
  }
  // y = L^-1 h_ray (rasterizer.py:470-473; tri_inv3_batch geometry.py:176-186)
  const double* L = st.L;
  double Li[9];
  {
    const double a = L[0], b = L[4], c = L[8];
    const double ra = 1.0 / a, rb = 1.0 / b, rc = 1.0 / c;
    Li[0] = ra; Li[1] = 0.0; Li[2] = 0.0;
    Li[3] = -L[3] * (ra * rb); Li[4] = rb; Li[5] = 0.0;
    Li[6] = (L[3] * L[7] - L[6] * b) * (ra * rb * rc); Li[7] = -L[7] * (rb * rc); Li[8] = rc;
  }
  double d_hr[3];
  for (int a = 0; a < 3; ++a) d_hr[a] = Li[a] * d_y[0] + Li[3 + a] * d_y[1] + Li[6 + a] * d_y[2];
  double dL[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) dL[3 * a + b] = -d_hr[a] * st.y[b];
  // whiten2d = inv(L[:2,:2]): d_L2 -= V^T dV V^T (rasterizer.py:475-484)
  {
    const double V00 = st.v00, V10 = st.v10, V11 = st.v11;
    // X = V^T dV with V^T = [[V00, V10],[0, V11]], dV = [[d_v00, 0],[d_v10, d_v11]]
    const double X00 = V00 * d_v00 + V10 * d_v10, X01 = V10 * d_v11;
    const double X10 = V11 * d_v10, X11 = V11 * d_v11;
    // Y = X V^T
    dL[0] -= X00 * V00;
    dL[1] -= X00 * V10 + X01 * V11;
    dL[3] -= X10 * V00;
    dL[4] -= X10 * V10 + X11 * V11;
  }
  dL[1] = 0.0; dL[2] = 0.0; dL[5] = 0.0;  // np.tril
  // chol3_vjp (geometry.py:163-173)
  double dC[9];
  {
    double P[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        P[3 * a + b] = L[a] * dL[b] + L[3 + a] * dL[3 + b] + L[6 + a] * dL[6 + b];
    double phi[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) phi[3 * a + b] = b < a ? P[3 * a + b] : (a == b ? 0.5 * P[3 * a + b] : 0.0);
    double S[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) S[3 * a + b] = phi[3 * a + b] + phi[3 * b + a];
    double tmp[9];  // S @ Li
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        tmp[3 * a + b] = S[3 * a] * Li[b] + S[3 * a + 1] * Li[3 + b] + S[3 * a + 2] * Li[6 + b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        dC[3 * a + b] = 0.5 * (Li[a] * tmp[b] + Li[3 + a] * tmp[3 + b] + Li[6 + a] * tmp[6 + b]);
  }
  // conic = inverse of the dilated 2x2 (rasterizer.py:489-500)
  {
    const double a = st.a, b = st.b, c = st.c, det = st.det, det2 = det * det;
    const double rd2 = 1.0 / det2;
    dC[0] += (-d_ca * c * c + d_cb * b * c - d_cc * b * b) * rd2;
    dC[1] += (2.0 * d_ca * b * c - d_cb * (det + 2.0 * b * b) + 2.0 * d_cc * a * b) * rd2;
    dC[4] += (-d_ca * b * b + d_cb * a * b - d_cc * a * a) * rd2;
  }
  // cov_ray = J cov_cam J^T, h_ray = J h_cam (rasterizer.py:503-507)
  const double* J = st.J;
  double dJ[9], dCc[9], d_hc[3];
  {
    double S[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) S[3 * a + b] = dC[3 * a + b] + dC[3 * b + a];
    double SJ[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        SJ[3 * a + b] = S[3 * a] * J[b] + S[3 * a + 1] * J[3 + b] + S[3 * a + 2] * J[6 + b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        dJ[3 * a + b] = SJ[3 * a] * st.ccam[b] + SJ[3 * a + 1] * st.ccam[3 + b] +
                        SJ[3 * a + 2] * st.ccam[6 + b] + d_hr[a] * st.hc[b];
    double tmp[9];  // dC @ J
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        tmp[3 * a + b] = dC[3 * a] * J[b] + dC[3 * a + 1] * J[3 + b] + dC[3 * a + 2] * J[6 + b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        dCc[3 * a + b] = J[a] * tmp[b] + J[3 + a] * tmp[3 + b] + J[6 + a] * tmp[6 + b];
    for (int a = 0; a < 3; ++a) d_hc[a] = J[a] * d_hr[0] + J[3 + a] * d_hr[1] + J[6 + a] * d_hr[2];
  }
  // cov_cam = W cov W^T, h_cam = W h (rasterizer.py:510-511)
  const double* Wr = cam.R;
  double dS[9], d_h[3];
  {
    double tmp[9];  // dCc @ W
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        tmp[3 * a + b] = dCc[3 * a] * Wr[b] + dCc[3 * a + 1] * Wr[3 + b] + dCc[3 * a + 2] * Wr[6 + b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        dS[3 * a + b] = Wr[a] * tmp[b] + Wr[3 + a] * tmp[3 + b] + Wr[6 + a] * tmp[6 + b];
    for (int a = 0; a < 3; ++a) d_h[a] = d_hc[0] * Wr[a] + d_hc[1] * Wr[3 + a] + d_hc[2] * Wr[6 + a];
  }
  // h = cov n_unit (rasterizer.py:514-515)
  double d_nu[3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) dS[3 * a + b] += d_h[a] * st.nu[b];
  for (int a = 0; a < 3; ++a)
    d_nu[a] = st.cov[a] * d_h[0] + st.cov[3 + a] * d_h[1] + st.cov[6 + a] * d_h[2];
  // projected mean and Jacobian w.r.t. the camera-space centre (rasterizer.py:518-538)
  double d_t[3];
  {
    const double tx = st.t[0], ty = st.t[1], tz = st.t[2];
    const double invz = 1.0 / tz;
    d_t[0] = d_mux * cam.fx * invz;
    d_t[1] = d_muy * cam.fy * invz;
    d_t[2] = -d_mux * cam.fx * tx * invz * invz - d_muy * cam.fy * ty * invz * invz;
    const double ell = sqrt(tx * tx + ty * ty + tz * tz);
    d_t[2] += dJ[0] * (-cam.fx * invz * invz);
    d_t[0] += dJ[2] * (-cam.fx * invz * invz);
    d_t[2] += dJ[2] * (2.0 * cam.fx * tx * invz * invz * invz);
    d_t[2] += dJ[4] * (-cam.fy * invz * invz);
    d_t[1] += dJ[5] * (-cam.fy * invz * invz);
    d_t[2] += dJ[5] * (2.0 * cam.fy * ty * invz * invz * invz);
    const double rell = 1.0 / ell;
    const double rh[3] = {tx * rell, ty * rell, tz * rell};
    const double dot = dJ[6] * rh[0] + dJ[7] * rh[1] + dJ[8] * rh[2];
    for (int k = 0; k < 3; ++k) d_t[k] += (dJ[6 + k] - dot * rh[k]) * rell;
  }
  double d_mu[3];
  for (int a = 0; a < 3; ++a) d_mu[a] = d_t[0] * Wr[a] + d_t[1] * Wr[3 + a] + d_t[2] * Wr[6 + a];
  // spherical harmonics colour, clamped at zero (rasterizer.py:543-552): the
  // clamp is already applied to d_rgb (merge_rows_kernel); well conditioned, so
  // FP32 (sh_bwd_f32); only the direction's normalisation is chained in FP64
  {
    const float dpre[3] = {(float)d_rgb[0], (float)d_rgb[1], (float)d_rgb[2]};
    const float dirf[3] = {(float)st.vdir[0], (float)st.vdir[1], (float)st.vdir[2]};
    float d_dir[3];
    // d_sh overwrites this thread's staged SH row (read first for d_basis)
    sh_bwd_f32<DEG, ACC>(dirf, dpre, sm.sh + t * St::SHS, d_dir,
                         ACC ? acc->sh + t * St::SHS : nullptr);
    if (DEG > 0) {
      const double dd[3] = {d_dir[0], d_dir[1], d_dir[2]};
      const double dot = dd[0] * st.vdir[0] + dd[1] * st.vdir[1] + dd[2] * st.vdir[2];
      const double rv = 1.0 / st.vdist;
      for (int d = 0; d < 3; ++d) d_mu[d] += (dd[d] - dot * st.vdir[d]) * rv;
    }
  }
  // covariance build: cov = M M^T, M = R diag(s) (rasterizer.py:555-562)
  {
    double Mf[9];
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) Mf[3 * r + k] = st.R[3 * r + k] * st.s[k];
    double dM[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int c = 0; c < 3; ++c) acc += (dS[3 * a + c] + dS[3 * c + a]) * Mf[3 * c + b];
        dM[3 * a + b] = acc;
      }
    double dR[9], d_s[3];
    for (int k = 0; k < 3; ++k) d_s[k] = 0.0;
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) {
        dR[3 * r + k] = dM[3 * r + k] * st.s[k];
        d_s[k] += dM[3 * r + k] * st.R[3 * r + k];
      }
    for (int k = 0; k < 3; ++k) K7_PUT(ls, 3 * t + k, d_s[k] * st.s[k]);
    // quat_rot_vjp (geometry.py:76-107) at the unit quaternion
    const double w = st.qu[0], x = st.qu[1], y = st.qu[2], z = st.qu[3];
    const double Dw[9] = {0, -z, y, z, 0, -x, -y, x, 0};
    const double Dx[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
    const double Dy[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
    const double Dz[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
    double dq[4] = {0, 0, 0, 0};
    for (int k = 0; k < 9; ++k) {
      dq[0] += 2 * Dw[k] * dR[k];
      dq[1] += 2 * Dx[k] * dR[k];
      dq[2] += 2 * Dy[k] * dR[k];
      dq[3] += 2 * Dz[k] * dR[k];
    }
    const double dot = dq[0] * w + dq[1] * x + dq[2] * y + dq[3] * z;
    const double rq = 1.0 / st.qnorm;
    for (int k = 0; k < 4; ++k) K7_PUT(rot, 4 * t + k, (dq[k] - dot * st.qu[k]) * rq);
  }
  // splitting normal through its normalisation (rasterizer.py:565-566)
  {
    const double dot = d_nu[0] * st.nu[0] + d_nu[1] * st.nu[1] + d_nu[2] * st.nu[2];
    const double rnn = 1.0 / st.nnorm;
    for (int k = 0; k < 3; ++k) K7_PUT(nrm, 3 * t + k, (d_nu[k] - dot * st.nu[k]) * rnn);
  }
  for (int k = 0; k < 3; ++k) K7_PUT(mu, 3 * t + k, d_mu[k]);
  if constexpr (ACC) {
    acc->pgn[t] = add_rn(acc->pgn[t], T(sqrt(d_mux * d_mux + d_muy * d_muy)));
    touch_s[t] += 1;
  } else {
    pgn_s[t] = T(sqrt(d_mux * d_mux + d_muy * d_muy));
    touch_s[t] = 1;
  }
#undef K7_PUT
}

template <typename E> struct Vec16;
template <> struct Vec16<float> { using type = float4; };
template <> struct Vec16<double> { using type = double2; };
template <> struct Vec16<int32_t> { using type = int4; };

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem));
}

// Which of the CTA's primitives this view touched, as a bit mask (one ballot per
// warp) plus an all-touched flag: the vectorised copies below test a 16-B vector's
// primitives with two word loads and a shift instead of a per-primitive loop with
// divisions, which was 18% of K7's instructions at c4 (ncu source view).
template <int NT>
struct LiveMask {
  uint32_t w[NT / 32 + 1];  // a zero word past the end: 64-bit windows never overrun
  int all;
};

// after touch_s is final and a __syncthreads()
template <int NT>
__device__ __forceinline__ void build_live_mask(LiveMask<NT>& m, const int32_t* touch_s) {
  const unsigned b = __ballot_sync(0xffffffffu, touch_s[threadIdx.x] != 0);
  if ((threadIdx.x & 31) == 0) m.w[threadIdx.x >> 5] = b;
  if (threadIdx.x == 0) m.w[NT / 32] = 0u;
  const int full = __syncthreads_and(b == 0xffffffffu);
  if (threadIdx.x == 0) m.all = full;
  __syncthreads();
}

// Does any primitive of elements [e0, e0 + len) (S elements per primitive) have
// a non-zero flag?  (len < 32 * S)
template <int S, int NT>
__device__ __forceinline__ bool any_live(bool all, const LiveMask<NT>& m, int e0, int len) {
  if (all) return true;
  const int p0 = e0 / S, p1 = (e0 + len - 1) / S;
  const int wi = p0 >> 5;
  const uint64_t win = ((uint64_t)m.w[wi + 1] << 32) | m.w[wi];
  const int n = p1 - p0 + 1;
  return ((win >> (p0 & 31)) & ((1ull << n) - 1ull)) != 0ull;
}

// Accumulation targets of one CTA, prefetched into shared memory while the
// geometry backward runs (field order and layout as in global memory, so both
// copies move in 16-B pieces).
template <typename T, int K, int NT>
struct GradStage {
  T mu[NT * 3], ls[NT * 3], nrm[NT * 3], rot[NT * 4], ra[NT], rb[NT], pgn[NT];
  int32_t touch[NT];
  T sh[NT * 3 * K];
};

// One field of the CTA's `cnt` primitives (S elements each, contiguous from
// `src`): global -> shared with cp.async, skipping primitives this view does
// not touch.  16-B copies when `src` is 16-B aligned, element copies otherwise.
template <int NT, int S, typename E>
__device__ __forceinline__ void prefetch_block(E* smem, const E* src, int cnt,
                                               const int32_t* live, const LiveMask<NT>& lm) {
  constexpr int kV = 16 / sizeof(E);
  const int n = cnt * S;
  const int nv = ((uintptr_t)src & 15) ? 0 : n / kV;
  const bool all = lm.all;
  for (int v = threadIdx.x; v < nv; v += NT)
    if (any_live<S>(all, lm, v * kV, kV)) cp_async16(smem + v * kV, src + v * kV);
  for (int e = nv * kV + threadIdx.x; e < n; e += NT)
    if (live[e / S]) cp_async_elem(smem + e, src + e);
}

// Write one field of the CTA's primitives from `get(e)`, or with `old` (the
// prefetched targets) add into it, skipping primitives this view did not touch
// (their gradient is zero).  16-B stores when `dst` is 16-B aligned.
template <int NT, int S, typename E, typename Get>
__device__ __forceinline__ void store_block(E* __restrict__ dst, int cnt, const E* old,
                                            const int32_t* live, const LiveMask<NT>& lm,
                                            Get get) {
  using V = typename Vec16<E>::type;
  constexpr int kV = 16 / sizeof(E);
  const int n = cnt * S;
  const int nv = ((uintptr_t)dst & 15) ? 0 : n / kV;
  V* dv = reinterpret_cast<V*>(dst);
  const bool all = lm.all;
  for (int v = threadIdx.x; v < nv; v += NT) {
    if (old && !any_live<S>(all, lm, v * kV, kV)) continue;
    V nw;
    E* ne = reinterpret_cast<E*>(&nw);
#pragma unroll
    for (int j = 0; j < kV; ++j) ne[j] = get(v * kV + j) + (old ? old[v * kV + j] : E(0));
    dv[v] = nw;
  }
  for (int e = nv * kV + threadIdx.x; e < n; e += NT) {
    if (old && !live[e / S]) continue;
    dst[e] = get(e) + (old ? old[e] : E(0));
  }
}

template <typename T, int K, int NT>
constexpr size_t k7_dynamic_smem() { return sizeof(GradStage<T, K, NT>); }

// Reduction stores (hs_grads.accumulate 2 / 3): add into the destination with a
// relaxed device-scope atomic, or -- when the destination is an NVLS multicast
// address of a buffer shared by every rank -- with multimem.red, which the
// NVSwitch reduces into every rank's copy: K7 then IS the cross-GPU all-reduce.
__device__ __forceinline__ void red_add(float* p, float v, bool mc) {
  if (mc)
    asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
  else
    asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add(double* p, double v, bool mc) {
  if (mc)
    asm volatile("multimem.red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
  else
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void red_add(int32_t* p, int32_t v, bool mc) {
  if (mc)
    asm volatile("multimem.red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add4(float* p, float4 v, bool mc) {
  if (mc)
    asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  else
    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// store_block for a field staged in padded shared-memory rows (row r of R elements
// at rows + r * STRIDE) whose rows are whole 16-B vectors: each vector's row and
// column come from one division instead of one per element.
template <int NT, int R, int STRIDE, typename E>
__device__ __forceinline__ void store_rows(E* __restrict__ dst, int cnt, const E* old,
                                           const int32_t* live, const LiveMask<NT>& lm,
                                           const E* rows) {
  using V = typename Vec16<E>::type;
  constexpr int kV = 16 / sizeof(E);
  static_assert(R % kV == 0, "rows must be whole vectors");
  const int n = cnt * R;
  if ((uintptr_t)dst & 15) {
    for (int e = threadIdx.x; e < n; e += NT) {
      const int r = e / R;
      if (old && !live[r]) continue;
      dst[e] = rows[r * STRIDE + (e - r * R)] + (old ? old[e] : E(0));
    }
    return;
  }
  V* dv = reinterpret_cast<V*>(dst);
  for (int v = threadIdx.x; v < n / kV; v += NT) {
    const int r = (v * kV) / R, c = v * kV - r * R;
    if (old && !live[r]) continue;
    V nw;
    E* ne = reinterpret_cast<E*>(&nw);
#pragma unroll
    for (int j = 0; j < kV; ++j) ne[j] = rows[r * STRIDE + c + j] + (old ? old[v * kV + j] : E(0));
    dv[v] = nw;
  }
}

// One field of the CTA's primitives reduced into `dst` (only touched ones: the
// others add zero).  float fields move in 16-B vector reductions when aligned.
template <int NT, int S, typename E, typename Get>
__device__ __forceinline__ void reduce_block(E* __restrict__ dst, int cnt, const int32_t* live,
                                             const LiveMask<NT>& lm, bool mc, Get get) {
  const int n = cnt * S;
  int done = 0;
  if constexpr (sizeof(E) == 4 && !std::is_same<E, int32_t>::value) {
    const int nv = ((uintptr_t)dst & 15) ? 0 : n / 4;
    const bool all = lm.all;
    for (int v = threadIdx.x; v < nv; v += NT) {
      if (!any_live<S>(all, lm, v * 4, 4)) continue;
      red_add4(dst + 4 * v, make_float4(get(4 * v), get(4 * v + 1), get(4 * v + 2),
                                        get(4 * v + 3)), mc);
    }
    done = nv * 4;
  }
  for (int e = done + threadIdx.x; e < n; e += NT)
    if (live[e / S]) red_add(dst + e, get(e), mc);
}

template <typename T, int DEG, int NT, int MODE>
#ifndef HS_K7_MINB
#define HS_K7_MINB 3
#endif
__global__ void __launch_bounds__(NT, HS_K7_MINB) preprocess_bwd_kernel(
    SceneArgs<T> sc, CamArgs cam, int kernel, int64_t n, const int32_t* __restrict__ count,
    const float4* __restrict__ merged, GradArgs<T> out) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  using St = Staged<T, K, NT>;
  using Gs = GradStage<T, K, NT>;
  __shared__ St sm;
  __shared__ T pgn_s[NT];
  __shared__ int32_t touch_s[NT];
  __shared__ LiveMask<NT> lm;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  const int64_t base = out.begin + (int64_t)blockIdx.x * NT;
  const int ncta = (int)(n - base < NT ? n - base : NT);
  const int t = threadIdx.x;
  // accumulate: 0 overwrite, 1 read-modify-write, 2 atomic add, 3 multimem add.
  // MODE (0, 1, or 2 for both reductions) compiles only that store path: the
  // unused ones cost ~30% of the kernel's code (c3 K7a + K7 0.304 -> 0.295 ms)
  constexpr bool acc = MODE == 1;
  constexpr bool red = MODE == 2;
  const bool mc = red && out.accumulate == 3;
  const bool bulk = stage_in(sm, sc, base, ncta, /*wait=*/false);
  Gs* g = acc ? reinterpret_cast<Gs*>(dyn_smem) : nullptr;
  if (acc) {
    // touch_s = visible in this view (count > 0); preprocess_bwd_one rewrites
    // the same value.  The targets of visible primitives stream in behind the
    // scene staging and are waited for only before the final stores.
    touch_s[t] = t < ncta ? (count[base + t] != 0) : 0;
    __syncthreads();
    build_live_mask(lm, touch_s);
    prefetch_block<NT, 3>(g->mu, out.d_mu + base * 3, ncta, touch_s, lm);
    prefetch_block<NT, 3>(g->ls, out.d_log_scale + base * 3, ncta, touch_s, lm);
    prefetch_block<NT, 3>(g->nrm, out.d_normal + base * 3, ncta, touch_s, lm);
    prefetch_block<NT, 4>(g->rot, out.d_rotation + base * 4, ncta, touch_s, lm);
    prefetch_block<NT, 1>(g->ra, out.d_ra + base, ncta, touch_s, lm);
    prefetch_block<NT, 1>(g->rb, out.d_rb + base, ncta, touch_s, lm);
    prefetch_block<NT, 1>(g->pgn, out.pos_grad_norm + base, ncta, touch_s, lm);
    prefetch_block<NT, 1>(g->touch, out.touch + base, ncta, touch_s, lm);
    prefetch_block<NT, 3 * K>(g->sh, out.d_sh + base * 3 * K, ncta, touch_s, lm);
    asm volatile("cp.async.commit_group;\n" ::);
    // the scene: its bulk copies, or every cp.async group but the targets'
    if (bulk)
      bulk_wait(&sm.bar);
    else
      asm volatile("cp.async.wait_group 1;\n" ::);
  } else {
    stage_wait(sm, bulk);
  }
  __syncthreads();
  if (t < ncta)
    preprocess_bwd_one<T, DEG, NT>(sm, pgn_s, touch_s, t, base + t, cam, kernel, count, merged);
  else
    touch_s[t] = 0;
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  if (!acc) build_live_mask(lm, touch_s);  // (acc: built from the same values above)
  if (red) {
    reduce_block<NT, 3>(out.d_mu + base * 3, ncta, touch_s, lm, mc, [&](int e) { return sm.mu[e]; });
    reduce_block<NT, 3>(out.d_log_scale + base * 3, ncta, touch_s, lm, mc,
                        [&](int e) { return sm.ls[e]; });
    reduce_block<NT, 3>(out.d_normal + base * 3, ncta, touch_s, lm, mc,
                        [&](int e) { return sm.nrm[e]; });
    reduce_block<NT, 4>(out.d_rotation + base * 4, ncta, touch_s, lm, mc,
                        [&](int e) { return sm.rot[e]; });
    reduce_block<NT, 1>(out.d_ra + base, ncta, touch_s, lm, mc, [&](int e) { return sm.ra[e]; });
    reduce_block<NT, 1>(out.d_rb + base, ncta, touch_s, lm, mc, [&](int e) { return sm.rb[e]; });
    reduce_block<NT, 1>(out.pos_grad_norm + base, ncta, touch_s, lm, mc,
                        [&](int e) { return pgn_s[e]; });
    reduce_block<NT, 1>(out.touch + base, ncta, touch_s, lm, mc, [&](int e) { return touch_s[e]; });
    reduce_block<NT, 3 * K>(out.d_sh + base * 3 * K, ncta, touch_s, lm, mc, [&](int e) {
      const int tt = e / (3 * K);
      return sm.sh[tt * St::SHS + (e - tt * 3 * K)];
    });
    // multimem.red is relaxed: release this thread's reductions at system scope
    // before the kernel ends, so the host-side cross-rank barrier that closes the
    // batch (FusedGradientReduce.end) orders them before any rank reads its copy
    if (mc) asm volatile("fence.acq_rel.sys;\n" ::: "memory");
    return;
  }
  store_block<NT, 3>(out.d_mu + base * 3, ncta, acc ? g->mu : nullptr, touch_s, lm,
                     [&](int e) { return sm.mu[e]; });
  store_block<NT, 3>(out.d_log_scale + base * 3, ncta, acc ? g->ls : nullptr, touch_s, lm,
                     [&](int e) { return sm.ls[e]; });
  store_block<NT, 3>(out.d_normal + base * 3, ncta, acc ? g->nrm : nullptr, touch_s, lm,
                     [&](int e) { return sm.nrm[e]; });
  store_block<NT, 4>(out.d_rotation + base * 4, ncta, acc ? g->rot : nullptr, touch_s, lm,
                     [&](int e) { return sm.rot[e]; });
  store_block<NT, 1>(out.d_ra + base, ncta, acc ? g->ra : nullptr, touch_s, lm,
                     [&](int e) { return sm.ra[e]; });
  store_block<NT, 1>(out.d_rb + base, ncta, acc ? g->rb : nullptr, touch_s, lm,
                     [&](int e) { return sm.rb[e]; });
  store_block<NT, 1>(out.pos_grad_norm + base, ncta, acc ? g->pgn : nullptr, touch_s, lm,
                     [&](int e) { return pgn_s[e]; });
  store_block<NT, 1>(out.touch + base, ncta, acc ? g->touch : nullptr, touch_s, lm,
                     [&](int e) { return touch_s[e]; });
  if constexpr ((3 * K) % (16 / sizeof(T)) == 0) {
    store_rows<NT, 3 * K, St::SHS>(out.d_sh + base * 3 * K, ncta, acc ? g->sh : nullptr,
                                   touch_s, lm, sm.sh);
  } else {
    store_block<NT, 3 * K>(out.d_sh + base * 3 * K, ncta, acc ? g->sh : nullptr, touch_s, lm,
                           [&](int e) {
                             const int tt = e / (3 * K);
                             return sm.sh[tt * St::SHS + (e - tt * 3 * K)];
                           });
  }
}


#endif  // HS_GEOMETRY_BWD_TU

// ---------------------------------------------------------------------------
#ifndef HS_GEOMETRY_BWD_TU
template <typename T>
cudaError_t launch_preprocess_fwd_t(const SceneArgs<T>& sc, const CamArgs& cam, int kernel,
                                    int64_t n, float4* rec, SteepRec* side, int4* rect,
                                    int32_t* count, uint64_t* dkey, uint32_t* dval,
                                    int32_t* radii, uint32_t* depth_range, cudaStream_t stream) {
  // staging holds NT primitives in shared memory: 128 float or 64 double ones
  constexpr int NT = sizeof(T) == 4 ? 128 : 64;
  const int64_t grid = (n + NT - 1) / NT;
  switch (sc.deg) {
#define HS_K1(D)                                                                               \
  case D:                                                                                      \
    preprocess_fwd_kernel<T, D, NT><<<(unsigned)grid, NT, 0, stream>>>(sc, cam, kernel, n, rec, \
                                                                       side, rect, count, dkey, \
                                                                       dval, radii,            \
                                                                       depth_range);           \
    break;
    HS_K1(0) HS_K1(1) HS_K1(2) HS_K1(3)
#undef HS_K1
    default: return cudaErrorInvalidValue;
  }
  note_launch();
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_preprocess_fwd_views_t(const SceneArgs<T>& sc, const FwdViewsArgs& va,
                                          int kernel, int64_t n, cudaStream_t stream) {
  constexpr int NT = sizeof(T) == 4 ? 128 : 64;
  const int64_t grid = (n + NT - 1) / NT;
  switch (sc.deg) {
#define HS_K1V(D)                                                                              \
  case D:                                                                                      \
    preprocess_fwd_views_kernel<T, D, NT><<<(unsigned)grid, NT, 0, stream>>>(sc, va, kernel, n); \
    break;
    HS_K1V(0) HS_K1V(1) HS_K1V(2) HS_K1V(3)
#undef HS_K1V
    default: return cudaErrorInvalidValue;
  }
  note_launch();
  return cudaGetLastError();
}
template cudaError_t launch_preprocess_fwd_views_t<float>(const SceneArgs<float>&,
                                                          const FwdViewsArgs&, int, int64_t,
                                                          cudaStream_t);
template cudaError_t launch_preprocess_fwd_views_t<double>(const SceneArgs<double>&,
                                                           const FwdViewsArgs&, int, int64_t,
                                                           cudaStream_t);

template cudaError_t launch_preprocess_fwd_t<float>(const SceneArgs<float>&, const CamArgs&, int,
                                                    int64_t, float4*, SteepRec*, int4*, int32_t*,
                                                    uint64_t*, uint32_t*, int32_t*, uint32_t*,
                                                    cudaStream_t);
template cudaError_t launch_preprocess_fwd_t<double>(const SceneArgs<double>&, const CamArgs&, int,
                                                     int64_t, float4*, SteepRec*, int4*, int32_t*,
                                                     uint64_t*, uint32_t*, int32_t*, uint32_t*,
                                                     cudaStream_t);
#else
template <typename T>
cudaError_t launch_preprocess_bwd_t(const SceneArgs<T>& sc, const CamArgs& cam, int kernel,
                                    int64_t n, int tiles_x, const float4* rec,
                                    const int32_t* row_origin, const int4* rect,
                                    const int32_t* count, const uint32_t* rank_of,
                                    const int32_t* last_rank, const float* rows, float4* merged,
                                    int64_t num_pairs, const GradArgs<T>& out,
                                    cudaStream_t stream) {
  // the launch covers primitives [out.begin, out.end): K7a and K7 over that range only
  const int64_t end = out.end < n ? out.end : n;
  if (end <= out.begin) return cudaSuccess;
  const int64_t cnt = end - out.begin;
  // wide splats (c5: ~134 rows per primitive) take 8 lanes each; at c1-c4
  // (3-4 rows) one lane per splat is faster (measured)
#ifndef HS_K7A_WIDE_ROWS
#define HS_K7A_WIDE_ROWS 32
#endif
  if (num_pairs >= (int64_t)HS_K7A_WIDE_ROWS * n)
    merge_rows_kernel<8><<<(unsigned)((cnt * 8 + 255) / 256), 256, 0, stream>>>(
        end, tiles_x, rec, row_origin, rect, count, rank_of, last_rank, rows, merged, out.begin,
        0);
  else
    merge_rows_kernel<1><<<(unsigned)((cnt + 255) / 256), 256, 0, stream>>>(
        end, tiles_x, rec, row_origin, rect, count, rank_of, last_rank, rows, merged, out.begin,
        0);
  note_launch();
#ifndef HS_K7_NT_F32
#define HS_K7_NT_F32 128
#endif
  constexpr int NT = sizeof(T) == 4 ? HS_K7_NT_F32 : 64;
  const int64_t grid = (cnt + NT - 1) / NT;
  switch (sc.deg) {
#define HS_K7_MODE(D, M)                                                                       \
  {                                                                                            \
    constexpr size_t dyn = M == 1 ? k7_dynamic_smem<T, (D + 1) * (D + 1), NT>() : 0;           \
    if (M == 1) {                                                                              \
      const cudaError_t attr = set_dynamic_smem<preprocess_bwd_kernel<T, D, NT, M>>((int)dyn); \
      if (attr != cudaSuccess) return attr;                                                    \
    }                                                                                          \
    preprocess_bwd_kernel<T, D, NT, M><<<(unsigned)grid, NT, dyn, stream>>>(                  \
        sc, cam, kernel, end, count, merged, out);                                             \
  }
#define HS_K7(D)                                                                               \
  case D:                                                                                      \
    if (out.accumulate == 0) HS_K7_MODE(D, 0)                                                  \
    else if (out.accumulate == 1) HS_K7_MODE(D, 1)                                             \
    else HS_K7_MODE(D, 2)                                                                      \
    break;
    HS_K7(0) HS_K7(1) HS_K7(2) HS_K7(3)
#undef HS_K7
#undef HS_K7_MODE
    default: return cudaErrorInvalidValue;
  }
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// The multi-view K7 (a batch of views of one scene): the CTA stages
// its primitives' parameters once, walks every view's merged rows (hs_merge_rows,
// one 64-B row per primitive and view), runs the geometry backward of each view the
// primitive is visible in and adds the gradients into shared-memory accumulators,
// then stores once.  Against one K7 per view this reads the scene once instead of
// per view and writes the gradient buffer once instead of a read-modify-write per
// view (about 1.5 GB per c4 view).  The sum runs in view order, as GradientSet.add
// (rasterizer.py:100-105) does.
template <typename T, int DEG, int NT, bool RED>
__global__ void __launch_bounds__(NT, HS_K7_MINB) preprocess_bwd_views_kernel(
    SceneArgs<T> sc, ViewsArgs va, int kernel, int64_t n, GradArgs<T> out) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  using St = Staged<T, K, NT>;
  using Ac = AccStage<T, K, NT>;
  __shared__ St sm;
  __shared__ int32_t touch_s[NT];
  __shared__ LiveMask<NT> lm;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  Ac* acc = reinterpret_cast<Ac*>(dyn_smem);
  const int64_t base = out.begin + (int64_t)blockIdx.x * NT;
  const int ncta = (int)(n - base < NT ? n - base : NT);
  const int t = threadIdx.x;
  const bool bulk = stage_in(sm, sc, base, ncta, /*wait=*/false);
  // the accumulators start at zero, or (accumulate == 1: an earlier batch or group of
  // views already wrote) at the stored sums, so every view adds onto the running sum
  // in view order exactly as K7 per view does
  if (out.accumulate == 1) {
    for (int e = t; e < ncta * 3; e += NT) {
      acc->mu[e] = out.d_mu[base * 3 + e];
      acc->ls[e] = out.d_log_scale[base * 3 + e];
      acc->nrm[e] = out.d_normal[base * 3 + e];
    }
    for (int e = t; e < ncta * 4; e += NT) acc->rot[e] = out.d_rotation[base * 4 + e];
    for (int e = t; e < ncta * 3 * K; e += NT) {
      const int tt = e / (3 * K);
      acc->sh[tt * St::SHS + (e - tt * 3 * K)] = out.d_sh[base * 3 * K + e];
    }
    if (t < ncta) {
      acc->ra[t] = out.d_ra[base + t];
      acc->rb[t] = out.d_rb[base + t];
      acc->pgn[t] = out.pos_grad_norm[base + t];
    }
    touch_s[t] = t < ncta ? out.touch[base + t] : 0;
  } else {
    T* z = reinterpret_cast<T*>(acc);
    for (int e = t; e < (int)(sizeof(Ac) / sizeof(T)); e += NT) z[e] = T(0);
    touch_s[t] = 0;
  }
  stage_wait(sm, bulk);
  __syncthreads();
  if (t < ncta)
    for (int v = 0; v < va.n_views; ++v)
      preprocess_bwd_one<T, DEG, NT, true>(sm, nullptr, touch_s, t, base + t, va.cam[v], kernel,
                                           nullptr, va.merged[v], acc);
  __syncthreads();
  build_live_mask(lm, touch_s);
  constexpr bool red = RED;  // the store path compiled alone, as in K7
  const bool mc = RED && out.accumulate == 3;
  if (red) {
    reduce_block<NT, 3>(out.d_mu + base * 3, ncta, touch_s, lm, mc, [&](int e) { return acc->mu[e]; });
    reduce_block<NT, 3>(out.d_log_scale + base * 3, ncta, touch_s, lm, mc,
                        [&](int e) { return acc->ls[e]; });
    reduce_block<NT, 3>(out.d_normal + base * 3, ncta, touch_s, lm, mc,
                        [&](int e) { return acc->nrm[e]; });
    reduce_block<NT, 4>(out.d_rotation + base * 4, ncta, touch_s, lm, mc,
                        [&](int e) { return acc->rot[e]; });
    reduce_block<NT, 1>(out.d_ra + base, ncta, touch_s, lm, mc, [&](int e) { return acc->ra[e]; });
    reduce_block<NT, 1>(out.d_rb + base, ncta, touch_s, lm, mc, [&](int e) { return acc->rb[e]; });
    reduce_block<NT, 1>(out.pos_grad_norm + base, ncta, touch_s, lm, mc,
                        [&](int e) { return acc->pgn[e]; });
    reduce_block<NT, 1>(out.touch + base, ncta, touch_s, lm, mc, [&](int e) { return touch_s[e]; });
    reduce_block<NT, 3 * K>(out.d_sh + base * 3 * K, ncta, touch_s, lm, mc, [&](int e) {
      const int tt = e / (3 * K);
      return acc->sh[tt * St::SHS + (e - tt * 3 * K)];
    });
    if (mc) asm volatile("fence.acq_rel.sys;\n" ::: "memory");
    return;
  }
  // accumulate 0 / 1: the accumulators hold the final values of every primitive
  const T* none = nullptr;
  store_block<NT, 3>(out.d_mu + base * 3, ncta, none, touch_s, lm,
                     [&](int e) { return acc->mu[e]; });
  store_block<NT, 3>(out.d_log_scale + base * 3, ncta, none, touch_s, lm,
                     [&](int e) { return acc->ls[e]; });
  store_block<NT, 3>(out.d_normal + base * 3, ncta, none, touch_s, lm,
                     [&](int e) { return acc->nrm[e]; });
  store_block<NT, 4>(out.d_rotation + base * 4, ncta, none, touch_s, lm,
                     [&](int e) { return acc->rot[e]; });
  store_block<NT, 1>(out.d_ra + base, ncta, none, touch_s, lm,
                     [&](int e) { return acc->ra[e]; });
  store_block<NT, 1>(out.d_rb + base, ncta, none, touch_s, lm,
                     [&](int e) { return acc->rb[e]; });
  store_block<NT, 1>(out.pos_grad_norm + base, ncta, none, touch_s, lm,
                     [&](int e) { return acc->pgn[e]; });
  store_block<NT, 1>(out.touch + base, ncta, (const int32_t*)nullptr, touch_s, lm,
                     [&](int e) { return touch_s[e]; });
  if constexpr ((3 * K) % (16 / sizeof(T)) == 0) {
    store_rows<NT, 3 * K, St::SHS>(out.d_sh + base * 3 * K, ncta, none, touch_s, lm, acc->sh);
  } else {
    store_block<NT, 3 * K>(out.d_sh + base * 3 * K, ncta, none, touch_s, lm, [&](int e) {
      const int tt = e / (3 * K);
      return acc->sh[tt * St::SHS + (e - tt * 3 * K)];
    });
  }
}

template <typename T>
cudaError_t launch_preprocess_bwd_views_t(const SceneArgs<T>& sc, const CamArgs* cams,
                                          const float4* const* merged, int n_views, int kernel,
                                          int64_t n, const GradArgs<T>& out_in,
                                          cudaStream_t stream) {
  const int64_t end = out_in.end < n ? out_in.end : n;
  if (end <= out_in.begin || n_views <= 0) return cudaSuccess;
  const int64_t cnt = end - out_in.begin;
  constexpr int NT = sizeof(T) == 4 ? HS_K7_NT_F32 : 64;
  const int64_t grid = (cnt + NT - 1) / NT;
  for (int v0 = 0; v0 < n_views; v0 += kMaxViews) {
    ViewsArgs va;
    va.n_views = n_views - v0 < kMaxViews ? n_views - v0 : kMaxViews;
    for (int v = 0; v < va.n_views; ++v) {
      va.cam[v] = cams[v0 + v];
      va.merged[v] = merged[v0 + v];
    }
    GradArgs<T> out = out_in;
    if (v0 > 0 && out.accumulate == 0) out.accumulate = 1;  // later groups add
    switch (sc.deg) {
#define HS_K7V(D)                                                                              \
  case D: {                                                                                    \
    constexpr size_t dyn = sizeof(AccStage<T, (D + 1) * (D + 1), NT>);                          \
    if (out.accumulate >= 2) {                                                                 \
      const cudaError_t attr =                                                                 \
          set_dynamic_smem<preprocess_bwd_views_kernel<T, D, NT, true>>((int)dyn);             \
      if (attr != cudaSuccess) return attr;                                                    \
      preprocess_bwd_views_kernel<T, D, NT, true><<<(unsigned)grid, NT, dyn, stream>>>(        \
          sc, va, kernel, end, out);                                                           \
    } else {                                                                                   \
      const cudaError_t attr =                                                                 \
          set_dynamic_smem<preprocess_bwd_views_kernel<T, D, NT, false>>((int)dyn);            \
      if (attr != cudaSuccess) return attr;                                                    \
      preprocess_bwd_views_kernel<T, D, NT, false><<<(unsigned)grid, NT, dyn, stream>>>(       \
          sc, va, kernel, end, out);                                                           \
    }                                                                                          \
    break;                                                                                     \
  }
      HS_K7V(0) HS_K7V(1) HS_K7V(2) HS_K7V(3)
#undef HS_K7V
      default: return cudaErrorInvalidValue;
    }
    note_launch();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
template cudaError_t launch_preprocess_bwd_views_t<float>(const SceneArgs<float>&, const CamArgs*,
                                                          const float4* const*, int, int, int64_t,
                                                          const GradArgs<float>&, cudaStream_t);
template cudaError_t launch_preprocess_bwd_views_t<double>(const SceneArgs<double>&,
                                                           const CamArgs*, const float4* const*,
                                                           int, int, int64_t,
                                                           const GradArgs<double>&, cudaStream_t);

// K7a alone into a caller buffer with culled markers (hs_merge_rows)
cudaError_t launch_merge_rows(int64_t n, int tiles_x, const float4* rec,
                              const int32_t* row_origin, const int4* rect,
                              const int32_t* count, const uint32_t* rank_of,
                              const int32_t* last_rank, const float* rows, float4* merged,
                              int64_t num_pairs, cudaStream_t stream) {
  if (num_pairs >= (int64_t)HS_K7A_WIDE_ROWS * n)
    merge_rows_kernel<8><<<(unsigned)((n * 8 + 255) / 256), 256, 0, stream>>>(
        n, tiles_x, rec, row_origin, rect, count, rank_of, last_rank, rows, merged, 0, 1);
  else
    merge_rows_kernel<1><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(
        n, tiles_x, rec, row_origin, rect, count, rank_of, last_rank, rows, merged, 0, 1);
  note_launch();
  return cudaGetLastError();
}

template cudaError_t launch_preprocess_bwd_t<float>(const SceneArgs<float>&, const CamArgs&, int,
                                                    int64_t, int, const float4*, const int32_t*,
                                                    const int4*,
                                                    const int32_t*, const uint32_t*, const int32_t*,
                                                    const float*, float4*, int64_t,
                                                    const GradArgs<float>&, cudaStream_t);
template cudaError_t launch_preprocess_bwd_t<double>(const SceneArgs<double>&, const CamArgs&, int,
                                                     int64_t, int, const float4*, const int32_t*,
                                                     const int4*,
                                                     const int32_t*, const uint32_t*,
                                                     const int32_t*, const float*, float4*,
                                                     int64_t, const GradArgs<double>&,
                                                     cudaStream_t);
#endif  // HS_GEOMETRY_BWD_TU

}  // namespace hs
