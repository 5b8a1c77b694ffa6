// hs_io.cu -- scene I/O on the device: the PLY vertex payload (one row per
// half-Gaussian pair, properties interleaved) <-> the scene's struct-of-arrays
// tensors (scene_io.py:136-269).
//
// The host moves the raw payload in ONE contiguous copy; these kernels do the
// (de)interleave, the per-property type conversion and the SH transpose
// (f_rest is channel-major in the file, coefficient-major in the scene).  A CTA
// stages kRows rows through shared memory so that both the row-major payload and
// the per-field outputs are read / written coalesced.
//
//   U  ply_unpack   payload (any of float / double / uchar / int per property)
//                   -> scene fields; a column map gives each scene component's
//                   source property (load_scene 171-197, import_3dgs 200-239)
//   P  ply_pack     scene fields -> payload rows of float or double in the
//                   native order (save_scene 136-168) or the 3D-GS order with
//                   zero normals and the alpha-collapsed opacity
//                   logit(clip((a1 + a2) / 2, 1e-6, 1 - 1e-6)) (export_3dgs
//                   242-269)
#include <cmath>
#include <cstdint>

#include "hs_common.cuh"
#include "hs_internal.h"
#include "hs_numpy_order.cuh"

namespace hs {

constexpr int kIoRows = 32;      // rows staged per CTA
constexpr int kIoThreads = 256;

// CTA-cooperative copy: 16-B pieces when both ends are 16-B aligned, bytes for
// the tail (a CTA's payload block starts at a multiple of 32 rows).
__device__ __forceinline__ void cta_copy(unsigned char* dst, const unsigned char* src, int bytes) {
  int done = 0;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const int nv = bytes / 16;
    for (int v = threadIdx.x; v < nv; v += kIoThreads)
      reinterpret_cast<uint4*>(dst)[v] = reinterpret_cast<const uint4*>(src)[v];
    done = nv * 16;
  }
  for (int b = done + threadIdx.x; b < bytes; b += kIoThreads) dst[b] = src[b];
}

__device__ __forceinline__ double load_prop(const unsigned char* row, int off, int type) {
  switch (type) {
    case kPlyF32: { float v; memcpy(&v, row + off, 4); return (double)v; }
    case kPlyF64: { double v; memcpy(&v, row + off, 8); return v; }
    case kPlyU8: return (double)row[off];
    default: { int32_t v; memcpy(&v, row + off, 4); return (double)v; }
  }
}

// Scene component c of a row (components in field order: mu 3, log_scale 3,
// rotation 4, sh 3K (k, channel), normal 3, ra, rb) -> (field, index in row).
struct CompRef {
  int field, idx, width;
};
__device__ __forceinline__ CompRef comp_ref(int c, int K3) {
  const int w[7] = {3, 3, 4, K3, 3, 1, 1};
  int f = 0;
  while (c >= w[f]) c -= w[f++];
  return {f, c, w[f]};
}

template <typename T>
__global__ void __launch_bounds__(kIoThreads) ply_unpack_kernel(PlyUnpackArgs a, SceneOut<T> out) {
  extern __shared__ __align__(16) unsigned char rows[];
  const int64_t r0 = (int64_t)blockIdx.x * kIoRows;
  const int nr = (int)(a.n - r0 < kIoRows ? a.n - r0 : kIoRows);
  const unsigned char* src = static_cast<const unsigned char*>(a.payload) + r0 * a.stride;
  cta_copy(rows, src, nr * a.stride);
  __syncthreads();
  const int K3 = 3 * a.K;
  const int ncomp = 3 + 3 + 4 + K3 + 3 + 1 + 1;
  T* fields[7] = {out.mu, out.ls, out.rot, out.sh, out.nrm, out.ra, out.rb};
  // consecutive threads: consecutive rows of one component -> coalesced per field
  for (int e = threadIdx.x; e < nr * ncomp; e += kIoThreads) {
    const int c = e / nr, r = e - c * nr;
    const CompRef cr = comp_ref(c, K3);
    const int col = a.column[c];
    if (col < 0) continue;  // left to the caller (e.g. import_3dgs normals)
    const double v = load_prop(rows + r * a.stride, a.offset[col], a.type[col]);
    fields[cr.field][(r0 + r) * cr.width + cr.idx] = (T)v;
  }
}

// export_3dgs opacity (scene_io.py:246-250): logit of the clipped mean alpha
__device__ __forceinline__ double collapsed_logit(double ra, double rb) {
  double p = 0.5 * (sigmoid_ref(ra) + sigmoid_ref(rb));
  p = fmin(fmax(p, 1e-6), 1 - 1e-6);  // np.clip
  return log(p) - log1p(-p);          // logit, geometry.py:355-358
}

template <typename T, typename O>
__global__ void __launch_bounds__(kIoThreads) ply_pack_kernel(PlyPackArgs a, SceneIn<T> in) {
  extern __shared__ __align__(16) unsigned char rows[];
  const int64_t r0 = (int64_t)blockIdx.x * kIoRows;
  const int nr = (int)(a.n - r0 < kIoRows ? a.n - r0 : kIoRows);
  const int K = a.K, nrest = 3 * (K - 1);
  // native: x y z nx ny nz f_dc_0..2 f_rest_* opacity opacity_2 scale_0..2 rot_0..3
  // 3dgs:   same with one opacity (collapsed) and zero normals
  const int ncol = 9 + nrest + (a.gs3d ? 1 : 2) + 3 + 4;
  O* orow = reinterpret_cast<O*>(rows);
  for (int e = threadIdx.x; e < nr * ncol; e += kIoThreads) {
    const int col = e / nr, r = e - col * nr;
    const int64_t i = r0 + r;
    double v;
    if (col < 3) {
      v = in.mu[3 * i + col];
    } else if (col < 6) {
      v = a.gs3d ? 0.0 : (double)in.nrm[3 * i + col - 3];
    } else if (col < 9) {
      v = in.sh[3 * K * i + (col - 6)];  // coefficient 0, channel col-6
    } else if (col < 9 + nrest) {
      // f_rest channel-major: j = channel * (K-1) + (k-1)
      const int j = col - 9, ch = j / (K - 1), k = 1 + j - ch * (K - 1);
      v = in.sh[3 * K * i + 3 * k + ch];
    } else {
      int c = col - 9 - nrest;
      if (a.gs3d) {
        if (c == 0) {
          v = a.opacity_first ? (double)in.ra[i] : collapsed_logit(in.ra[i], in.rb[i]);
          goto store;
        }
        c += 1;  // skip opacity_2
      }
      if (c == 0)
        v = in.ra[i];
      else if (c == 1)
        v = in.rb[i];
      else if (c < 5)
        v = in.ls[3 * i + c - 2];
      else
        v = in.rot[4 * i + c - 5];
    }
  store:
    orow[r * ncol + col] = (O)v;
  }
  __syncthreads();
  unsigned char* dst = static_cast<unsigned char*>(a.payload) + r0 * ncol * (int64_t)sizeof(O);
  cta_copy(dst, rows, nr * ncol * (int)sizeof(O));
}

cudaError_t launch_ply_unpack(const PlyUnpackArgs& a, const void* const* fields, int dtype,
                              cudaStream_t s) {
  const unsigned grid = (unsigned)((a.n + kIoRows - 1) / kIoRows);
  const size_t smem = (size_t)kIoRows * a.stride;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;  // rows wider than ~6 KB
  constexpr int kMaxSmem = 200 * 1024;
  if (dtype == 0) {
    auto k = ply_unpack_kernel<float>;
    const cudaError_t e = set_dynamic_smem<ply_unpack_kernel<float>>(kMaxSmem);
    if (e != cudaSuccess) return e;
    SceneOut<float> o{(float*)fields[0], (float*)fields[1], (float*)fields[2], (float*)fields[3],
                      (float*)fields[4], (float*)fields[5], (float*)fields[6]};
    k<<<grid, kIoThreads, smem, s>>>(a, o);
  } else {
    auto k = ply_unpack_kernel<double>;
    const cudaError_t e = set_dynamic_smem<ply_unpack_kernel<double>>(kMaxSmem);
    if (e != cudaSuccess) return e;
    SceneOut<double> o{(double*)fields[0], (double*)fields[1], (double*)fields[2],
                       (double*)fields[3], (double*)fields[4], (double*)fields[5],
                       (double*)fields[6]};
    k<<<grid, kIoThreads, smem, s>>>(a, o);
  }
  note_launch();
  return cudaGetLastError();
}

template <typename T>
static cudaError_t pack_t(const PlyPackArgs& a, const void* const* f, cudaStream_t s) {
  const SceneIn<T> in{(const T*)f[0], (const T*)f[1], (const T*)f[2], (const T*)f[3],
                      (const T*)f[4], (const T*)f[5], (const T*)f[6]};
  const int ncol = 9 + 3 * (a.K - 1) + (a.gs3d ? 1 : 2) + 7;
  const unsigned grid = (unsigned)((a.n + kIoRows - 1) / kIoRows);
  if (a.out_f64) {
    const size_t smem = (size_t)kIoRows * ncol * 8;
    auto k = ply_pack_kernel<T, double>;
    const cudaError_t e = set_dynamic_smem<ply_pack_kernel<T, double>>((int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, kIoThreads, smem, s>>>(a, in);
  } else {
    const size_t smem = (size_t)kIoRows * ncol * 4;
    auto k = ply_pack_kernel<T, float>;
    const cudaError_t e = set_dynamic_smem<ply_pack_kernel<T, float>>((int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, kIoThreads, smem, s>>>(a, in);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_ply_pack(const PlyPackArgs& a, const void* const* fields, int dtype,
                            cudaStream_t s) {
  return dtype == 0 ? pack_t<float>(a, fields, s) : pack_t<double>(a, fields, s);
}

}  // namespace hs
