// hs_binning.cu -- depth-rank sort (K3a), pair counts and their scan,
// duplicate-with-keys (K2), the stable tile sort (K3b) and tile ranges (K4);
// plus the FrameGeometry export used by the parity tests.
//
// The reference orders pairs with np.lexsort((prim index, depth f64, tile))
// (rasterizer.py:318-323).  Here the primitives are first ranked once by
// (depth f64 bits, index) with a stable 64-bit radix sort, pairs are emitted in
// that rank order, and a stable radix sort on the tile id alone (tile_bits =
// ceil(log2 n_tiles) bits, two 8-bit passes at 1080p) yields exactly the
// lexsort order without ever materialising a 64-bit (tile|depth) key.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

size_t depth_sort_temp_bytes(int64_t n) {
  size_t bytes = 0, hi = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 64);
  cub::DeviceRadixSort::SortPairs(nullptr, hi, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 32, 64);
  return bytes > hi ? bytes : hi;
}

size_t scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                (int)(n + 1));
  return bytes;
}

size_t pair_sort_temp_bytes(int64_t p, int tile_bits) {
  size_t bytes = 0;
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr), v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, (int)(p > 0 ? p : 1), 0,
                                  tile_bits > 0 ? tile_bits : 1);
  return bytes;
}

cudaError_t run_depth_sort(void* temp, size_t temp_bytes, const uint64_t* keys_in,
                           uint64_t* keys_out, const uint32_t* vals_in, uint32_t* order,
                           int64_t n, cudaStream_t stream) {
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in,
                                                  order, (int)n, 0, 64, stream);
  note_launch(9);  // onesweep: histogram + one pass per 8-bit digit
  return e;
}

// Depth ranks in two steps (the default; run_depth_sort is the fallback).  A
// stable sort on the upper 32 bits of the f64 depth (4 one-sweep passes instead
// of 8) leaves splats whose depths share those bits -- a bucket 2^-20 of the
// depth wide -- in index order.  Each such run is then put in full-key order:
// every element counts the run's elements that precede it in (full key, current
// position) order -- its rank in the run, a stable order, so equal depths keep
// index order as np.lexsort's tie-break does -- and a second kernel scatters the
// run into those ranks.  Runs are about one splat long at c3 and ~200 in c5's
// clustered depths (O(run) work per element, all in parallel).  A run longer
// than kMaxDepthRun sets *overflow and the host redoes the full 64-bit sort
// (hs_frame_read_num_pairs).  Culled splats share the key ~0 and are already in
// index order.
#ifndef HS_MAX_DEPTH_RUN
#define HS_MAX_DEPTH_RUN 2048
#endif
constexpr int kMaxDepthRun = HS_MAX_DEPTH_RUN;

// newpos[k] = position of sorted element k after its run is ordered by the full
// key; val[k] = its order value (copied, so the scatter does not race)
__global__ void depth_run_rank_kernel(const uint64_t* __restrict__ keys,
                                      const uint32_t* __restrict__ order, int64_t n,
                                      uint32_t* __restrict__ newpos, uint32_t* __restrict__ val,
                                      int* __restrict__ overflow) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint64_t key = keys[k];
  const uint32_t hi = (uint32_t)(key >> 32);
  val[k] = order[k];
  if (hi == 0xffffffffu) {  // culled
    newpos[k] = (uint32_t)k;
    return;
  }
  // The run's bounds by galloping then bisecting over the sorted upper bits:
  // O(log run) dependent loads instead of O(run).  s = first index >= lo with
  // this hi; e = first index in (k, cap) with another hi, else cap -- the same
  // bounds a linear walk capped at kMaxDepthRun finds.
  auto same = [&](int64_t j) { return (uint32_t)(keys[j] >> 32) == hi; };
  const int64_t lo = k - kMaxDepthRun > 0 ? k - kMaxDepthRun : 0;
  int64_t good = k, bad = lo - 1;
  for (int64_t step = 1;; step <<= 1) {
    const int64_t c = good - step;
    if (c < lo) break;
    if (same(c)) {
      good = c;
    } else {
      bad = c;
      break;
    }
  }
  while (good - bad > 1) {
    const int64_t mid = bad + (good - bad) / 2;
    if (same(mid)) good = mid; else bad = mid;
  }
  const int64_t s = good;
  const int64_t cap = s + kMaxDepthRun + 1 < n ? s + kMaxDepthRun + 1 : n;
  int64_t in = k, out = cap;  // same(in); out = cap or an index with another hi
  for (int64_t step = 1;; step <<= 1) {
    const int64_t c = in + step;
    if (c >= cap) break;
    if (same(c)) {
      in = c;
    } else {
      out = c;
      break;
    }
  }
  while (out - in > 1) {
    const int64_t mid = in + (out - in) / 2;
    if (same(mid)) in = mid; else out = mid;
  }
  const int64_t e = out;
  if (e - s > kMaxDepthRun || k - s >= kMaxDepthRun) {
    atomicExch(overflow, 1);
    newpos[k] = (uint32_t)k;
    return;
  }
  int64_t r = 0;
  for (int64_t j = s; j < e; ++j) {
    const uint64_t kj = keys[j];
    r += (kj < key || (kj == key && j < k)) ? 1 : 0;
  }
  newpos[k] = (uint32_t)(s + r);
}

__global__ void depth_run_scatter_kernel(const uint32_t* __restrict__ newpos,
                                         const uint32_t* __restrict__ val, int64_t n,
                                         uint32_t* __restrict__ order) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) order[newpos[k]] = val[k];
}

cudaError_t run_depth_sort_hi(void* temp, size_t temp_bytes, const uint64_t* keys_in,
                              uint64_t* keys_out, const uint32_t* vals_in, uint32_t* order,
                              int64_t n, uint32_t* scratch_pos, uint32_t* scratch_val,
                              int* overflow, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(overflow, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, order, (int)n,
                                      32, 64, stream);
  note_launch(5);
  if (e != cudaSuccess) return e;
  const int block = 256;
  const unsigned grid = (unsigned)((n + block - 1) / block);
  depth_run_rank_kernel<<<grid, block, 0, stream>>>(keys_out, order, n, scratch_pos, scratch_val,
                                                    overflow);
  depth_run_scatter_kernel<<<grid, block, 0, stream>>>(scratch_pos, scratch_val, n, order);
  note_launch(2);
  return cudaGetLastError();
}

__global__ void gather_counts_kernel(const int32_t* __restrict__ count,
                                     const uint32_t* __restrict__ order, int32_t* __restrict__ cnt_r,
                                     uint32_t* __restrict__ rank_of, int64_t n) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r > n) return;
  if (r == n) {
    cnt_r[n] = 0;
    return;
  }
  const uint32_t i = order[r] & kIndexMask;
  cnt_r[r] = count[i];
  rank_of[i] = (uint32_t)r;
}

cudaError_t run_count_scan(void* temp, size_t temp_bytes, const int32_t* count,
                           const uint32_t* order, int32_t* cnt_r, int32_t* off_r,
                           uint32_t* rank_of, int64_t n, cudaStream_t stream) {
  const int block = 256;
  gather_counts_kernel<<<(unsigned)((n + 1 + block - 1) / block), block, 0, stream>>>(
      count, order, cnt_r, rank_of, n);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, cnt_r, off_r, (int)(n + 1), stream);
  note_launch(2);
  return e;
}

// K2: one thread per depth rank; a splat's pairs are contiguous, row-major over
// its tile rect (the reference's `local % spans_x` order, rasterizer.py:312-317),
// and splats appear in depth-rank order.
// One warp per 32 consecutive depth ranks.  Their pairs form one contiguous run
// of the output (off_r is the exclusive scan in rank order), so the warp writes
// that run with consecutive lanes on consecutive pairs: each lane finds the
// splat owning pair j by a binary search over the warp's exclusive counts
// (shuffles) and the tile from the pair's index inside the splat's rect.
__global__ void __launch_bounds__(256) duplicate_kernel(
    const uint32_t* __restrict__ order, const int32_t* __restrict__ cnt_r,
    const int32_t* __restrict__ off_r, const int4* __restrict__ rect, float* __restrict__ rec,
    int tiles_x, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t r0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane;
  if (r0 >= n) return;  // whole warp
  const int64_t r = r0 + lane;
  const int c = r < n ? cnt_r[r] : 0;
  uint32_t v = 0;
  int4 rc = make_int4(0, 0, 0, 0);
  int spans_x = 1;
  if (c > 0) {
    v = order[r];  // index | steep flag, carried into the pair value
    const uint32_t i = v & kIndexMask;
    rc = rect[i];
    spans_x = rc.y - rc.x + 1;
    rec[(size_t)i * kRecordFloats + R_ROW_ORIGIN] =
        __int_as_float(off_r[r] - rc.z * spans_x - rc.x);
  }
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int excl = incl - c;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  const int64_t wbase = __shfl_sync(0xffffffffu, r < n ? (int64_t)off_r[r] : 0, 0);
  for (int j0 = 0; j0 < total; j0 += 32) {
    const int j = j0 + lane;
    // largest s with excl[s] <= j (splats with c == 0 share their successor's
    // excl and are skipped by taking the largest)
    int sidx = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int cand = sidx + step;
      const int e = __shfl_sync(0xffffffffu, excl, cand & 31);
      if (cand < 32 && e <= j) sidx = cand;
    }
    const int es = __shfl_sync(0xffffffffu, excl, sidx);
    const int sx = __shfl_sync(0xffffffffu, spans_x, sidx);
    const int x0 = __shfl_sync(0xffffffffu, rc.x, sidx);
    const int y0 = __shfl_sync(0xffffffffu, rc.z, sidx);
    const uint32_t vs = __shfl_sync(0xffffffffu, v, sidx);
    if (j < total) {
      const int l = j - es, ly = l / sx, lx = l - ly * sx;
      keys[wbase + j] = (uint32_t)(y0 + ly) * (uint32_t)tiles_x + (uint32_t)(x0 + lx);
      vals[wbase + j] = vs;
    }
  }
}

cudaError_t run_duplicate(const uint32_t* order, const int32_t* cnt_r, const int32_t* off_r,
                          const int4* rect, float4* rec, int tiles_x, uint32_t* keys,
                          uint32_t* vals, int64_t n, cudaStream_t stream) {
  const int block = 256;
  duplicate_kernel<<<(unsigned)((n + block - 1) / block), block, 0, stream>>>(
      order, cnt_r, off_r, rect, reinterpret_cast<float*>(rec), tiles_x, keys, vals, n);
  note_launch();
  return cudaGetLastError();
}

cudaError_t run_pair_sort(void* temp, size_t temp_bytes, uint32_t* keys0, uint32_t* keys1,
                          uint32_t* vals0, uint32_t* vals1, int64_t p, int tile_bits,
                          int* selector, cudaStream_t stream) {
  cub::DoubleBuffer<uint32_t> k(keys0, keys1), v(vals0, vals1);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, (int)p, 0,
                                                  tile_bits > 0 ? tile_bits : 1, stream);
  note_launch(1 + (tile_bits + 7) / 8);
  *selector = k.selector;
  return e;
}

// K4: CSR tile offsets (np.searchsorted(tile_sorted, arange(T+1)),
// rasterizer.py:324-325).  Every entry is written exactly once.
// K4: tile_starts[u] = first sorted pair of tile >= u.  Each thread takes four
// consecutive keys with one 16-B load (the sorted keys come from CUB's 256-B
// aligned buffers) and writes the starts of the tiles that begin at them.
__device__ __forceinline__ void tile_starts_at(int64_t k, int t, int& prev,
                                               int32_t* __restrict__ starts) {
  for (int u = prev + 1; u <= t; ++u) starts[u] = (int32_t)k;
  prev = t;
}

__global__ void tile_ranges_kernel(const uint32_t* __restrict__ keys, int64_t p, int n_tiles,
                                   int32_t* __restrict__ starts) {
  const int64_t k0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (k0 >= p) return;
  int prev = k0 == 0 ? -1 : (int)keys[k0 - 1];
  if (k0 + 4 <= p && !((uintptr_t)keys & 15)) {
    const uint4 v = reinterpret_cast<const uint4*>(keys)[k0 >> 2];
    tile_starts_at(k0, (int)v.x, prev, starts);
    tile_starts_at(k0 + 1, (int)v.y, prev, starts);
    tile_starts_at(k0 + 2, (int)v.z, prev, starts);
    tile_starts_at(k0 + 3, (int)v.w, prev, starts);
  } else {
    for (int64_t k = k0; k < p && k < k0 + 4; ++k) tile_starts_at(k, (int)keys[k], prev, starts);
  }
  if (k0 + 4 >= p)  // the thread holding the last pair closes the table
    for (int u = prev + 1; u <= n_tiles; ++u) starts[u] = (int32_t)p;
}

__global__ void fill_i32_kernel(int32_t* __restrict__ a, int64_t n, int32_t v) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) a[k] = v;
}

cudaError_t run_tile_ranges(const uint32_t* sorted_keys, int64_t p, int n_tiles,
                            int32_t* tile_starts, cudaStream_t stream) {
  const int block = 256;
  if (p == 0) {
    fill_i32_kernel<<<(unsigned)((n_tiles + 1 + block - 1) / block), block, 0, stream>>>(
        tile_starts, n_tiles + 1, 0);
  } else {
    const int64_t threads = (p + 3) / 4;
    tile_ranges_kernel<<<(unsigned)((threads + block - 1) / block), block, 0, stream>>>(
        sorted_keys, p, n_tiles, tile_starts);
  }
  note_launch();
  return cudaGetLastError();
}

// ---- FrameGeometry export (introspection / parity only) ------------------
__global__ void visible_flags_kernel(const int32_t* __restrict__ count, int32_t* __restrict__ flags,
                                     int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  flags[i] = (i < n && count[i] > 0) ? 1 : 0;
}

__global__ void export_splats_kernel(const int32_t* __restrict__ count,
                                     const int32_t* __restrict__ local_of,
                                     const float4* __restrict__ rec, const int4* __restrict__ rect,
                                     int64_t n, int32_t* __restrict__ valid,
                                     int64_t* __restrict__ m_out, float* __restrict__ packed,
                                     int8_t* __restrict__ mode, int32_t* __restrict__ tile_rect) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == n - 1) *m_out = (int64_t)local_of[n];
  if (count[i] == 0) return;
  const int64_t l = local_of[i];
  if (valid) valid[l] = (int32_t)i;
  const float* r = reinterpret_cast<const float*>(rec + 4 * i);
  if (packed) {
    for (int c = 0; c < 13; ++c) packed[l * 13 + c] = r[c];
    // large splats carry the stable conic form (hs_common.cuh kFlagNoWin)
    conic_abc(r[R_CA], r[R_CB], r[R_CC], __float_as_uint(r[R_FLAGS]), packed[l * 13 + R_CB],
              packed[l * 13 + R_CC]);
  }
  if (mode) mode[l] = (int8_t)(__float_as_uint(r[R_FLAGS]) & 3u);
  if (tile_rect) {
    const int4 rc = rect[i];
    tile_rect[4 * l + 0] = rc.x;
    tile_rect[4 * l + 1] = rc.y;
    tile_rect[4 * l + 2] = rc.z;
    tile_rect[4 * l + 3] = rc.w;
  }
}

__global__ void export_pairs_kernel(const uint32_t* __restrict__ pair_src,
                                    const int32_t* __restrict__ local_of, int64_t p,
                                    int32_t* __restrict__ pair_splat) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < p) pair_splat[k] = local_of[pair_src[k] & kIndexMask];
}

__global__ void widen_kernel(const int32_t* __restrict__ a, int64_t* __restrict__ b, int64_t n) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) b[k] = a[k];
}

cudaError_t run_export(void* temp, size_t temp_bytes, const int32_t* count, const float4* rec,
                       const int4* rect, const uint32_t* pair_src, const int32_t* tile_starts32,
                       int64_t n, int64_t p, int n_tiles, int32_t* local_of, int32_t* flags,
                       int32_t* valid, int64_t* m_out, float* packed, int8_t* mode, int32_t* tile_rect,
                       int32_t* pair_splat, int64_t* tile_starts, cudaStream_t stream) {
  const int block = 256;
  visible_flags_kernel<<<(unsigned)((n + 1 + block - 1) / block), block, 0, stream>>>(count, flags,
                                                                                      n);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, flags, local_of, (int)(n + 1),
                                                stream);
  if (e != cudaSuccess) return e;
  export_splats_kernel<<<(unsigned)((n + block - 1) / block), block, 0, stream>>>(
      count, local_of, rec, rect, n, valid, m_out, packed, mode, tile_rect);
  if (pair_splat && p > 0)
    export_pairs_kernel<<<(unsigned)((p + block - 1) / block), block, 0, stream>>>(
        pair_src, local_of, p, pair_splat);
  if (tile_starts)
    widen_kernel<<<(unsigned)((n_tiles + 1 + block - 1) / block), block, 0, stream>>>(
        tile_starts32, tile_starts, n_tiles + 1);
  note_launch(5);
  return cudaGetLastError();
}

}  // namespace hs
