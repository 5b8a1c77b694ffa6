// hs_binning.cu -- depth-rank sort (K3a), pair counts and their scan, and the
// tile binning: duplicate-with-keys (K2) fused with a stable two-level counting
// sort by tile (row buckets, then columns) that also yields the tile ranges (K4);
// plus the FrameGeometry export used by the parity tests.
//
// The reference orders pairs with np.lexsort((prim index, depth f64, tile))
// (rasterizer.py:318-323).  Here the primitives are first ranked once by
// (depth f64 bits, index), pairs are generated in that rank order, and a STABLE
// sort on the tile id alone yields exactly the lexsort order without ever
// materialising a 64-bit (tile|depth) key.  The stable tile sort is the
// row-bucket counting sort below (no host round trip: P stays on the device);
// images wider than kBinMaxCols or taller than kBinMaxRows tiles use a CUB radix
// sort on the tile id after a host read of P instead.
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
  size_t k24 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, k24, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0,
                                  kDepthKeyBits);
  if (k24 > bytes) bytes = k24;
  return bytes > hi ? bytes : hi;
}

size_t scan_temp_bytes(int64_t n) {  // n scan entries
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                (int)n);
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
// key; val[k] = its order value (copied, so the scatter does not race).  The runs
// are runs of equal 24-bit keys (= equal upper 32 bits of the depth, see
// depth_key24_kernel); the full keys are read from the unsorted array by index.
__global__ void depth_run_rank_kernel(const uint32_t* __restrict__ key24,
                                      const uint64_t* __restrict__ full,
                                      const uint32_t* __restrict__ order, int64_t n,
                                      uint32_t* __restrict__ newpos, uint32_t* __restrict__ val,
                                      int* __restrict__ overflow) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t hk = key24[k];
  const uint32_t vk = order[k];
  val[k] = vk;
  if (hk == kDepthKeyCulled) {  // culled: one run, already in index order
    newpos[k] = (uint32_t)k;
    return;
  }
  // The run's bounds by galloping then bisecting over the sorted keys: O(log run)
  // dependent loads instead of O(run).  s = first index >= lo with this key; e =
  // first index in (k, cap) with another key, else cap -- the same bounds a linear
  // walk capped at kMaxDepthRun finds.
  auto same = [&](int64_t j) { return key24[j] == hk; };
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
  int64_t in = k, out = cap;  // same(in); out = cap or an index with another key
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
  if (e - s == 1) {  // the usual case: a run of one
    newpos[k] = (uint32_t)k;
    return;
  }
  const uint64_t key = full[vk & kIndexMask];
  int64_t r = 0;
  // (independent iterations: unrolled so several gathers are in flight)
#pragma unroll 8
  for (int64_t j = s; j < e; ++j) {
    const uint64_t kj = full[order[j] & kIndexMask];
    r += (kj < key || (kj == key && j < k)) ? 1 : 0;
  }
  newpos[k] = (uint32_t)(s + r);
}

// The sort key: the upper 32 bits of a visible splat's f64 depth minus the
// frame's smallest (K1 reduces the range), which fits 24 bits unless the depths
// span a factor ~2^16 -- then the overflow flag sends the frame to the full
// 64-bit sort (the clamped keys would still rank right while the farthest run
// fits the fixup).  Culled splats take the largest key.  3 radix passes of 8 bits on
// 4-byte keys instead of 4 passes on 8-byte ones.
__global__ void depth_key24_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                   const uint32_t* __restrict__ range, uint32_t* __restrict__ out,
                                   int* __restrict__ overflow) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t lo = range[0], hi_max = range[1];
  if (k == 0 && lo <= hi_max && hi_max - lo >= kDepthKeyCulled) atomicExch(overflow, 1);
  const uint32_t hi = (uint32_t)(keys[k] >> 32);
  if (hi == 0xffffffffu) {
    out[k] = kDepthKeyCulled;
    return;
  }
  const uint32_t d = hi - lo;
  out[k] = d < kDepthKeyCulled ? d : kDepthKeyCulled - 1;
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
                              int* overflow, const uint32_t* range, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(overflow, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  const int block = 256;
  const unsigned grid = (unsigned)((n + block - 1) / block);
  // keys_out (8 bytes per splat) holds the 24-bit keys, unsorted then sorted
  uint32_t* k24_in = reinterpret_cast<uint32_t*>(keys_out);
  uint32_t* k24_out = k24_in + n;
  depth_key24_kernel<<<grid, block, 0, stream>>>(keys_in, n, range, k24_in, overflow);
  e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k24_in, k24_out, vals_in, order, (int)n, 0,
                                      kDepthKeyBits, stream);
  note_launch(5);
  if (e != cudaSuccess) return e;
  depth_run_rank_kernel<<<grid, block, 0, stream>>>(k24_out, keys_in, order, n, scratch_pos,
                                                    scratch_val, overflow);
  depth_run_scatter_kernel<<<grid, block, 0, stream>>>(scratch_pos, scratch_val, n, order);
  note_launch(3);
  return cudaGetLastError();
}

// cnt_r[r] = count[order[r]] and rank_of; P accumulates as int64 next to the
// int32 scan (which may wrap).  With the segment path (SEGS) each CTA -- one
// block of kBinRanks ranks, 4 per thread -- also histograms its segments by
// (tile row, column block) key into cnt_r[n + 1 + key * nb + block] and adds its
// pairs per key into key_pairs.
template <bool SEGS>
__global__ void __launch_bounds__(kBinThreads) gather_counts_kernel(
    const int32_t* __restrict__ count, const uint32_t* __restrict__ order,
    const int4* __restrict__ rect, int32_t* __restrict__ cnt_r, uint32_t* __restrict__ rank_of,
    int64_t n, int tiles_y, int nblk, int32_t* __restrict__ key_pairs,
    BinStatusDev* __restrict__ status, int4* __restrict__ rect_r) {
  extern __shared__ int smem_cnt[];  // [keys] segments, then [keys] pairs
  __shared__ long long csum[kBinThreads / 32][2];
  const int keys = tiles_y * nblk;
  int* keys_s = smem_cnt;
  int* pairs_s = smem_cnt + keys;
  if (SEGS) {
    for (int e = threadIdx.x; e < 2 * keys; e += kBinThreads) smem_cnt[e] = 0;
    __syncthreads();
  }
  long long v = 0, vs = 0;
#pragma unroll
  for (int q = 0; q < kBinRanks / kBinThreads; ++q) {
    const int64_t r = (int64_t)blockIdx.x * kBinRanks + q * kBinThreads + threadIdx.x;
    if (r >= n) continue;
    const uint32_t i = order[r] & kIndexMask;
    const int c = count[i];
    cnt_r[r] = c;
    rank_of[i] = (uint32_t)r;
    v += c;
    if (SEGS && c > 0) {
      const int4 rc = rect[i];
      rect_r[r] = rc;  // in rank order: the emit pass reads it coalesced
      const int b0 = rc.x / kSegCols, b1 = rc.y / kSegCols;
      vs += (rc.w - rc.z + 1) * (b1 - b0 + 1);
      for (int ty = rc.z; ty <= rc.w; ++ty)
        for (int b = b0; b <= b1; ++b) {
          const int lo = max(rc.x, b * kSegCols), hi = min(rc.y, b * kSegCols + kSegCols - 1);
          atomicAdd(&keys_s[ty * nblk + b], 1);
          atomicAdd(&pairs_s[ty * nblk + b], hi - lo + 1);
        }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt_r[n] = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    vs += __shfl_xor_sync(0xffffffffu, vs, o);
  }
  if ((threadIdx.x & 31) == 0) {
    csum[threadIdx.x >> 5][0] = v;
    csum[threadIdx.x >> 5][1] = vs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0, ts = 0;
    for (int w = 0; w < kBinThreads / 32; ++w) {
      t += csum[w][0];
      ts += csum[w][1];
    }
    if (t) atomicAdd(reinterpret_cast<unsigned long long*>(&status->pairs),
                     (unsigned long long)t);
    if (ts) atomicAdd(reinterpret_cast<unsigned long long*>(&status->segs),
                      (unsigned long long)ts);
  }
  if (!SEGS) return;
  const int64_t nb = gridDim.x;
  for (int k = threadIdx.x; k < keys; k += kBinThreads) {
    cnt_r[n + 1 + k * nb + blockIdx.x] = keys_s[k];
    if (pairs_s[k]) atomicAdd(&key_pairs[k], pairs_s[k]);
  }
}

cudaError_t run_count_scan(void* temp, size_t temp_bytes, const int32_t* count,
                           const uint32_t* order, const int4* rect, int32_t* cnt_r,
                           int32_t* off_r, uint32_t* rank_of, int64_t n, int tiles_x,
                           int tiles_y, int32_t* key_pairs, BinStatusDev* status,
                           int4* rect_r, cudaStream_t stream) {
  const bool segs = tiles_x > 0;
  const int nblk = segs ? seg_blocks(tiles_x) : 0;
  const int keys = segs ? tiles_y * nblk : 0;
  const unsigned nb = (unsigned)bin_row_blocks(n);
  cudaError_t e = cudaMemsetAsync(status, 0, sizeof(BinStatusDev), stream);
  if (e != cudaSuccess) return e;
  if (segs) {
    e = cudaMemsetAsync(key_pairs, 0, keys * sizeof(int32_t), stream);
    if (e != cudaSuccess) return e;
    gather_counts_kernel<true><<<nb, kBinThreads, 2 * keys * sizeof(int), stream>>>(
        count, order, rect, cnt_r, rank_of, n, tiles_y, nblk, key_pairs, status, rect_r);
  } else {
    gather_counts_kernel<false><<<nb, kBinThreads, 0, stream>>>(count, order, rect, cnt_r,
                                                                rank_of, n, 0, 0, key_pairs,
                                                                status, rect_r);
  }
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, cnt_r, off_r,
                                    (int)count_scan_len(n, keys, segs), stream);
  note_launch(2);
  return e;
}

// ---- segment binning (no host round trip) -----------------------------------
// 256-thread exclusive scan of one int per thread; returns the CTA total.
__device__ __forceinline__ int block_exclusive_scan(int v, int* excl, int* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  int before = 0, total = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
    const int t = warp_tot[k];
    before += k < w ? t : 0;
    total += t;
  }
  *excl = before + x - v;
  __syncthreads();
  return total;
}

// Lanes of the warp holding the same key (0 <= key < 2^nbits), from one ballot per
// key bit: the multisplit form of __match_any_sync.  MATCH.ANY issues on the ADU
// pipe, whose throughput capped a per-pair version of these passes at c5 (ncu: ADU
// 96% busy).
__device__ __forceinline__ unsigned warp_peers(int key, int nbits) {
  unsigned peers = 0xffffffffu;
  for (int b = 0; b < nbits; ++b) {
    const bool bit = (key >> b) & 1;
    const unsigned vote = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? vote : ~vote;
  }
  return peers;
}

__device__ __forceinline__ int bit_width(int v) { return 32 - __clz(v); }

__device__ __forceinline__ bool bin_overflowed(const RowBinArgs& a, long long* p_out) {
  const long long p = *reinterpret_cast<volatile long long*>(&a.status->pairs);
  *p_out = p;
  return p > a.capacity || p > 0x7fffffffll;
}

// first segment of key k's bucket (the histograms' scan entries are offset by P)
__device__ __forceinline__ int key_start(const RowBinArgs& a, int k, int p) {
  return k < a.keys ? a.off_r[a.n + 1 + (int64_t)k * a.nb] - p
                    : (int)*reinterpret_cast<volatile long long*>(&a.status->segs);
}

// a / b for 0 <= a < 2^24, 1 <= b: a float estimate corrected by one step (exact)
__device__ __forceinline__ int div_small(int a, int b, float inv_b) {
  int q = __float2int_rz((float)a * inv_b);
  if (q * b > a) --q;
  if ((q + 1) * b <= a) ++q;
  return q;
}

// Emit: one CTA per block of kBinRanks depth ranks, 8 warps x 128 ranks (4
// sub-blocks of 32), the count pass's blocks.  Warp w's segments, in generation
// order (splat-major, then tile row, then column block), go to
//   the key's bucket base (the scan) + the earlier warps' segments of that key +
//   the warp's earlier segments of that key (ballot peers, in segment order),
// so every bucket holds its segments in depth-rank order.
// CTA 0 also lays out the fill passes' chunks (kSegChunk segments, key-aligned).
__global__ void __launch_bounds__(kBinThreads) seg_emit_kernel(RowBinArgs a) {
  extern __shared__ int wkey[];  // [8][keys]
  __shared__ int scan_tot[kBinThreads / 32];
  constexpr int kSub = kBinRanks / kBinThreads;  // sub-blocks of 32 ranks per warp
  long long p64;
  if (bin_overflowed(a, &p64)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) a.status->flags |= kBinFlagOverflow;
    return;
  }
  const int p = (int)p64;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int K = a.keys;
  if (blockIdx.x == 0) {
    constexpr int kPer = kBinMaxKeys / kBinThreads;
    int nch[kPer], tot = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int k = threadIdx.x * kPer + q;
      nch[q] = k < K ? (key_start(a, k + 1, p) - key_start(a, k, p) + kSegChunk - 1) / kSegChunk
                     : 0;
      tot += nch[q];
    }
    int excl;
    const int all = block_exclusive_scan(tot, &excl, scan_tot);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int k = threadIdx.x * kPer + q;
      if (k < K) a.chunk_first[k] = excl;
      excl += nch[q];
    }
    if (threadIdx.x == 0) a.chunk_first[K] = all;
  }
  for (int e = threadIdx.x; e < 8 * K; e += kBinThreads) wkey[e] = 0;
  __syncthreads();
  // this lane's splat of each sub-block: rank base + w * 128 + sub * 32 + lane
  const int64_t r0 = (int64_t)blockIdx.x * kBinRanks + w * (32 * kSub) + lane;
  uint32_t v[kSub];
  int4 rc[kSub];
  int nbl[kSub], b0[kSub], ns[kSub];
#pragma unroll
  for (int q = 0; q < kSub; ++q) {
    const int64_t r = r0 + 32 * q;
    const int c = r < a.n ? a.cnt_r[r] : 0;
    v[q] = 0;
    rc[q] = make_int4(0, 0, 0, 0);
    nbl[q] = 1;
    b0[q] = 0;
    ns[q] = 0;
    if (c > 0) {
      v[q] = a.order[r];
      const uint32_t i = v[q] & kIndexMask;
      rc[q] = a.rect_r[r];
      const int spans_x = rc[q].y - rc[q].x + 1;
      // pair (tx, ty) of this splat has generation index origin + ty * spans_x + tx
      // (a dense array: a 4-byte store into each 64-B record cost a partial-sector
      // read-modify-write of the record in DRAM, c3 binning 0.088 -> 0.108 ms)
      a.row_origin[i] = a.off_r[r] - rc[q].z * spans_x - rc[q].x;
      b0[q] = rc[q].x / kSegCols;
      nbl[q] = rc[q].y / kSegCols - b0[q] + 1;
      ns[q] = (rc[q].w - rc[q].z + 1) * nbl[q];
      for (int ty = rc[q].z; ty <= rc[q].w; ++ty)
        for (int b = 0; b < nbl[q]; ++b) atomicAdd(&wkey[w * K + ty * a.nblk + b0[q] + b], 1);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += kBinThreads) {
    int base = a.off_r[a.n + 1 + (int64_t)k * a.nb + blockIdx.x] - p;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int t = wkey[q * K + k];
      wkey[q * K + k] = base;
      base += t;
    }
  }
  __syncthreads();
  int* cur = wkey + w * K;
  const unsigned lt = (1u << lane) - 1u;
  const int kbits = bit_width(K);  // keys 0..K (K: no segment)
#pragma unroll
  for (int q = 0; q < kSub; ++q) {
    int incl = ns[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int excl = incl - ns[q];
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const float inv_nbl = 1.0f / (float)nbl[q];
    for (int j0 = 0; j0 < total; j0 += 32) {
      const int j = j0 + lane;
      int sidx = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int cand = sidx + step;
        const int e = __shfl_sync(0xffffffffu, excl, cand & 31);
        if (cand < 32 && e <= j) sidx = cand;
      }
      const int es = __shfl_sync(0xffffffffu, excl, sidx);
      const int sn = __shfl_sync(0xffffffffu, nbl[q], sidx);
      const float sinv = __shfl_sync(0xffffffffu, inv_nbl, sidx);
      const int sb0 = __shfl_sync(0xffffffffu, b0[q], sidx);
      const int x0 = __shfl_sync(0xffffffffu, rc[q].x, sidx);
      const int x1 = __shfl_sync(0xffffffffu, rc[q].y, sidx);
      const int y0 = __shfl_sync(0xffffffffu, rc[q].z, sidx);
      const uint32_t vs = __shfl_sync(0xffffffffu, v[q], sidx);
      const bool live = j < total;
      const int l = j - es;
      const int row = div_small(l, sn, sinv);
      const int b = sb0 + (l - row * sn);
      const int key = live ? (y0 + row) * a.nblk + b : K;
      const unsigned peers = warp_peers(key, kbits);
      const int pos = live ? cur[key] + __popc(peers & lt) : 0;
      __syncwarp();
      if (live && lane == __ffs(peers) - 1) cur[key] += __popc(peers);
      __syncwarp();
      if (live) {
        const int lo = max(x0, b * kSegCols) - b * kSegCols;
        const int hi = min(x1, b * kSegCols + kSegCols - 1) - b * kSegCols;
        a.segs[pos] = make_uint2(vs, (uint32_t)(lo | ((hi - lo + 1) << 5)));
      }
    }
  }
}

// The chunk a fill warp owns: its key and [begin, end) in the segment buckets.
__device__ __forceinline__ bool seg_chunk_of(const RowBinArgs& a, int p, int c, int* key,
                                             int* begin, int* end) {
  const int K = a.keys;
  if (c >= a.chunk_first[K]) return false;
  int lo = 0, hi = K;  // last key with chunk_first[key] <= c
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a.chunk_first[mid] <= c) lo = mid; else hi = mid;
  }
  *key = lo;
  *begin = key_start(a, lo, p) + (c - a.chunk_first[lo]) * kSegChunk;
  *end = min(*begin + kSegChunk, key_start(a, lo + 1, p));
  return true;
}

// Fill pass 1: per chunk (one warp), lane L counts the chunk's segments covering
// tile column L of the key's block -> seg_cnt[chunk][L].  Each segment adds +1 at
// its first column and -1 past its last in a per-warp difference array in shared
// memory; one 32-wide prefix sum at the end gives the counts.
__global__ void __launch_bounds__(256) seg_count_kernel(RowBinArgs a) {
  __shared__ int diff_all[8][33];
  long long p64;
  if (bin_overflowed(a, &p64)) return;
  const int lane = threadIdx.x & 31;
  int* diff = diff_all[threadIdx.x >> 5];
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
  int key, begin, end;
  if (!seg_chunk_of(a, (int)p64, c, &key, &begin, &end)) return;
  diff[lane] = 0;
  if (lane == 0) diff[32] = 0;
  __syncwarp();
  for (int s = begin + lane; s < end; s += 32) {
    const uint32_t sg = a.segs[s].y;
    const int lo = (int)(sg & 31u), len = (int)(sg >> 5);
    atomicAdd(&diff[lo], 1);
    atomicAdd(&diff[lo + len], -1);
  }
  __syncwarp();
  int cnt = diff[lane];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, cnt, o);
    if (lane >= o) cnt += t;
  }
  a.seg_cnt[(int64_t)c * 32 + lane] = cnt;
}

// Fill pass 2: one CTA per key (tile row, column block); lane L of each warp is
// tile column L of the block.  Each tile's chunk counts become exclusive prefixes
// over the key's chunks (in place; the 8 warps take consecutive chunk ranges);
// the tile totals, scanned across the block from the pairs of every earlier key
// (row-major, the count pass's per-key pair totals), are the block's tile_starts
// (np.searchsorted's CSR, rasterizer.py:324-325).  On overflow every tile list is
// left empty, so the blends and K7 see no pairs.
__global__ void __launch_bounds__(256) tile_scan_kernel(RowBinArgs a) {
  __shared__ int part[8][32];
  __shared__ int red[8];
  long long p64;
  const int key = blockIdx.x, X = a.tiles_x;
  const int ty = key / a.nblk, b = key - ty * a.nblk;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = b * kSegCols + lane;
  if (bin_overflowed(a, &p64)) {
    if (w == 0 && tx < X) a.tile_starts[ty * X + tx] = 0;
    if (key == a.keys - 1 && threadIdx.x == 0) a.tile_starts[a.tiles_y * X] = 0;
    return;
  }
  const int p = (int)p64;
  const int c0 = a.chunk_first[key], c1 = a.chunk_first[key + 1];
  const int per = (c1 - c0 + 7) / 8;
  const int w0 = c0 + min(c1 - c0, w * per), w1 = c0 + min(c1 - c0, (w + 1) * per);
  int32_t* h = a.seg_cnt + (int64_t)w0 * 32 + lane;
  int run = 0;
  for (int c = w0; c < w1; ++c, h += 32) run += *h;
  part[w][lane] = run;
  // pairs of every earlier key: the rows above and this row's earlier blocks
  int above = 0;
  for (int k = threadIdx.x; k < key; k += 256) above += a.key_pairs[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) above += __shfl_xor_sync(0xffffffffu, above, o);
  if (lane == 0) red[w] = above;
  __syncthreads();
  int before = 0, total = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int t = part[q][lane];
    before += q < w ? t : 0;
    total += t;
  }
  // second pass: exclusive prefixes in place
  run = before;
  h = a.seg_cnt + (int64_t)w0 * 32 + lane;
  for (int c = w0; c < w1; ++c, h += 32) {
    const int t = *h;
    *h = run;
    run += t;
  }
  if (w == 0) {
    int base = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) base += red[q];
    int incl = total;  // tile totals scanned across the block's 32 columns
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (tx < X) a.tile_starts[ty * X + tx] = base + incl - total;
    if (key == a.keys - 1 && lane == 0) a.tile_starts[a.tiles_y * X] = p;
  }
}

// Fill pass 3: per chunk (one warp), lane L owns tile column L of the key's block;
// the values of the segments covering it are appended, in segment (= depth rank)
// order, at tile_starts[tile] + the chunk's prefix: a stable counting sort by
// tile, so each tile list equals np.lexsort((index, depth, tile))
// (rasterizer.py:318-323).  The warp loads 32 segments at a time (one per lane).
// Two ways to write them, chosen per key by its mean segment length:
// * narrow segments (small splats, c3/c4): the segments are broadcast in order and
//   each lane stores for its own column -- a few instructions per segment;
// * wide segments (c5): the columns are walked, a ballot names the segments that
//   cover a column and they store at consecutive positions of its list -- one
//   coalesced store per column, but two population counts per lane (XU pipe).
// Measured per view: narrow c3 0.110 / c4 0.330 / c5 0.81 ms; wide 0.139 / 0.37 /
// 0.52 ms (binning stage).
#ifndef HS_FILL_WIDE
#define HS_FILL_WIDE 6  // mean pairs per segment from which the column walk is used
#endif
__global__ void __launch_bounds__(256) seg_fill_kernel(RowBinArgs a) {
  long long p64;
  if (bin_overflowed(a, &p64)) return;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
  int key, begin, end;
  if (!seg_chunk_of(a, (int)p64, c, &key, &begin, &end)) return;
  const int ty = key / a.nblk, tx = (key - ty * a.nblk) * kSegCols + lane;
  int pos = tx < a.tiles_x ? a.tile_starts[ty * a.tiles_x + tx] +
                                 a.seg_cnt[(int64_t)c * 32 + lane]
                           : 0;
  const int key_segs = key_start(a, key + 1, (int)p64) - key_start(a, key, (int)p64);
  const bool wide = a.key_pairs[key] >= HS_FILL_WIDE * key_segs;
  for (int s0 = begin; s0 < end; s0 += 32) {
    const uint2 sg = s0 + lane < end ? a.segs[s0 + lane] : make_uint2(0u, 0u);
    const uint32_t len = sg.y >> 5;
    const uint32_t span = len ? (0xffffffffu >> (32 - len)) << (sg.y & 31u) : 0u;
    if (wide) {
      unsigned cols = __reduce_or_sync(0xffffffffu, span);
      while (cols) {
        const int L = __ffs(cols) - 1;
        cols &= cols - 1;
        const unsigned m = __ballot_sync(0xffffffffu, (span >> L) & 1u);
        const int b = __shfl_sync(0xffffffffu, pos, L);
        if ((span >> L) & 1u) a.pair_src[b + __popc(m & lt)] = sg.x;
        if (lane == L) pos += __popc(m);
      }
    } else {
      const int m = min(32, end - s0);
      for (int k = 0; k < m; ++k) {
        const uint32_t sk = __shfl_sync(0xffffffffu, span, k);
        const uint32_t vk = __shfl_sync(0xffffffffu, sg.x, k);
        if ((sk >> lane) & 1u) a.pair_src[pos++] = vk;
      }
    }
  }
}

cudaError_t run_row_binning(const RowBinArgs& a, cudaStream_t stream) {
  const int64_t chunks = bin_chunk_capacity(a.capacity, a.keys);
  const unsigned fill_grid = (unsigned)((chunks + 7) / 8);
  // the attribute is set once per device: set it for the largest key count
  cudaError_t e = set_dynamic_smem<seg_emit_kernel>(8 * kBinMaxKeys * (int)sizeof(int));
  if (e != cudaSuccess) return e;
  seg_emit_kernel<<<(unsigned)a.nb, kBinThreads, 8 * a.keys * sizeof(int), stream>>>(a);
  seg_count_kernel<<<fill_grid, 256, 0, stream>>>(a);
  tile_scan_kernel<<<(unsigned)a.keys, 256, 0, stream>>>(a);
  seg_fill_kernel<<<fill_grid, 256, 0, stream>>>(a);
  note_launch(4);
  return cudaGetLastError();
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
    const int32_t* __restrict__ off_r, const int4* __restrict__ rect,
    int32_t* __restrict__ row_origin,
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
    row_origin[i] = off_r[r] - rc.z * spans_x - rc.x;
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
                          const int4* rect, int32_t* row_origin, int tiles_x, uint32_t* keys,
                          uint32_t* vals, int64_t n, cudaStream_t stream) {
  const int block = 256;
  duplicate_kernel<<<(unsigned)((n + block - 1) / block), block, 0, stream>>>(
      order, cnt_r, off_r, rect, row_origin, tiles_x, keys, vals, n);
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
