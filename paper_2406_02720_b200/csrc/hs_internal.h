// hs_internal.h -- kernel argument structs and launcher prototypes shared by
// the translation units of libhalfsplat_b200.so (not part of the public ABI).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "hs_common.cuh"

namespace hs {

template <typename T>
struct SceneArgs {
  const T* mu;
  const T* ls;
  const T* rot;
  const T* sh;
  const T* nrm;
  const T* ra;
  const T* rb;
  int K;    // SH coefficients per channel, (deg+1)^2
  int deg;  // SH degree 0..3
};

struct CamArgs {
  double R[9];   // world_to_cam rotation, row-major
  double tr[3];  // world_to_cam translation
  double center[3];
  double fx, fy, cx, cy, near_clip;
  int width, height;
};

template <typename T>
struct GradArgs {
  T* d_mu;
  T* d_log_scale;
  T* d_rotation;
  T* d_sh;
  T* d_normal;
  T* d_ra;
  T* d_rb;
  T* pos_grad_norm;
  int32_t* touch;
  int accumulate;
  int64_t begin, end;  // primitive range [begin, end) of this launch (begin % 128 == 0)
};

// ---- hs_preprocess.cu -----------------------------------------------------
template <typename T>
cudaError_t launch_preprocess_fwd_t(const SceneArgs<T>& sc, const CamArgs& cam, int kernel,
                                    int64_t n, float4* rec, SteepRec* side, int4* rect,
                                    int32_t* count, uint64_t* dkey, uint32_t* dval,
                                    int32_t* radii, uint32_t* depth_range, cudaStream_t stream);
template <typename T>
cudaError_t launch_preprocess_bwd_t(const SceneArgs<T>& sc, const CamArgs& cam, int kernel,
                                    int64_t n, int tiles_x, const float4* rec,
                                    const int32_t* row_origin, const int4* rect,
                                    const int32_t* count, const uint32_t* rank_of,
                                    const int32_t* last_rank, const float* rows, float4* merged,
                                    int64_t num_pairs, const GradArgs<T>& out,
                                    cudaStream_t stream);
// the multi-view K7 (and K1): views in groups of kMaxViews per launch
constexpr int kMaxViews = 8;
// K1's per-view outputs
struct FwdOut {
  float4* rec;
  SteepRec* side;
  int4* rect;
  int32_t* count;
  uint64_t* dkey;
  uint32_t* dval;
  int32_t* radii;
  uint32_t* range;  // the visible depths' upper-word range, or nullptr
};
struct FwdViewsArgs {
  CamArgs cam[kMaxViews];
  FwdOut out[kMaxViews];
  int n_views;
};
template <typename T>
cudaError_t launch_preprocess_fwd_views_t(const SceneArgs<T>& sc, const FwdViewsArgs& va,
                                          int kernel, int64_t n, cudaStream_t stream);
struct ViewsArgs {
  CamArgs cam[kMaxViews];
  const float4* merged[kMaxViews];
  int n_views;
};
template <typename T>
cudaError_t launch_preprocess_bwd_views_t(const SceneArgs<T>& sc, const CamArgs* cams,
                                          const float4* const* merged, int n_views, int kernel,
                                          int64_t n, const GradArgs<T>& out, cudaStream_t stream);
cudaError_t launch_merge_rows(int64_t n, int tiles_x, const float4* rec,
                              const int32_t* row_origin, const int4* rect,
                              const int32_t* count, const uint32_t* rank_of,
                              const int32_t* last_rank, const float* rows, float4* merged,
                              int64_t num_pairs, cudaStream_t stream);

template <typename T>
cudaError_t launch_screen_splats_t(const SceneArgs<T>& sc, const CamArgs& cam, int kernel,
                                   int64_t n, double* out, cudaStream_t stream);

// ---- hs_blend.cu ------------------------------------------------------------
struct BlendGeom {
  const int32_t* tile_starts;  // (n_tiles+1) CSR offsets into pair_src
  const uint32_t* pair_src;    // sorted pair -> record index
  const float4* rec;           // 4 float4 per record
  const int32_t* row_origin;   // K6: each splat's pair-row origin (nullptr: Seam 1 rows)
  const SteepRec* side;        // FP64 side records of steep splats (flag: bit 31 of pair_src)
  int width, height, tiles_x;
  int tile_lo, n_work;         // tiles [tile_lo, tile_lo + n_work)
  const int32_t* tile_order;   // optional work order (nullptr = natural)
  int* work_counter;           // the unit queue (UnitQueue below); zeroed by the launcher
  int32_t* tile_work;          // optional (K5): per-tile largest terminal count
  int sub_tiles;               // K5 work units per tile: 1 (16x16), 2 (16x8) or 4 (16x4)
  int spread;                  // 1: first wave spread over the SMs (work_counter holds
                               // kQueueInts ints), 0: plain dynamic queue (1 int)
  int n_sm, per_sm, n_first;   // set by the launcher
  // Split backward (small frames, see hs_blend.cu "K6 segments"): K5 leaves per-pixel
  // checkpoints every kCkpt list positions, K6 runs (tile, segment) units
  float4* ckpt;                // nullptr: off
  const int2* units;           // K6: (tile, segment) units, *n_units of them
  const int* n_units;
  int ckpt_shift;              // log2 of the list positions per segment / checkpoint
};
// checkpoint slots hold a tile's 256 pixels; segments of 2^shift list positions,
// shift in [kCkptMinShift, 8]
constexpr int kCkptMinShift = 6;
constexpr int kCkptSlot = 256;
cudaError_t launch_bwd_units(const int32_t* tile_work, const int32_t* order, int n_tiles,
                             int ckpt_shift, int2* units, int* n_units, cudaStream_t stream);
// The blends' unit queue with an SM-spread first wave: [0] dynamic counter, [1]
// sweep counter, [2, 2 + kQueueMaxSms) per-SM slot counters, then one claim flag per
// first-wave unit.
constexpr int kQueueMaxSms = 256;
constexpr int kQueueMaxFirst = 4096;
constexpr int kQueueInts = 2 + kQueueMaxSms + kQueueMaxFirst;
int blend_fwd_slots();
int blend_bwd_slots();
// longest-first tile order: work = list length (starts != nullptr) or work[t]
cudaError_t launch_tile_order(const int32_t* starts, const int32_t* work, int n_tiles,
                              int32_t* order, cudaStream_t stream);

cudaError_t launch_blend_fwd(const BlendGeom& g, float bg0, float bg1, float bg2, float* color,
                             float* alpha, float* depth, float* trans, int32_t* terminal,
                             cudaStream_t stream);
// rows_by_sorted_pos: write pair row at the sorted position (reference layout,
// Seam 1) instead of at the generation-order index from the record.
cudaError_t launch_blend_bwd(const BlendGeom& g, float bg0, float bg1, float bg2,
                             const float* d_color, const float* trans, const int32_t* terminal,
                             float* rows, int32_t* last_rank, const uint32_t* rank_of,
                             bool rows_by_sorted_pos, cudaStream_t stream);
// diagnostic: strip window codes (hs_blend.cu strip_window) over all pairs -> hist[4]
cudaError_t launch_window_stats(const BlendGeom& g, unsigned long long* hist, cudaStream_t stream);
// Seam 1: reference packed (M,13) f64 + mode -> records + side records; marks
// steep splats in bit 31 of pair_splat (in place, device copy).
cudaError_t launch_pack_records(const double* packed, const int8_t* mode, int64_t m,
                                float4* rec, SteepRec* side, uint32_t* pairs, int64_t p,
                                cudaStream_t stream);

// ---- hs_binning.cu --------------------------------------------------------
size_t depth_sort_temp_bytes(int64_t n);
size_t scan_temp_bytes(int64_t n);
size_t pair_sort_temp_bytes(int64_t p, int tile_bits);

cudaError_t run_depth_sort(void* temp, size_t temp_bytes, const uint64_t* keys_in,
                           uint64_t* keys_out, const uint32_t* vals_in, uint32_t* order,
                           int64_t n, cudaStream_t stream);
// upper-32-bit sort + per-run fixup (two n-element u32 scratch arrays); *overflow =
// 1 when a run was too long (then run_depth_sort must redo the ranks)
// range: the visible splats' smallest and largest upper depth word (K1)
cudaError_t run_depth_sort_hi(void* temp, size_t temp_bytes, const uint64_t* keys_in,
                              uint64_t* keys_out, const uint32_t* vals_in, uint32_t* order,
                              int64_t n, uint32_t* scratch_pos, uint32_t* scratch_val,
                              int* overflow, const uint32_t* range, cudaStream_t stream);
constexpr int kDepthKeyBits = 24;
constexpr uint32_t kDepthKeyCulled = (1u << kDepthKeyBits) - 1u;
// ---- tile binning without a host round trip -------------------
// A splat's pairs in one tile row and one block of 32 tile columns form a
// SEGMENT (value, first column, length).  The count pass histograms every block
// of kBinRanks depth ranks' segments by (tile row, column block) key and its pairs
// by tile row; the emit pass writes each segment straight into its key's bucket
// (rank order within the key, so stable); the fill passes give each warp a chunk
// of one bucket, lane L = tile column L of the block, and every lane appends the
// values of the segments that cover it -- a stable counting sort by tile whose
// per-pair cost is one predicated store.  P stays on the device: the caller sizes
// the binning workspace for a pair capacity, and a frame whose P exceeds it is
// flagged (kBinFlagOverflow) with every tile list left empty.
#ifndef HS_BIN_RANKS
#define HS_BIN_RANKS 256
#endif
constexpr int kBinRanks = HS_BIN_RANKS;  // depth ranks per CTA of the count and emit passes
constexpr int kBinThreads = 256;  // 8 warps, each kBinRanks / 8 ranks (sub-blocks of 32)
constexpr int kSegCols = 32;        // tile columns per block (one warp's lanes)
constexpr int kBinMaxCols = 2048;   // tiles_x limit (larger images: CUB pair sort)
constexpr int kBinMaxRows = 1024;   // tiles_y limit
constexpr int kBinMaxKeys = 2048;   // tile rows x column blocks limit
#ifndef HS_SEG_CHUNK
#define HS_SEG_CHUNK 256
#endif
constexpr int kSegChunk = HS_SEG_CHUNK;  // segments per warp in the fill passes
constexpr int kBinFlagOverflow = 1;
constexpr int kBinFlagDepth = 2;    // the depth-run fixup overflowed: ranks need the full sort
inline int seg_blocks(int tiles_x) { return (tiles_x + kSegCols - 1) / kSegCols; }
inline int seg_keys(int tiles_x, int tiles_y) { return tiles_y * seg_blocks(tiles_x); }
inline bool row_binning_ok(int tiles_x, int tiles_y) {
  return tiles_x <= kBinMaxCols && tiles_y <= kBinMaxRows &&
         seg_keys(tiles_x, tiles_y) <= kBinMaxKeys;
}
inline int64_t bin_row_blocks(int64_t n) { return (n + kBinRanks - 1) / kBinRanks; }
inline int64_t bin_chunk_capacity(int64_t capacity, int keys) {
  return capacity / kSegChunk + keys + 1;
}
// scan entries of the count pass: pair counts by rank (n + 1), then, with the
// segment path, the segment histograms [key][rank block]
inline int64_t count_scan_len(int64_t n, int keys, bool rows) {
  return n + 1 + (rows ? (int64_t)keys * bin_row_blocks(n) : 0);
}
struct BinStatusDev {   // in the frame's counters
  long long pairs;      // P as int64 (the int32 scan may wrap)
  long long segs;       // segments
  int flags;
  int pad;
};

// cnt_r[r] = count[order[r]], off_r = exclusive scan (count_scan_len entries),
// rank_of[order[r]] = r, P as int64 in *status (zeroed here); with the segment
// path (tiles_x > 0) also the segment histograms and key_pairs[keys] (pairs per
// (tile row, column block) key, zeroed here).
cudaError_t run_count_scan(void* temp, size_t temp_bytes, const int32_t* count,
                           const uint32_t* order, const int4* rect, int32_t* cnt_r,
                           int32_t* off_r, uint32_t* rank_of, int64_t n, int tiles_x,
                           int tiles_y, int32_t* key_pairs, BinStatusDev* status,
                           int4* rect_r, cudaStream_t stream);
struct RowBinArgs {
  const uint32_t* order;
  const int4* rect;
  const int4* rect_r;    // rects in depth-rank order (the count pass writes them)
  int32_t* row_origin;   // [n] each splat's pair-row origin (K6, K7a)
  const int32_t* cnt_r;
  const int32_t* off_r;
  BinStatusDev* status;
  const int32_t* key_pairs;  // [keys] pairs per (tile row, column block)
  int64_t n;
  int nb;  // rank blocks
  int tiles_x, tiles_y, nblk, keys;
  int64_t capacity;
  uint2* segs;           // [capacity] buckets: (index | steep, first column | length << 5)
  int32_t* chunk_first;  // [keys + 1]
  int32_t* seg_cnt;      // [chunk capacity][32]
  int32_t* tile_starts;  // [n_tiles + 1]
  uint32_t* pair_src;    // [capacity] final order
};
// emit + column passes (4 launches); no host synchronisation
cudaError_t run_row_binning(const RowBinArgs& a, cudaStream_t stream);
cudaError_t run_duplicate(const uint32_t* order, const int32_t* cnt_r, const int32_t* off_r,
                          const int4* rect, int32_t* row_origin, int tiles_x, uint32_t* keys,
                          uint32_t* vals, int64_t n, cudaStream_t stream);
// returns selector (0/1) of the buffer holding the sorted result
cudaError_t run_pair_sort(void* temp, size_t temp_bytes, uint32_t* keys0, uint32_t* keys1,
                          uint32_t* vals0, uint32_t* vals1, int64_t p, int tile_bits,
                          int* selector, cudaStream_t stream);
cudaError_t run_tile_ranges(const uint32_t* sorted_keys, int64_t p, int n_tiles,
                            int32_t* tile_starts, cudaStream_t stream);
cudaError_t run_export(void* temp, size_t temp_bytes, const int32_t* count, const float4* rec,
                       const int4* rect, const uint32_t* pair_src, const int32_t* tile_starts32,
                       int64_t n, int64_t p, int n_tiles, int32_t* local_of, int32_t* flags,
                       int32_t* valid, int64_t* m_out, float* packed, int8_t* mode, int32_t* tile_rect,
                       int32_t* pair_splat, int64_t* tile_starts, cudaStream_t stream);

// ---- hs_loss.cu -------------------------------------------------------------
struct LossArgs {
  const float* x;  // rendered (H,W,C) float32
  const float* y;  // target   (H,W,C) float32
  const double* x64;  // float64 images instead (hs_loss_f64); x, y unused then
  const double* y64;
  int width, height, channels;
  double lambda;   // lambda_ssim
  double n;        // H*W*C
  double inv_n;    // 1 / n
  double* adj_m;   // ssim_with_grad adjoint maps, (C,H,W) float64 each
  double* adj_s1;
  double* adj_s12;
  double* partial;  // 3 per CTA: sum |x-y|, sum SSIM map, sum (x-y)^2
  int n_partials;
  double* loss;     // [loss, l1, mean ssim, mse]
  float* d_f32;     // d loss / d rendered (nullable)
  double* d_f64;    // same in float64 (nullable)
  int ssim;         // lambda > 0
  int group0;       // first channel group of a launch (internal)
  double win[11];   // Gaussian window, loss.py:19-23 (kernel parameter space)
};
cudaError_t launch_loss(const LossArgs& a, cudaStream_t stream);
int64_t loss_partials(int width, int height, int channels);

// ---- hs_adam.cu -------------------------------------------------------------
enum AdamKind { kAdamPlain = 0, kAdamSh = 1, kAdamNormal = 2, kAdamOpacity = 3 };
struct AdamSeg {
  void* param[2];  // [1] used by kAdamOpacity (raw_opacity_b)
  void* m[2];
  void* v[2];
  const void* grad[2];
  double lr[2];    // kAdamSh: [0] sh_dc, [1] sh_rest
  double bc1[2];   // 1 - beta1^t of the group
  double bc2[2];   // 1 - beta2^t
  int active[2];
  int kind;
  int K;           // SH coefficients per channel (kAdamSh)
  int vec;         // units are 16-B vectors (plain / sh segments, aligned, divisible)
  int64_t units;   // work units of the segment
};
constexpr int kAdamMaxSeg = 6;
struct AdamArgs {
  AdamSeg seg[kAdamMaxSeg];
  int cta_start[kAdamMaxSeg + 1];  // CTA prefix over segments (set by launch_adam)
  int nseg;
  int tie_opacities;
};
cudaError_t launch_adam(AdamArgs a, int dtype, cudaStream_t stream);

// ---- hs_densify.cu ----------------------------------------------------------
struct DensifyStatsArgs {
  double* grad_sum;     // (n,)
  double* mu_grad_sum;  // (n,3)
  int64_t* count;       // (n,)
};
struct DensifyParams {
  double densify_grad_threshold, prune_opacity_threshold, percent_dense, prune_extent_factor,
      scene_extent;
};
struct DensifyBufs {
  uint8_t* flags;
  int32_t *f_surv, *f_clone, *f_split;           // n + 1 each
  int32_t *surv_rank, *clone_rank, *split_rank;  // exclusive scans, n + 1 each
  void* temp;
  size_t temp_bytes;
};
template <typename T>
struct DensifyEmitArgs {
  int64_t n;
  int K;
  const uint8_t* flags;
  const int32_t *surv_rank, *clone_rank, *split_rank;
  int64_t acc_clone, acc_split, n_surv;
  const double* mu_grad_sum;
  const double* offsets;  // (2, acc_split, 3) standard normals or nullptr (Philox)
  uint64_t seed;
  double log_split_scale;
  struct { const T *mu, *ls, *rot, *sh, *nrm, *ra, *rb; } in;
  struct { T *mu, *ls, *rot, *sh, *nrm, *ra, *rb; } out;
  const void* m_in[7];
  const void* v_in[7];
  void* m_out[7];
  void* v_out[7];
};
cudaError_t launch_densify_stats(const DensifyStatsArgs& st, const void* pgn, const void* d_mu,
                                 const int32_t* touch, int64_t n, int dtype, cudaStream_t s);
size_t densify_scan_temp_bytes(int64_t n);
cudaError_t launch_densify_classify(const DensifyStatsArgs& st, const void* log_scale,
                                    const void* ra, const void* rb, int64_t n, int dtype,
                                    const DensifyParams& p, DensifyBufs& b, cudaStream_t s);
template <typename T>
cudaError_t launch_densify_emit_t(const DensifyEmitArgs<T>& a, cudaStream_t s);
cudaError_t opacity_disparity_sum(const void* ra, const void* rb, int64_t n, int dtype,
                                  double* out, void* temp, size_t* temp_bytes, cudaStream_t s);
cudaError_t launch_reset_opacity(void* ra, void* rb, void* ma, void* va, void* mb, void* vb,
                                 int64_t n, double cap, int dtype, cudaStream_t s);

// ---- hs_io.cu ----------------------------------------------------------------
enum PlyType { kPlyF32 = 0, kPlyF64 = 1, kPlyU8 = 2, kPlyI32 = 3 };
constexpr int kPlyMaxProps = 128;
constexpr int kPlyMaxComps = 3 + 3 + 4 + 48 + 3 + 1 + 1;
struct PlyUnpackArgs {
  const void* payload;  // device, n rows of `stride` bytes
  int64_t n;
  int stride;
  int K;                       // SH coefficients per channel
  int16_t offset[kPlyMaxProps];  // byte offset of each property in a row
  int8_t type[kPlyMaxProps];     // PlyType of each property
  int16_t column[kPlyMaxComps];  // source property of each scene component, -1 = skip
};
struct PlyPackArgs {
  void* payload;  // device, n rows
  int64_t n;
  int K;
  int gs3d;           // export_3dgs layout (zero normals, one opacity)
  int opacity_first;  // export_3dgs(opacity="first")
  int out_f64;        // double properties (native) / float
};
template <typename T>
struct SceneOut { T *mu, *ls, *rot, *sh, *nrm, *ra, *rb; };
template <typename T>
struct SceneIn { const T *mu, *ls, *rot, *sh, *nrm, *ra, *rb; };
cudaError_t launch_ply_unpack(const PlyUnpackArgs& a, const void* const* fields, int dtype,
                              cudaStream_t s);
cudaError_t launch_ply_pack(const PlyPackArgs& a, const void* const* fields, int dtype,
                            cudaStream_t s);

}  // namespace hs
