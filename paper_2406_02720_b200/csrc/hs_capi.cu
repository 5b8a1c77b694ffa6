// hs_capi.cu -- extern "C" entry points of libhalfsplat_b200.so
// (declared in include/halfsplat_b200.h).
#include <atomic>
#include <map>
#include <mutex>
#include <shared_mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/halfsplat_b200.h"
#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

static std::atomic<int64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static thread_local char g_err[256] = "";

static int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return HS_OK;
  snprintf(g_err, sizeof(g_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return HS_ERR_CUDA;
}

#define HS_CUDA(expr)                          \
  do {                                         \
    cudaError_t _e = (expr);                   \
    if (_e != cudaSuccess) return cuda_status(_e); \
  } while (0)

static size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Carves a workspace into typed sub-buffers; the same walk computes the size.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off = align_up(off + count * sizeof(T));
    return p;
  }
};

// counters[]: 48 depth-fixup overflow flag, 60-61 depth range (K1 -> rank sort),
// 52-57 the binning status (BinStatusDev: P and segments as int64, flags)
constexpr int kDepthOverflowSlot = 48;
constexpr int kDepthRangeSlot = 60;  // 60-61: the visible depths' upper-word range
constexpr int kBinStatusSlot = 52;

struct FrameBufs {
  float4* rec;
  SteepRec* side;
  int4* rect;
  int32_t* count;
  uint64_t* dkey_in;
  uint64_t* dkey_out;
  uint32_t* dval;
  uint32_t* order;
  int32_t* cnt_r;
  int32_t* off_r;
  uint32_t* rank_of;
  int32_t* tile_starts;
  int32_t* last_rank;
  int* counters;
  int32_t* xflags;
  int32_t* xlocal;
  float4* merged;
  int32_t* chunk_first;
  int32_t* key_pairs;
  int4* rect_r;
  int32_t* order_fwd;   // longest-first tile orders of K5 / K6
  int32_t* order_bwd;
  int32_t* tile_work;   // K5 -> K6: per-tile largest terminal count
  int32_t* row_origin;  // binning -> K6 / K7a: each splat's pair-row origin
  int* queue_fwd;       // the blends' unit queues (kQueueInts each)
  int* queue_bwd;
  BinStatusDev* status;
  void* temp;
  size_t temp_bytes;
};

// CUB temp-storage queries cost tens of microseconds (device attribute and
// occupancy lookups), and every entry point validates its workspace, so the
// sizes are memoised.  Counts are rounded up to a power of two: CUB's temp
// storage is monotone in the item count, so the bucket's size is an upper bound.
static int64_t pow2_bucket(int64_t n) {
  int64_t b = 1024;
  while (b < n) b <<= 1;
  return b;
}

static std::mutex g_size_mu;
static std::map<int64_t, size_t> g_frame_temp;
static std::map<std::pair<int64_t, int>, size_t> g_pair_temp;

static size_t frame_temp_bytes(int64_t n, int64_t scan_len) {
  const int64_t b = pow2_bucket(n), bs = pow2_bucket(scan_len);
  std::lock_guard<std::mutex> lock(g_size_mu);
  const int64_t key = b * 4096 + (bs / 1024 > 4095 ? 4095 : bs / 1024);
  auto it = g_frame_temp.find(key);
  if (it != g_frame_temp.end()) return it->second;
  const size_t x = depth_sort_temp_bytes(b), y = scan_temp_bytes(bs), z = scan_temp_bytes(b + 1);
  size_t m = x > y ? x : y;
  return g_frame_temp[key] = m > z ? m : z;
}

static size_t pair_temp_bytes(int64_t p, int tile_bits) {
  const auto key = std::make_pair(pow2_bucket(p), tile_bits);
  std::lock_guard<std::mutex> lock(g_size_mu);
  auto it = g_pair_temp.find(key);
  if (it != g_pair_temp.end()) return it->second;
  return g_pair_temp[key] = pair_sort_temp_bytes(key.first, tile_bits);
}

static FrameBufs carve_frame(void* ws, int64_t n, int tiles_x, int tiles_y, size_t* total) {
  Carver c(ws);
  FrameBufs f;
  const int n_tiles = tiles_x * tiles_y;
  const bool rows = row_binning_ok(tiles_x, tiles_y);
  const int64_t scan_len = count_scan_len(n, seg_keys(tiles_x, tiles_y), rows);
  f.rec = c.take<float4>(4 * (size_t)n);
  f.side = c.take<SteepRec>(n);
  f.rect = c.take<int4>(n);
  f.count = c.take<int32_t>(n);
  f.dkey_in = c.take<uint64_t>(n);
  f.dkey_out = c.take<uint64_t>(n);
  f.dval = c.take<uint32_t>(n);
  f.order = c.take<uint32_t>(n);
  f.cnt_r = c.take<int32_t>(scan_len);
  f.off_r = c.take<int32_t>(scan_len);
  f.rank_of = c.take<uint32_t>(n);
  f.tile_starts = c.take<int32_t>(n_tiles + 1);
  f.last_rank = c.take<int32_t>(n_tiles);
  f.counters = c.take<int>(64);
  f.xflags = c.take<int32_t>(n + 1);
  f.xlocal = c.take<int32_t>(n + 1);
  f.merged = c.take<float4>(4 * (size_t)n);
  f.chunk_first = c.take<int32_t>(seg_keys(tiles_x, tiles_y) + 1);
  f.key_pairs = c.take<int32_t>(seg_keys(tiles_x, tiles_y));
  f.rect_r = c.take<int4>(rows ? n : 1);
  f.order_fwd = c.take<int32_t>(n_tiles);
  f.order_bwd = c.take<int32_t>(n_tiles);
  f.tile_work = c.take<int32_t>(n_tiles);
  f.row_origin = c.take<int32_t>(n);
  f.queue_fwd = c.take<int>(kQueueInts);
  f.queue_bwd = c.take<int>(kQueueInts);
  f.status = reinterpret_cast<BinStatusDev*>(f.counters ? f.counters + kBinStatusSlot : nullptr);
  f.temp_bytes = frame_temp_bytes(n, scan_len);
  f.temp = c.take<char>(f.temp_bytes);
  if (total) *total = c.off;
  return f;
}

// The binning workspace for a pair capacity p.  Row-bucket path: the row buckets
// (tile column u16 + value), the final pair order, the column histograms and K6's
// pair rows; CUB path (very large images): keys/values double buffers + temp.
struct BinBufs {
  uint32_t* keys[2];
  uint32_t* vals[2];
  uint2* segs;
  uint32_t* pair_src;
  int32_t* seg_cnt;
  float* rows;
  float4* ckpt;  // split backward only: K5's per-pixel checkpoints, K6's units
  int2* units;
  int* n_units;
  void* temp;
  size_t temp_bytes;
};

// Split backward (K6 segments, hs_blend.cu): frames of at most this many tiles --
// c1, c2, c4; c3 has 8160 tiles -- where a few long tiles, not the total work, set
// K6's time.  HS_K6_SPLIT=0 / 1 forces it off / on.
constexpr int kSplitMaxTiles = 6144;
#ifndef HS_CKPT_SMALL_TILES
#define HS_CKPT_SMALL_TILES 1024
#endif
static bool bwd_split(int64_t n_tiles) {
  static const int mode = [] {
    const char* e = getenv("HS_K6_SPLIT");
    return e ? (e[0] == '0' ? 0 : 1) : 2;
  }();
  return mode == 1 || (mode == 2 && n_tiles <= kSplitMaxTiles);
}

// list positions per K6 segment (a power of two, 64 .. 256): the fewer the tiles, the
// shorter the segments, so a frame still has several units per resident warp slot
// (HS_CKPT_SHIFT forces the log2)
static int ckpt_shift(int64_t n_tiles) {
  static const int forced = [] {
    const char* e = getenv("HS_CKPT_SHIFT");
    const int v = e ? atoi(e) : 0;
    return v >= kCkptMinShift && v <= 8 ? v : 0;
  }();
  if (forced) return forced;
  return n_tiles <= HS_CKPT_SMALL_TILES ? kCkptMinShift : 8;
}

static BinBufs carve_bin(void* ws, int64_t p, int tiles_x, int tiles_y, size_t* total) {
  Carver c(ws);
  BinBufs b{};
  const size_t pp = p > 0 ? (size_t)p : 1;
  if (row_binning_ok(tiles_x, tiles_y)) {
    b.segs = c.take<uint2>(pp);
    b.pair_src = c.take<uint32_t>(pp);
    b.seg_cnt = c.take<int32_t>((size_t)bin_chunk_capacity(p, seg_keys(tiles_x, tiles_y)) * 32);
  } else {
    int bits = 0;
    while ((1ll << bits) < (long long)tiles_x * tiles_y) ++bits;
    b.keys[0] = c.take<uint32_t>(pp);
    b.keys[1] = c.take<uint32_t>(pp);
    b.vals[0] = c.take<uint32_t>(pp);
    b.vals[1] = c.take<uint32_t>(pp);
    b.temp_bytes = pair_temp_bytes(p, bits);
    b.temp = c.take<char>(b.temp_bytes);
  }
  b.rows = c.take<float>(pp * kRowFloats);
  const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
  if (bwd_split(n_tiles)) {
    // one checkpoint slot (a tile's 256 pixels) per segment of pairs; one unit per
    // tile + per segment
    const int sh = ckpt_shift(n_tiles);
    b.ckpt = c.take<float4>(((pp >> sh) + 2) * (size_t)kCkptSlot);
    b.units = c.take<int2>((size_t)n_tiles + (pp >> sh) + 1);
    b.n_units = c.take<int>(1);
  }
  if (total) *total = c.off;
  return b;
}

// pair capacity the binning workspace is laid out for
static int64_t bin_capacity(const hs_frame* f) {
  return f->pair_capacity > 0 ? f->pair_capacity : (f->num_pairs > 0 ? f->num_pairs : 0);
}

static BinBufs frame_bin(const hs_frame* f) {
  return carve_bin(f->bin_ws, bin_capacity(f), f->tiles_x, f->tiles_y, nullptr);
}

static FrameBufs frame_bufs(const hs_frame* f) {
  return carve_frame(f->frame_ws, f->n, f->tiles_x, f->tiles_y, nullptr);
}

static int tiles_of(int32_t px) { return (px + kTile - 1) / kTile; }

static int bits_for(int n_tiles) {
  int b = 0;
  while ((1ll << b) < (long long)n_tiles) ++b;
  return b;
}

static CamArgs cam_args(const hs_camera* cam) {
  CamArgs c;
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) c.R[3 * r + k] = cam->world_to_cam[4 * r + k];
    c.tr[r] = cam->world_to_cam[4 * r + 3];
    c.center[r] = cam->center[r];
  }
  c.fx = cam->fx;
  c.fy = cam->fy;
  c.cx = cam->cx;
  c.cy = cam->cy;
  c.near_clip = cam->near_clip;
  c.width = cam->width;
  c.height = cam->height;
  return c;
}

template <typename T>
static SceneArgs<T> scene_args(const hs_scene* s) {
  SceneArgs<T> a;
  a.mu = static_cast<const T*>(s->mu);
  a.ls = static_cast<const T*>(s->log_scale);
  a.rot = static_cast<const T*>(s->rotation);
  a.sh = static_cast<const T*>(s->sh_coeffs);
  a.nrm = static_cast<const T*>(s->normal);
  a.ra = static_cast<const T*>(s->raw_opacity_a);
  a.rb = static_cast<const T*>(s->raw_opacity_b);
  a.deg = s->sh_degree;
  a.K = (s->sh_degree + 1) * (s->sh_degree + 1);
  return a;
}

template <typename T>
static GradArgs<T> grad_args(const hs_grads* g) {
  GradArgs<T> a;
  a.d_mu = static_cast<T*>(g->d_mu);
  a.d_log_scale = static_cast<T*>(g->d_log_scale);
  a.d_rotation = static_cast<T*>(g->d_rotation);
  a.d_sh = static_cast<T*>(g->d_sh);
  a.d_normal = static_cast<T*>(g->d_normal);
  a.d_ra = static_cast<T*>(g->d_raw_opacity_a);
  a.d_rb = static_cast<T*>(g->d_raw_opacity_b);
  a.pos_grad_norm = static_cast<T*>(g->pos_grad_norm);
  a.touch = g->touch_count;
  a.accumulate = g->accumulate;
  a.begin = 0;
  a.end = INT64_MAX;
  return a;
}

template <typename T>
static GradArgs<T> ranged(GradArgs<T> a, int64_t begin, int64_t end) {
  a.begin = begin;
  a.end = end;
  return a;
}


static int check_frame_ws(const hs_frame* f) {
  if (!f || !f->frame_ws) return HS_ERR_WORKSPACE;
  if (f->frame_ws_bytes < hs_frame_workspace_size(f->n, f->width, f->height))
    return HS_ERR_WORKSPACE;
  return HS_OK;
}

static int check_bin_ws(const hs_frame* f) {
  if (!f->bin_ws) return HS_ERR_WORKSPACE;
  if (f->bin_ws_bytes < hs_binning_workspace_size(f->n, bin_capacity(f), f->width, f->height))
    return HS_ERR_WORKSPACE;
  return HS_OK;
}

static int check_scene(const hs_scene* s, const hs_frame* f) {
  if (!s || s->n != f->n) return HS_ERR_MISMATCHED_FORWARD;
  if (s->sh_degree < 0 || s->sh_degree > 3) return HS_ERR_INVALID_ARG;
  if (s->dtype != HS_DTYPE_F32 && s->dtype != HS_DTYPE_F64) return HS_ERR_INVALID_ARG;
  if (!s->mu || !s->log_scale || !s->rotation || !s->sh_coeffs || !s->normal ||
      !s->raw_opacity_a || !s->raw_opacity_b)
    return HS_ERR_INVALID_ARG;
  return HS_OK;
}

}  // namespace hs

using namespace hs;

static int reset_depth_range(const hs_frame* frame, const FrameBufs& f, uint32_t** range,
                             cudaStream_t stream);
static int rank_and_count(hs_frame* frame, const FrameBufs& f, const uint32_t* range,
                          cudaStream_t stream);

extern "C" {

int32_t hs_abi_version(void) { return 2; }

int64_t hs_kernel_launch_count(void) { return g_launches.load(); }

const char* hs_last_cuda_error(void) { return g_err; }

const char* hs_status_string(int status) {
  switch (status) {
    case HS_OK: return "ok";
    case HS_ERR_EMPTY_SCENE: return "EmptyScene: cannot render an empty scene";
    case HS_ERR_IMAGE_TOO_LARGE: return "ImageTooLarge: render target exceeds the supported size";
    case HS_ERR_INVALID_KERNEL: return "ValueError: kernel must be 'half' or 'full'";
    case HS_ERR_MISMATCHED_FORWARD: return "MismatchedForward: forward bookkeeping does not match";
    case HS_ERR_INVALID_ARG: return "invalid argument";
    case HS_ERR_CUDA: return "CUDA error";
    case HS_ERR_WORKSPACE: return "workspace missing or too small";
    case HS_ERR_IMAGE_TOO_SMALL: return "ImageTooSmall: needs at least 11 pixels on each side";
    case HS_ERR_INVALID_LAMBDA: return "ValueError: lambda_ssim must lie in [0, 1]";
    default: return "unknown status";
  }
}

int hs_frame_init(hs_frame* frame, int64_t n, int32_t width, int32_t height, int32_t kernel) {
  if (!frame) return HS_ERR_INVALID_ARG;
  memset(frame, 0, sizeof(*frame));
  if (n <= 0) return HS_ERR_EMPTY_SCENE;
  if ((int64_t)width * (int64_t)height > (int64_t)1 << 31) return HS_ERR_IMAGE_TOO_LARGE;
  if (kernel != HS_KERNEL_HALF && kernel != HS_KERNEL_FULL) return HS_ERR_INVALID_KERNEL;
  if (width <= 0 || height <= 0) return HS_ERR_INVALID_ARG;
  if (n > 0x7fffffffll) return HS_ERR_INVALID_ARG;
  const int tx = tiles_of(width), ty = tiles_of(height);
  // tx0/ty0 are packed into 16 bits of the splat record
  if (tx > 0xffff || ty > 0xffff) return HS_ERR_IMAGE_TOO_LARGE;
  frame->n = n;
  frame->width = width;
  frame->height = height;
  frame->tiles_x = tx;
  frame->tiles_y = ty;
  frame->n_tiles = tx * ty;
  frame->kernel = kernel;
  frame->tile_bits = bits_for(tx * ty);
  frame->num_pairs = -1;
  return HS_OK;
}

size_t hs_frame_workspace_size(int64_t n, int32_t width, int32_t height) {
  size_t total = 0;
  carve_frame(nullptr, n, tiles_of(width), tiles_of(height), &total);
  return total;
}

size_t hs_binning_workspace_size(int64_t n, int64_t num_pairs, int32_t width, int32_t height) {
  (void)n;
  size_t total = 0;
  carve_bin(nullptr, num_pairs, tiles_of(width), tiles_of(height), &total);
  return total;
}

static cudaError_t count_scan(const hs_frame* frame, const FrameBufs& f, cudaStream_t stream) {
  const bool segs = row_binning_ok(frame->tiles_x, frame->tiles_y);
  return run_count_scan(f.temp, f.temp_bytes, f.count, f.order, f.rect, f.cnt_r, f.off_r,
                        f.rank_of, frame->n, segs ? frame->tiles_x : 0, frame->tiles_y,
                        f.key_pairs, f.status, f.rect_r, stream);
}

int hs_preprocess_fwd(hs_frame* frame, const hs_scene* scene, const hs_camera* cam,
                      int32_t* radii, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if ((st = check_scene(scene, frame))) return st;
  if (!cam || cam->width != frame->width || cam->height != frame->height) return HS_ERR_INVALID_ARG;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  FrameBufs f = frame_bufs(frame);
  const CamArgs ca = cam_args(cam);
  uint32_t* range = nullptr;
  if ((st = reset_depth_range(frame, f, &range, stream))) return st;
  if (scene->dtype == HS_DTYPE_F32) {
    HS_CUDA(launch_preprocess_fwd_t<float>(scene_args<float>(scene), ca, frame->kernel, frame->n,
                                           f.rec, f.side, f.rect, f.count, f.dkey_in, f.dval,
                                           radii, range, stream));
  } else {
    HS_CUDA(launch_preprocess_fwd_t<double>(scene_args<double>(scene), ca, frame->kernel,
                                            frame->n, f.rec, f.side, f.rect, f.count, f.dkey_in,
                                            f.dval, radii, range, stream));
  }
  return rank_and_count(frame, f, range, stream);
}

int hs_preprocess_fwd_views(hs_frame* const* frames, int32_t n_views, const hs_scene* scene,
                            const hs_camera* cams, int32_t* const* radii, int32_t rank,
                            void* stream_) {
  if (!frames || n_views <= 0 || !cams) return HS_ERR_INVALID_ARG;
  for (int v = 0; v < n_views; ++v) {
    hs_frame* fr = frames[v];
    int st = check_frame_ws(fr);
    if (st) return st;
    if ((st = check_scene(scene, fr))) return st;
    if (cams[v].width != fr->width || cams[v].height != fr->height ||
        fr->kernel != frames[0]->kernel)
      return HS_ERR_INVALID_ARG;
  }
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  std::vector<uint32_t*> ranges((size_t)n_views, nullptr);
  for (int v0 = 0; v0 < n_views; v0 += kMaxViews) {
    FwdViewsArgs va;
    va.n_views = n_views - v0 < kMaxViews ? n_views - v0 : kMaxViews;
    for (int k = 0; k < va.n_views; ++k) {
      hs_frame* fr = frames[v0 + k];
      FrameBufs f = frame_bufs(fr);
      int st = reset_depth_range(fr, f, &ranges[(size_t)(v0 + k)], stream);
      if (st) return st;
      va.cam[k] = cam_args(&cams[v0 + k]);
      va.out[k] = FwdOut{f.rec, f.side, f.rect, f.count, f.dkey_in, f.dval,
                         radii ? radii[v0 + k] : nullptr, ranges[(size_t)(v0 + k)]};
    }
    if (scene->dtype == HS_DTYPE_F32)
      HS_CUDA(launch_preprocess_fwd_views_t<float>(scene_args<float>(scene), va,
                                                   frames[0]->kernel, scene->n, stream));
    else
      HS_CUDA(launch_preprocess_fwd_views_t<double>(scene_args<double>(scene), va,
                                                    frames[0]->kernel, scene->n, stream));
  }
  if (!rank) return HS_OK;  // the caller ranks each frame (hs_frame_rank), e.g. per stream
  for (int v = 0; v < n_views; ++v) {
    const int st = rank_and_count(frames[v], frame_bufs(frames[v]), ranges[(size_t)v], stream);
    if (st) return st;
  }
  return HS_OK;
}

int hs_frame_rank(hs_frame* frame, void* stream_) {
  const int st = check_frame_ws(frame);
  if (st) return st;
  FrameBufs f = frame_bufs(frame);
  return rank_and_count(
      frame, f,
      frame->depth_sort_full ? nullptr
                             : reinterpret_cast<uint32_t*>(f.counters + kDepthRangeSlot),
      static_cast<cudaStream_t>(stream_));
}

}  // extern "C"

// the 24-bit rank sort's depth range: [min, max] of the visible upper words (none
// when the frame ranks with the full 64-bit sort)
static int reset_depth_range(const hs_frame* frame, const FrameBufs& f, uint32_t** range,
                             cudaStream_t stream) {
  *range = frame->depth_sort_full ? nullptr
                                  : reinterpret_cast<uint32_t*>(f.counters + kDepthRangeSlot);
  if (*range) {
    HS_CUDA(cudaMemsetAsync(*range, 0xff, sizeof(uint32_t), stream));
    HS_CUDA(cudaMemsetAsync(*range + 1, 0, sizeof(uint32_t), stream));
  }
  return HS_OK;
}

// after K1: the depth ranks and the count scan
static int rank_and_count(hs_frame* frame, const FrameBufs& f, const uint32_t* range,
                          cudaStream_t stream) {
  if (frame->depth_sort_full) {
    HS_CUDA(cudaMemsetAsync(f.counters + kDepthOverflowSlot, 0, sizeof(int), stream));
    HS_CUDA(run_depth_sort(f.temp, f.temp_bytes, f.dkey_in, f.dkey_out, f.dval, f.order,
                           frame->n, stream));
  } else {
    // rank_of and cnt_r are outputs of the count scan below: free as fixup scratch here
    HS_CUDA(run_depth_sort_hi(f.temp, f.temp_bytes, f.dkey_in, f.dkey_out, f.dval, f.order,
                              frame->n, f.rank_of, reinterpret_cast<uint32_t*>(f.cnt_r),
                              f.counters + kDepthOverflowSlot, range, stream));
  }
  HS_CUDA(count_scan(frame, f, stream));
  frame->num_pairs = -1;
  return HS_OK;
}

extern "C" {

// P (int64, it cannot wrap) and the flags, with a host synchronisation.
static int read_status(hs_frame* frame, const FrameBufs& f, int64_t* p, int32_t* flags,
                       cudaStream_t stream) {
  BinStatusDev bs;
  int depth = 0;
  HS_CUDA(cudaMemcpyAsync(&bs, f.status, sizeof(bs), cudaMemcpyDeviceToHost, stream));
  HS_CUDA(cudaMemcpyAsync(&depth, f.counters + kDepthOverflowSlot, sizeof(int),
                          cudaMemcpyDeviceToHost, stream));
  HS_CUDA(cudaStreamSynchronize(stream));
  *p = bs.pairs;
  *flags = bs.flags | (depth ? kBinFlagDepth : 0);
  return HS_OK;
}

int hs_frame_read_num_pairs(hs_frame* frame, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  FrameBufs f = frame_bufs(frame);
  int64_t p = 0;
  int32_t flags = 0;
  if ((st = read_status(frame, f, &p, &flags, stream))) return st;
  if (p > 0x7fffffffll) return HS_ERR_INVALID_ARG;  // more pairs than int32 offsets hold
  if (flags & kBinFlagDepth) {
    // a depth bucket held more than the fixup handles (e.g. thousands of equal
    // depths): redo the ranks with the full 64-bit sort; P is order-independent
    HS_CUDA(cudaMemsetAsync(f.counters + kDepthOverflowSlot, 0, sizeof(int), stream));
    HS_CUDA(run_depth_sort(f.temp, f.temp_bytes, f.dkey_in, f.dkey_out, f.dval, f.order,
                           frame->n, stream));
    HS_CUDA(count_scan(frame, f, stream));
    frame->depth_sort_full = 1;
  }
  frame->num_pairs = p;
  return HS_OK;
}

int hs_frame_status(hs_frame* frame, int64_t* num_pairs, int32_t* flags, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if (!num_pairs || !flags) return HS_ERR_INVALID_ARG;
  FrameBufs f = frame_bufs(frame);
  if ((st = read_status(frame, f, num_pairs, flags, static_cast<cudaStream_t>(stream_))))
    return st;
  if (!*flags) frame->num_pairs = *num_pairs;
  return HS_OK;
}

int hs_frame_status_async(const hs_frame* frame, void* host_status, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if (!host_status) return HS_ERR_INVALID_ARG;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  FrameBufs f = frame_bufs(frame);
  char* h = static_cast<char*>(host_status);
  HS_CUDA(cudaMemcpyAsync(h, f.status, sizeof(BinStatusDev), cudaMemcpyDeviceToHost, stream));
  HS_CUDA(cudaMemcpyAsync(h + sizeof(BinStatusDev), f.counters + kDepthOverflowSlot, sizeof(int),
                          cudaMemcpyDeviceToHost, stream));
  return HS_OK;
}

int hs_read_pairs_and_bin(hs_frame* frame, void* stream_) {
  int st = hs_frame_read_num_pairs(frame, stream_);
  if (st) return st;
  const int64_t cap = frame->pair_capacity > frame->num_pairs ? frame->pair_capacity
                                                              : frame->num_pairs;
  if (!frame->bin_ws ||
      frame->bin_ws_bytes < hs_binning_workspace_size(frame->n, cap, frame->width, frame->height))
    return HS_ERR_WORKSPACE;  // P is set: size the workspace, then hs_bin_and_sort
  return hs_bin_and_sort(frame, stream_);
}

static int row_bin(hs_frame* frame, const FrameBufs& f, const BinBufs& b, cudaStream_t stream) {
  RowBinArgs a;
  a.order = f.order;
  a.rect = f.rect;
  a.rect_r = f.rect_r;
  a.row_origin = f.row_origin;
  a.cnt_r = f.cnt_r;
  a.off_r = f.off_r;
  a.status = f.status;
  a.key_pairs = f.key_pairs;
  a.n = frame->n;
  a.nb = (int)bin_row_blocks(frame->n);
  a.tiles_x = frame->tiles_x;
  a.tiles_y = frame->tiles_y;
  a.nblk = seg_blocks(frame->tiles_x);
  a.keys = seg_keys(frame->tiles_x, frame->tiles_y);
  a.capacity = bin_capacity(frame);
  a.segs = b.segs;
  a.chunk_first = f.chunk_first;
  a.seg_cnt = b.seg_cnt;
  a.tile_starts = f.tile_starts;
  a.pair_src = b.pair_src;
  HS_CUDA(run_row_binning(a, stream));
  return HS_OK;
}

int hs_bin_and_sort(hs_frame* frame, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if (frame->num_pairs < 0) return HS_ERR_INVALID_ARG;
  if (frame->pair_capacity < frame->num_pairs) frame->pair_capacity = frame->num_pairs;
  if ((st = check_bin_ws(frame))) return st;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  FrameBufs f = frame_bufs(frame);
  BinBufs b = frame_bin(frame);
  if (row_binning_ok(frame->tiles_x, frame->tiles_y)) return row_bin(frame, f, b, stream);
  const int64_t p = frame->num_pairs;
  int sel = 0;
  if (p > 0) {
    HS_CUDA(run_duplicate(f.order, f.cnt_r, f.off_r, f.rect, f.row_origin, frame->tiles_x,
                          b.keys[0],
                          b.vals[0], frame->n, stream));
    HS_CUDA(run_pair_sort(b.temp, b.temp_bytes, b.keys[0], b.keys[1], b.vals[0], b.vals[1], p,
                          frame->tile_bits, &sel, stream));
  }
  frame->sort_selector = sel;
  HS_CUDA(run_tile_ranges(b.keys[sel], p, frame->n_tiles, f.tile_starts, stream));
  return HS_OK;
}

int hs_bin_async(hs_frame* frame, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if (!row_binning_ok(frame->tiles_x, frame->tiles_y)) {
    // the CUB path sizes its passes from P: read it (a host sync), then bin
    if ((st = hs_frame_read_num_pairs(frame, stream_))) return st;
    if (frame->pair_capacity < frame->num_pairs) return HS_ERR_WORKSPACE;
    return hs_bin_and_sort(frame, stream_);
  }
  if (frame->pair_capacity <= 0) return HS_ERR_INVALID_ARG;
  if ((st = check_bin_ws(frame))) return st;
  frame->num_pairs = -1;  // on the device until hs_frame_status
  return row_bin(frame, frame_bufs(frame), frame_bin(frame), static_cast<cudaStream_t>(stream_));
}

static const uint32_t* sorted_pairs(const hs_frame* frame, const BinBufs& b) {
  return row_binning_ok(frame->tiles_x, frame->tiles_y) ? b.pair_src
                                                        : b.vals[frame->sort_selector];
}

// P for launch heuristics (K7a's lanes per splat): exact once read, else the capacity
static int64_t pairs_hint(const hs_frame* frame) {
  return frame->num_pairs >= 0 ? frame->num_pairs : bin_capacity(frame) * 4 / 5;
}

// Longest-first tile order for the blends when the tiles are at least 1.5x the
// blend's resident warps (HS_LPT=0 never, HS_LPT=1 always).  Measured per view:
// c3 K5 0.807 -> 0.784 ms, K6 1.512 -> 1.475; c4 K6 1.314 -> 1.096; but c2, whose
// 2500 tiles about fill the resident warps once, K5 0.379 -> 0.457, K6 0.630 -> 0.695.
static bool lpt_order(int n_tiles, int slots) {
  static const int mode = [] {
    const char* e = getenv("HS_LPT");
    return e ? (e[0] == '0' ? 0 : 1) : 2;
  }();
  return mode == 1 || (mode == 2 && 2 * (int64_t)n_tiles >= 3 * (int64_t)slots);
}

// K5 work units per tile: whole tiles when the frame has enough of them to fill the
// resident warps 1.5 times, else 4 sub-tiles of 16x4 (HS_SUBTILE=1/2/4 forces a
// split).  Measured per view: c2 (2500 tiles, 2368 warps) K5 0.255 ms in 16x8 halves,
// 0.243 in 16x4 quarters; c4 (4346 tiles) 0.714 whole, 0.758 in halves.
static int fwd_sub_tiles(int n_tiles, int slots) {
  const char* env = getenv("HS_SUBTILE");  // read per call: tests switch it
  const int forced = env ? atoi(env) : 0;
  if (forced == 1 || forced == 2 || forced == 4) return forced;
  return 2 * (int64_t)n_tiles >= 3 * (int64_t)slots ? 1 : 4;
}

// K5/K6 queues with an SM-spread first wave (HS_SPREAD=0: a plain counter)
static int spread_queue() {
  static const int on = [] {
    const char* e = getenv("HS_SPREAD");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return on;
}

static BlendGeom frame_geom(const hs_frame* frame, const FrameBufs& f, const BinBufs& b) {
  BlendGeom g;
  g.tile_starts = f.tile_starts;
  g.pair_src = sorted_pairs(frame, b);
  g.rec = f.rec;
  g.row_origin = f.row_origin;
  g.side = f.side;
  g.width = frame->width;
  g.height = frame->height;
  g.tiles_x = frame->tiles_x;
  g.tile_lo = 0;
  g.n_work = frame->n_tiles;
  g.tile_order = nullptr;
  g.tile_work = nullptr;
  g.sub_tiles = 1;
  g.work_counter = f.queue_fwd;
  g.spread = spread_queue();
  g.ckpt = nullptr;
  g.units = nullptr;
  g.n_units = nullptr;
  g.ckpt_shift = ckpt_shift(frame->n_tiles);
  return g;
}

int hs_blend_fwd(hs_frame* frame, const double* bg, float* color, float* alpha, float* depth,
                 float* transmittance, int32_t* terminal, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if ((st = check_bin_ws(frame))) return st;
  if (!bg || !color || !alpha || !depth || !transmittance || !terminal) return HS_ERR_INVALID_ARG;
  FrameBufs f = frame_bufs(frame);
  BinBufs b = frame_bin(frame);
  BlendGeom g = frame_geom(frame, f, b);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  g.tile_work = f.tile_work;
  g.sub_tiles = fwd_sub_tiles(frame->n_tiles, blend_fwd_slots());
  if (bwd_split(frame->n_tiles)) g.ckpt = b.ckpt;
  if (lpt_order(frame->n_tiles * g.sub_tiles, blend_fwd_slots())) {
    HS_CUDA(launch_tile_order(f.tile_starts, nullptr, frame->n_tiles, f.order_fwd, stream));
    g.tile_order = f.order_fwd;
  }
  HS_CUDA(launch_blend_fwd(g, (float)bg[0], (float)bg[1], (float)bg[2], color, alpha, depth,
                           transmittance, terminal, stream));
  return HS_OK;
}

int hs_blend_bwd(hs_frame* frame, const double* bg, const float* d_color,
                 const float* transmittance, const int32_t* terminal, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if ((st = check_bin_ws(frame))) return st;
  if (!bg || !d_color || !transmittance || !terminal) return HS_ERR_INVALID_ARG;
  FrameBufs f = frame_bufs(frame);
  BinBufs b = frame_bin(frame);
  BlendGeom g = frame_geom(frame, f, b);
  g.work_counter = f.queue_bwd;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (lpt_order(frame->n_tiles, blend_bwd_slots())) {
    // K5 left each tile's largest terminal count: the positions K6 walks
    HS_CUDA(launch_tile_order(nullptr, f.tile_work, frame->n_tiles, f.order_bwd, stream));
    g.tile_order = f.order_bwd;
  }
  if (bwd_split(frame->n_tiles)) {
    // (tile, segment) units from K5's checkpoints, tiles in the order above
    HS_CUDA(launch_bwd_units(f.tile_work, g.tile_order, frame->n_tiles, g.ckpt_shift, b.units,
                             b.n_units, stream));
    g.ckpt = b.ckpt;
    g.units = b.units;
    g.n_units = b.n_units;
  }
  HS_CUDA(launch_blend_bwd(g, (float)bg[0], (float)bg[1], (float)bg[2], d_color, transmittance,
                           terminal, b.rows, f.last_rank, f.rank_of, false, stream));
  return HS_OK;
}

int hs_blend_window_stats(hs_frame* frame, unsigned long long* hist, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if ((st = check_bin_ws(frame))) return st;
  if (!hist) return HS_ERR_INVALID_ARG;
  FrameBufs f = frame_bufs(frame);
  BinBufs b = frame_bin(frame);
  BlendGeom g = frame_geom(frame, f, b);
  HS_CUDA(launch_window_stats(g, hist, static_cast<cudaStream_t>(stream_)));
  return HS_OK;
}

int hs_preprocess_bwd(hs_frame* frame, const hs_scene* scene, const hs_camera* cam,
                      const hs_grads* grads, void* stream_) {
  return hs_preprocess_bwd_range(frame, scene, cam, grads, 0, INT64_MAX, stream_);
}

int hs_preprocess_bwd_range(hs_frame* frame, const hs_scene* scene, const hs_camera* cam,
                            const hs_grads* grads, int64_t begin, int64_t end, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if ((st = check_bin_ws(frame))) return st;
  if ((st = check_scene(scene, frame))) return st;
  if (!cam || !grads || !grads->d_mu || !grads->d_log_scale || !grads->d_rotation ||
      !grads->d_sh || !grads->d_normal || !grads->d_raw_opacity_a || !grads->d_raw_opacity_b ||
      !grads->pos_grad_norm || !grads->touch_count || grads->accumulate < 0 ||
      grads->accumulate > 3 || begin < 0 || begin % 128 != 0 || end < begin)
    return HS_ERR_INVALID_ARG;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  FrameBufs f = frame_bufs(frame);
  BinBufs b = frame_bin(frame);
  const CamArgs ca = cam_args(cam);
  if (scene->dtype == HS_DTYPE_F32) {
    HS_CUDA(launch_preprocess_bwd_t<float>(scene_args<float>(scene), ca, frame->kernel, frame->n,
                                           frame->tiles_x, f.rec, f.row_origin, f.rect, f.count,
                                           f.rank_of,
                                           f.last_rank, b.rows, f.merged, pairs_hint(frame),
                                           ranged(grad_args<float>(grads), begin, end), stream));
  } else {
    HS_CUDA(launch_preprocess_bwd_t<double>(scene_args<double>(scene), ca, frame->kernel,
                                            frame->n, frame->tiles_x, f.rec, f.row_origin, f.rect,
                                            f.count,
                                            f.rank_of, f.last_rank, b.rows, f.merged,
                                            pairs_hint(frame),
                                            ranged(grad_args<double>(grads), begin, end),
                                            stream));
  }
  return HS_OK;
}

int hs_merge_rows(hs_frame* frame, float* merged_out, void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if ((st = check_bin_ws(frame))) return st;
  if (!merged_out || ((uintptr_t)merged_out & 15)) return HS_ERR_INVALID_ARG;
  FrameBufs f = frame_bufs(frame);
  BinBufs b = frame_bin(frame);
  HS_CUDA(launch_merge_rows(frame->n, frame->tiles_x, f.rec, f.row_origin, f.rect, f.count,
                            f.rank_of,
                            f.last_rank, b.rows, reinterpret_cast<float4*>(merged_out),
                            pairs_hint(frame), static_cast<cudaStream_t>(stream_)));
  return HS_OK;
}

int hs_preprocess_bwd_views(const hs_scene* scene, int32_t n_views, const hs_camera* cams,
                            const float* const* merged, int32_t kernel, const hs_grads* grads,
                            int64_t begin, int64_t end, void* stream_) {
  if (!scene || n_views <= 0 || !cams || !merged || kernel < 0 || kernel > 1)
    return HS_ERR_INVALID_ARG;
  hs_frame shape{};
  shape.n = scene->n;
  if (int st = check_scene(scene, &shape)) return st;
  if (!grads || !grads->d_mu || !grads->d_log_scale || !grads->d_rotation || !grads->d_sh ||
      !grads->d_normal || !grads->d_raw_opacity_a || !grads->d_raw_opacity_b ||
      !grads->pos_grad_norm || !grads->touch_count || grads->accumulate < 0 ||
      grads->accumulate > 3 || begin < 0 || begin % 128 != 0 || end < begin)
    return HS_ERR_INVALID_ARG;
  std::vector<CamArgs> ca((size_t)n_views);
  std::vector<const float4*> mg((size_t)n_views);
  for (int v = 0; v < n_views; ++v) {
    if (!merged[v] || ((uintptr_t)merged[v] & 15)) return HS_ERR_INVALID_ARG;
    ca[(size_t)v] = cam_args(&cams[v]);
    mg[(size_t)v] = reinterpret_cast<const float4*>(merged[v]);
  }
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (scene->dtype == HS_DTYPE_F32)
    HS_CUDA(launch_preprocess_bwd_views_t<float>(scene_args<float>(scene), ca.data(), mg.data(),
                                                 n_views, kernel, scene->n,
                                                 ranged(grad_args<float>(grads), begin, end),
                                                 stream));
  else
    HS_CUDA(launch_preprocess_bwd_views_t<double>(scene_args<double>(scene), ca.data(), mg.data(),
                                                  n_views, kernel, scene->n,
                                                  ranged(grad_args<double>(grads), begin, end),
                                                  stream));
  return HS_OK;
}

int hs_frame_export(const hs_frame* frame, int32_t* valid, int64_t* m_out, float* packed,
                    int8_t* mode, int32_t* tile_rect, int32_t* pair_splat, int64_t* tile_starts,
                    void* stream_) {
  int st = check_frame_ws(frame);
  if (st) return st;
  if (!m_out) return HS_ERR_INVALID_ARG;
  const bool binned = frame->bin_ws && frame->num_pairs >= 0;
  if ((pair_splat || tile_starts) && !binned) return HS_ERR_INVALID_ARG;
  FrameBufs f = frame_bufs(frame);
  const uint32_t* pair_src = nullptr;
  if (binned) {
    BinBufs b = frame_bin(frame);
    pair_src = sorted_pairs(frame, b);
  }
  HS_CUDA(run_export(f.temp, f.temp_bytes, f.count, f.rec, f.rect, pair_src, f.tile_starts,
                     frame->n, binned ? frame->num_pairs : 0, frame->n_tiles, f.xlocal, f.xflags,
                     valid, m_out, packed, mode, tile_rect, pair_splat, tile_starts,
                     static_cast<cudaStream_t>(stream_)));
  return HS_OK;
}

int hs_screen_splats(const hs_scene* scene, const hs_camera* cam, int32_t kernel, double* out,
                     void* stream_) {
  if (!scene || !cam || !out) return HS_ERR_INVALID_ARG;
  if (scene->n <= 0) return HS_ERR_EMPTY_SCENE;
  if (kernel != HS_KERNEL_HALF && kernel != HS_KERNEL_FULL) return HS_ERR_INVALID_KERNEL;
  const CamArgs ca = cam_args(cam);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (scene->dtype == HS_DTYPE_F32)
    HS_CUDA(launch_screen_splats_t<float>(scene_args<float>(scene), ca, kernel, scene->n, out,
                                          stream));
  else
    HS_CUDA(launch_screen_splats_t<double>(scene_args<double>(scene), ca, kernel, scene->n, out,
                                           stream));
  return HS_OK;
}

// ---- Seam 1 ----------------------------------------------------------------
namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes > 0 ? bytes : 16); }
};

int seam1_validate(const int64_t* tile_starts, int64_t num_pairs, int32_t height, int32_t width,
                   int32_t tiles_x, int32_t tile_lo, int32_t tile_hi) {
  if (height <= 0 || width <= 0 || tiles_x != tiles_of(width)) return HS_ERR_INVALID_ARG;
  const int n_tiles = tiles_x * tiles_of(height);
  if (tile_lo < 0 || tile_hi > n_tiles || tile_lo > tile_hi) return HS_ERR_INVALID_ARG;
  if (!tile_starts || tile_starts[n_tiles] != num_pairs) return HS_ERR_INVALID_ARG;
  if (num_pairs > 0x7fffffffll) return HS_ERR_INVALID_ARG;
  return HS_OK;
}
}  // namespace

}  // extern "C"

// Seam 1 under the reference's threaded chunk dispatch (rasterizer.py:373-378):
// every chunk call of one frame passes the same packed / mode / pair_splat /
// tile_starts (and, backward, the same cotangent and forward outputs).  The
// first call of a frame blends ALL tiles on the GPU and keeps the full result on
// the host; every later call whose inputs compare equal (memcmp against the kept
// copies, exact) only copies its tiles out.  Concurrent calls read the cache
// under a shared lock; a miss recomputes under the exclusive lock.
namespace {

struct HostCopy {
  std::vector<char> b;
  void set(const void* p, size_t n) {
    b.resize(n);
    if (n) memcpy(b.data(), p, n);
  }
  bool same(const void* p, size_t n) const {
    return b.size() == n && (n == 0 || memcmp(b.data(), p, n) == 0);
  }
};

struct Seam1Key {
  HostCopy packed, mode, pairs, starts;
  int32_t h = -1, w = -1, tx = -1;
  double bg[3] = {0, 0, 0};
  void set(const double* pk, const int8_t* md, const int32_t* ps, const int64_t* ts, int64_t m,
           int64_t p, int32_t hh, int32_t ww, int32_t t, const double* b, int n_tiles) {
    packed.set(pk, (size_t)m * 13 * sizeof(double));
    mode.set(md, (size_t)m);
    pairs.set(ps, (size_t)p * sizeof(int32_t));
    starts.set(ts, (size_t)(n_tiles + 1) * sizeof(int64_t));
    h = hh; w = ww; tx = t;
    for (int k = 0; k < 3; ++k) bg[k] = b[k];
  }
  bool same(const double* pk, const int8_t* md, const int32_t* ps, const int64_t* ts, int64_t m,
            int64_t p, int32_t hh, int32_t ww, int32_t t, const double* b, int n_tiles) const {
    return h == hh && w == ww && tx == t && bg[0] == b[0] && bg[1] == b[1] && bg[2] == b[2] &&
           starts.same(ts, (size_t)(n_tiles + 1) * sizeof(int64_t)) &&
           pairs.same(ps, (size_t)p * sizeof(int32_t)) && mode.same(md, (size_t)m) &&
           packed.same(pk, (size_t)m * 13 * sizeof(double));
  }
};

struct FwdCache {
  bool valid = false;
  Seam1Key key;
  std::vector<float> out;  // color (3 npx), alpha, depth, transmittance
  std::vector<int32_t> term;
};
struct BwdCache {
  bool valid = false;
  Seam1Key key;
  HostCopy d_color, trans, term;
  std::vector<float> rows;  // (P, 12), every pair of the frame
};
std::shared_mutex g_fwd_mu, g_bwd_mu;
FwdCache g_fwd;
BwdCache g_bwd;

struct Seam1Dev {
  cudaStream_t s = nullptr;
  DevBuf packed, mode, rec, side, pairs, ts, ctr;
  ~Seam1Dev() {
    if (s) cudaStreamDestroy(s);
  }
};

// upload + pack the reference's frame (shared by both directions)
int seam1_upload(Seam1Dev& d, const double* packed, const int8_t* mode,
                 const int32_t* pair_splat, const int64_t* tile_starts, int64_t m, int64_t p,
                 int n_tiles, BlendGeom& g, int32_t height, int32_t width, int32_t tiles_x) {
  std::vector<int32_t> ts32(n_tiles + 1);
  for (int t = 0; t <= n_tiles; ++t) ts32[t] = (int32_t)tile_starts[t];
  HS_CUDA(cudaStreamCreateWithFlags(&d.s, cudaStreamNonBlocking));
  HS_CUDA(d.packed.alloc(m * 13 * sizeof(double)));
  HS_CUDA(d.mode.alloc(m));
  HS_CUDA(d.rec.alloc(m * 64));
  HS_CUDA(d.side.alloc(m * sizeof(SteepRec)));
  HS_CUDA(d.pairs.alloc(p * 4));
  HS_CUDA(d.ts.alloc((n_tiles + 1) * 4));
  HS_CUDA(d.ctr.alloc(256));
  if (m > 0) {
    HS_CUDA(cudaMemcpyAsync(d.packed.p, packed, m * 13 * sizeof(double), cudaMemcpyHostToDevice,
                            d.s));
    HS_CUDA(cudaMemcpyAsync(d.mode.p, mode, m, cudaMemcpyHostToDevice, d.s));
  }
  if (p > 0) HS_CUDA(cudaMemcpyAsync(d.pairs.p, pair_splat, p * 4, cudaMemcpyHostToDevice, d.s));
  HS_CUDA(cudaMemcpyAsync(d.ts.p, ts32.data(), (n_tiles + 1) * 4, cudaMemcpyHostToDevice, d.s));
  HS_CUDA(launch_pack_records((const double*)d.packed.p, (const int8_t*)d.mode.p, m,
                              (float4*)d.rec.p, (SteepRec*)d.side.p, (uint32_t*)d.pairs.p, p, d.s));
  HS_CUDA(cudaStreamSynchronize(d.s));  // ts32 goes out of scope
  g.tile_starts = (const int32_t*)d.ts.p;
  g.pair_src = (const uint32_t*)d.pairs.p;
  g.rec = (const float4*)d.rec.p;
  g.row_origin = nullptr;
  g.side = (const SteepRec*)d.side.p;
  g.width = width;
  g.height = height;
  g.tiles_x = tiles_x;
  g.tile_lo = 0;
  g.n_work = n_tiles;
  g.tile_order = nullptr;
  g.tile_work = nullptr;
  g.sub_tiles = 1;
  g.work_counter = (int*)d.ctr.p;
  g.spread = 0;
  g.ckpt = nullptr;
  g.units = nullptr;
  g.n_units = nullptr;
  g.ckpt_shift = 8;
  return HS_OK;
}

}  // namespace

extern "C" {

int hs_forward_tiles(const double* packed, const int8_t* mode, const int32_t* pair_splat,
                     const int64_t* tile_starts, int64_t m, int64_t p, int32_t height,
                     int32_t width, int32_t tiles_x, const double* bg, double* color, double* alpha,
                     double* depth, double* transmittance, int32_t* terminal, int32_t tile_lo,
                     int32_t tile_hi) {
  int st = seam1_validate(tile_starts, p, height, width, tiles_x, tile_lo, tile_hi);
  if (st) return st;
  if (tile_hi == tile_lo) return HS_OK;
  const int n_tiles = tiles_x * tiles_of(height);
  const size_t npx = (size_t)height * width;
  auto copy_out = [&](const FwdCache& c) {
    const float* h = c.out.data();
    for (int t = tile_lo; t < tile_hi; ++t) {
      const int ty = t / tiles_x, tx = t - ty * tiles_x;
      for (int r = ty * kTile; r < ty * kTile + kTile && r < height; ++r)
        for (int col = tx * kTile; col < tx * kTile + kTile && col < width; ++col) {
          const size_t q = (size_t)r * width + col;
          for (int ch = 0; ch < 3; ++ch) color[3 * q + ch] = h[3 * q + ch];
          alpha[q] = h[3 * npx + q];
          depth[q] = h[4 * npx + q];
          transmittance[q] = h[5 * npx + q];
          terminal[q] = c.term[q];
        }
    }
  };
  {
    std::shared_lock<std::shared_mutex> lock(g_fwd_mu);
    if (g_fwd.valid && g_fwd.key.same(packed, mode, pair_splat, tile_starts, m, p, height, width,
                                      tiles_x, bg, n_tiles)) {
      copy_out(g_fwd);
      return HS_OK;
    }
  }
  std::unique_lock<std::shared_mutex> lock(g_fwd_mu);
  if (!(g_fwd.valid && g_fwd.key.same(packed, mode, pair_splat, tile_starts, m, p, height, width,
                                      tiles_x, bg, n_tiles))) {
    g_fwd.valid = false;
    Seam1Dev d;
    BlendGeom g;
    if ((st = seam1_upload(d, packed, mode, pair_splat, tile_starts, m, p, n_tiles, g, height,
                           width, tiles_x)))
      return st;
    DevBuf d_out, d_term;
    HS_CUDA(d_out.alloc(npx * 6 * sizeof(float)));
    HS_CUDA(d_term.alloc(npx * 4));
    float* o = (float*)d_out.p;
    HS_CUDA(launch_blend_fwd(g, (float)bg[0], (float)bg[1], (float)bg[2], o, o + 3 * npx,
                             o + 4 * npx, o + 5 * npx, (int32_t*)d_term.p, d.s));
    g_fwd.out.resize(npx * 6);
    g_fwd.term.resize(npx);
    HS_CUDA(cudaMemcpyAsync(g_fwd.out.data(), o, npx * 6 * sizeof(float), cudaMemcpyDeviceToHost,
                            d.s));
    HS_CUDA(cudaMemcpyAsync(g_fwd.term.data(), d_term.p, npx * 4, cudaMemcpyDeviceToHost, d.s));
    HS_CUDA(cudaStreamSynchronize(d.s));
    g_fwd.key.set(packed, mode, pair_splat, tile_starts, m, p, height, width, tiles_x, bg,
                  n_tiles);
    g_fwd.valid = true;
  }
  copy_out(g_fwd);
  return HS_OK;
}

int hs_backward_tiles(const double* packed, const int8_t* mode, const int32_t* pair_splat,
                      const int64_t* tile_starts, int64_t m, int64_t p, int32_t height,
                      int32_t width, int32_t tiles_x, const double* bg, const double* d_color,
                      const double* transmittance, const int32_t* terminal, double* pair_grads,
                      int32_t tile_lo, int32_t tile_hi) {
  int st = seam1_validate(tile_starts, p, height, width, tiles_x, tile_lo, tile_hi);
  if (st) return st;
  if (tile_hi == tile_lo || p == 0) return HS_OK;
  const int n_tiles = tiles_x * tiles_of(height);
  const size_t npx = (size_t)height * width;
  auto same = [&](const BwdCache& c) {
    return c.valid && c.term.same(terminal, npx * 4) &&
           c.trans.same(transmittance, npx * sizeof(double)) &&
           c.d_color.same(d_color, npx * 3 * sizeof(double)) &&
           c.key.same(packed, mode, pair_splat, tile_starts, m, p, height, width, tiles_x, bg,
                      n_tiles);
  };
  auto add_rows = [&](const BwdCache& c) {  // pair rows of this chunk's tiles, +=
    const int64_t r0 = tile_starts[tile_lo], r1 = tile_starts[tile_hi];
    for (int64_t k = r0; k < r1; ++k)
      for (int col = 0; col < 12; ++col) pair_grads[k * 12 + col] += c.rows[k * 12 + col];
  };
  {
    std::shared_lock<std::shared_mutex> lock(g_bwd_mu);
    if (same(g_bwd)) {
      add_rows(g_bwd);
      return HS_OK;
    }
  }
  std::unique_lock<std::shared_mutex> lock(g_bwd_mu);
  if (!same(g_bwd)) {
    g_bwd.valid = false;
    std::vector<float> hin(npx * 4);
    for (size_t q = 0; q < npx * 3; ++q) hin[q] = (float)d_color[q];
    for (size_t q = 0; q < npx; ++q) hin[3 * npx + q] = (float)transmittance[q];
    Seam1Dev d;
    BlendGeom g;
    if ((st = seam1_upload(d, packed, mode, pair_splat, tile_starts, m, p, n_tiles, g, height,
                           width, tiles_x)))
      return st;
    DevBuf d_in, d_term, d_rows;
    HS_CUDA(d_in.alloc(npx * 4 * sizeof(float)));
    HS_CUDA(d_term.alloc(npx * 4));
    HS_CUDA(d_rows.alloc(p * 12 * sizeof(float)));
    HS_CUDA(cudaMemcpyAsync(d_in.p, hin.data(), npx * 4 * sizeof(float), cudaMemcpyHostToDevice,
                            d.s));
    HS_CUDA(cudaMemcpyAsync(d_term.p, terminal, npx * 4, cudaMemcpyHostToDevice, d.s));
    HS_CUDA(cudaMemsetAsync(d_rows.p, 0, p * 12 * sizeof(float), d.s));
    const float* in = (const float*)d_in.p;
    HS_CUDA(launch_blend_bwd(g, (float)bg[0], (float)bg[1], (float)bg[2], in, in + 3 * npx,
                             (const int32_t*)d_term.p, (float*)d_rows.p, nullptr, nullptr, true,
                             d.s));
    g_bwd.rows.resize((size_t)p * 12);
    HS_CUDA(cudaMemcpyAsync(g_bwd.rows.data(), d_rows.p, p * 12 * sizeof(float),
                            cudaMemcpyDeviceToHost, d.s));
    HS_CUDA(cudaStreamSynchronize(d.s));
    g_bwd.key.set(packed, mode, pair_splat, tile_starts, m, p, height, width, tiles_x, bg, n_tiles);
    g_bwd.d_color.set(d_color, npx * 3 * sizeof(double));
    g_bwd.trans.set(transmittance, npx * sizeof(double));
    g_bwd.term.set(terminal, npx * 4);
    g_bwd.valid = true;
  }
  add_rows(g_bwd);
  return HS_OK;
}

void hs_seam1_cache_clear(void) {
  {
    std::unique_lock<std::shared_mutex> lock(g_fwd_mu);
    g_fwd = FwdCache();
  }
  std::unique_lock<std::shared_mutex> lock(g_bwd_mu);
  g_bwd = BwdCache();
}

}  // extern "C"

// ---- training loss (loss.py:48-106) -----------------------------------------
namespace {
struct LossBufs {
  double* adj_m;
  double* adj_s1;
  double* adj_s12;
  double* partial;
};
LossBufs carve_loss(void* ws, int32_t height, int32_t width, int32_t channels, size_t* bytes) {
  Carver c(ws);
  const size_t n = (size_t)height * width * channels;
  LossBufs b;
  b.adj_m = c.take<double>(n);
  b.adj_s1 = c.take<double>(n);
  b.adj_s12 = c.take<double>(n);
  b.partial = c.take<double>(3 * (size_t)hs::loss_partials(width, height, channels));
  *bytes = c.off;
  return b;
}
}  // namespace

extern "C" size_t hs_loss_workspace_size(int32_t height, int32_t width, int32_t channels) {
  if (height <= 0 || width <= 0 || channels <= 0) return 0;
  size_t bytes = 0;
  carve_loss(nullptr, height, width, channels, &bytes);
  return bytes;
}

static int loss_impl(const float* rendered, const float* target, const double* rendered64,
                     const double* target64, int32_t height, int32_t width, int32_t channels,
                     double lambda_ssim, double* loss4, float* d_rendered,
                     double* d_rendered_f64, void* ws, size_t ws_bytes, void* stream_) {
  if (!((rendered && target) || (rendered64 && target64)) || !loss4 || height <= 0 ||
      width <= 0 || channels <= 0)
    return HS_ERR_INVALID_ARG;
  if (!(lambda_ssim >= 0.0 && lambda_ssim <= 1.0)) return HS_ERR_INVALID_LAMBDA;
  const bool ssim = lambda_ssim != 0.0;  // loss.py:97-103: lambda 0 skips SSIM
  if (ssim && (height < 11 || width < 11)) return HS_ERR_IMAGE_TOO_SMALL;
  size_t need = 0;
  carve_loss(nullptr, height, width, channels, &need);
  if (!ws || ws_bytes < need) return HS_ERR_WORKSPACE;
  const LossBufs b = carve_loss(ws, height, width, channels, &need);
  hs::LossArgs a;
  a.x = rendered;
  a.y = target;
  a.x64 = rendered64;
  a.y64 = target64;
  a.width = width;
  a.height = height;
  a.channels = channels;
  a.lambda = lambda_ssim;
  a.n = (double)height * width * channels;
  a.inv_n = 1.0 / a.n;
  a.adj_m = b.adj_m;
  a.adj_s1 = b.adj_s1;
  a.adj_s12 = b.adj_s12;
  a.partial = b.partial;
  a.n_partials = (int)hs::loss_partials(width, height, channels);
  a.loss = loss4;
  a.d_f32 = d_rendered;
  a.d_f64 = d_rendered_f64;
  a.ssim = ssim;
  a.group0 = 0;
  // _window(), loss.py:19-23
  for (int k = 0; k < 11; ++k) {
    const double t = (double)(k - 5) / 1.5;
    a.win[k] = std::exp(-0.5 * (t * t));
  }
  // numpy's pairwise sum order for 11 elements: 8 lanes, tree, then the tail
  const double* w = a.win;
  double sum = ((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7]));
  sum += w[8];
  sum += w[9];
  sum += w[10];
  for (int k = 0; k < 11; ++k) a.win[k] /= sum;
  HS_CUDA(hs::launch_loss(a, static_cast<cudaStream_t>(stream_)));
  return HS_OK;
}

extern "C" int hs_loss(const float* rendered, const float* target, int32_t height, int32_t width,
                       int32_t channels, double lambda_ssim, double* loss4, float* d_rendered,
                       double* d_rendered_f64, void* ws, size_t ws_bytes, void* stream_) {
  if (!rendered || !target) return HS_ERR_INVALID_ARG;
  return loss_impl(rendered, target, nullptr, nullptr, height, width, channels, lambda_ssim,
                   loss4, d_rendered, d_rendered_f64, ws, ws_bytes, stream_);
}

extern "C" int hs_loss_f64(const double* rendered, const double* target, int32_t height,
                           int32_t width, int32_t channels, double lambda_ssim, double* loss4,
                           float* d_rendered, double* d_rendered_f64, void* ws, size_t ws_bytes,
                           void* stream_) {
  if (!rendered || !target) return HS_ERR_INVALID_ARG;
  return loss_impl(nullptr, nullptr, rendered, target, height, width, channels, lambda_ssim,
                   loss4, d_rendered, d_rendered_f64, ws, ws_bytes, stream_);
}

// ---- optimizer (trainer.py:192-224) -------------------------------------------
extern "C" int hs_adam_step(const hs_scene* scene, const hs_grads* grads, hs_adam_state* state,
                            const double lr[HS_ADAM_GROUPS], int32_t tie_opacities,
                            void* stream_) {
  if (!scene || !grads || !state || !lr) return HS_ERR_INVALID_ARG;
  if (scene->n <= 0) return HS_ERR_EMPTY_SCENE;
  if (scene->sh_degree < 0 || scene->sh_degree > 3) return HS_ERR_INVALID_ARG;
  for (int g = 0; g < HS_ADAM_GROUPS; ++g)
    if (!(lr[g] >= 0.0)) return HS_ERR_INVALID_ARG;
  const int64_t n = scene->n;
  const int K = (scene->sh_degree + 1) * (scene->sh_degree + 1);
  bool on[HS_ADAM_GROUPS];
  double bc1[HS_ADAM_GROUPS], bc2[HS_ADAM_GROUPS];
  for (int g = 0; g < HS_ADAM_GROUPS; ++g) {
    on[g] = lr[g] != 0.0;
    // sh_rest has no coefficients at degree 0: the reference still counts its step
    const int64_t t = state->t[g] + (on[g] ? 1 : 0);
    bc1[g] = 1.0 - std::pow(0.9, (double)t);  // 1 - ADAM_BETA1**t (trainer.py:210)
    bc2[g] = 1.0 - std::pow(0.999, (double)t);
  }
  hs::AdamArgs a;
  memset(&a, 0, sizeof(a));
  int s = 0;
  auto add = [&](int kind, int field, int64_t count, int g0, int g1, const void* p1, void* m1,
                 void* v1, const void* gr1, void* grad0) {
    hs::AdamSeg& sg = a.seg[s];
    const void* params[7] = {scene->mu, scene->log_scale, scene->rotation, scene->sh_coeffs,
                             scene->normal, scene->raw_opacity_a, scene->raw_opacity_b};
    sg.kind = kind;
    sg.K = K;
    sg.param[0] = const_cast<void*>(params[field]);
    sg.m[0] = state->m[field];
    sg.v[0] = state->v[field];
    sg.grad[0] = grad0;
    sg.param[1] = const_cast<void*>(p1);
    sg.m[1] = m1;
    sg.v[1] = v1;
    sg.grad[1] = gr1;
    const int gs[2] = {g0, g1};
    for (int j = 0; j < 2; ++j) {
      if (gs[j] < 0) continue;
      sg.lr[j] = lr[gs[j]];
      sg.bc1[j] = bc1[gs[j]];
      sg.bc2[j] = bc2[gs[j]];
      sg.active[j] = on[gs[j]];
    }
    // elementwise segments move in 16-B vectors when every array allows it
    const int esz = scene->dtype == HS_DTYPE_F64 ? 8 : 4, per = 16 / esz;
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    sg.vec = (kind == hs::kAdamPlain || kind == hs::kAdamSh) && count % per == 0 &&
             al(sg.param[0]) && al(sg.m[0]) && al(sg.v[0]) && al(sg.grad[0]);
    if (sg.vec) count /= per;
    sg.units = count;
    ++s;
  };
  if (on[HS_GROUP_MU]) add(hs::kAdamPlain, 0, 3 * n, HS_GROUP_MU, -1, nullptr, nullptr, nullptr, nullptr, grads->d_mu);
  if (on[HS_GROUP_LOG_SCALE])
    add(hs::kAdamPlain, 1, 3 * n, HS_GROUP_LOG_SCALE, -1, nullptr, nullptr, nullptr, nullptr,
        grads->d_log_scale);
  if (on[HS_GROUP_ROTATION])
    add(hs::kAdamPlain, 2, 4 * n, HS_GROUP_ROTATION, -1, nullptr, nullptr, nullptr, nullptr,
        grads->d_rotation);
  if (on[HS_GROUP_SH_DC] || on[HS_GROUP_SH_REST])
    add(hs::kAdamSh, 3, 3 * (int64_t)K * n, HS_GROUP_SH_DC, HS_GROUP_SH_REST, nullptr, nullptr,
        nullptr, nullptr, grads->d_sh);
  if (on[HS_GROUP_NORMAL])
    add(hs::kAdamNormal, 4, n, HS_GROUP_NORMAL, -1, nullptr, nullptr, nullptr, nullptr,
        grads->d_normal);
  if (on[HS_GROUP_OPACITY_A] || on[HS_GROUP_OPACITY_B] || tie_opacities)
    add(hs::kAdamOpacity, 5, n, HS_GROUP_OPACITY_A, HS_GROUP_OPACITY_B, scene->raw_opacity_b,
        state->m[6], state->v[6], grads->d_raw_opacity_b, grads->d_raw_opacity_a);
  a.nseg = s;
  a.tie_opacities = tie_opacities != 0;
  HS_CUDA(hs::launch_adam(a, scene->dtype == HS_DTYPE_F64 ? 1 : 0,
                          static_cast<cudaStream_t>(stream_)));
  for (int g = 0; g < HS_ADAM_GROUPS; ++g)
    if (on[g]) state->t[g] += 1;
  return HS_OK;
}

// ---- density control (trainer.py:229-350) --------------------------------------
namespace {
hs::DensifyStatsArgs stats_args(const hs_densify_stats* s) {
  return {s->grad_sum, s->mu_grad_sum, s->count};
}
hs::DensifyBufs carve_densify(void* ws, int64_t n, size_t* bytes) {
  Carver c(ws);
  hs::DensifyBufs b;
  b.flags = c.take<uint8_t>(n + 1);
  b.f_surv = c.take<int32_t>(n + 1);
  b.f_clone = c.take<int32_t>(n + 1);
  b.f_split = c.take<int32_t>(n + 1);
  b.surv_rank = c.take<int32_t>(n + 1);
  b.clone_rank = c.take<int32_t>(n + 1);
  b.split_rank = c.take<int32_t>(n + 1);
  b.temp_bytes = hs::densify_scan_temp_bytes(n);
  b.temp = c.take<char>(b.temp_bytes);
  *bytes = c.off;
  return b;
}
}  // namespace

extern "C" int hs_densify_stats_update(const hs_densify_stats* stats, const hs_grads* grads,
                                       int64_t n, int32_t dtype, void* stream_) {
  if (!stats || !grads || n < 0) return HS_ERR_INVALID_ARG;
  if (n == 0) return HS_OK;
  HS_CUDA(hs::launch_densify_stats(stats_args(stats), grads->pos_grad_norm, grads->d_mu,
                                   grads->touch_count, n, dtype == HS_DTYPE_F64 ? 1 : 0,
                                   static_cast<cudaStream_t>(stream_)));
  return HS_OK;
}

extern "C" size_t hs_densify_workspace_size(int64_t n) {
  if (n < 0 || n >= ((int64_t)1 << 31) - 1) return 0;
  size_t bytes = 0;
  carve_densify(nullptr, n, &bytes);
  return bytes;
}

extern "C" int hs_densify_plan_compute(const hs_scene* scene, const hs_densify_stats* stats,
                                       const hs_densify_config* cfg, hs_densify_plan* plan,
                                       void* ws, size_t ws_bytes, void* stream_) {
  if (!scene || !stats || !cfg || !plan) return HS_ERR_INVALID_ARG;
  const int64_t n = scene->n;
  if (n < 0 || n >= ((int64_t)1 << 31) - 1) return HS_ERR_INVALID_ARG;
  size_t need = 0;
  carve_densify(nullptr, n, &need);
  if (!ws || ws_bytes < need) return HS_ERR_WORKSPACE;
  hs::DensifyBufs b = carve_densify(ws, n, &need);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  memset(plan, 0, sizeof(*plan));
  plan->n_in = n;
  if (n == 0) return HS_OK;
  const hs::DensifyParams p{cfg->densify_grad_threshold, cfg->prune_opacity_threshold,
                            cfg->percent_dense, cfg->prune_extent_factor, cfg->scene_extent};
  HS_CUDA(hs::launch_densify_classify(stats_args(stats), scene->log_scale, scene->raw_opacity_a,
                                      scene->raw_opacity_b, n,
                                      scene->dtype == HS_DTYPE_F64 ? 1 : 0, p, b, stream));
  int32_t tot[3];
  HS_CUDA(cudaMemcpyAsync(&tot[0], b.surv_rank + n, 4, cudaMemcpyDeviceToHost, stream));
  HS_CUDA(cudaMemcpyAsync(&tot[1], b.clone_rank + n, 4, cudaMemcpyDeviceToHost, stream));
  HS_CUDA(cudaMemcpyAsync(&tot[2], b.split_rank + n, 4, cudaMemcpyDeviceToHost, stream));
  HS_CUDA(cudaStreamSynchronize(stream));
  const int64_t surv0 = tot[0], nc = tot[1], ns = tot[2];
  // the reference's budget loops (trainer.py:268-288): clones first, then splits,
  // each in index order; over-budget split parents are kept unsplit
  int64_t acc_c = nc, acc_s = ns;
  if (cfg->max_primitives > 0) {
    const int64_t base = surv0 + ns;
    int64_t budget = cfg->max_primitives - base;
    if (budget < 0) budget = 0;
    acc_c = nc < budget ? nc : budget;
    budget -= acc_c;
    acc_s = ns < budget ? ns : budget;
  }
  plan->kept = surv0 + (ns - acc_s);
  plan->cloned = acc_c;
  plan->split = acc_s;
  plan->pruned = n - surv0 - ns;
  plan->n_out = plan->kept + acc_c + 2 * acc_s;
  return HS_OK;
}

namespace {
template <typename T>
int densify_apply_t(const hs_scene* scene, const hs_densify_stats* stats,
                    const hs_densify_config* cfg, const hs_densify_plan* plan,
                    const hs::DensifyBufs& b, const double* offsets, uint64_t seed,
                    const hs_adam_state* sin, hs_scene* out, hs_adam_state* sout,
                    cudaStream_t stream) {
  hs::DensifyEmitArgs<T> a;
  memset(&a, 0, sizeof(a));
  a.n = scene->n;
  a.K = (scene->sh_degree + 1) * (scene->sh_degree + 1);
  a.flags = b.flags;
  a.surv_rank = b.surv_rank;
  a.clone_rank = b.clone_rank;
  a.split_rank = b.split_rank;
  a.acc_clone = plan->cloned;
  a.acc_split = plan->split;
  a.n_surv = plan->kept;
  a.mu_grad_sum = stats->mu_grad_sum;
  a.offsets = offsets;
  a.seed = seed;
  a.log_split_scale = cfg->log_split_scale;
  a.in = {(const T*)scene->mu, (const T*)scene->log_scale, (const T*)scene->rotation,
          (const T*)scene->sh_coeffs, (const T*)scene->normal, (const T*)scene->raw_opacity_a,
          (const T*)scene->raw_opacity_b};
  a.out = {(T*)out->mu, (T*)out->log_scale, (T*)out->rotation, (T*)out->sh_coeffs,
           (T*)out->normal, (T*)out->raw_opacity_a, (T*)out->raw_opacity_b};
  for (int f = 0; f < 7; ++f) {
    const bool have = sin && sout && sin->m[f] && sin->v[f] && sout->m[f] && sout->v[f];
    a.m_in[f] = have ? sin->m[f] : nullptr;
    a.v_in[f] = have ? sin->v[f] : nullptr;
    a.m_out[f] = have ? sout->m[f] : nullptr;
    a.v_out[f] = have ? sout->v[f] : nullptr;
  }
  HS_CUDA(hs::launch_densify_emit_t<T>(a, stream));
  return HS_OK;
}
}  // namespace

extern "C" int hs_densify_apply(const hs_scene* scene, const hs_densify_stats* stats,
                                const hs_densify_config* cfg, const hs_densify_plan* plan,
                                const void* ws, size_t ws_bytes, const double* split_offsets,
                                uint64_t seed, const hs_adam_state* state_in, hs_scene* out,
                                hs_adam_state* state_out, void* stream_) {
  if (!scene || !stats || !cfg || !plan || !out) return HS_ERR_INVALID_ARG;
  if (plan->n_in != scene->n || out->n != plan->n_out || out->dtype != scene->dtype ||
      out->sh_degree != scene->sh_degree)
    return HS_ERR_INVALID_ARG;
  size_t need = 0;
  carve_densify(nullptr, scene->n, &need);
  if (!ws || ws_bytes < need) return HS_ERR_WORKSPACE;
  const hs::DensifyBufs b = carve_densify(const_cast<void*>(ws), scene->n, &need);
  if (state_in && state_out)
    for (int g = 0; g < HS_ADAM_GROUPS; ++g) state_out->t[g] = state_in->t[g];
  if (scene->n == 0 || plan->n_out == 0) return HS_OK;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (scene->dtype == HS_DTYPE_F64)
    return densify_apply_t<double>(scene, stats, cfg, plan, b, split_offsets, seed, state_in, out,
                                   state_out, stream);
  return densify_apply_t<float>(scene, stats, cfg, plan, b, split_offsets, seed, state_in, out,
                                state_out, stream);
}

extern "C" int hs_reset_opacity(const hs_scene* scene, double cap, hs_adam_state* state,
                                void* stream_) {
  if (!scene) return HS_ERR_INVALID_ARG;
  if (scene->n == 0) return HS_OK;
  HS_CUDA(hs::launch_reset_opacity(const_cast<void*>(scene->raw_opacity_a),
                                   const_cast<void*>(scene->raw_opacity_b),
                                   state ? state->m[5] : nullptr, state ? state->v[5] : nullptr,
                                   state ? state->m[6] : nullptr, state ? state->v[6] : nullptr,
                                   scene->n, cap, scene->dtype == HS_DTYPE_F64 ? 1 : 0,
                                   static_cast<cudaStream_t>(stream_)));
  if (state) state->t[HS_GROUP_OPACITY_A] = state->t[HS_GROUP_OPACITY_B] = 0;
  return HS_OK;
}

// ---- scene I/O (scene_io.py:136-269) -------------------------------------------
static_assert(HS_PLY_MAX_PROPS == hs::kPlyMaxProps, "PLY property table size");
static_assert(66 >= hs::kPlyMaxComps, "PLY component table size");

extern "C" int hs_ply_unpack(const void* payload, const hs_ply_layout* layout, hs_scene* out,
                             void* stream_) {
  if (!payload || !layout || !out) return HS_ERR_INVALID_ARG;
  if (layout->n != out->n || layout->sh_degree != out->sh_degree || layout->stride <= 0 ||
      layout->n_props <= 0 || layout->n_props > HS_PLY_MAX_PROPS)
    return HS_ERR_INVALID_ARG;
  if (out->sh_degree < 0 || out->sh_degree > 3) return HS_ERR_INVALID_ARG;
  if (layout->n == 0) return HS_OK;
  hs::PlyUnpackArgs a;
  memset(&a, 0, sizeof(a));
  a.payload = payload;
  a.n = layout->n;
  a.stride = layout->stride;
  a.K = (out->sh_degree + 1) * (out->sh_degree + 1);
  for (int p = 0; p < layout->n_props; ++p) {
    if (layout->offset[p] < 0 || layout->type[p] < 0 || layout->type[p] > HS_PLY_INT)
      return HS_ERR_INVALID_ARG;
    a.offset[p] = layout->offset[p];
    a.type[p] = layout->type[p];
  }
  const int ncomp = 3 + 3 + 4 + 3 * a.K + 3 + 1 + 1;
  for (int c = 0; c < ncomp; ++c) {
    if (layout->column[c] >= layout->n_props) return HS_ERR_INVALID_ARG;
    a.column[c] = layout->column[c];
  }
  const void* fields[7] = {out->mu, out->log_scale, out->rotation, out->sh_coeffs, out->normal,
                           out->raw_opacity_a, out->raw_opacity_b};
  HS_CUDA(hs::launch_ply_unpack(a, fields, out->dtype == HS_DTYPE_F64 ? 1 : 0,
                                static_cast<cudaStream_t>(stream_)));
  return HS_OK;
}

extern "C" int32_t hs_ply_row_bytes(int32_t sh_degree, int32_t kind) {
  if (sh_degree < 0 || sh_degree > 3 || kind < HS_PLY_NATIVE || kind > HS_PLY_3DGS_FIRST)
    return 0;
  const int K = (sh_degree + 1) * (sh_degree + 1);
  const int ncol = 9 + 3 * (K - 1) + (kind == HS_PLY_NATIVE ? 2 : 1) + 7;
  return ncol * (kind == HS_PLY_NATIVE ? 8 : 4);
}

extern "C" int hs_ply_pack(const hs_scene* scene, void* payload, int32_t kind, void* stream_) {
  if (!scene || !payload) return HS_ERR_INVALID_ARG;
  if (hs_ply_row_bytes(scene->sh_degree, kind) == 0) return HS_ERR_INVALID_ARG;
  if (scene->n == 0) return HS_OK;
  hs::PlyPackArgs a;
  a.payload = payload;
  a.n = scene->n;
  a.K = (scene->sh_degree + 1) * (scene->sh_degree + 1);
  a.gs3d = kind != HS_PLY_NATIVE;
  a.opacity_first = kind == HS_PLY_3DGS_FIRST;
  a.out_f64 = kind == HS_PLY_NATIVE;
  const void* fields[7] = {scene->mu, scene->log_scale, scene->rotation, scene->sh_coeffs,
                           scene->normal, scene->raw_opacity_a, scene->raw_opacity_b};
  HS_CUDA(hs::launch_ply_pack(a, fields, scene->dtype == HS_DTYPE_F64 ? 1 : 0,
                              static_cast<cudaStream_t>(stream_)));
  return HS_OK;
}

extern "C" size_t hs_opacity_disparity_workspace_size(int64_t n) {
  if (n <= 0 || n >= ((int64_t)1 << 31)) return 0;
  size_t bytes = 0;
  hs::opacity_disparity_sum(nullptr, nullptr, n, 0, nullptr, nullptr, &bytes, 0);
  size_t b64 = 0;
  hs::opacity_disparity_sum(nullptr, nullptr, n, 1, nullptr, nullptr, &b64, 0);
  return bytes > b64 ? bytes : b64;
}

extern "C" int hs_opacity_disparity(const hs_scene* scene, double* out_sum, void* ws,
                                    size_t ws_bytes, void* stream_) {
  if (!scene || !out_sum) return HS_ERR_INVALID_ARG;
  if (scene->n <= 0) return HS_ERR_EMPTY_SCENE;
  if (scene->n >= ((int64_t)1 << 31)) return HS_ERR_INVALID_ARG;
  if (!ws || ws_bytes < hs_opacity_disparity_workspace_size(scene->n)) return HS_ERR_WORKSPACE;
  size_t bytes = ws_bytes;
  HS_CUDA(hs::opacity_disparity_sum(scene->raw_opacity_a, scene->raw_opacity_b, scene->n,
                                    scene->dtype == HS_DTYPE_F64 ? 1 : 0, out_sum, ws, &bytes,
                                    static_cast<cudaStream_t>(stream_)));
  return HS_OK;
}
