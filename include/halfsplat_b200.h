/*
 * halfsplat_b200.h -- C ABI of the B200-native half-Gaussian rasterizer.
 *
 * This is the drop-in boundary for the reference's hot path
 * (halfsplat.rasterizer.prepare -> render -> render_backward and its blend-core
 * plugin).  Every entry point is extern "C", takes plain pointers and sizes,
 * returns an int status (HS_OK or one of the HS_ERR_* codes that mirror the
 * reference's exceptions) and never throws.  Citations are into the reference
 * tree (/root/reference/pkg/src/halfsplat/...).
 *
 * Two seams are exported:
 *
 *  Seam 1 -- blend-core plugin (host pointers, float64, reference layout).
 *    hs_forward_tiles / hs_backward_tiles replace the Cython module's
 *    forward_tiles / backward_tiles (_blend_cy.pyx:74-83, 190-199; the contract
 *    is documented in _blend_py.py:1-19).  The backend seam that selects them
 *    is backend.py:26-48.  Arrays are the caller's; only pixels and pair rows of
 *    tiles in [tile_lo, tile_hi) are written (pair rows are accumulated, +=).
 *
 *  Seam 2 -- staged device pipeline (device pointers, one cudaStream_t).
 *    hs_preprocess_fwd      <- rasterizer.prepare projection/cull/SH part
 *                              (rasterizer.py:159-298)
 *    hs_bin_and_sort        <- pair expansion + np.lexsort + searchsorted
 *                              (rasterizer.py:300-325)
 *    hs_blend_fwd           <- render's forward_tiles calls (rasterizer.py:351-383)
 *    hs_blend_bwd           <- render_backward's backward_tiles calls
 *                              (rasterizer.py:386-418)
 *    hs_preprocess_bwd      <- np.add.at merge + _geometry_backward
 *                              (rasterizer.py:419-575)
 *    Workspaces are caller-allocated from the *_workspace_size queries; the
 *    library never allocates on this seam.  Calls on distinct frames/streams are
 *    independent (re-entrant).
 *
 *  Training-iteration entry points around the path, same
 *  conventions (device pointers, caller stream, caller workspaces):
 *    hs_loss                 <- loss.compute_loss / ssim_with_grad (loss.py:48-106)
 *    hs_adam_step            <- the Adam block of trainer.step (trainer.py:192-224)
 *    hs_densify_*            <- DensifyStats / densify_and_prune (trainer.py:229-340)
 *    hs_reset_opacity, hs_opacity_disparity (trainer.py:343-358)
 *    hs_ply_pack / unpack    <- scene_io save/load/import/export payloads
 *                               (scene_io.py:136-269)
 *  hs_grads.accumulate = 3 lets K7 reduce its gradients straight into an NVLS
 *  multicast buffer: the multi-GPU all-reduce fused into the kernel.
 */
#ifndef HALFSPLAT_B200_H
#define HALFSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror errors.py) ---------------------------------- */
#define HS_OK 0
#define HS_ERR_EMPTY_SCENE 1        /* errors.EmptyScene      (rasterizer.py:161-162) */
#define HS_ERR_IMAGE_TOO_LARGE 2    /* errors.ImageTooLarge   (rasterizer.py:163-164) */
#define HS_ERR_INVALID_KERNEL 3     /* ValueError on kernel   (rasterizer.py:165-166) */
#define HS_ERR_MISMATCHED_FORWARD 4 /* errors.MismatchedForward (rasterizer.py:390-398) */
#define HS_ERR_INVALID_ARG 5
#define HS_ERR_CUDA 6
#define HS_ERR_WORKSPACE 7          /* workspace missing or too small */
#define HS_ERR_IMAGE_TOO_SMALL 8    /* errors.ImageTooSmall   (loss.py:52-53) */
#define HS_ERR_INVALID_LAMBDA 9     /* ValueError on lambda_ssim (loss.py:91-92) */

#define HS_DTYPE_F32 0
#define HS_DTYPE_F64 1

#define HS_KERNEL_HALF 0
#define HS_KERNEL_FULL 1

#define HS_TILE 16
#define HS_PAIR_GRAD_COLS 12

/* Pinhole camera, geometry.py:210-273 (world_to_cam row-major 4x4). */
typedef struct hs_camera {
  double world_to_cam[16];
  double fx, fy, cx, cy;
  double near_clip;
  double center[3]; /* camera centre in world coords, -R^T t (geometry.py:266-269) */
  int32_t width, height;
} hs_camera;

/* Struct-of-arrays scene, geometry.py:364-383.  Device pointers, all of one
 * dtype (HS_DTYPE_F32 or HS_DTYPE_F64), C-contiguous:
 *   mu (n,3)  log_scale (n,3)  rotation (n,4) wxyz unnormalised
 *   sh_coeffs (n,(deg+1)^2,3)  normal (n,3)  raw_opacity_a/b (n,)          */
typedef struct hs_scene {
  int64_t n;
  int32_t sh_degree;
  int32_t dtype;
  const void* mu;
  const void* log_scale;
  const void* rotation;
  const void* sh_coeffs;
  const void* normal;
  const void* raw_opacity_a;
  const void* raw_opacity_b;
  double background[3];
} hs_scene;

/* Per-view frame state.  Filled by hs_frame_init / hs_preprocess_fwd /
 * hs_bin_and_sort; the caller owns the two workspaces it points into. */
typedef struct hs_frame {
  int64_t n;            /* primitives in the scene */
  int32_t width, height;
  int32_t tiles_x, tiles_y, n_tiles;
  int32_t kernel;       /* HS_KERNEL_HALF / HS_KERNEL_FULL */
  int32_t tile_bits;    /* significant bits of the pair sort key */
  int32_t sort_selector;/* internal: which pair double-buffer holds the result */
  int64_t num_pairs;    /* P once read (hs_frame_read_num_pairs / hs_frame_status),
                           else -1 */
  void* frame_ws;       /* size hs_frame_workspace_size(n, width, height) */
  size_t frame_ws_bytes;
  void* bin_ws;         /* size hs_binning_workspace_size(n, pair_capacity, ...) */
  size_t bin_ws_bytes;
  int64_t pair_capacity;/* pairs bin_ws is laid out for (0: num_pairs) */
  int32_t depth_sort_full;/* in: 1 ranks depths with the full 64-bit sort (no
                           run fixup, so no depth fallback can be pending); out:
                           hs_frame_read_num_pairs sets it when it had to */
} hs_frame;

/* ---- Seam 2: staged device pipeline ----------------------------------- */

/* Validates sizes (EmptyScene / ImageTooLarge / kernel) and fills the static
 * fields of *frame.  Workspace pointers are left for the caller to set. */
int hs_frame_init(hs_frame* frame, int64_t n, int32_t width, int32_t height,
                  int32_t kernel);
size_t hs_frame_workspace_size(int64_t n, int32_t width, int32_t height);
size_t hs_binning_workspace_size(int64_t n, int64_t num_pairs, int32_t width,
                                 int32_t height);

/* K1 preprocess (one thread per Gaussian, FP64 geometry) + depth-rank sort +
 * per-splat tile counts and their scan.  radii (n,) int32 is optional
 * (ceil of the 3.5-sigma radius, 0 when culled). */
int hs_preprocess_fwd(hs_frame* frame, const hs_scene* scene,
                      const hs_camera* cam, int32_t* radii, void* stream);

/* hs_preprocess_fwd for a batch of views of one scene (rasterizer.py:159-298 per
 * camera): frames[v] (each with its own workspaces) gets view cams[v].  One K1
 * pass stages each Gaussian once and computes its camera-independent state
 * (rotation, covariance, normal, opacities) once for all the views; every output
 * is bit-identical to hs_preprocess_fwd's.  radii may be NULL, or hold NULL
 * entries.  rank = 1: each frame's depth ranks and pair counts follow on
 * `stream`; rank = 0: the caller runs hs_frame_rank per frame (after this call's
 * work, e.g. on one stream per view) before binning it. */
int hs_preprocess_fwd_views(hs_frame* const* frames, int32_t n_views, const hs_scene* scene,
                            const hs_camera* cams, int32_t* const* radii, int32_t rank,
                            void* stream);
int hs_frame_rank(hs_frame* frame, void* stream);

/* Synchronises `stream` and reads P (the number of (tile, splat) pairs).  The
 * depth ranks of hs_preprocess_fwd come from a 32-bit sort plus a per-run fixup;
 * when a depth bucket was too long for the fixup this call redoes them with the
 * full 64-bit sort before returning, so it must precede every use of the ranks. */
int hs_frame_read_num_pairs(hs_frame* frame, void* stream);

/* K2 duplicate-with-keys, K3 stable tile sort, K4 tile ranges, once P is known.
 * Needs frame->bin_ws of hs_binning_workspace_size(n, max(P, pair_capacity), ...)
 * bytes. */
int hs_bin_and_sort(hs_frame* frame, void* stream);

/* The same binning with no host round trip: P stays on the device and the
 * workspace is laid out for frame->pair_capacity pairs (set by the caller, e.g.
 * from an earlier view's P with headroom).  K2 writes each splat's pairs as
 * segments (one per tile row and block of 32 tile columns) straight into
 * per-(row, block) buckets in depth-rank order, and a warp per bucket chunk
 * appends them to the tile lists (a stable counting sort by tile); tile_starts
 * come out of the same scans.  If P exceeds the capacity nothing is binned
 * (every tile list is empty, so the blends and K7 do no work) and the status
 * says so: check it with hs_frame_status at the caller's next sync point and
 * re-bin with a larger workspace.  Images wider than 2048 tiles, taller than
 * 1024 tiles, or with more than 2048 (tile row, 32-column block) pairs (beyond
 * 4K UHD) take the synchronous path inside this call. */
int hs_bin_async(hs_frame* frame, void* stream);

/* Binning status flags (hs_frame_status) */
#define HS_FRAME_PAIR_OVERFLOW 1 /* P > pair_capacity: re-bin (hs_bin_and_sort) */
#define HS_FRAME_DEPTH_FALLBACK 2 /* a depth run was too long for the fixup:
                                    hs_frame_read_num_pairs redoes the ranks */
/* Synchronises `stream` and reads P (int64: more pairs than int32 offsets hold
 * is reported, not wrapped) and the flags; with no flag set, frame->num_pairs
 * becomes P. */
int hs_frame_status(hs_frame* frame, int64_t* num_pairs, int32_t* flags, void* stream);
/* The same status without waiting: enqueues on `stream` a copy of it into
 * host_status (24 bytes of host memory, pinned for an asynchronous copy):
 * int64 P at byte 0, int64 segment count at byte 8, int32 binning flags at
 * byte 16 (bit 0: HS_FRAME_PAIR_OVERFLOW), int32 depth-fallback flag at byte 24
 * (non-zero: HS_FRAME_DEPTH_FALLBACK); 32 bytes.
 * Valid once the stream has passed this point (e.g. an event recorded after it). */
int hs_frame_status_async(const hs_frame* frame, void* host_status, void* stream);

/* hs_frame_read_num_pairs followed by hs_bin_and_sort in one call, so the GPU
 * is not left idle while the caller sizes the binning workspace: with a
 * frame->bin_ws already large enough (e.g. the previous view's) it bins right
 * after the sync; otherwise it returns HS_ERR_WORKSPACE with num_pairs set, and
 * the caller sizes the workspace and calls hs_bin_and_sort. */
int hs_read_pairs_and_bin(hs_frame* frame, void* stream);

/* K5 forward blend.  Outputs (device, float32 / int32):
 * color (H,W,3), alpha (H,W), depth (H,W), transmittance (H,W), terminal (H,W). */
int hs_blend_fwd(hs_frame* frame, const double* background, float* color,
                 float* alpha, float* depth, float* transmittance,
                 int32_t* terminal, void* stream);

/* K6 backward blend for cotangent d_color (H,W,3) float32; consumes the
 * forward's transmittance and terminal. Writes per-pair partial rows. */
int hs_blend_bwd(hs_frame* frame, const double* background,
                 const float* d_color, const float* transmittance,
                 const int32_t* terminal, void* stream);

/* Diagnostic: histogram over every (tile, pair) of the blend's strip window
 * codes (0 none, 1 rows 0-7, 2 rows 8-15, 3 all; hs_blend.cu strip_window).
 * hist: device array of 4 uint64. */
int hs_blend_window_stats(hs_frame* frame, unsigned long long* hist, void* stream);

/* K7: merge pair rows per splat and chain to the primitive parameters
 * (GradientSet, rasterizer.py:72-105).  Output pointers are device arrays of
 * the scene dtype (touch_count int32); culled primitives get zeros. */
typedef struct hs_grads {
  void* d_mu;           /* (n,3) */
  void* d_log_scale;    /* (n,3) */
  void* d_rotation;     /* (n,4) w.r.t. the raw quaternion */
  void* d_sh;           /* (n,K,3) */
  void* d_normal;       /* (n,3) w.r.t. the raw normal */
  void* d_raw_opacity_a;/* (n,) */
  void* d_raw_opacity_b;/* (n,) */
  void* pos_grad_norm;  /* (n,) */
  int32_t* touch_count; /* (n,) */
  int32_t accumulate;   /* 0: overwrite; 1: add into the buffers (multi-view
                           batches, GradientSet.add rasterizer.py:100-105);
                           2: add with device atomics (red.global.add);
                           3: the pointers are NVLS multicast addresses of a
                           buffer every rank of a node maps (e.g. torch
                           symmetric memory): K7 adds with multimem.red, so
                           the switch sums all ranks' gradients into every
                           rank's copy -- the all-reduce fused into K7.  With
                           2 / 3 the caller zeroes the buffers first and, for
                           3, brackets the batch with a cross-rank barrier. */
} hs_grads;

int hs_preprocess_bwd(hs_frame* frame, const hs_scene* scene,
                      const hs_camera* cam, const hs_grads* grads, void* stream);

/* hs_preprocess_bwd restricted to primitives [begin, end) (begin a multiple of
 * 128; end clamped to n): K7 in buckets, so a bucket's gradients can be
 * all-reduced while the next bucket computes. */
int hs_preprocess_bwd_range(hs_frame* frame, const hs_scene* scene, const hs_camera* cam,
                            const hs_grads* grads, int64_t begin, int64_t end, void* stream);

/* Multi-view geometry backward (a batch of views of one scene, the reference's
 * per-view K7 loop of train.py / GradientSet.add, rasterizer.py:100-105, fused):
 *   hs_merge_rows      -- after hs_blend_bwd of a view: that view's per-primitive
 *                         merged blend gradients into merged_out ((n,16) float32,
 *                         16-B aligned; culled primitives marked), so the frame's
 *                         workspace can be reused by the next view;
 *   hs_preprocess_bwd_views -- one pass over the scene for all the views: each
 *                         primitive's parameters are read once, the gradients of
 *                         every view it is visible in are summed on chip (in view
 *                         order) and stored once.  grads->accumulate as for
 *                         hs_preprocess_bwd; begin a multiple of 128. */
int hs_merge_rows(hs_frame* frame, float* merged_out, void* stream);
int hs_preprocess_bwd_views(const hs_scene* scene, int32_t n_views, const hs_camera* cams,
                            const float* const* merged, int32_t kernel, const hs_grads* grads,
                            int64_t begin, int64_t end, void* stream);

/* Introspection for parity: the reference's FrameGeometry integers and packed
 * columns (rasterizer.py:108-147).  Device outputs:
 *   valid (n,) int32 -- original indices of surviving primitives, first M used
 *   m_out (1,) int64 -- M
 *   packed (n,13) float32, mode (n,) int8, tile_rect (n,4) int32 in valid order
 *   pair_splat (P,) int32 splat-local, tile_starts (n_tiles+1,) int64        */
int hs_frame_export(const hs_frame* frame, int32_t* valid, int64_t* m_out,
                    float* packed, int8_t* mode, int32_t* tile_rect,
                    int32_t* pair_splat, int64_t* tile_starts, void* stream);

/* ScreenSplat export (rasterizer.py:578-603): for every primitive 20 doubles
 * (zeros when culled): mu_hat x,y; conic a,b,c; whiten2d v00,v10,v11;
 * n_ray x,y,z; alpha1, alpha2; rgb (3); depth; radius; za, zb.  `out` is a
 * device array of n*20 doubles. */
int hs_screen_splats(const hs_scene* scene, const hs_camera* cam, int32_t kernel, double* out,
                     void* stream);

/* ---- Seam 1: blend-core plugin (host float64 arrays) ------------------- */
int hs_forward_tiles(const double* packed, const int8_t* mode,
                     const int32_t* pair_splat, const int64_t* tile_starts,
                     int64_t num_splats, int64_t num_pairs, int32_t height,
                     int32_t width, int32_t tiles_x, const double* background,
                     double* color, double* alpha, double* depth,
                     double* transmittance, int32_t* terminal, int32_t tile_lo,
                     int32_t tile_hi);

int hs_backward_tiles(const double* packed, const int8_t* mode,
                      const int32_t* pair_splat, const int64_t* tile_starts,
                      int64_t num_splats, int64_t num_pairs, int32_t height,
                      int32_t width, int32_t tiles_x, const double* background,
                      const double* d_color, const double* transmittance,
                      const int32_t* terminal, double* pair_grads,
                      int32_t tile_lo, int32_t tile_hi);

/* Seam 1 keeps the last frame's full GPU result (and a host copy of its inputs)
 * so the reference's concurrent chunk calls on one frame blend it once; a call
 * whose inputs differ (exact byte compare) recomputes.  This releases it. */
void hs_seam1_cache_clear(void);

/* ---- training loss: the cotangent producer between K5 and K6 ---------- */

/* Device workspace for hs_loss on an (height, width, channels) image. */
size_t hs_loss_workspace_size(int32_t height, int32_t width, int32_t channels);

/* compute_loss (loss.py:88-106): (1 - lambda) L1 + lambda (1 - SSIM) of
 * `rendered` against `target`, both device float32 (H,W,C) C-contiguous, and
 * its exact gradient w.r.t. `rendered` (ssim_with_grad, loss.py:48-79).
 * loss4 (device, 4 doubles) receives [loss, L1, mean SSIM, MSE] (the MSE is
 * metrics.psnr's, metrics.py:13-22); the gradient goes
 * to d_rendered (float32, the cotangent hs_blend_bwd takes) and/or
 * d_rendered_f64 (float64); either may be NULL.  FP64 arithmetic.  lambda 0
 * skips SSIM as the reference does (and then accepts images under 11 px).
 * Errors: HS_ERR_INVALID_LAMBDA outside [0, 1]; HS_ERR_IMAGE_TOO_SMALL when
 * lambda > 0 and min(H, W) < 11; HS_ERR_WORKSPACE.  Asynchronous on `stream`. */
int hs_loss(const float* rendered, const float* target, int32_t height, int32_t width,
            int32_t channels, double lambda_ssim, double* loss4, float* d_rendered,
            double* d_rendered_f64, void* ws, size_t ws_bytes, void* stream);
/* hs_loss on float64 images (a reference caller's arrays, e.g. uint8/255
 * targets): same outputs, workspace and errors; the FP64 arithmetic then sees
 * the inputs unrounded, as loss.py does. */
int hs_loss_f64(const double* rendered, const double* target, int32_t height, int32_t width,
                int32_t channels, double lambda_ssim, double* loss4, float* d_rendered,
                double* d_rendered_f64, void* ws, size_t ws_bytes, void* stream);

/* ---- optimizer: per-group Adam, the step after K7 ----------------------- */

/* Parameter groups in the reference's order (trainer.py:81-82). */
#define HS_ADAM_GROUPS 8
#define HS_GROUP_MU 0
#define HS_GROUP_LOG_SCALE 1
#define HS_GROUP_ROTATION 2
#define HS_GROUP_SH_DC 3
#define HS_GROUP_SH_REST 4
#define HS_GROUP_NORMAL 5
#define HS_GROUP_OPACITY_A 6
#define HS_GROUP_OPACITY_B 7

/* AdamState (trainer.py:110-136).  m / v: device arrays of the scene's dtype
 * and shapes, in scene-field order mu, log_scale, rotation, sh_coeffs (both SH
 * groups), normal, raw_opacity_a, raw_opacity_b.  t: per-group step counts,
 * advanced by hs_adam_step for every group it updates. */
typedef struct hs_adam_state {
  void* m[7];
  void* v[7];
  int64_t t[HS_ADAM_GROUPS];
} hs_adam_state;

/* The Adam part of trainer.step (trainer.py:192-224): for every group g with
 * lr[g] > 0 (the caller passes 0 for groups its mode freezes, active_groups
 * trainer.py:161-168), t[g] += 1 and
 *   m = b1 m + (1-b1) grad;  v = b2 v + (1-b2) grad^2;
 *   param -= lr m/(1-b1^t) / (sqrt(v/(1-b2^t)) + 1e-15)
 * with b1 0.9, b2 0.999; normals whose update is non-zero are renormalised;
 * tie_opacities (the 'full' kernel) then sets raw_opacity_b = raw_opacity_a.
 * The SCENE'S PARAMETER ARRAYS ARE UPDATED IN PLACE (the const in hs_scene is
 * the renderer's view).  grads: the hs_grads buffers of the same scene/dtype.
 * One kernel launch; a float64 scene steps bit-identically to the reference. */
int hs_adam_step(const hs_scene* scene, const hs_grads* grads, hs_adam_state* state,
                 const double lr[HS_ADAM_GROUPS], int32_t tie_opacities, void* stream);

/* ---- density control (trainer.py:229-350) ------------------------------- */

/* DensifyStats (trainer.py:229-244): device float64 / int64 accumulators. */
typedef struct hs_densify_stats {
  double* grad_sum;     /* (n,)   sum of pos_grad_norm */
  double* mu_grad_sum;  /* (n,3)  sum of d_mu */
  int64_t* count;       /* (n,)   sum of touch_count */
} hs_densify_stats;

/* TrainConfig's density fields (trainer.py:47-53) plus the scene extent. */
typedef struct hs_densify_config {
  double densify_grad_threshold;
  double prune_opacity_threshold;
  double percent_dense;
  double prune_extent_factor;
  double scene_extent;
  double log_split_scale;  /* log(split_scale_factor), as numpy computes it */
  int64_t max_primitives;  /* 0 = unlimited */
} hs_densify_config;

/* Filled by hs_densify_plan; read by hs_densify_apply. */
typedef struct hs_densify_plan {
  int64_t n_in, n_out;
  int64_t kept;    /* survivors, including over-budget split parents */
  int64_t cloned;  /* report["cloned"] */
  int64_t split;   /* report["split"] (parents; 2 children each) */
  int64_t pruned;  /* report["pruned"] */
} hs_densify_plan;

/* DensifyStats.update (trainer.py:241-244) from one step's gradients. */
int hs_densify_stats_update(const hs_densify_stats* stats, const hs_grads* grads, int64_t n,
                            int32_t dtype, void* stream);

size_t hs_densify_workspace_size(int64_t n);

/* First half of densify_and_prune (trainer.py:254-288): classify every
 * primitive, rank the candidates, apply the max_primitives budget.  Fills
 * `plan` (so the caller can allocate n_out rows); SYNCHRONISES `stream`.
 * The workspace carries the classification to hs_densify_apply. */
int hs_densify_plan_compute(const hs_scene* scene, const hs_densify_stats* stats,
                            const hs_densify_config* cfg, hs_densify_plan* plan, void* ws,
                            size_t ws_bytes, void* stream);

/* Second half (trainer.py:290-340): write the new scene into `out` (device
 * arrays of plan->n_out rows, same dtype/degree; the const in hs_scene is the
 * renderer's view, these ARE WRITTEN) and the re-aligned Adam moments into
 * state_out (survivor rows copied, new rows zero; NULL entries skipped).
 * split_offsets: device float64 (2, plan->split, 3) standard normals, the
 * reference's two rng.normal draws; NULL draws them on the device (Philox,
 * keyed by `seed`). */
int hs_densify_apply(const hs_scene* scene, const hs_densify_stats* stats,
                     const hs_densify_config* cfg, const hs_densify_plan* plan, const void* ws,
                     size_t ws_bytes, const double* split_offsets, uint64_t seed,
                     const hs_adam_state* state_in, hs_scene* out, hs_adam_state* state_out,
                     void* stream);

/* reset_opacity (trainer.py:343-350): raw opacities = min(raw, cap) with
 * cap = logit(ceiling); zeroes the opacity groups' moments and steps when
 * `state` is given.  Writes the scene's opacity arrays. */
int hs_reset_opacity(const hs_scene* scene, double cap, hs_adam_state* state, void* stream);

/* opacity_disparity (trainer.py:353-358): the SUM of |sigmoid(a) - sigmoid(b)|
 * over the scene into *out_sum (device double; divide by n for the mean).
 * Deterministic; EmptyScene for n == 0. */
size_t hs_opacity_disparity_workspace_size(int64_t n);
int hs_opacity_disparity(const hs_scene* scene, double* out_sum, void* ws, size_t ws_bytes,
                         void* stream);

/* ---- scene I/O: PLY payload <-> device scene (scene_io.py:136-269) ----- */

#define HS_PLY_FLOAT 0   /* property float / float32 */
#define HS_PLY_DOUBLE 1  /* property double / float64 */
#define HS_PLY_UCHAR 2   /* property uchar / uint8 */
#define HS_PLY_INT 3     /* property int / int32 */
#define HS_PLY_MAX_PROPS 128

#define HS_PLY_NATIVE 0       /* save_scene: double, x y z nx ny nz f_dc f_rest opacity opacity_2 scale rot */
#define HS_PLY_3DGS_MEAN 1    /* export_3dgs(opacity="mean"): float, zero normals, one opacity */
#define HS_PLY_3DGS_FIRST 2   /* export_3dgs(opacity="first") */

/* The vertex payload of a parsed PLY header: `n` rows of `stride` bytes.
 * offset/type: byte offset and HS_PLY_* type of each property.  column: for each
 * scene component in field order (mu 3, log_scale 3, rotation 4, sh 3K as
 * (coefficient, channel), normal 3, raw_opacity_a, raw_opacity_b) the source
 * property index, or -1 to leave that component untouched. */
typedef struct hs_ply_layout {
  int64_t n;
  int32_t stride;
  int32_t n_props;
  int32_t sh_degree;
  int16_t offset[HS_PLY_MAX_PROPS];
  int8_t type[HS_PLY_MAX_PROPS];
  int16_t column[66];
} hs_ply_layout;

/* load_scene / import_3dgs payload step: de-interleave the device payload into
 * the scene's device arrays (`out`, n rows, written), converting types and
 * transposing f_rest from channel-major.  One launch. */
int hs_ply_unpack(const void* payload, const hs_ply_layout* layout, hs_scene* out,
                  void* stream);

/* Bytes per payload row of hs_ply_pack's output for a layout kind. */
int32_t hs_ply_row_bytes(int32_t sh_degree, int32_t kind);

/* save_scene / export_3dgs payload step: interleave the scene into `payload`
 * (device, n * hs_ply_row_bytes bytes) in the reference's property order.
 * HS_PLY_3DGS_MEAN writes logit(clip((a1 + a2) / 2, 1e-6, 1 - 1e-6)). */
int hs_ply_pack(const hs_scene* scene, void* payload, int32_t kind, void* stream);

/* ---- multi-GPU: the gradient exchange ------------------
 * View-sharded training: every rank renders its views against a replica of
 * the Gaussians and accumulates their gradients (hs_grads.accumulate = 1);
 * the batch gradient is the sum over ranks (GradientSet.add,
 * rasterizer.py:100-105).  A communicator is an NCCL communicator (NCCL is
 * loaded at run time; these return HS_ERR_CUDA without it).  Rank 0 calls
 * hs_comm_unique_id, the host hands the HS_COMM_ID_BYTES bytes to every rank
 * (any channel), and every rank calls hs_comm_init on its own device. */
#define HS_COMM_ID_BYTES 128
int hs_comm_unique_id(void* id);
int hs_comm_init(void** comm, int32_t world, int32_t rank, const void* id);
int hs_comm_destroy(void* comm);
/* Ranks in / this rank of `comm`, and the NCCL version loaded (comm may be
 * NULL for the version only). */
int hs_comm_info(void* comm, int32_t* world, int32_t* rank, int32_t* nccl_version);
/* Sums primitive rows [begin, end) of every gradient field of `grads` (n
 * primitives, SH degree, dtype HS_DTYPE_F32/F64) over the ranks of `comm`, in
 * place, as one NCCL group on `stream`; with_touch also sums the int32 touch
 * counts.  Issued on a side stream after each K7 bucket
 * (hs_preprocess_bwd_range), bucket b's exchange overlaps bucket b+1's K7. */
int hs_grad_allreduce(void* comm, const hs_grads* grads, int64_t n, int32_t sh_degree,
                      int32_t dtype, int64_t begin, int64_t end, int32_t with_touch,
                      void* stream);

/* ---- misc --------------------------------------------------------------- */
const char* hs_status_string(int status);
const char* hs_last_cuda_error(void);
/* Number of kernels this library launched so far (process-wide counter). */
int64_t hs_kernel_launch_count(void);
int32_t hs_abi_version(void);
/* FP32 FMA (TFLOP/s, FMA = 2 flops) and MUFU.EX2 (Gop/s) throughput of the
 * current device, measured by two probe kernels: the roofline denominators for
 * the FP32/SFU-bound blend kernels. */
int hs_measure_fp32_peaks(double* fma_tflops, double* ex2_gops);
/* Packed FP32 (fma.rn.f32x2) throughput measured by the last
 * hs_measure_fp32_peaks call, TFLOP/s. */
double hs_last_fma2_tflops(void);
/* Evaluates the blend kernels' FP32 erf (the one K5/K6 use, on MUFU.EX2) at n
 * device points z -> out: a test probe for its accuracy and oddness. */
int hs_probe_erf32(const float* z, float* out, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HALFSPLAT_B200_H */
