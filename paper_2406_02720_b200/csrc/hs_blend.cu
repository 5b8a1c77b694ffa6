// hs_blend.cu -- K5 forward blend and K6 backward blend.
//
// Semantics follow the reference blend core exactly (_blend_cy.pyx:86-187 and
// 202-347): every pair in a tile list is evaluated until the pixel terminates
// (no alpha skip), w = min((c1 + c2*E) * g, 0.99), termination *before*
// compositing when T*(1-w) < 1e-4, terminal = committed count, depth = sum of
// w*T*z, gradient gating on w_raw <= 0.99, pixel centres at +0.5.
//
// Mapping (B200): one warp owns one 16x16 tile; lane l owns column l&15 and the
// eight rows (l>>4) + 2i.  Because the column is shared, every per-splat term
// that depends only on dx (A*dx^2, B*dx, za*dx) is hoisted out of the 8-pixel
// loop, leaving ~2 FMAs of Gaussian power per pixel.  Splat records (64 B) are
// gathered 32 at a time with cp.async into a per-warp double buffer and read back
// as broadcast LDS.128.  Warps pull tiles from a global counter (persistent
// grid), so long tile lists do not stall a whole CTA.
//
// Precision: pixel offsets use mu_hat = hi + lo (float + half residual), so dx
// is exact to ~3e-8 px at any resolution; "steep" splats (see hs_common.cuh)
// evaluate the erf argument in FP64 from a side record staged with the record.
#include <cstdint>
#include <type_traits>

#include <cuda_fp16.h>

#include <mutex>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

// Warps per CTA and the minimum resident CTAs per SM (a register cap) of each
// blend.  One-warp CTAs (each warp is independent: its own tile queue pulls,
// staging and shared memory) let the SM fill to the register limit exactly:
// K5 at 124 registers runs 16 warps/SM, K6 at 153 runs 12.  Measured on c3
// (tools/build_variant.sh + tools/variant_bench.sh): one-warp CTAs took K5 0.856
// -> 0.840 ms and K6 1.693 -> 1.651 ms; with the current bodies, capping K6 at 13
// or 14 warps (MINB 13/14) or K5 at 12/14 is slower.  MINB 0 = no cap.
#ifndef HS_FWD_WARPS
#define HS_FWD_WARPS 1
#endif
#ifndef HS_FWD_MINB
#define HS_FWD_MINB 16
#endif
#ifndef HS_BWD_WARPS
#define HS_BWD_WARPS 1
#endif
#ifndef HS_BWD_MINB
#define HS_BWD_MINB 12
#endif
constexpr int kFwdWarps = HS_FWD_WARPS;
constexpr int kBwdWarps = HS_BWD_WARPS;
#if HS_FWD_MINB > 0
#define HS_FWD_BOUNDS __launch_bounds__(kFwdWarps * 32, HS_FWD_MINB)
#else
#define HS_FWD_BOUNDS __launch_bounds__(kFwdWarps * 32)
#endif
#if HS_BWD_MINB > 0
#define HS_BWD_BOUNDS __launch_bounds__(kBwdWarps * 32, HS_BWD_MINB)
#else
#define HS_BWD_BOUNDS __launch_bounds__(kBwdWarps * 32)
#endif
constexpr int kBatch = 32;

constexpr int kPx = 8;  // pixels per lane
constexpr float kNegHalfLog2e = -0.5f * kLog2e;
constexpr float kNegLog2e = -kLog2e;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct WarpStage {
  float4 rec[2][kBatch][4];
  SteepRec side[2][kBatch];
  int win[2][kBatch];  // strip window code of each staged splat in the current tile
  int org[2][kBatch];  // K6: each staged splat's pair-row origin
};

// Gather the records of `count` (<= 32) pairs, pair j at sorted index
// k0 + pos(j), into stage slot j (one lane per record); steep splats also get
// their FP64 side record.  In two halves, so a batch's sorted indices can be
// loaded one batch ahead (a register prefetch) and the gather of its records
// issued without waiting on them: a warp alone on its SM (a frame's longest
// tiles) otherwise stalls a full global round trip per batch.
template <typename PosFn>
__device__ __forceinline__ uint32_t batch_index(const BlendGeom& g, int k0, int count,
                                                PosFn pos, int lane) {
  return lane < count ? g.pair_src[k0 + pos(lane)] : 0u;
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}

// ORG (K6): also the splat's pair-row origin
template <bool ORG = false>
__device__ __forceinline__ void issue_records(const BlendGeom& g, uint32_t v, int count,
                                              WarpStage& st, int stage, int lane) {
  if (lane < count) {
    const uint32_t idx = v & kIndexMask;
    const float4* src = g.rec + 4 * (size_t)idx;
#pragma unroll
    for (int c = 0; c < 4; ++c) cp_async16(&st.rec[stage][lane][c], src + c);
    if (ORG) cp_async4(&st.org[stage][lane], g.row_origin + idx);
    if (v & kSteepBit) {
      const char* s = reinterpret_cast<const char*>(g.side + idx);
      char* d = reinterpret_cast<char*>(&st.side[stage][lane]);
      cp_async16(d, s);
      cp_async16(d + 16, s + 16);
    }
  }
  cp_async_commit();
}

// The persistent blends' work queue.  Units come in longest-first order, and the
// warps of one SM share its issue slots, so what has to balance is the work per
// SM: a plain counter hands the first (longest) units to consecutive warps, i.e. to
// the same few SMs (c2: 16 of the longest tiles on SM 0, the kernel 2.3x its
// balanced time).  So the first wave is spread: the k-th warp to start on SM s
// takes unit k * n_sm + s (snake order over k), claimed with a flag; later units
// come from a dynamic counter over [n_first, n_units); a first-wave unit nobody
// claimed (an SM that hosts fewer warps than planned) is picked up by a final
// sweep over the flags, so every unit runs exactly once whatever the placement.
// Returns -1 when the queue is empty; `phase` is per warp, starting at 0.
__device__ __forceinline__ int next_unit(const BlendGeom& g, int n_units, int& phase, int lane) {
  int t = -1;
  if (lane == 0) {
    int* q = g.work_counter;
    const int n_first = g.spread ? min(g.n_first, n_units) : 0;
    if (phase == 0) {
      phase = 1;
      if (n_first > 0) {
        int s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        if (s < g.n_sm && s < kQueueMaxSms) {
          const int k = atomicAdd(q + 2 + s, 1);
          const int r = k * g.n_sm + ((k & 1) ? g.n_sm - 1 - s : s);
          if (k < g.per_sm && r < n_first && atomicExch(q + 2 + kQueueMaxSms + r, 1) == 0) t = r;
        }
      }
    }
    if (t < 0 && phase == 1) {
      const int d = n_first + atomicAdd(q, 1);
      if (d < n_units) t = d;
      else phase = n_first > 0 ? 2 : 3;
    }
    while (t < 0 && phase == 2) {
      const int i = atomicAdd(q + 1, 1);
      if (i >= n_first) phase = 3;
      else if (atomicExch(q + 2 + kQueueMaxSms + i, 1) == 0) t = i;
    }
  }
  phase = __shfl_sync(0xffffffffu, phase, 0);
  return __shfl_sync(0xffffffffu, t, 0);
}


// Per-(splat, lane) constants shared by the forward and backward pixel loops.
struct SplatLane {
  float dx, dy0;       // pixel offsets of row 0 (dy of row i = dy0 + 2i)
  float A, B, C;       // conic scaled to log2: power = dx*(A dx + B dy) + C dy^2
  float P0, Bx;        // A dx^2, B dx
  float za, zb, Z0;    // erf coefficients, za*dx
  // steep splats: z(row offset o) = zK * (fma(zt_hi, o, zc_hi) + zc_lo + zt_lo o)
  float zK, zc_hi, zc_lo, zt_hi, zt_lo;
};

// PRE: the staged record was already transformed by prescale_record (K5).
template <bool STEEP, bool PRE = false>
__device__ __forceinline__ SplatLane splat_lane(const float4 (&q)[4], const SteepRec& side,
                                                float px, float py0) {
  SplatLane s;
  const __half2 lo = *reinterpret_cast<const __half2*>(&q[3].w);
  const float2 lof = __half22float2(lo);
  s.dx = (px - q[0].x) - lof.x;
  s.dy0 = (py0 - q[0].y) - lof.y;
  s.A = PRE ? q[0].z : q[0].z * kNegHalfLog2e;
  s.B = PRE ? q[0].w : q[0].w * kNegLog2e;
  s.C = PRE ? q[1].x : q[1].x * kNegHalfLog2e;
  s.P0 = s.A * s.dx * s.dx;
  s.Bx = s.B * s.dx;
  s.za = q[1].y;
  s.zb = q[1].z;
  s.Z0 = s.za * s.dx;
  if (STEEP) {
    // the bracket at this lane's column and first row, in FP64 (SteepRec)
    const double dxd = (double)px - side.mux, dyd = (double)py0 - side.muy;
    const double c = side.xform ? fma(side.r, dyd, dxd) : fma(side.r, dxd, dyd);
    const double t = side.xform ? side.r : 1.0;
    s.zK = side.K;
    s.zc_hi = (float)c;
    s.zc_lo = (float)(c - (double)s.zc_hi);
    s.zt_hi = (float)t;
    s.zt_lo = (float)(t - (double)s.zt_hi);
  }
  return s;
}

// Pixel pairs.  Lane pixel i (row offset 2i) lives in pair i>>1, slot i&1, so
// every per-pixel quantity is a float2 and the fast paths run on the packed
// FP32 pipe instructions of sm_100 (FFMA2/FMUL2/FADD2: one issue slot for two
// pixels; negated, broadcast-scalar and immediate operands fold into the
// instruction).  The MUFU ops (ex2, rcp) stay scalar.
constexpr int kPairs = kPx / 2;
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 ex2x2(float2 x) {
  return make_float2(ex2_approx(x.x), ex2_approx(x.y));
}
__device__ __forceinline__ float& slot(float2& v, int h) { return h ? v.y : v.x; }
__device__ __forceinline__ float slot(const float2& v, int h) { return h ? v.y : v.x; }

// erf32 on a pixel pair: same arithmetic as erf32 (fma.rn per lane), so the
// packed and scalar paths agree bit for bit.
__device__ __forceinline__ float2 erf32x2(float2 z) {
  const float2 a = make_float2(fminf(fabsf(z.x), 3.92f), fminf(fabsf(z.y), 3.92f));
  float2 r = ffma2(f2(1.420475164e-04f), a, f2(-3.664300777e-03f));
  r = ffma2(r, a, f2(3.089622408e-02f));
  r = ffma2(r, a, f2(-1.496994644e-01f));
  r = ffma2(r, a, f2(-9.181654453e-01f));
  r = ffma2(r, a, f2(-1.627925038e+00f));
  r = fmul2(r, a);
  const float2 om = fadd2(f2(1.0f), neg2(ex2x2(r)));
  return make_float2(copysignf(om.x, z.x), copysignf(om.y, z.y));
}

// dy of pair p: rows (row0 + 4p, row0 + 4p + 2)
__device__ __forceinline__ float2 pair_dy(float dy0, int p) {
  return fadd2(f2(dy0), make_float2(4.0f * p, 4.0f * p + 2.0f));
}

// steep z of a pixel pair (row offsets o = 4p, 4p + 2) and of one pixel; the
// same operation sequence, so packed and scalar paths agree bit for bit
__device__ __forceinline__ float2 steep_z2(const SplatLane& s, int p) {
  const float2 o = make_float2(4.0f * p, 4.0f * p + 2.0f);
  float2 b = fadd2(ffma2(f2(s.zt_hi), o, f2(s.zc_hi)), f2(s.zc_lo));
  b = ffma2(f2(s.zt_lo), o, b);
  return fmul2(f2(s.zK), b);
}

// erf argument z of pixel i: FP32 for ordinary splats, the side-record form
// for steep ones.
__device__ __forceinline__ float erf_arg(const SplatLane& s, bool steep, int i) {
  if (steep) {
    const float o = 2.0f * i;
    return s.zK * fmaf(s.zt_lo, o, fmaf(s.zt_hi, o, s.zc_hi) + s.zc_lo);
  }
  return fmaf(s.zb, s.dy0 + 2.0f * i, s.Z0);
}

// Blend factor E of the three modes (_blend_cy.pyx:156-161); mode 2 records
// carry za = zb = 0, so erf32(0) = 0 serves it too.
__device__ __forceinline__ float mode_factor(int mode, float z) {
  return mode == kModeSign ? sign32(z) : erf32(z);
}

// packed fast paths: mode 0 or 2 and no clamp (steep or not)
__device__ __forceinline__ bool fast_flags(uint32_t flags) {
  return (flags & kFlagClamp) == 0 && (flags & 3u) != (uint32_t)kModeSign;
}

// ---------------------------------------------------------------------------
// Strip windows.  Strip p of a tile is rows 4p..4p+3, i.e. pixel pair p of every
// lane.  A splat whose Gaussian is below 2^-27 at every pixel centre of a strip
// cannot change that strip in FP32: w <= g (u <= max(alpha1, alpha2) < 1), so
// w T is below half an ulp of T and T (1 - w) rounds to T, every alive pixel
// still commits (T >= 1e-4 already held), 1 - w rounds to 1 so the backward's
// T / (1 - w) is T, and the skipped colour, depth and gradient terms are below
// 2^-27 of their scale per pair.  The fast paths therefore evaluate only the
// strips the splat reaches (the forward still counts the commit of the others):
// about a third of the (splat, strip) work at c3-c4 (small splats straddling
// tile borders).  The reached strips of a convex superlevel set are contiguous;
// they are evaluated in one of three windows (code 1: pairs 0-1, code 2: pairs
// 2-3, code 3: all four; code 0: none), which keeps 22 of the 31 points of
// skippable work at c3 with two extra pair bodies per path (finer windows cost
// more in instruction-cache misses than they save).
// The staging lane of each splat computes its code once per tile.  The FP32
// bound uses 2^-27 against the 2^-25 the argument needs (a factor 4 of margin for
// its own rounding); NaN keeps every strip.
constexpr int kWinNone = 0;
constexpr int kWinAll = 3;
constexpr float kSkipQ = 37.42994775f;  // q = a dx^2 + 2b dx dy + c dy^2 > 54 ln 2  <=>  g < 2^-27

// min over t in [lo, hi] of a X^2 + 2 b X t + c t^2 (c > 0)
__device__ __forceinline__ float edge_min_q(float a, float b, float c, float X, float lo,
                                            float hi) {
  const float t = fminf(fmaxf(__fdividef(-b * X, c), lo), hi);
  return fmaf(a * X, X, t * fmaf(2.0f * b, X, c * t));
}

// min of the conic's quadratic form over the box [xl, xh] x [yl, yh] of offsets:
// 0 if the centre is inside, else the least of the four edge minima (convexity)
__device__ __forceinline__ float box_min_q(float a, float b, float c, float xl, float xh,
                                           float yl, float yh) {
  if (xl <= 0.f && xh >= 0.f && yl <= 0.f && yh >= 0.f) return 0.f;
  float m = fminf(edge_min_q(a, b, c, xl, yl, yh), edge_min_q(a, b, c, xh, yl, yh));
  m = fminf(m, edge_min_q(c, b, a, yl, xl, xh));
  return fminf(m, edge_min_q(c, b, a, yh, xl, xh));
}

// window code of a staged record (raw conic, before any prescale) in the tile
// (or sub-tile of 2 H rows: H = pixels per lane) whose first pixel centre is (x0, y0)
template <int H = kPx>
__device__ __forceinline__ int strip_window(const float4 (&q)[4], float x0, float y0) {
  if (__float_as_uint(q[3].y) & kFlagNoWin) return kWinAll;
  const float2 lo = __half22float2(*reinterpret_cast<const __half2*>(&q[3].w));
  const float xl = (x0 - q[0].x) - lo.x, xh = xl + (float)(kTile - 1);
  const float a = q[0].z, b = q[0].w, c = q[1].x;
  // the windows are halves: one box per half, rows 0..H-1 and H..2H-1
  const float yl = (y0 - q[0].y) - lo.y;
  const bool low = !(box_min_q(a, b, c, xl, xh, yl, yl + (float)(H - 1)) > kSkipQ);
  const bool high = !(box_min_q(a, b, c, xl, xh, yl + (float)H, yl + (float)(2 * H - 1)) > kSkipQ);
  if (H <= 2) return (low || high) ? kWinAll : 0;  // one pixel pair: no half windows
  return (low ? 1 : 0) | (high ? 2 : 0);
}

// calls f(P0, NP) with the window as compile-time constants
template <typename F>
__device__ __forceinline__ void with_window(int win, F&& f) {
  switch (win) {
    case 1: f(std::integral_constant<int, 0>{}, std::integral_constant<int, 2>{}); break;
    case 2: f(std::integral_constant<int, 2>{}, std::integral_constant<int, 2>{}); break;
    default: f(std::integral_constant<int, 0>{}, std::integral_constant<int, 4>{}); break;
  }
}

// ---------------------------------------------------------------------------
// K5 forward.  Each pixel carries T and a 0/1 float "alive" mask A; a splat
// commits with m = A * [T (1 - w) >= 1e-4], and every update is an exact
// multiply by m: nw m is -w or 0, so T <- fma(nw m, T, T) is T (1 - w) or T
// unchanged, the colour term is (nw m) T, the count adds m, and A <- m (a pixel
// that fails the test is dead for good).  No selects or integer ops per pixel;
// pixels outside the image start dead.  The colour/depth accumulators hold the
// NEGATED sums (T - w T = fma(-w, T, T) needs -w; the sign is restored at the
// store).  Dead pixels compute and discard.
template <int NPX = kPx>
struct FwdPix {
  static constexpr int NP = NPX / 2;
  float2 T[NP], A[NP], C[NP], ar[NP], ag[NP], ab[NP], ad[NP];
};

__device__ __forceinline__ float ge_mask(float v) { return v >= kTerminationT ? 1.0f : 0.0f; }

// one pixel: the termination rule and compositing of _blend_cy.pyx:162-176
__device__ __forceinline__ void fwd_commit(float nw, float& T, float& A, float& C, float& ar,
                                           float& ag, float& ab, float& ad, float cr, float cg,
                                           float cb, float z) {
  const float tn = fmaf(nw, T, T);  // T * (1 - w)
  const float m = A * ge_mask(tn);
  const float nwm = nw * m;
  const float nwt = nwm * T;
  ar = fmaf(nwt, cr, ar);
  ag = fmaf(nwt, cg, ag);
  ab = fmaf(nwt, cb, ab);
  ad = fmaf(nwt, z, ad);
  C += m;
  A = m;
  T = fmaf(nwm, T, T);
}

// FAST: mode 0 or 2, weight provably below the 0.99 clamp; STEEP takes z from
// the side-record form.
// Pairs [P0, P0 + NP) are evaluated; the others are outside the splat's strip
// window and only count the commit of their alive pixels (see strip_window).
// -w of pixel pair p (independent of the pixels' state)
template <bool STEEP>
__device__ __forceinline__ float2 fwd_pair_nw(const SplatLane& s, const float4 (&q)[4], int p) {
  const float nc1 = q[1].w, nc2 = q[2].x;  // negated by prescale_record
  const float2 dy = pair_dy(s.dy0, p);
  const float2 g = ex2x2(ffma2(ffma2(f2(s.C), dy, f2(s.Bx)), dy, f2(s.P0)));
  const float2 e = erf32x2(STEEP ? steep_z2(s, p) : ffma2(f2(s.zb), dy, f2(s.Z0)));
  return fmul2(ffma2(f2(nc2), e, f2(nc1)), g);
}

// the termination test and compositing of pair p given its -w
template <int NPX>
__device__ __forceinline__ void fwd_pair_commit(FwdPix<NPX>& P, int p, float2 nw,
                                                const float4 (&q)[4]) {
  const float cr = q[2].y, cg = q[2].z, cb = q[2].w, z = q[3].x;
  const float2 tn = ffma2(nw, P.T[p], P.T[p]);  // T * (1 - w)
  const float2 m = fmul2(P.A[p], make_float2(ge_mask(tn.x), ge_mask(tn.y)));
  const float2 nwm = fmul2(nw, m);
  const float2 nwt = fmul2(nwm, P.T[p]);
  P.ar[p] = ffma2(nwt, f2(cr), P.ar[p]);
  P.ag[p] = ffma2(nwt, f2(cg), P.ag[p]);
  P.ab[p] = ffma2(nwt, f2(cb), P.ab[p]);
  P.ad[p] = ffma2(nwt, f2(z), P.ad[p]);
  P.C[p] = fadd2(P.C[p], m);
  P.A[p] = m;
  P.T[p] = ffma2(nwm, P.T[p], P.T[p]);
}

template <bool STEEP, int P0, int NP, int NPX>
__device__ __forceinline__ void fwd_splat_fast(const float4 (&q)[4], const SteepRec& side,
                                               float px, float py0, FwdPix<NPX>& P) {
  const SplatLane s = splat_lane<STEEP, true>(q, side, px, py0);
#pragma unroll
  for (int p = 0; p < NPX / 2; ++p) {
    if (p < P0 || p >= P0 + NP) {
      P.C[p] = fadd2(P.C[p], P.A[p]);
      continue;
    }
    fwd_pair_commit(P, p, fwd_pair_nw<STEEP>(s, q, p), q);
  }
}

// N consecutive plain fast splats with the same window (pairs [P0, P0 + NPR)): every
// weight first, then the commits in list order.  The same operations as N
// fwd_splat_fast calls, but in one block, so the later splats' weight chains
// (record, exponent, erf) overlap the earlier ones' -- a warp alone on its scheduler
// (small frames, the long tails of a frame) waits out every splat's latency otherwise.
// (Pairs outside the window only count their alive pixels; those counts are exact
// small integers, so their order does not matter.)
template <int N, int P0, int NPR, int NPX>
__device__ __forceinline__ void fwd_splats_ilp(const WarpStage& st, int s, int j,
                                               float px, float py0, FwdPix<NPX>& P) {
  constexpr int NP = NPX / 2;
  float2 nw[N][NPR];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const float4 q[4] = {st.rec[s][j + k][0], st.rec[s][j + k][1], st.rec[s][j + k][2],
                         st.rec[s][j + k][3]};
    const SplatLane sl = splat_lane<false, true>(q, st.side[s][j], px, py0);
#pragma unroll
    for (int p = 0; p < NPR; ++p) nw[k][p] = fwd_pair_nw<false>(sl, q, P0 + p);
  }
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const float4 q[4] = {st.rec[s][j + k][0], st.rec[s][j + k][1], st.rec[s][j + k][2],
                         st.rec[s][j + k][3]};
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (p >= P0 && p < P0 + NPR)
        fwd_pair_commit(P, p, nw[k][p - P0], q);
      else
        P.C[p] = fadd2(P.C[p], P.A[p]);
    }
  }
}

// Generic: steep (FP64 z), sign mode, clamped weights; scalar per pixel.
template <int NPX>
__device__ __forceinline__ void fwd_splat_generic(const float4 (&q)[4], const SteepRec& side,
                                                  uint32_t flags, float px, float py0,
                                                  FwdPix<NPX>& P) {
  const bool steep = flags & kFlagSteep;
  const SplatLane s = steep ? splat_lane<true, true>(q, side, px, py0)
                            : splat_lane<false, true>(q, side, px, py0);
  const int mode = (int)(flags & 3u);
  const float c1 = -q[1].w, c2 = -q[2].x;  // prescale_record negated them
  const float cr = q[2].y, cg = q[2].z, cb = q[2].w, z = q[3].x;
  const bool large = flags & kFlagNoWin;  // s.A, s.C = scaled a, D; q[0].w = r
#pragma unroll
  for (int i = 0; i < NPX; ++i) {
    const int p = i >> 1, h = i & 1;
    const float dy = s.dy0 + 2.0f * i;
    const float u = fmaf(q[0].w, dy, s.dx);
    const float g = ex2_approx(large ? fmaf(s.A * u, u, s.C * dy * dy)
                                     : fmaf(fmaf(s.C, dy, s.Bx), dy, s.P0));
    const float e = mode_factor(mode, erf_arg(s, steep, i));
    const float w = fminf(fmaf(c2, e, c1) * g, kWeightClamp);
    fwd_commit(-w, slot(P.T[p], h), slot(P.A[p], h), slot(P.C[p], h), slot(P.ar[p], h),
               slot(P.ag[p], h), slot(P.ab[p], h), slot(P.ad[p], h), cr, cg, cb, z);
  }
}

// K5 staging transform, once per splat instead of once per lane: conic to the
// log2 scale of the exponent and -c1, -c2 (the forward composites with -w).
__device__ __forceinline__ void prescale_record(float4 (&r)[4]) {
  r[0].z *= kNegHalfLog2e;
  if (!(__float_as_uint(r[3].y) & kFlagNoWin)) r[0].w *= kNegLog2e;  // large: r = b/a stays
  r[1].x *= kNegHalfLog2e;
  r[1].w = -r[1].w;
  r[2].x = -r[2].x;
}

// Window mask (strip_window codes are a 2-bit mask: 1 first half of the pairs, 2
// second half) of the halves of the (sub-)tile that still have an alive pixel in
// some lane.  A dead half never changes again, so it joins the windows as skipped
// work.  With one pixel pair per lane there are no halves: 3 or 0.
template <int NPX>
__device__ __forceinline__ int alive_halves(const FwdPix<NPX>& P) {
  constexpr int NP = NPX / 2;
  float lo = 0.f, hi = 0.f;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const float a = fmaxf(P.A[p].x, P.A[p].y);
    if (NP == 1 || p < NP / 2) lo = fmaxf(lo, a); else hi = fmaxf(hi, a);
  }
  if (NP == 1) return __any_sync(0xffffffffu, lo > 0.0f) ? kWinAll : 0;
  return (__any_sync(0xffffffffu, lo > 0.0f) ? 1 : 0) | (__any_sync(0xffffffffu, hi > 0.0f) ? 2 : 0);
}

#if defined(HS_K5_PROBE) || defined(HS_K6_PROBE)
// experiments only (tools/k5_probe.py): per work unit {start ns, end ns, splats
// evaluated, SM id}
__device__ long long g_k5_probe[65536 * 4];
__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int sm_id() {
  int s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
extern "C" int hs_k5_probe_read(long long* out, int n_units) {
  if (cudaDeviceSynchronize() != cudaSuccess) return 1;
  return cudaMemcpyFromSymbol(out, g_k5_probe, sizeof(long long) * 4 * (size_t)n_units) !=
         cudaSuccess;
}
#endif

// A forward work unit: a 16-column by 2 * NPX-row sub-tile (the whole 16 x 16 tile
// at NPX = 8).  Small frames (c1's 64 tiles, c2's 2500 against 2368 resident warps)
// split their tiles into 2 or 4 sub-tiles, so more warps share the work and each
// stops when its own pixels are done.
template <int NPX, bool CKPT>
__global__ void HS_FWD_BOUNDS blend_fwd_kernel(
    BlendGeom g, float bg0, float bg1, float bg2, float* __restrict__ color,
    float* __restrict__ alpha, float* __restrict__ depth, float* __restrict__ trans,
    int32_t* __restrict__ terminal) {
  constexpr int NP = NPX / 2;
  constexpr int SUB = kPx / NPX;  // sub-tiles per tile
  __shared__ WarpStage stage_all[kFwdWarps];
  const int lane = threadIdx.x & 31;
  WarpStage& st = stage_all[threadIdx.x >> 5];
  int phase = 0;
  for (;;) {
    const int t = next_unit(g, g.n_work * SUB, phase, lane);
    if (t < 0) break;
    const int tr = t / SUB, sub = t - tr * SUB;
    const int tile = g.tile_order ? g.tile_order[tr] : g.tile_lo + tr;
    const int ty = tile / g.tiles_x, tx = tile - ty * g.tiles_x;
#ifdef HS_K5_PROBE
    const long long probe_t0 = global_ns();
    int probe_splats = 0;
#endif
    const int col = tx * kTile + (lane & 15);
    const int sy0 = ty * kTile + sub * 2 * NPX;  // first row of the sub-tile
    const int row0 = sy0 + (lane >> 4);
    const float px = (float)col + 0.5f;
    const float py0 = (float)row0 + 0.5f;
    const float x0 = (float)(tx * kTile) + 0.5f, y0 = (float)sy0 + 0.5f;
    FwdPix<NPX> P;
#pragma unroll
    for (int i = 0; i < NPX; ++i) {
      const int p = i >> 1, h = i & 1;
      slot(P.T[p], h) = 1.f;
      slot(P.A[p], h) = (col < g.width && row0 + 2 * i < g.height) ? 1.f : 0.f;
      slot(P.C[p], h) = 0.f;
      slot(P.ar[p], h) = 0.f; slot(P.ag[p], h) = 0.f; slot(P.ab[p], h) = 0.f;
      slot(P.ad[p], h) = 0.f;
    }
    const int k0 = g.tile_starts[tile];
    const int nk = g.tile_starts[tile + 1] - k0;
    auto fwd_pos = [](int j) { return j; };
    auto count_of = [&](int b) { return min(kBatch, nk - b * kBatch); };
    if (nk > 0)
      issue_records(g, batch_index(g, k0, count_of(0), fwd_pos, lane), count_of(0), st, 0, lane);
    uint32_t vnext = nk > kBatch ? batch_index(g, k0 + kBatch, count_of(1), fwd_pos, lane) : 0u;
    bool any = true;
    int alive = kWinAll;
    // pixel id within the tile (checkpoint layout: row * 16 + column) of pixel 0;
    // pixel i is 32 i further
    const int ck_pid0 = CKPT ? (sy0 - ty * kTile + (lane >> 4)) * kTile + (lane & 15) : 0;
    for (int b = 0; b * kBatch < nk && any; ++b) {
      const int nb = min(kBatch, nk - b * kBatch);
      if ((b + 1) * kBatch < nk) {
        issue_records(g, vnext, count_of(b + 1), st, (b + 1) & 1, lane);
        if ((b + 2) * kBatch < nk)
          vnext = batch_index(g, k0 + (b + 2) * kBatch, count_of(b + 2), fwd_pos, lane);
      } else {
        cp_async_commit();
      }
      cp_async_wait<1>();
      __syncwarp();
      const int s = b & 1;
      if (lane < nb) {
        // one dispatch key per staged splat: 4 * kind + window, kind 0 fast, 1 fast
        // steep, 2 generic (the window mask then only selects among the fast bodies)
        const uint32_t fl = __float_as_uint(st.rec[s][lane][3].y);
        const int kind = (!fast_flags(fl) || (fl & kFlagNoWin)) ? 2 : ((fl & kFlagSteep) ? 1 : 0);
        st.win[s][lane] =
            4 * kind + (kind == 2 ? kWinAll : strip_window<NPX>(st.rec[s][lane], x0, y0));
        prescale_record(st.rec[s][lane]);
      }
      __syncwarp();
      for (int j = 0; j < nb; ++j) {
        // dead pixels never change again: stop once the whole (sub-)tile is dead,
        // skip a dead half (checked every 8 splats; the reference checks per
        // splat, same result)
        if ((j & 7) == 0) {
          alive = alive_halves(P);
          if (!(any = alive != 0)) break;
          if (CKPT && j == 0 && b > 0 && ((b * kBatch) & ((1 << g.ckpt_shift) - 1)) == 0) {
            // K6 segment checkpoint at list position m = b * kBatch: the state of
            // every pixel still alive before splat m (T, negated colour sums so far)
            // (scalar stores: a 16-B store would want the four values in an aligned
            // register quad, which reshuffles the packed pixel pairs all over the loop)
            float* ck = reinterpret_cast<float*>(
                g.ckpt + (size_t)((k0 + b * kBatch) >> g.ckpt_shift) * kCkptSlot);
#pragma unroll
            for (int i = 0; i < NPX; ++i) {
              const int p = i >> 1, h = i & 1;
              if (slot(P.A[p], h) > 0.f) {
                float* e = ck + 4 * (ck_pid0 + 32 * i);
                e[0] = slot(P.T[p], h);
                e[1] = slot(P.ar[p], h);
                e[2] = slot(P.ag[p], h);
                e[3] = slot(P.ab[p], h);
              }
            }
          }
        }
#ifdef HS_K5_PROBE
        ++probe_splats;
#endif
        const int key = st.win[s][j] & (~3 | alive);  // generic keeps its window bits: 8+
#ifndef HS_K5_TWO
#define HS_K5_TWO 2
#endif
// (HS_K5_TWO8: the same on full 16x16 tiles, off: c5 K5 -3%, c3 +1.2%, c4 -0.5%)
#ifndef HS_K5_TWO8
#define HS_K5_TWO8 0
#endif
        constexpr int H = NP > 1 ? NP / 2 : NP;  // pairs per half window
        if constexpr (HS_K5_TWO > 1 && (NPX == 2 || HS_K5_TWO8)) {
          // two plain fast splats with the same window inside one group of 8 (same
          // alive mask)
          if (key >= 1 && key <= 3 && (j & 7) != 7 && j + 1 < nb &&
              (st.win[s][j + 1] & (~3 | alive)) == key) {
            if constexpr (NP == 1) {
              fwd_splats_ilp<2, 0, 1>(st, s, j, px, py0, P);
            } else {
              if (key == 1) fwd_splats_ilp<2, 0, H>(st, s, j, px, py0, P);
              else if (key == 2) fwd_splats_ilp<2, NP - H, H>(st, s, j, px, py0, P);
              else fwd_splats_ilp<2, 0, NP>(st, s, j, px, py0, P);
            }
            ++j;
#ifdef HS_K5_PROBE
            ++probe_splats;
#endif
            continue;
          }
        }
        const float4 q[4] = {st.rec[s][j][0], st.rec[s][j][1], st.rec[s][j][2], st.rec[s][j][3]};
        const uint32_t flags = __float_as_uint(q[3].y);
        switch (key) {
          case 1: fwd_splat_fast<false, 0, H>(q, st.side[s][j], px, py0, P); break;
          case 2: fwd_splat_fast<false, NP - H, H>(q, st.side[s][j], px, py0, P); break;
          case 3: fwd_splat_fast<false, 0, NP>(q, st.side[s][j], px, py0, P); break;
          case 5: fwd_splat_fast<true, 0, H>(q, st.side[s][j], px, py0, P); break;
          case 6: fwd_splat_fast<true, NP - H, H>(q, st.side[s][j], px, py0, P); break;
          case 7: fwd_splat_fast<true, 0, NP>(q, st.side[s][j], px, py0, P); break;
          case 0:
          case 4:
#pragma unroll
            for (int p = 0; p < NP; ++p) P.C[p] = fadd2(P.C[p], P.A[p]);
            break;
          default: fwd_splat_generic(q, st.side[s][j], flags, px, py0, P); break;
        }
      }
      __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NPX; ++i) {
      const int p = i >> 1, h = i & 1;
      const int row = row0 + 2 * i;
      if (col < g.width && row < g.height) {
        const size_t o = (size_t)row * g.width + col;
        const float t = slot(P.T[p], h);
        color[3 * o + 0] = fmaf(t, bg0, -slot(P.ar[p], h));
        color[3 * o + 1] = fmaf(t, bg1, -slot(P.ag[p], h));
        color[3 * o + 2] = fmaf(t, bg2, -slot(P.ab[p], h));
        alpha[o] = 1.0f - t;
        depth[o] = -slot(P.ad[p], h);
        trans[o] = t;
        terminal[o] = (int32_t)slot(P.C[p], h);
      }
    }
    if (CKPT) {
      // the checkpoints become (T_m, S_m): S_m = the pixel's final colour minus its
      // colour before position m = background term + everything from m on, which K6
      // needs there (its dC . S).  Written for count >= m (the pixel was alive
      // before splat m), m < the list length.
#pragma unroll
      for (int i = 0; i < NPX; ++i) {
        const int p = i >> 1, h = i & 1;
        const int c = (int)slot(P.C[p], h);
        const int ck_len = 1 << g.ckpt_shift;
        if (c < ck_len || col >= g.width || row0 + 2 * i >= g.height) continue;
        const float t = slot(P.T[p], h);
        const float fr = fmaf(t, bg0, -slot(P.ar[p], h)), fg = fmaf(t, bg1, -slot(P.ag[p], h)),
                    fb = fmaf(t, bg2, -slot(P.ab[p], h));
        for (int m = ck_len; m <= c && m < nk; m += ck_len) {
          float4* ck =
              g.ckpt + (size_t)((k0 + m) >> g.ckpt_shift) * kCkptSlot + ck_pid0 + 32 * i;
          float4 v = *ck;
          v.y = fr + v.y;
          v.z = fg + v.z;
          v.w = fb + v.w;
          *ck = v;
        }
      }
    }
#ifdef HS_K5_PROBE
    if (lane == 0 && t < 65536) {
      long long* pr = g_k5_probe + 4 * (size_t)t;
      pr[0] = probe_t0;
      pr[1] = global_ns();
      pr[2] = probe_splats;
      pr[3] = sm_id() | ((long long)tile << 16);
    }
#endif
    if (g.tile_work) {
      // the backward's work on this tile: its largest terminal count (K6 walks
      // positions maxc-1 .. 0), for K6's longest-first tile order
      float mc = 0.f;
#pragma unroll
      for (int p = 0; p < NP; ++p) mc = fmaxf(mc, fmaxf(P.C[p].x, P.C[p].y));
      const int m = __reduce_max_sync(0xffffffffu, (int)mc);
      if (lane == 0) {
        if (SUB == 1) g.tile_work[tile] = m;
        else atomicMax(g.tile_work + tile, m);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K6 backward
struct BwdAcc {
  float s0, s1, s2;  // sum d_pow, d_pow*dy, d_pow*dy^2 (dx is constant per lane)
  float q0, q1, qz;  // sum d_z, d_z*dy, d_z*z
  float c1, c2, r, g, b;
  float dx;          // the lane's pixel offset from the splat centre (for the row columns)
  float cb, cc;      // the conic's b and c (the generic path rebuilds them for kFlagNoWin)
};

struct BwdPix {
  float2 T[kPairs], D[kPairs], dr[kPairs], dg[kPairs], db[kPairs];
  const int* cnt;  // this lane's terminal counts, cnt[i * 32] (shared memory; read
                   // by the generic path only)
};

// FAST: mode 0 or 2, FP32 z, no clamp.  Packed pixel pairs, no per-pixel masks:
// pixels past their terminal count are inert (T = D = 0, see blend_bwd_kernel)
// and contribute exact zeros.  Pairs [P0, P0 + NP) are evaluated; the others are
// outside the splat's strip window and unchanged (see strip_window).
template <bool STEEP, int P0 = 0, int NP = kPairs>
__device__ __forceinline__ void bwd_splat_fast(const float4 (&q)[4], const SteepRec& side,
                                               int pos, float px, float py0, BwdPix& P,
                                               BwdAcc& out) {
  const SplatLane s = splat_lane<STEEP>(q, side, px, py0);
  const float c1 = q[1].w, c2 = q[2].x;
  const float cr = q[2].y, cg = q[2].z, cb = q[2].w;
  // Row-offset basis: pixel dy = dy0 + o with o = 2i the offset from row 0, so the
  // exponent is (C o + Lg) o + Kg, z = zb o + Zc, and the dy-moments are kept as
  // o-moments and shifted by dy0 once per splat (no per-pixel dy).
  const float Lg = fmaf(2.0f * s.C, s.dy0, s.Bx);
  const float Kg = fmaf(fmaf(s.C, s.dy0, s.Bx), s.dy0, s.P0);
  const float Zc = fmaf(s.zb, s.dy0, s.Z0);
  float2 s0 = f2(0.f), s1 = f2(0.f), s2 = f2(0.f), q0 = f2(0.f), q1 = f2(0.f), qz = f2(0.f);
  float2 a1 = f2(0.f), a2 = f2(0.f), ar = f2(0.f), ag = f2(0.f), ab = f2(0.f);
#pragma unroll
  for (int p = P0; p < P0 + NP; ++p) {
    const float2 o = make_float2(4.0f * p, 4.0f * p + 2.0f);
    const float2 o2 = make_float2(16.0f * p * p, (4.0f * p + 2.0f) * (4.0f * p + 2.0f));
    const float2 gg = ex2x2(ffma2(ffma2(f2(s.C), o, f2(Lg)), o, f2(Kg)));
    const float2 zz = STEEP ? steep_z2(s, p) : ffma2(f2(s.zb), o, f2(Zc));
    const float2 e = erf32x2(zz);
    const float2 u = ffma2(f2(c2), e, f2(c1));
    const float2 w = fmul2(u, gg);
    const float2 om = fadd2(f2(1.0f), neg2(w));
    const float2 inv = make_float2(rcp_approx(om.x), rcp_approx(om.y));  // 1 - w >= 0.01
    const float2 Tp = fmul2(P.T[p], inv);
    float2 wt = fmul2(w, Tp);
    const float2 dcr = ffma2(P.dr[p], f2(cr), ffma2(P.dg[p], f2(cg), fmul2(P.db[p], f2(cb))));
    ar = ffma2(P.dr[p], wt, ar);
    ag = ffma2(P.dg[p], wt, ag);
    ab = ffma2(P.db[p], wt, ab);
    // d_w = T_prev*(dC.rgb) - (dC.S)/(1-w) = inv*(T*dcr - D) (_blend_cy.pyx:310-312)
    float2 d_w = fmul2(inv, ffma2(P.T[p], dcr, neg2(P.D[p])));
    const float2 dwg = fmul2(d_w, gg);
    const float2 d_pow = fmul2(dwg, u);
    s0 = fadd2(s0, d_pow);
    s1 = ffma2(d_pow, o, s1);
    s2 = ffma2(d_pow, o2, s2);
    a1 = fadd2(a1, dwg);
    a2 = ffma2(dwg, e, a2);
    // d_z / c2k (the constant factor is applied once per splat below)
    const float2 ez = ex2x2(fmul2(fmul2(zz, zz), f2(-kLog2e)));
    const float2 dz = fmul2(dwg, ez);
    q0 = fadd2(q0, dz);
    q1 = ffma2(dz, o, q1);
    qz = ffma2(dz, zz, qz);
    P.D[p] = ffma2(wt, dcr, P.D[p]);
    P.T[p] = Tp;
  }
  const float c2k = c2 * (2.0f * kInvSqrtPi);
  const float S0 = s0.x + s0.y, S1 = s1.x + s1.y, S2 = s2.x + s2.y;
  const float Q0 = q0.x + q0.y, Q1 = q1.x + q1.y;
  // back to dy-moments: sum d (dy0 + o) = dy0 S0 + S1; sum d (dy0 + o)^2 = dy0 (dy0 S0 + 2 S1) + S2
  out.s0 = S0;
  out.s1 = fmaf(s.dy0, S0, S1);
  out.s2 = fmaf(s.dy0, fmaf(s.dy0, S0, 2.0f * S1), S2);
  out.q0 = c2k * Q0; out.q1 = c2k * fmaf(s.dy0, Q0, Q1); out.qz = c2k * (qz.x + qz.y);
  out.c1 = a1.x + a1.y; out.c2 = a2.x + a2.y;
  out.r = ar.x + ar.y; out.g = ag.x + ag.y; out.b = ab.x + ab.y;
  out.dx = s.dx;
  out.cb = q[0].w;
  out.cc = q[1].x;
}

// Generic: sign mode, clamped weights, large splats (kFlagNoWin).  Scalar;
// inert pixels (T = D = 0) compute and contribute exact zeros.
__device__ __forceinline__ void bwd_splat_generic(const float4 (&q)[4], const SteepRec& side,
                                                  uint32_t flags, int pos, float px, float py0,
                                                  BwdPix& P, BwdAcc& a) {
  const bool steep = flags & kFlagSteep;
  const SplatLane s = steep ? splat_lane<true>(q, side, px, py0)
                            : splat_lane<false>(q, side, px, py0);
  const int mode = (int)(flags & 3u);
  const float c1 = q[1].w, c2 = q[2].x;
  const float cr = q[2].y, cg = q[2].z, cb = q[2].w;
  // d erf/dz = 2/sqrt(pi) exp(-z^2); only the erf mode has a z derivative
  const float c2k = mode == kModeErf ? c2 * (2.0f * kInvSqrtPi) : 0.0f;
  const bool large = flags & kFlagNoWin;  // s.A, s.C = scaled a, D; q[0].w = r
  a = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, s.dx, 0.f, 0.f};
  conic_abc(q[0].z, q[0].w, q[1].x, flags, a.cb, a.cc);
#pragma unroll
  for (int i = 0; i < kPx; ++i) {
    const int p = i >> 1, h = i & 1;
    float& T = slot(P.T[p], h);
    float& D = slot(P.D[p], h);
    const float dr = slot(P.dr[p], h), dg = slot(P.dg[p], h), db = slot(P.db[p], h);
    const float dy = s.dy0 + 2.0f * i;
    const float ul = fmaf(q[0].w, dy, s.dx);
    const float gg = ex2_approx(large ? fmaf(s.A * ul, ul, s.C * dy * dy)
                                      : fmaf(fmaf(s.C, dy, s.Bx), dy, s.P0));
    const float zz = erf_arg(s, steep, i);
    const float e = mode_factor(mode, zz);
    const float u = fmaf(c2, e, c1);
    const float w_raw = u * gg;
    const float w = fminf(w_raw, kWeightClamp);
    const float inv = rcp_approx(1.0f - w);
    const float Tp = T * inv;
    const float wt = w * Tp;  // inert pixels (T = D = 0) give exact zeros throughout
    const float dcr = fmaf(dr, cr, fmaf(dg, cg, db * cb));
    a.r = fmaf(dr, wt, a.r);
    a.g = fmaf(dg, wt, a.g);
    a.b = fmaf(db, wt, a.b);
    // gated on the unclamped weight (_blend_cy.pyx:309)
    const float d_w = w_raw <= kWeightClamp ? inv * fmaf(T, dcr, -D) : 0.0f;
    const float dwg = d_w * gg;
    const float d_pow = dwg * u;
    a.s0 += d_pow;
    a.s1 = fmaf(d_pow, dy, a.s1);
    a.s2 = fmaf(d_pow * dy, dy, a.s2);
    a.c1 += dwg;
    a.c2 = fmaf(dwg, e, a.c2);
    const float d_z = dwg * c2k * ex2_approx(-(zz * zz) * kLog2e);
    a.q0 += d_z;
    a.q1 = fmaf(d_z, dy, a.q1);
    a.qz = fmaf(d_z, zz, a.qz);
    D = fmaf(wt, dcr, D);
    T = Tp;
  }
}

// Pair rows are written once and read once, by K7a after the whole blend: a
// streaming (evict-first) store keeps them from evicting the splat records the
// blend gathers again for neighbouring tiles (HS_ROWS_STREAM=0: plain stores).
#ifndef HS_ROWS_STREAM
#define HS_ROWS_STREAM 1
#endif
__device__ __forceinline__ void row_store(float* p, float v) {
#if HS_ROWS_STREAM
  __stcs(p, v);
#else
  *p = v;
#endif
}

// Sum 16 per-lane values over the warp with 16 shuffles (recursive halving):
// afterwards lanes 2m and 2m+1 both hold the warp total of value m.
__device__ __forceinline__ float warp_transpose_reduce16(float (&v)[16], int lane) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const bool h = lane & 16;
    const float keep = h ? v[8 + j] : v[j];
    const float send = h ? v[j] : v[8 + j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool h = lane & 8;
    const float keep = h ? v[4 + j] : v[j];
    const float send = h ? v[j] : v[4 + j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool h = lane & 4;
    const float keep = h ? v[2 + j] : v[j];
    const float send = h ? v[j] : v[2 + j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  {
    const bool h = lane & 2;
    const float keep = h ? v[1] : v[0];
    const float send = h ? v[0] : v[1];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Sum 13 per-lane values over the warp through shared memory: every lane writes
// its values as column `lane` of a 13 x 36 buffer (rows padded to 36 floats: the
// 16-B reads below hit distinct bank groups), then lane 2m + h sums the 16 values
// of row m in columns 16h..16h+15 (four LDS.128 and a 4-level add tree) and the
// two halves are combined with one shuffle: lanes 2m and 2m + 1 both hold the warp
// total of value m.  ~35 instructions against the 61 of the shuffle transpose.
#ifndef HS_SMEM_REDUCE
#define HS_SMEM_REDUCE 1
#endif
constexpr int kRedStride = 36;
__device__ __forceinline__ float warp_reduce13_smem(const float (&v)[16], float* red, int lane) {
  __syncwarp();  // the previous splat's reads are done
#pragma unroll
  for (int k = 0; k < 13; ++k) red[k * kRedStride + lane] = v[k];
  __syncwarp();
  const int m = lane >> 1, h = lane & 1;
  float t = 0.f;
  if (m < 13) {
    const float4* row = reinterpret_cast<const float4*>(red + m * kRedStride + 16 * h);
    const float4 a = row[0], b = row[1], c = row[2], d = row[3];
    t = ((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w)) +
        (((c.x + c.y) + (c.z + c.w)) + ((d.x + d.y) + (d.z + d.w)));
  }
  return t + __shfl_xor_sync(0xffffffffu, t, 1);
}

// kRowsBySortedPos: Seam 1 layout (row k = sorted pair index, 12 reference
// columns).  Otherwise the generation-order layout: row = record origin +
// ty*spans_x + tx, kRowFloats columns, consumed by K7.
// Inert pixels.  A pixel whose terminal count c is below the tile's largest is
// inactive at the positions >= c that the reverse walk visits first.  Instead of
// masking it per splat, it starts "inert": T = 0 and D = 0, which makes every
// body contribute exact zeros for it (T_prev = 0, w T = 0, d_w = inv (0 - 0)) and
// keeps it inert.  Its real T and D wait in shared memory and are restored at
// position c - 1, when the warp reaches the next activation level (a warp-uniform
// check per splat; the restore itself runs once per distinct count).  So every
// position runs the all-active bodies with their strip windows, masked further by
// the halves (pairs 0-1, 2-3) in which every pixel is still inert.
template <bool kRowsBySortedPos, bool SPLIT>
__global__ void HS_BWD_BOUNDS blend_bwd_kernel(
    BlendGeom g, float bg0, float bg1, float bg2, const float* __restrict__ d_color,
    const float* __restrict__ trans, const int32_t* __restrict__ terminal,
    float* __restrict__ rows, int32_t* __restrict__ last_rank,
    const uint32_t* __restrict__ rank_of) {
  constexpr int kStride = kRowsBySortedPos ? 12 : kRowFloats;
  constexpr int kCols = kRowsBySortedPos ? 12 : 13;
  // generation-order rows are stored whole (columns 13-15 zero): a row's second
  // 32-B sector written in part would cost a read-modify-write in DRAM
  constexpr int kStoreCols = kRowsBySortedPos ? kCols : kStride;
  __shared__ WarpStage stage_all[kBwdWarps];
  __shared__ int cnt_all[kBwdWarps][kPx][32];
  __shared__ float tfin_all[kBwdWarps][kPx][32], dini_all[kBwdWarps][kPx][32];
  __shared__ __align__(16) float red_all[kBwdWarps][13 * kRedStride];
  float* red = red_all[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  WarpStage& st = stage_all[threadIdx.x >> 5];
  int* cnt = &cnt_all[threadIdx.x >> 5][0][lane];
  float* tfin = &tfin_all[threadIdx.x >> 5][0][lane];
  float* dini = &dini_all[threadIdx.x >> 5][0][lane];
  int phase = 0;
  const int n_units = SPLIT ? *g.n_units : g.n_work;
  for (;;) {
    const int u = next_unit(g, n_units, phase, lane);
    if (u < 0) break;
    int tile, seg = -1;
    if (SPLIT) {
      const int2 un = g.units[u];
      tile = un.x;
      seg = un.y;
    } else {
      tile = g.tile_order ? g.tile_order[u] : g.tile_lo + u;
    }
#ifdef HS_K6_PROBE
    const long long probe_t0 = global_ns();
#endif
    const int ty = tile / g.tiles_x, tx = tile - ty * g.tiles_x;
    const int col = tx * kTile + (lane & 15);
    const int row0 = ty * kTile + (lane >> 4);
    const float px = (float)col + 0.5f;
    const float py0 = (float)row0 + 0.5f;
    const float x0 = (float)(tx * kTile) + 0.5f, y0 = (float)(ty * kTile) + 0.5f;
    BwdPix P;
    P.cnt = cnt;
    int maxc = 0;
#pragma unroll
    for (int i = 0; i < kPx; ++i) {
      const int p = i >> 1, h = i & 1;
      const int row = row0 + 2 * i;
      if (col < g.width && row < g.height) {
        const size_t o = (size_t)row * g.width + col;
        const float t = trans[o];
        const float dr = d_color[3 * o + 0], dg = d_color[3 * o + 1], db = d_color[3 * o + 2];
        slot(P.T[p], h) = t;
        cnt[i * 32] = terminal[o];
        slot(P.dr[p], h) = dr;
        slot(P.dg[p], h) = dg;
        slot(P.db[p], h) = db;
        // suffix S starts at T_final * background; only dC.S is needed
        slot(P.D[p], h) = t * fmaf(dr, bg0, fmaf(dg, bg1, db * bg2));
        maxc = max(maxc, cnt[i * 32]);
      } else {
        // outside the image: inert for good (T = 0, zero cotangent; count "infinite"
        // so no activation level ever picks it)
        slot(P.T[p], h) = 0.f; cnt[i * 32] = 0x7fffffff; slot(P.dr[p], h) = 0.f;
        slot(P.dg[p], h) = 0.f; slot(P.db[p], h) = 0.f; slot(P.D[p], h) = 0.f;
      }
    }
    maxc = __reduce_max_sync(0xffffffffu, maxc);
    const int k0 = g.tile_starts[tile];
    // K6 segments: this unit walks positions top-1 .. lo.  Below the tile's top
    // segment, the pixels alive at `top` start from K5's checkpoint there (T before
    // position top, S = everything blended from top on).
    const int lo = SPLIT ? seg << g.ckpt_shift : 0;
    const int top = SPLIT ? min((seg + 1) << g.ckpt_shift, maxc) : maxc;
    if (SPLIT && top < maxc) {
      const float4* ck = g.ckpt + (size_t)((k0 + top) >> g.ckpt_shift) * kCkptSlot;
#pragma unroll
      for (int i = 0; i < kPx; ++i) {
        const int p = i >> 1, h = i & 1;
        const int c = cnt[i * 32];
        if (c >= top && c != 0x7fffffff) {
          const float4 v = ck[((lane >> 4) + 2 * i) * kTile + (lane & 15)];
          // parked values first: a pixel is restored from them only below its count
          slot(P.T[p], h) = v.x;
          slot(P.D[p], h) = fmaf(slot(P.dr[p], h), v.y,
                                 fmaf(slot(P.dg[p], h), v.z, slot(P.db[p], h) * v.w));
        }
      }
    }
    // park the pixels that start inactive; nxt = the next activation level (the
    // largest count below top), hmax_* = each half's largest count
    int nxt = -1, hmax_lo = 0, hmax_hi = 0;
#pragma unroll
    for (int i = 0; i < kPx; ++i) {
      const int p = i >> 1, h = i & 1;
      const int c = cnt[i * 32];
      if (c < top) {
        tfin[i * 32] = slot(P.T[p], h);
        dini[i * 32] = slot(P.D[p], h);
        slot(P.T[p], h) = 0.f;
        slot(P.D[p], h) = 0.f;
        nxt = max(nxt, c);
      }
      const int cm = c == 0x7fffffff ? 0 : c;
      if (i < kPx / 2) hmax_lo = max(hmax_lo, cm); else hmax_hi = max(hmax_hi, cm);
    }
    nxt = __reduce_max_sync(0xffffffffu, nxt);
    hmax_lo = __reduce_max_sync(0xffffffffu, hmax_lo);
    hmax_hi = __reduce_max_sync(0xffffffffu, hmax_hi);
    if (!kRowsBySortedPos && lane == 0 && top == maxc)
      last_rank[tile] =
          maxc > 0 ? (int32_t)rank_of[g.pair_src[k0 + maxc - 1] & kIndexMask] : -1;
    if (maxc == 0 || top <= lo) continue;
    // positions top-1 .. lo; batch b holds positions hi_b - j for j < nb
    const int len = top - lo;
    auto batch_hi = [&](int b) { return top - 1 - b * kBatch; };
    auto bwd_index = [&](int b) {
      const int hi = batch_hi(b);
      return batch_index(g, k0, min(kBatch, hi - lo + 1), [hi](int j) { return hi - j; }, lane);
    };
    issue_records<!kRowsBySortedPos>(g, bwd_index(0), min(kBatch, len), st, 0, lane);
    uint32_t vnext = kBatch < len ? bwd_index(1) : 0u;
    for (int b = 0; b * kBatch < len; ++b) {
      const int hi = batch_hi(b);
      const int nb = min(kBatch, hi - lo + 1);
      if ((b + 1) * kBatch < len) {
        issue_records<!kRowsBySortedPos>(g, vnext, min(kBatch, batch_hi(b + 1) - lo + 1), st,
                                         (b + 1) & 1, lane);
        if ((b + 2) * kBatch < len) vnext = bwd_index(b + 2);
      } else {
        cp_async_commit();
      }
      cp_async_wait<1>();
      __syncwarp();
      const int s = b & 1;
      if (lane < nb) {
        // dispatch key 4 * kind + window, as in K5 (kind 0 fast, 1 fast steep, 2 generic)
        const uint32_t fl = __float_as_uint(st.rec[s][lane][3].y);
        const int kind = (!fast_flags(fl) || (fl & kFlagNoWin)) ? 2 : ((fl & kFlagSteep) ? 1 : 0);
        st.win[s][lane] = 4 * kind + (kind == 2 ? kWinAll : strip_window(st.rec[s][lane], x0, y0));
        // the pair's generation-order row in this tile, once per splat instead of per lane
        if (!kRowsBySortedPos) {
          const int spans_x = (int)(fl >> kFlagSpanShift);
          st.rec[s][lane][3].z = __int_as_float(st.org[s][lane] + ty * spans_x + tx);
        }
      }
      __syncwarp();
      for (int j = 0; j < nb; ++j) {
        const int pos = hi - j;
        if (pos < nxt) {
          // activation level nxt: its pixels are active from this position on
#pragma unroll
          for (int i = 0; i < kPx; ++i) {
            const int p = i >> 1, h = i & 1;
            if (cnt[i * 32] == nxt) {
              slot(P.T[p], h) = tfin[i * 32];
              slot(P.D[p], h) = dini[i * 32];
            }
          }
          int m = -1;
#pragma unroll
          for (int i = 0; i < kPx; ++i) {
            const int c = cnt[i * 32];
            if (c < nxt) m = max(m, c);
          }
          nxt = __reduce_max_sync(0xffffffffu, m);
        }
        const float4 q[4] = {st.rec[s][j][0], st.rec[s][j][1], st.rec[s][j][2], st.rec[s][j][3]};
        const SteepRec& side = st.side[s][j];
        const uint32_t flags = __float_as_uint(q[3].y);
        BwdAcc a;
        // kRowsBySortedPos: the sorted position; else the row staged above
        const size_t row = kRowsBySortedPos ? (size_t)(k0 + pos) : (size_t)__float_as_int(q[3].z);
        const int vi = lane >> 1;
        // halves in which every pixel is still inert contribute nothing: skip them
        const int key = st.win[s][j] & (~3 | (pos < hmax_lo ? 1 : 0) | (pos < hmax_hi ? 2 : 0));
        if (key == 0 || key == 4) {
          // fast splat below 2^-27 on every live strip: a zero pair row, no reduction
          if (!(lane & 1) && vi < kStoreCols) row_store(rows + row * kStride + vi, 0.f);
          continue;
        }
        switch (key) {
          case 1: bwd_splat_fast<false, 0, 2>(q, side, pos, px, py0, P, a); break;
          case 2: bwd_splat_fast<false, 2, 2>(q, side, pos, px, py0, P, a); break;
          case 3: bwd_splat_fast<false, 0, 4>(q, side, pos, px, py0, P, a); break;
          case 5: bwd_splat_fast<true, 0, 2>(q, side, pos, px, py0, P, a); break;
          case 6: bwd_splat_fast<true, 2, 2>(q, side, pos, px, py0, P, a); break;
          case 7: bwd_splat_fast<true, 0, 4>(q, side, pos, px, py0, P, a); break;
          default: bwd_splat_generic(q, side, flags, pos, px, py0, P, a); break;
        }
        // per-lane partials -> the pair-row columns (_blend_py.py:16-18)
        const float ca = q[0].z, cb = a.cb, cc = a.cc, za = q[1].y, zb = q[1].z;
        const float dx = a.dx;
        float v[16];
        v[0] = fmaf(ca * dx, a.s0, fmaf(cb, a.s1, -za * a.q0));
        v[1] = fmaf(cc, a.s1, fmaf(cb * dx, a.s0, -zb * a.q0));
        v[2] = -0.5f * dx * dx * a.s0;
        v[3] = -dx * a.s1;
        v[4] = -0.5f * a.s2;
        // za/zb gradients exist only in the erf mode (_blend_cy.pyx:322-329)
        const bool erf_mode = (flags & 3u) == (uint32_t)kModeErf;
        v[5] = erf_mode ? dx * a.q0 : 0.f;
        v[6] = erf_mode ? a.q1 : 0.f;
        v[7] = a.c1;
        v[8] = a.c2;
        v[9] = a.r;
        v[10] = a.g;
        v[11] = a.b;
        v[12] = erf_mode ? a.qz : 0.f;
        v[13] = v[14] = v[15] = 0.f;
        const float total = HS_SMEM_REDUCE ? warp_reduce13_smem(v, red, lane)
                                           : warp_transpose_reduce16(v, lane);
        if (!(lane & 1) && vi < kStoreCols) row_store(rows + row * kStride + vi, total);
      }
      __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
#ifdef HS_K6_PROBE
    if (lane == 0 && tile < 65536) {
      long long* pr = g_k5_probe + 4 * (size_t)tile;
      pr[0] = probe_t0;
      pr[1] = global_ns();
      pr[2] = maxc;
      pr[3] = sm_id() | ((long long)tile << 16);
    }
#endif
  }
}

// Diagnostic: histogram of the strip window codes over every (tile, pair).
__global__ void window_stats_kernel(BlendGeom g, unsigned long long* __restrict__ hist) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.n_work) return;
  const int tile = g.tile_lo + t;
  const int ty = tile / g.tiles_x, tx = tile - ty * g.tiles_x;
  const float x0 = (float)(tx * kTile) + 0.5f, y0 = (float)(ty * kTile) + 0.5f;
  unsigned long long h[4] = {0, 0, 0, 0};
  for (int k = g.tile_starts[tile]; k < g.tile_starts[tile + 1]; ++k) {
    const float4* r = g.rec + 4 * (size_t)(g.pair_src[k] & kIndexMask);
    const float4 q[4] = {r[0], r[1], r[2], r[3]};
    ++h[strip_window(q, x0, y0)];
  }
  for (int i = 0; i < 4; ++i)
    if (h[i]) atomicAdd(hist + i, h[i]);
}

cudaError_t launch_window_stats(const BlendGeom& g, unsigned long long* hist, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(hist, 0, 4 * sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  window_stats_kernel<<<(g.n_work + 127) / 128, 128, 0, stream>>>(g, hist);
  note_launch();
  return cudaGetLastError();
}

// Seam 1: reference packed (M,13) float64 + mode int8 -> records; steep splats
// get side records and bit 31 in their pair values.
__global__ void pack_records_kernel(const double* __restrict__ packed,
                                    const int8_t* __restrict__ mode, int64_t m,
                                    float* __restrict__ rec, SteepRec* __restrict__ side,
                                    uint8_t* __restrict__ steep_flag) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= m) return;
  const double* p = packed + l * 13;
  float* r = rec + l * kRecordFloats;
  for (int c = 0; c < 13; ++c) r[c] = (float)p[c];
  const int md = mode[l] & 3;
  // reach from the dilated covariance = inverse of the conic (rasterizer.py:194-200)
  const double a = p[2], b = p[3], c = p[4], det = a * c - b * b;
  const double ia = c / det, ic = a / det, idet = ia * ic - (b / det) * (b / det);
  const double mid = 0.5 * (ia + ic);
  const double lam = mid + sqrt(fmax(mid * mid - idet, 0.0));
  const double reach = kRadiusSigmas * sqrt(fmax(lam, 0.0)) + 24.0;
  const bool steep = md != kModePlain && is_steep(p[5], p[6], reach);
  const float mux = (float)p[0], muy = (float)p[1];
  const __half2 lo = __floats2half2_rn((float)(p[0] - (double)mux), (float)(p[1] - (double)muy));
  const bool large = reach - 24.0 > kWinMaxRadius;
  if (large) {  // the stable conic form (hs_common.cuh kFlagNoWin)
    r[R_CB] = (float)(p[3] / p[2]);
    r[R_CC] = (float)(p[4] - p[3] * p[3] / p[2]);
  }
  r[R_FLAGS] = __uint_as_float(pack_flags(md, steep, may_clamp(p[7], p[8]), 0, false, large));
  r[R_ROW_ORIGIN] = __int_as_float(0);
  r[R_MU_LO] = __uint_as_float(*reinterpret_cast<const uint32_t*>(&lo));
  if (steep) side[l] = make_steep(p[0], p[1], p[5], p[6]);
  steep_flag[l] = steep ? 1 : 0;
}

__global__ void mark_steep_pairs_kernel(const uint8_t* __restrict__ steep_flag,
                                        uint32_t* __restrict__ pairs, int64_t p) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < p && steep_flag[pairs[k]]) pairs[k] |= kSteepBit;
}

// K6 segments: the (tile, segment) units of a split backward, segments of kCkpt
// list positions below each tile's largest terminal count (one unit for a tile
// with nothing to walk, which still writes its last_rank), tiles in `order` (K6's
// longest-first order) or natural order.  One CTA: a block scan per 1024 tiles.
__global__ void __launch_bounds__(1024) bwd_units_kernel(const int32_t* __restrict__ work,
                                                         const int32_t* __restrict__ order,
                                                         int n_tiles, int shift,
                                                         int2* __restrict__ units,
                                                         int* __restrict__ n_units) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < n_tiles; base += 1024) {
    const int i = base + threadIdx.x;
    int t = 0, ns = 0;
    if (i < n_tiles) {
      t = order ? order[i] : i;
      const int mc = work[t];
      ns = mc > (1 << shift) ? (mc + (1 << shift) - 1) >> shift : 1;
    }
    int x = ns;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += v;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      int y = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += v;
      }
      warp_tot[lane] = y;  // inclusive over warps
    }
    __syncthreads();
    const int excl = carry + (w > 0 ? warp_tot[w - 1] : 0) + x - ns;
    for (int k = 0; k < ns; ++k) units[excl + k] = make_int2(t, k);
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + ns;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_units = carry;
}

cudaError_t launch_bwd_units(const int32_t* tile_work, const int32_t* order, int n_tiles,
                             int ckpt_shift, int2* units, int* n_units, cudaStream_t stream) {
  bwd_units_kernel<<<1, 1024, 0, stream>>>(tile_work, order, n_tiles, ckpt_shift, units,
                                           n_units);
  note_launch();
  return cudaGetLastError();
}

// Longest-first tile order for the persistent blends (LPT): one CTA buckets the
// tiles by their work estimate -- the list length from tile_starts for K5, K5's
// largest terminal count per tile for K6 -- into 256 buckets, longest first, so
// the long tiles start first and the queue's tail holds short ones.  Order within
// a bucket is arbitrary: every tile's result is independent of when it runs.
__global__ void __launch_bounds__(1024) tile_order_kernel(const int32_t* __restrict__ starts,
                                                          const int32_t* __restrict__ work,
                                                          int n_tiles,
                                                          int32_t* __restrict__ order) {
  __shared__ int off[256];
  __shared__ int wmax;
  // (clamped: a K6 whose frame never ran K5 orders arbitrary values -- still a
  // permutation, so still correct)
  auto w_of = [&](int t) {
    return min(max(starts ? starts[t + 1] - starts[t] : work[t], 0), 1 << 30);
  };
  if (threadIdx.x == 0) wmax = 0;
  if (threadIdx.x < 256) off[threadIdx.x] = 0;
  __syncthreads();
  int m = 0;
  for (int t = threadIdx.x; t < n_tiles; t += 1024) m = max(m, w_of(t));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(&wmax, m);
  __syncthreads();
  const int shift = max(0, 24 - __clz(wmax));  // (w >> shift) < 256
  auto bucket = [&](int t) { return 255 - (w_of(t) >> shift); };
  for (int t = threadIdx.x; t < n_tiles; t += 1024) atomicAdd(&off[bucket(t)], 1);
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the 256 bucket sizes, 8 per lane
    int v[8], s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = off[threadIdx.x * 8 + k];
      s += v[k];
    }
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, incl, o);
      if (threadIdx.x >= o) incl += x;
    }
    int e = incl - s;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      off[threadIdx.x * 8 + k] = e;
      e += v[k];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += 1024) order[atomicAdd(&off[bucket(t)], 1)] = t;
}

cudaError_t launch_tile_order(const int32_t* starts, const int32_t* work, int n_tiles,
                              int32_t* order, cudaStream_t stream) {
  tile_order_kernel<<<1, 1024, 0, stream>>>(starts, work, n_tiles, order);
  note_launch();
  return cudaGetLastError();
}

// Persistent grid: resident CTAs per SM x SMs of that kernel (queried once).
template <typename Kernel>
static int blend_grid(Kernel kernel, int warps, int n_work, int* cache) {
  // (filled once per kernel; Seam 1 calls arrive from several host threads)
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (*cache == 0) {
    int dev = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, warps * 32, 0);
    *cache = sms * (per_sm < 1 ? 1 : per_sm);
  }
  const int want = (n_work + warps - 1) / warps;
  return want < *cache ? (want > 0 ? want : 1) : *cache;
}
static int g_fwd_grid[3][2] = {{0, 0}, {0, 0}, {0, 0}}, g_bwd_grid[2][2] = {{0, 0}, {0, 0}};

// resident warps of the persistent blends (the longest-first order pays only when
// the tiles are several times these)
int blend_fwd_slots() {
  return blend_grid(blend_fwd_kernel<kPx, false>, kFwdWarps, 1 << 30, &g_fwd_grid[0][0]) *
         kFwdWarps;
}
int blend_bwd_slots() {
  return blend_grid(blend_bwd_kernel<false, false>, kBwdWarps, 1 << 30, &g_bwd_grid[0][0]) *
         kBwdWarps;
}

static int sm_count() {
  static const int n = [] {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }();
  return n;
}

// the unit queue of a launch of `grid` CTAs of `warps` warps (see next_unit)
static cudaError_t reset_queue(BlendGeom& g, int grid, int warps, cudaStream_t stream) {
  int ints = 1;
  if (g.spread) {
    const int slots = grid * warps;
    g.n_sm = sm_count();
    g.per_sm = (slots + g.n_sm - 1) / g.n_sm;
    g.n_first = slots < kQueueMaxFirst ? slots : kQueueMaxFirst;
    ints = 2 + kQueueMaxSms + g.n_first;
  }
  return cudaMemsetAsync(g.work_counter, 0, sizeof(int) * (size_t)ints, stream);
}

template <int NPX, bool CKPT>
static cudaError_t launch_fwd_variant(BlendGeom& g, int units, int* cache, float bg0, float bg1,
                                      float bg2, float* color, float* alpha, float* depth,
                                      float* trans, int32_t* terminal, cudaStream_t stream) {
  const int grid = blend_grid(blend_fwd_kernel<NPX, CKPT>, kFwdWarps, units, cache);
  const cudaError_t e = reset_queue(g, grid, kFwdWarps, stream);
  if (e != cudaSuccess) return e;
  blend_fwd_kernel<NPX, CKPT><<<grid, kFwdWarps * 32, 0, stream>>>(g, bg0, bg1, bg2, color, alpha,
                                                                   depth, trans, terminal);
  return cudaSuccess;
}

cudaError_t launch_blend_fwd(const BlendGeom& g_in, float bg0, float bg1, float bg2, float* color,
                             float* alpha, float* depth, float* trans, int32_t* terminal,
                             cudaStream_t stream) {
  BlendGeom g = g_in;
  const int sub = g.sub_tiles == 2 || g.sub_tiles == 4 ? g.sub_tiles : 1;
  cudaError_t e;
  if (sub > 1 && g.tile_work) {  // max-reduced by the sub-tiles
    e = cudaMemsetAsync(g.tile_work, 0, (size_t)g.n_work * sizeof(int32_t), stream);
    if (e != cudaSuccess) return e;
  }
  const int units = g.n_work * sub;
  const bool ck = g.ckpt != nullptr;
#define HS_FWD_LAUNCH(NPX, SLOT)                                                               \
  (ck ? launch_fwd_variant<NPX, true>(g, units, &g_fwd_grid[SLOT][1], bg0, bg1, bg2, color,   \
                                      alpha, depth, trans, terminal, stream)                  \
      : launch_fwd_variant<NPX, false>(g, units, &g_fwd_grid[SLOT][0], bg0, bg1, bg2, color,  \
                                       alpha, depth, trans, terminal, stream))
  switch (sub) {
    case 4: e = HS_FWD_LAUNCH(2, 2); break;
    case 2: e = HS_FWD_LAUNCH(4, 1); break;
    default: e = HS_FWD_LAUNCH(kPx, 0); break;
  }
#undef HS_FWD_LAUNCH
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

template <bool SORTED, bool SPLIT>
static cudaError_t launch_bwd_variant(BlendGeom& g, int* cache, float bg0, float bg1, float bg2,
                                      const float* d_color, const float* trans,
                                      const int32_t* terminal, float* rows, int32_t* last_rank,
                                      const uint32_t* rank_of, cudaStream_t stream) {
  // a split backward's unit count is only known on the device: the persistent grid
  const int grid = blend_grid(blend_bwd_kernel<SORTED, SPLIT>, kBwdWarps,
                              SPLIT ? (1 << 30) : g.n_work, cache);
  const cudaError_t e = reset_queue(g, grid, kBwdWarps, stream);
  if (e != cudaSuccess) return e;
  blend_bwd_kernel<SORTED, SPLIT><<<grid, kBwdWarps * 32, 0, stream>>>(
      g, bg0, bg1, bg2, d_color, trans, terminal, rows, last_rank, rank_of);
  return cudaSuccess;
}

cudaError_t launch_blend_bwd(const BlendGeom& g_in, float bg0, float bg1, float bg2,
                             const float* d_color, const float* trans, const int32_t* terminal,
                             float* rows, int32_t* last_rank, const uint32_t* rank_of,
                             bool rows_by_sorted_pos, cudaStream_t stream) {
  BlendGeom g = g_in;
  const bool split = g.units != nullptr;
  cudaError_t e;
  if (rows_by_sorted_pos)
    e = split ? launch_bwd_variant<true, true>(g, &g_bwd_grid[1][1], bg0, bg1, bg2, d_color,
                                                trans, terminal, rows, last_rank, rank_of, stream)
              : launch_bwd_variant<true, false>(g, &g_bwd_grid[1][0], bg0, bg1, bg2, d_color,
                                                 trans, terminal, rows, last_rank, rank_of,
                                                 stream);
  else
    e = split ? launch_bwd_variant<false, true>(g, &g_bwd_grid[0][1], bg0, bg1, bg2, d_color,
                                                 trans, terminal, rows, last_rank, rank_of,
                                                 stream)
              : launch_bwd_variant<false, false>(g, &g_bwd_grid[0][0], bg0, bg1, bg2, d_color,
                                                  trans, terminal, rows, last_rank, rank_of,
                                                  stream);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pack_records(const double* packed, const int8_t* mode, int64_t m, float4* rec,
                                SteepRec* side, uint32_t* pairs, int64_t p, cudaStream_t stream) {
  if (m == 0) return cudaSuccess;
  const int block = 256;
  uint8_t* flag = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&flag), m, stream);
  if (e != cudaSuccess) return e;
  pack_records_kernel<<<(unsigned)((m + block - 1) / block), block, 0, stream>>>(
      packed, mode, m, reinterpret_cast<float*>(rec), side, flag);
  if (p > 0)
    mark_steep_pairs_kernel<<<(unsigned)((p + block - 1) / block), block, 0, stream>>>(flag, pairs,
                                                                                      p);
  note_launch(2);
  e = cudaGetLastError();
  cudaFreeAsync(flag, stream);
  return e;
}

}  // namespace hs
