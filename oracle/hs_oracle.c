/*
 * hs_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * CPU restatement (float64, OpenMP) of the reference's hot path, used only as the
 * parity checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg.  Nothing in paper_2406_02720_b200/ links or calls it.
 *
 *   oracle_prepare        rasterizer.py:159-341 (prepare)
 *   oracle_forward_tiles  _blend_cy.pyx:86-187  (_forward)
 *   oracle_backward_tiles _blend_cy.pyx:202-347 (_backward)
 *   oracle_backward       rasterizer.py:386-575 (render_backward: add.at merge +
 *                         _geometry_backward)
 *
 * Numerics: compiled with -ffp-contract=off; fma() is used exactly where the
 * reference's numpy kernels fuse (OpenBLAS (N,3)@(3,3) and batched 3x3 matmul),
 * and the einsum reductions are summed in numpy's order.  The blend loops use
 * libm exp and the reference's piecewise erf, so they reproduce the compiled
 * Cython core bit for bit.  Pinned against the reference's own outputs by the
 * golden fixtures in tests/golden/ (tests/test_oracle_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TILE 16

/* kernels.py:34-72 */
static const double ERF_A[8] = {
    1.12837916701112384e+00, -3.76126382909789891e-01, 1.12837808616513241e-01,
    -2.68653686626153521e-02, 5.22092079952539076e-03, -8.48317008549591932e-04,
    1.12635153599516605e-04, -9.67013017894719878e-06};
static const double ERF_B[12] = {
    9.83790458267390644e-01, 6.27110407795858915e-02, -1.06608717154423910e-01,
    9.99195736486563901e-02, -4.93967225258238121e-02, 3.61330218115488502e-03,
    1.11371212802822434e-02, -6.26603860062541380e-03, 2.26018291841496854e-04,
    1.12165288159421766e-03, -3.25562507513530439e-04, -6.62957189382834869e-05};
static const double ERF_C[13] = {
    1.06604446603597580e-06, -7.64436843295190904e-06, 2.63691391003892384e-05,
    -5.80627943074455560e-05, 9.14210397499398350e-05, -1.09033436115601448e-04,
    1.00745516147541982e-04, -7.23964850830453220e-05, 4.14900304640991566e-05,
    -1.92305757609595023e-05, 5.10217603715594495e-06, 1.07793806577579218e-06,
    -9.03744268830116947e-07};

static const double INV_SQRT_PI = 0.5641895835477563;
static const double TERMINATION_T = 1e-4;
static const double WEIGHT_CLAMP = 0.99;

/* _blend_cy.pyx:40-63 */
double oracle_erf(double z) {
  double az = fabs(z), acc, t;
  int i;
  if (az < 1.0) {
    t = az * az;
    acc = ERF_A[7];
    for (i = 6; i >= 0; --i) acc = acc * t + ERF_A[i];
    acc = az * acc;
  } else if (az < 2.4) {
    t = az - 1.7;
    acc = ERF_B[11];
    for (i = 10; i >= 0; --i) acc = acc * t + ERF_B[i];
  } else if (az < 4.5) {
    t = az - 3.45;
    acc = ERF_C[12];
    for (i = 11; i >= 0; --i) acc = acc * t + ERF_C[i];
    acc = 1.0 - acc;
  } else {
    acc = 1.0;
  }
  return z < 0.0 ? -acc : acc;
}

static double sgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

static int resolve_threads(int threads) {
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#endif
  return threads > 0 ? threads : 1;
}

/* ------------------------------------------------------------------------- */
/* Blend core: one tile at a time, same recurrence and order as _blend_cy.   */
/* ------------------------------------------------------------------------- */

typedef struct {
  const double* packed; /* (M,13) */
  const int8_t* mode;
  const int32_t* pair_splat;
  const int64_t* tile_starts;
  int height, width, tiles_x;
  const double* bg;
} blend_in;

static void forward_one_tile(const blend_in* in, int tile, double* color, double* alpha,
                             double* depth, double* trans, int32_t* terminal) {
  double px[256], py[256], T[256], ar[256], ag[256], ab[256], dep[256];
  int cnt[256];
  signed char alive[256];
  const int ty = tile / in->tiles_x, tx = tile - ty * in->tiles_x;
  const int r0 = ty * TILE, c0 = tx * TILE;
  const int r1 = r0 + TILE < in->height ? r0 + TILE : in->height;
  const int c1 = c0 + TILE < in->width ? c0 + TILE : in->width;
  int npx = 0;
  for (int row = r0; row < r1; ++row)
    for (int col = c0; col < c1; ++col, ++npx) {
      px[npx] = col + 0.5;
      py[npx] = row + 0.5;
      T[npx] = 1.0;
      ar[npx] = ag[npx] = ab[npx] = dep[npx] = 0.0;
      cnt[npx] = 0;
      alive[npx] = 1;
    }
  int n_alive = npx;
  for (int64_t k = in->tile_starts[tile]; k < in->tile_starts[tile + 1]; ++k) {
    if (n_alive == 0) break;
    const double* s = in->packed + 13 * (int64_t)in->pair_splat[k];
    const int md = in->mode[in->pair_splat[k]];
    for (int p = 0; p < npx; ++p) {
      if (!alive[p]) continue;
      const double dx = px[p] - s[0], dy = py[p] - s[1];
      const double g = exp(-0.5 * (s[2] * dx * dx + s[4] * dy * dy) - s[3] * dx * dy);
      double e;
      if (md == 0)
        e = oracle_erf(s[5] * dx + s[6] * dy);
      else if (md == 1)
        e = sgn(s[5] * dx + s[6] * dy);
      else
        e = 0.0;
      double w = (s[7] + s[8] * e) * g;
      if (w > WEIGHT_CLAMP) w = WEIGHT_CLAMP;
      const double tn = T[p] * (1.0 - w);
      if (tn < TERMINATION_T) {
        alive[p] = 0;
        --n_alive;
        continue;
      }
      const double wt = w * T[p];
      ar[p] += wt * s[9];
      ag[p] += wt * s[10];
      ab[p] += wt * s[11];
      dep[p] += wt * s[12];
      cnt[p] += 1;
      T[p] = tn;
    }
  }
  npx = 0;
  for (int row = r0; row < r1; ++row)
    for (int col = c0; col < c1; ++col, ++npx) {
      const int64_t q = (int64_t)row * in->width + col;
      color[3 * q + 0] = ar[npx] + T[npx] * in->bg[0];
      color[3 * q + 1] = ag[npx] + T[npx] * in->bg[1];
      color[3 * q + 2] = ab[npx] + T[npx] * in->bg[2];
      alpha[q] = 1.0 - T[npx];
      depth[q] = dep[npx];
      trans[q] = T[npx];
      terminal[q] = cnt[npx];
    }
}

static void backward_one_tile(const blend_in* in, int tile, const double* d_color,
                              const double* trans, const int32_t* terminal, double* pair_grads) {
  double px[256], py[256], T[256], sr[256], sg_[256], sb[256], dr[256], dg[256], db[256];
  int cnt[256];
  const int64_t k0 = in->tile_starts[tile], k1 = in->tile_starts[tile + 1];
  if (k0 == k1) return;
  const int ty = tile / in->tiles_x, tx = tile - ty * in->tiles_x;
  const int r0 = ty * TILE, c0 = tx * TILE;
  const int r1 = r0 + TILE < in->height ? r0 + TILE : in->height;
  const int c1 = c0 + TILE < in->width ? c0 + TILE : in->width;
  int npx = 0, max_cnt = 0;
  for (int row = r0; row < r1; ++row)
    for (int col = c0; col < c1; ++col, ++npx) {
      const int64_t q = (int64_t)row * in->width + col;
      px[npx] = col + 0.5;
      py[npx] = row + 0.5;
      cnt[npx] = terminal[q];
      if (cnt[npx] > max_cnt) max_cnt = cnt[npx];
      T[npx] = trans[q];
      sr[npx] = T[npx] * in->bg[0];
      sg_[npx] = T[npx] * in->bg[1];
      sb[npx] = T[npx] * in->bg[2];
      dr[npx] = d_color[3 * q];
      dg[npx] = d_color[3 * q + 1];
      db[npx] = d_color[3 * q + 2];
    }
  for (int64_t pos = max_cnt - 1; pos >= 0; --pos) {
    const int64_t k = k0 + pos;
    const double* s = in->packed + 13 * (int64_t)in->pair_splat[k];
    const int md = in->mode[in->pair_splat[k]];
    double a[12] = {0};
    for (int p = 0; p < npx; ++p) {
      if (pos >= cnt[p]) continue;
      const double dx = px[p] - s[0], dy = py[p] - s[1];
      const double g = exp(-0.5 * (s[2] * dx * dx + s[4] * dy * dy) - s[3] * dx * dy);
      double e;
      if (md == 0)
        e = oracle_erf(s[5] * dx + s[6] * dy);
      else if (md == 1)
        e = sgn(s[5] * dx + s[6] * dy);
      else
        e = 0.0;
      const double w_raw = (s[7] + s[8] * e) * g;
      const double w = w_raw > WEIGHT_CLAMP ? WEIGHT_CLAMP : w_raw;
      const double om = 1.0 - w;
      const double tp = T[p] / om;
      const double wt = w * tp;
      a[9] += dr[p] * wt;
      a[10] += dg[p] * wt;
      a[11] += db[p] * wt;
      if (w_raw <= WEIGHT_CLAMP) {
        const double d_w = dr[p] * (tp * s[9] - sr[p] / om) + dg[p] * (tp * s[10] - sg_[p] / om) +
                           db[p] * (tp * s[11] - sb[p] / om);
        const double d_g = d_w * (s[7] + s[8] * e);
        const double d_pow = d_g * g;
        a[2] += d_pow * (-0.5) * dx * dx;
        a[3] += d_pow * (-dx * dy);
        a[4] += d_pow * (-0.5) * dy * dy;
        a[7] += d_w * g;
        a[8] += d_w * e * g;
        double ddx = d_pow * (-(s[2] * dx + s[3] * dy));
        double ddy = d_pow * (-(s[4] * dy + s[3] * dx));
        if (md == 0) {
          const double z = s[5] * dx + s[6] * dy;
          const double d_e = d_w * s[8] * g;
          const double d_z = d_e * 2.0 * INV_SQRT_PI * exp(-z * z);
          a[5] += d_z * dx;
          a[6] += d_z * dy;
          ddx += d_z * s[5];
          ddy += d_z * s[6];
        }
        a[0] -= ddx;
        a[1] -= ddy;
      }
      sr[p] += wt * s[9];
      sg_[p] += wt * s[10];
      sb[p] += wt * s[11];
      T[p] = tp;
    }
    for (int c = 0; c < 12; ++c) pair_grads[12 * k + c] += a[c];
  }
}

void oracle_forward_tiles(const double* packed, const int8_t* mode, const int32_t* pair_splat,
                          const int64_t* tile_starts, int height, int width, int tiles_x,
                          const double* bg, double* color, double* alpha, double* depth,
                          double* trans, int32_t* terminal, int tile_lo, int tile_hi,
                          int threads) {
  blend_in in = {packed, mode, pair_splat, tile_starts, height, width, tiles_x, bg};
  threads = resolve_threads(threads);
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads)
  for (int t = tile_lo; t < tile_hi; ++t) forward_one_tile(&in, t, color, alpha, depth, trans, terminal);
}

void oracle_backward_tiles(const double* packed, const int8_t* mode, const int32_t* pair_splat,
                           const int64_t* tile_starts, int height, int width, int tiles_x,
                           const double* bg, const double* d_color, const double* trans,
                           const int32_t* terminal, double* pair_grads, int tile_lo, int tile_hi,
                           int threads) {
  blend_in in = {packed, mode, pair_splat, tile_starts, height, width, tiles_x, bg};
  threads = resolve_threads(threads);
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads)
  for (int t = tile_lo; t < tile_hi; ++t)
    backward_one_tile(&in, t, d_color, trans, terminal, pair_grads);
}

/* ------------------------------------------------------------------------- */
/* prepare                                                                   */
/* ------------------------------------------------------------------------- */

typedef struct {
  double R[9], tr[3], center[3];
  double fx, fy, cx, cy, near_clip;
  int width, height;
} cam_t;

typedef struct {
  const double *mu, *ls, *rot, *sh, *nrm, *ra, *rb;
  int64_t n;
  int deg, K;
} scene_t;

/* every FP64 quantity prepare() saves in FrameGeometry (rasterizer.py:108-147) */
typedef struct {
  double t[3], qu[4], qnorm, R[9], s[3], cov[9];
  double ccam[9], J[9], cray[9], mux, muy, a, b, c, det, radius;
  int64_t x0, x1, y0, y1;
  double L[9];
  int bad, mode;
  double v00, v10, v11, nnorm, nu[3], hc[3], hr[3], y[3], ynorm, nray[3];
  double a1, a2, c1, c2, za, zb;
  double vdir[3], vdist, basis[16], rgbu[3];
} splat_t;

static int64_t f2i(double x) {
  if (!(x > -9.2233720368547758e18 && x < 9.2233720368547758e18)) return INT64_MIN;
  return (int64_t)x;
}

static double sigmoid(double x) { return x >= 0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x)); }

/* sh.py:32-61 */
static void sh_basis(const double d[3], int deg, double* o) {
  const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
  const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                        -1.0925484305920792, 0.5462742152960396};
  const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                        0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                        -0.5900435899266435};
  const double x = d[0], y = d[1], z = d[2];
  o[0] = C0;
  if (deg < 1) return;
  o[1] = -C1 * y;
  o[2] = C1 * z;
  o[3] = -C1 * x;
  if (deg < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  o[4] = C2[0] * x * y;
  o[5] = C2[1] * y * z;
  o[6] = C2[2] * (2.0 * zz - xx - yy);
  o[7] = C2[3] * x * z;
  o[8] = C2[4] * (xx - yy);
  if (deg < 3) return;
  o[9] = C3[0] * y * (3.0 * xx - yy);
  o[10] = C3[1] * x * y * z;
  o[11] = C3[2] * y * (4.0 * zz - xx - yy);
  o[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  o[13] = C3[4] * x * (4.0 * zz - xx - yy);
  o[14] = C3[5] * z * (xx - yy);
  o[15] = C3[6] * x * (xx - 3.0 * yy);
}

/* sh.py:64-98, g is (K,3) */
static void sh_basis_grad(const double d[3], int deg, double* g) {
  const double C1 = 0.4886025119029199;
  const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                        -1.0925484305920792, 0.5462742152960396};
  const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                        0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                        -0.5900435899266435};
  const double x = d[0], y = d[1], z = d[2];
  memset(g, 0, sizeof(double) * 48);
  if (deg >= 1) {
    g[1 * 3 + 1] = -C1;
    g[2 * 3 + 2] = C1;
    g[3 * 3 + 0] = -C1;
  }
  if (deg >= 2) {
    double r[5][3] = {{y, x, 0}, {0, z, y}, {-2 * x, -2 * y, 4 * z}, {z, 0, x}, {2 * x, -2 * y, 0}};
    for (int k = 0; k < 5; ++k)
      for (int j = 0; j < 3; ++j) g[(4 + k) * 3 + j] = C2[k] * r[k][j];
  }
  if (deg >= 3) {
    const double xx = x * x, yy = y * y, zz = z * z;
    double r[7][3] = {{6 * x * y, 3 * xx - 3 * yy, 0},
                      {y * z, x * z, x * y},
                      {-2 * x * y, 4 * zz - xx - 3 * yy, 8 * y * z},
                      {-6 * x * z, -6 * y * z, 6 * zz - 3 * xx - 3 * yy},
                      {4 * zz - 3 * xx - yy, -2 * x * y, 8 * x * z},
                      {2 * x * z, -2 * y * z, xx - yy},
                      {3 * xx - 3 * yy, -6 * x * y, 0}};
    for (int k = 0; k < 7; ++k)
      for (int j = 0; j < 3; ++j) g[(9 + k) * 3 + j] = C3[k] * r[k][j];
  }
}

/* Returns 1 when the primitive survives (in front, on screen, det > 0). */
static int splat_state(const scene_t* sc, const cam_t* cam, int kernel, int64_t i, splat_t* s) {
  const double* m = sc->mu + 3 * i;
  /* t_all = mu @ rot.T + t  (OpenBLAS: fma chain, then + t) */
  for (int a = 0; a < 3; ++a)
    s->t[a] = fma(m[2], cam->R[3 * a + 2], fma(m[1], cam->R[3 * a + 1], m[0] * cam->R[3 * a])) +
              cam->tr[a];
  const double* q = sc->rot + 4 * i;
  {
    double acc = 0.0;
    for (int k = 0; k < 4; ++k) acc += q[k] * q[k];
    s->qnorm = sqrt(acc);
  }
  for (int k = 0; k < 4; ++k) s->qu[k] = q[k] / s->qnorm;
  {
    /* quat_to_rot normalises again (geometry.py:35-38) */
    double acc = 0.0;
    for (int k = 0; k < 4; ++k) acc += s->qu[k] * s->qu[k];
    const double nn = sqrt(acc);
    const double w = s->qu[0] / nn, x = s->qu[1] / nn, y = s->qu[2] / nn, z = s->qu[3] / nn;
    double* R = s->R;
    R[0] = 1 - 2 * (y * y + z * z);
    R[1] = 2 * (x * y - w * z);
    R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);
    R[4] = 1 - 2 * (x * x + z * z);
    R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);
    R[7] = 2 * (y * z + w * x);
    R[8] = 1 - 2 * (x * x + y * y);
  }
  for (int k = 0; k < 3; ++k) s->s[k] = exp(sc->ls[3 * i + k]);
  double M[9];
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) M[3 * r + k] = s->R[3 * r + k] * s->s[k];
  for (int a = 0; a < 3; ++a)
    for (int d = 0; d < 3; ++d)
      s->cov[3 * a + d] =
          fma(M[3 * a + 2], M[3 * d + 2], fma(M[3 * a + 1], M[3 * d + 1], M[3 * a] * M[3 * d]));
  if (!(s->t[2] > cam->near_clip)) return 0;
  /* einsum "ab,nbc,dc->nad" and "nab,nbc,ndc->nad": b outer, c inner */
  for (int a = 0; a < 3; ++a)
    for (int d = 0; d < 3; ++d) {
      double acc = 0.0;
      for (int b = 0; b < 3; ++b)
        for (int c = 0; c < 3; ++c) acc += cam->R[3 * a + b] * s->cov[3 * b + c] * cam->R[3 * d + c];
      s->ccam[3 * a + d] = acc;
    }
  const double tx = s->t[0], ty = s->t[1], tz = s->t[2];
  const double invz = 1.0 / tz, ell = sqrt(tx * tx + ty * ty + tz * tz);
  double* J = s->J;
  J[0] = cam->fx * invz; J[1] = 0.0; J[2] = -cam->fx * tx * invz * invz;
  J[3] = 0.0; J[4] = cam->fy * invz; J[5] = -cam->fy * ty * invz * invz;
  J[6] = tx / ell; J[7] = ty / ell; J[8] = tz / ell;
  for (int a = 0; a < 3; ++a)
    for (int d = 0; d < 3; ++d) {
      double acc = 0.0;
      for (int b = 0; b < 3; ++b)
        for (int c = 0; c < 3; ++c) acc += J[3 * a + b] * s->ccam[3 * b + c] * J[3 * d + c];
      s->cray[3 * a + d] = acc;
    }
  s->mux = cam->fx * tx * invz + cam->cx;
  s->muy = cam->fy * ty * invz + cam->cy;
  s->a = s->cray[0] + 0.3;
  s->b = s->cray[1];
  s->c = s->cray[4] + 0.3;
  s->det = s->a * s->c - s->b * s->b;
  const double mid = 0.5 * (s->a + s->c);
  const double lam = mid + sqrt(fmax(mid * mid - s->det, 0.0));
  s->radius = 3.5 * sqrt(fmax(lam, 0.0));
  const int64_t x0 = f2i(ceil(s->mux - s->radius - 0.5)), x1 = f2i(floor(s->mux + s->radius - 0.5));
  const int64_t y0 = f2i(ceil(s->muy - s->radius - 0.5)), y1 = f2i(floor(s->muy + s->radius - 0.5));
  const int64_t W1 = cam->width - 1, H1 = cam->height - 1;
  if (!((x1 >= 0) && (x0 <= W1) && (y1 >= 0) && (y0 <= H1) && (x1 >= x0) && (y1 >= y0) &&
        (s->det > 0)))
    return 0;
  s->x0 = x0 < 0 ? 0 : (x0 > W1 ? W1 : x0);
  s->x1 = x1 < 0 ? 0 : (x1 > W1 ? W1 : x1);
  s->y0 = y0 < 0 ? 0 : (y0 > H1 ? H1 : y0);
  s->y1 = y1 < 0 ? 0 : (y1 > H1 ? H1 : y1);
  /* chol3_batch (geometry.py:126-160) */
  {
    const double* A = s->cray;
    const double d0 = A[0], l00 = sqrt(fmax(d0, 0.0));
    const double l10 = A[3] / l00, l20 = A[6] / l00;
    const double d1 = A[4] - l10 * l10, l11 = sqrt(fmax(d1, 0.0));
    const double l21 = (A[7] - l20 * l10) / l11;
    const double d2 = A[8] - l20 * l20 - l21 * l21, l22 = sqrt(fmax(d2, 0.0));
    const int finite = isfinite(l00) && isfinite(l11) && isfinite(l22);
    const double mn = fmin(fmin(l00, l11), l22), mx = fmax(fmax(l00, l11), l22);
    s->bad = (d0 <= 0.0) || (d1 <= 0.0) || (d2 <= 0.0) || !finite || (mn * 1e8 < mx);
    memset(s->L, 0, sizeof(s->L));
    if (s->bad) {
      s->L[0] = s->L[4] = s->L[8] = 1.0;
    } else {
      s->L[0] = l00; s->L[3] = l10; s->L[4] = l11; s->L[6] = l20; s->L[7] = l21; s->L[8] = l22;
    }
  }
  s->v00 = 1.0 / s->L[0];
  s->v11 = 1.0 / s->L[4];
  s->v10 = -s->L[3] * s->v00 * s->v11;
  const double* nr = sc->nrm + 3 * i;
  s->nnorm = sqrt(nr[0] * nr[0] + nr[1] * nr[1] + nr[2] * nr[2]);
  for (int k = 0; k < 3; ++k) s->nu[k] = nr[k] / s->nnorm;
  double hw[3];
  for (int a = 0; a < 3; ++a) /* einsum "nab,nb->na": (x0 + x2) + x1 */
    hw[a] = (s->cov[3 * a] * s->nu[0] + s->cov[3 * a + 2] * s->nu[2]) + s->cov[3 * a + 1] * s->nu[1];
  for (int a = 0; a < 3; ++a)
    s->hc[a] = fma(hw[2], cam->R[3 * a + 2], fma(hw[1], cam->R[3 * a + 1], hw[0] * cam->R[3 * a]));
  for (int a = 0; a < 3; ++a)
    s->hr[a] = (J[3 * a] * s->hc[0] + J[3 * a + 2] * s->hc[2]) + J[3 * a + 1] * s->hc[1];
  s->y[0] = s->hr[0] * s->v00;
  s->y[1] = (s->hr[1] - s->L[3] * s->y[0]) / s->L[4];
  s->y[2] = (s->hr[2] - s->L[6] * s->y[0] - s->L[7] * s->y[1]) / s->L[8];
  const double yn = sqrt(s->y[0] * s->y[0] + s->y[1] * s->y[1] + s->y[2] * s->y[2]);
  s->bad = s->bad || (yn < 1e-12) || !isfinite(yn);
  s->ynorm = s->bad ? 1.0 : yn;
  if (s->bad) {
    s->nray[0] = 0.0; s->nray[1] = 0.0; s->nray[2] = 1.0;
  } else {
    for (int k = 0; k < 3; ++k) s->nray[k] = s->y[k] / s->ynorm;
  }
  s->a1 = sigmoid(sc->ra[i]);
  s->a2 = sigmoid(sc->rb[i]);
  s->c1 = 0.5 * (s->a1 + s->a2);
  if (kernel == 1) {
    s->c2 = 0.0;
    s->mode = 2;
  } else {
    s->c2 = 0.5 * (s->a1 - s->a2);
    s->mode = fabs(s->nray[2]) < 1e-6 ? 1 : 0;
    if (s->bad) s->mode = 2;
  }
  s->za = s->zb = 0.0;
  if (s->mode == 0) {
    const double inv = 1.0 / (sqrt(2.0) * fabs(s->nray[2]));
    s->za = inv * (s->nray[0] * s->v00 + s->nray[1] * s->v10);
    s->zb = inv * (s->nray[1] * s->v11);
  } else if (s->mode == 1) {
    s->za = s->nray[0] * s->v00 + s->nray[1] * s->v10;
    s->zb = s->nray[1] * s->v11;
  }
  double vv[3];
  for (int k = 0; k < 3; ++k) vv[k] = m[k] - cam->center[k];
  s->vdist = sqrt(vv[0] * vv[0] + vv[1] * vv[1] + vv[2] * vv[2]);
  for (int k = 0; k < 3; ++k) s->vdir[k] = vv[k] / s->vdist;
  sh_basis(s->vdir, sc->deg, s->basis);
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0.0;
    for (int k = 0; k < sc->K; ++k) acc += s->basis[k] * sc->sh[(i * sc->K + k) * 3 + ch];
    s->rgbu[ch] = acc + 0.5;
  }
  return 1;
}

typedef struct {
  scene_t sc;
  cam_t cam;
  int kernel;
  int tiles_x, tiles_y;
  int64_t m, p;
  int64_t* valid;
  double* packed;
  int8_t* mode;
  int32_t* tile_rect;
  int32_t* pair_splat;
  int64_t* tile_starts;
  int32_t* radii; /* (n,) ceil(3.5 sqrt(lambda_max)) of rasterizer.py:194-200, 0 if culled */
} oracle_frame;

static const double* g_sort_depth;
static int cmp_depth_rank(const void* pa, const void* pb) {
  const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  const double da = g_sort_depth[a], db = g_sort_depth[b];
  if (da < db) return -1;
  if (da > db) return 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}

void oracle_frame_free(oracle_frame* f) {
  if (!f) return;
  free(f->valid);
  free(f->packed);
  free(f->mode);
  free(f->tile_rect);
  free(f->pair_splat);
  free(f->tile_starts);
  free(f->radii);
  free(f);
}

/* rasterizer.py:159-341.  Input arrays must outlive the frame (backward reuses them). */
oracle_frame* oracle_prepare(const double* mu, const double* log_scale, const double* rotation,
                             const double* sh_coeffs, const double* normal, const double* raw_a,
                             const double* raw_b, int64_t n, int sh_degree, const double* w2c,
                             double fx, double fy, double cx, double cy, double near_clip,
                             const double* center, int width, int height, int kernel,
                             int threads) {
  oracle_frame* f = (oracle_frame*)calloc(1, sizeof(oracle_frame));
  f->sc = (scene_t){mu, log_scale, rotation, sh_coeffs, normal, raw_a, raw_b, n, sh_degree,
                    (sh_degree + 1) * (sh_degree + 1)};
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) f->cam.R[3 * r + k] = w2c[4 * r + k];
    f->cam.tr[r] = w2c[4 * r + 3];
    f->cam.center[r] = center[r];
  }
  f->cam.fx = fx; f->cam.fy = fy; f->cam.cx = cx; f->cam.cy = cy;
  f->cam.near_clip = near_clip;
  f->cam.width = width;
  f->cam.height = height;
  f->kernel = kernel;
  f->tiles_x = (width + TILE - 1) / TILE;
  f->tiles_y = (height + TILE - 1) / TILE;
  threads = resolve_threads(threads);

  char* vis = (char*)malloc(n > 0 ? n : 1);
  double* rec = (double*)malloc(sizeof(double) * 13 * (n > 0 ? n : 1));
  int8_t* md = (int8_t*)malloc(n > 0 ? n : 1);
  int32_t* rect = (int32_t*)malloc(sizeof(int32_t) * 4 * (n > 0 ? n : 1));
  f->radii = (int32_t*)calloc(n > 0 ? n : 1, sizeof(int32_t));
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t i = 0; i < n; ++i) {
    splat_t s;
    vis[i] = (char)splat_state(&f->sc, &f->cam, kernel, i, &s);
    if (!vis[i]) continue;
    f->radii[i] = (int32_t)ceil(s.radius);
    double* r = rec + 13 * i;
    r[0] = s.mux; r[1] = s.muy;
    r[2] = s.c / s.det; r[3] = -s.b / s.det; r[4] = s.a / s.det;
    r[5] = s.za; r[6] = s.zb; r[7] = s.c1; r[8] = s.c2;
    for (int ch = 0; ch < 3; ++ch) r[9 + ch] = fmax(s.rgbu[ch], 0.0);
    r[12] = s.t[2];
    md[i] = (int8_t)s.mode;
    rect[4 * i + 0] = (int32_t)(s.x0 / TILE);
    rect[4 * i + 1] = (int32_t)(s.x1 / TILE);
    rect[4 * i + 2] = (int32_t)(s.y0 / TILE);
    rect[4 * i + 3] = (int32_t)(s.y1 / TILE);
  }
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) m += vis[i];
  f->m = m;
  f->valid = (int64_t*)malloc(sizeof(int64_t) * (m > 0 ? m : 1));
  f->packed = (double*)malloc(sizeof(double) * 13 * (m > 0 ? m : 1));
  f->mode = (int8_t*)malloc(m > 0 ? m : 1);
  f->tile_rect = (int32_t*)malloc(sizeof(int32_t) * 4 * (m > 0 ? m : 1));
  int64_t l = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!vis[i]) continue;
    f->valid[l] = i;
    memcpy(f->packed + 13 * l, rec + 13 * i, sizeof(double) * 13);
    f->mode[l] = md[i];
    memcpy(f->tile_rect + 4 * l, rect + 4 * i, sizeof(int32_t) * 4);
    ++l;
  }
  free(vis);
  free(rec);
  free(md);
  free(rect);
  /* pair order = np.lexsort((valid, depth, tile)): rank splats by (depth, index),
     then a stable bucket sort of the rank-ordered pairs by tile. */
  const int n_tiles = f->tiles_x * f->tiles_y;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (m > 0 ? m : 1));
  double* dep = (double*)malloc(sizeof(double) * (m > 0 ? m : 1));
  for (int64_t j = 0; j < m; ++j) {
    order[j] = j;
    dep[j] = f->packed[13 * j + 12];
  }
  g_sort_depth = dep;
  qsort(order, (size_t)m, sizeof(int64_t), cmp_depth_rank);
  int64_t* tcount = (int64_t*)calloc(n_tiles + 1, sizeof(int64_t));
  int64_t p = 0;
  for (int64_t j = 0; j < m; ++j) {
    const int32_t* rc = f->tile_rect + 4 * j;
    for (int ty = rc[2]; ty <= rc[3]; ++ty)
      for (int tx = rc[0]; tx <= rc[1]; ++tx) tcount[ty * f->tiles_x + tx]++;
    p += (int64_t)(rc[1] - rc[0] + 1) * (rc[3] - rc[2] + 1);
  }
  f->p = p;
  f->tile_starts = (int64_t*)malloc(sizeof(int64_t) * (n_tiles + 1));
  f->tile_starts[0] = 0;
  for (int t = 0; t < n_tiles; ++t) f->tile_starts[t + 1] = f->tile_starts[t] + tcount[t];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (n_tiles > 0 ? n_tiles : 1));
  memcpy(fill, f->tile_starts, sizeof(int64_t) * n_tiles);
  f->pair_splat = (int32_t*)malloc(sizeof(int32_t) * (p > 0 ? p : 1));
  for (int64_t r = 0; r < m; ++r) {
    const int64_t j = order[r];
    const int32_t* rc = f->tile_rect + 4 * j;
    for (int ty = rc[2]; ty <= rc[3]; ++ty)
      for (int tx = rc[0]; tx <= rc[1]; ++tx) f->pair_splat[fill[ty * f->tiles_x + tx]++] = (int32_t)j;
  }
  free(fill);
  free(tcount);
  free(order);
  free(dep);
  return f;
}

int64_t oracle_frame_m(const oracle_frame* f) { return f->m; }
int64_t oracle_frame_p(const oracle_frame* f) { return f->p; }

void oracle_frame_get(const oracle_frame* f, int64_t* valid, double* packed, int8_t* mode,
                      int32_t* tile_rect, int32_t* pair_splat, int64_t* tile_starts) {
  const int n_tiles = f->tiles_x * f->tiles_y;
  if (valid) memcpy(valid, f->valid, sizeof(int64_t) * f->m);
  if (packed) memcpy(packed, f->packed, sizeof(double) * 13 * f->m);
  if (mode) memcpy(mode, f->mode, f->m);
  if (tile_rect) memcpy(tile_rect, f->tile_rect, sizeof(int32_t) * 4 * f->m);
  if (pair_splat) memcpy(pair_splat, f->pair_splat, sizeof(int32_t) * f->p);
  if (tile_starts) memcpy(tile_starts, f->tile_starts, sizeof(int64_t) * (n_tiles + 1));
}

/* radii (N,): int32 ceil of the influence radius (rasterizer.py:194-200), 0 when culled */
void oracle_frame_radii(const oracle_frame* f, int32_t* radii) {
  memcpy(radii, f->radii, sizeof(int32_t) * f->sc.n);
}

/* render (rasterizer.py:351-383) over all tiles */
void oracle_forward(const oracle_frame* f, const double* bg, double* color, double* alpha,
                    double* depth, double* trans, int32_t* terminal, int threads) {
  oracle_forward_tiles(f->packed, f->mode, f->pair_splat, f->tile_starts, f->cam.height,
                       f->cam.width, f->tiles_x, bg, color, alpha, depth, trans, terminal, 0,
                       f->tiles_x * f->tiles_y, threads);
}

/* ------------------------------------------------------------------------- */
/* geometry backward (rasterizer.py:424-575), written with 3x3 helpers        */
/* ------------------------------------------------------------------------- */
static void mm(const double* A, const double* B, double* C) { /* C = A B */
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
  memcpy(C, t, sizeof(t));
}
static void tr3(const double* A, double* B) { /* B = A^T */
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[3 * i + j] = A[3 * j + i];
  memcpy(B, t, sizeof(t));
}
static void mtv(const double* A, const double* v, double* o) { /* o = A^T v */
  double t[3];
  for (int j = 0; j < 3; ++j) t[j] = A[j] * v[0] + A[3 + j] * v[1] + A[6 + j] * v[2];
  memcpy(o, t, sizeof(t));
}
static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void tri_inv(const double* L, double* I) { /* geometry.py:176-186 */
  const double a = L[0], b = L[4], c = L[8];
  memset(I, 0, 9 * sizeof(double));
  I[0] = 1.0 / a; I[4] = 1.0 / b; I[8] = 1.0 / c;
  I[3] = -L[3] / (a * b);
  I[7] = -L[7] / (b * c);
  I[6] = (L[3] * L[7] - L[6] * b) / (a * b * c);
}

typedef struct {
  double *d_mu, *d_log_scale, *d_rotation, *d_sh, *d_normal, *d_ra, *d_rb, *pos_grad_norm;
  int64_t* touch;
} grads_t;

static void geometry_backward_one(const oracle_frame* f, int64_t i, const double* g12,
                                  grads_t* out) {
  splat_t s;
  splat_state(&f->sc, &f->cam, f->kernel, i, &s);
  const int K = f->sc.K;
  const double *d_muhat = g12, *d_conic = g12 + 2;
  const double d_za = g12[5], d_zb = g12[6], d_c1 = g12[7], d_c2 = g12[8];
  const double* d_rgb = g12 + 9;
  const double d_a1 = 0.5 * (d_c1 + d_c2), d_a2 = 0.5 * (d_c1 - d_c2);
  out->d_ra[i] = d_a1 * s.a1 * (1.0 - s.a1);
  out->d_rb[i] = d_a2 * s.a2 * (1.0 - s.a2);
  const int m0 = s.mode == 0;
  const double n1 = s.nray[0], n2 = s.nray[1], n3 = s.nray[2];
  const double inv = m0 ? 1.0 / (sqrt(2.0) * fabs(n3)) : 0.0;
  const double za0 = m0 ? d_za : 0.0, zb0 = m0 ? d_zb : 0.0;
  const double d_inv = za0 * (n1 * s.v00 + n2 * s.v10) + zb0 * (n2 * s.v11);
  double dn[3] = {za0 * inv * s.v00, za0 * inv * s.v10 + zb0 * inv * s.v11,
                  m0 ? -d_inv * sgn(n3) / (sqrt(2.0) * n3 * n3) : 0.0};
  const double dv00 = za0 * inv * n1, dv10 = za0 * inv * n2, dv11 = zb0 * inv * n2;
  double dy[3];
  const double dd = dot3(dn, s.nray);
  for (int k = 0; k < 3; ++k) dy[k] = (dn[k] - dd * s.nray[k]) / s.ynorm;
  double Li[9], dh[3], dL[9];
  tri_inv(s.L, Li);
  mtv(Li, dy, dh);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) dL[3 * a + b] = -dh[a] * s.y[b];
  { /* d_L2 += -(V^T dV V^T) */
    double V[9] = {s.v00, 0, 0, s.v10, s.v11, 0, 0, 0, 0}, dV[9] = {dv00, 0, 0, dv10, dv11, 0, 0, 0, 0};
    double Vt[9], t[9];
    tr3(V, Vt);
    mm(Vt, dV, t);
    mm(t, Vt, t);
    dL[0] -= t[0]; dL[1] -= t[1]; dL[3] -= t[3]; dL[4] -= t[4];
  }
  dL[1] = dL[2] = dL[5] = 0.0;
  double dC[9];
  { /* chol3_vjp, geometry.py:163-173 */
    double Lt[9], P[9], phi[9] = {0}, S[9], Lit[9];
    tr3(s.L, Lt);
    mm(Lt, dL, P);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b <= a; ++b) phi[3 * a + b] = a == b ? 0.5 * P[3 * a + b] : P[3 * a + b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) S[3 * a + b] = phi[3 * a + b] + phi[3 * b + a];
    tr3(Li, Lit);
    mm(Lit, S, dC);
    mm(dC, Li, dC);
    for (int k = 0; k < 9; ++k) dC[k] *= 0.5;
  }
  {
    const double a = s.a, b = s.b, c = s.c, det = s.det, det2 = det * det;
    const double dca = d_conic[0], dcb = d_conic[1], dcc = d_conic[2];
    dC[0] += (-dca * c * c + dcb * b * c - dcc * b * b) / det2;
    dC[1] += (2.0 * dca * b * c - dcb * (det + 2.0 * b * b) + 2.0 * dcc * a * b) / det2;
    dC[4] += (-dca * b * b + dcb * a * b - dcc * a * a) / det2;
  }
  double dJ[9], dCc[9], dhc[3];
  {
    double S[9], Jt[9], t[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) S[3 * a + b] = dC[3 * a + b] + dC[3 * b + a];
    mm(S, s.J, t);
    mm(t, s.ccam, dJ);
    tr3(s.J, Jt);
    mm(Jt, dC, t);
    mm(t, s.J, dCc);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) dJ[3 * a + b] += dh[a] * s.hc[b];
    mtv(s.J, dh, dhc);
  }
  double dS[9], dhw[3], dnu[3];
  {
    double Rt[9], t[9];
    tr3(f->cam.R, Rt);
    mm(Rt, dCc, t);
    mm(t, f->cam.R, dS);
    mtv(f->cam.R, dhc, dhw);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) dS[3 * a + b] += dhw[a] * s.nu[b];
    mtv(s.cov, dhw, dnu);
  }
  double dt[3];
  {
    const double tx = s.t[0], ty = s.t[1], tz = s.t[2], invz = 1.0 / tz;
    const double fx = f->cam.fx, fy = f->cam.fy;
    dt[0] = d_muhat[0] * fx * invz;
    dt[1] = d_muhat[1] * fy * invz;
    dt[2] = -d_muhat[0] * fx * tx * invz * invz - d_muhat[1] * fy * ty * invz * invz;
    const double ell = sqrt(tx * tx + ty * ty + tz * tz);
    dt[2] += dJ[0] * (-fx * invz * invz);
    dt[0] += dJ[2] * (-fx * invz * invz);
    dt[2] += dJ[2] * (2.0 * fx * tx * invz * invz * invz);
    dt[2] += dJ[4] * (-fy * invz * invz);
    dt[1] += dJ[5] * (-fy * invz * invz);
    dt[2] += dJ[5] * (2.0 * fy * ty * invz * invz * invz);
    const double rh[3] = {tx / ell, ty / ell, tz / ell};
    const double dd3 = dot3(dJ + 6, rh);
    for (int k = 0; k < 3; ++k) dt[k] += (dJ[6 + k] - dd3 * rh[k]) / ell;
  }
  double dmu[3];
  mtv(f->cam.R, dt, dmu);
  {
    double pre[3];
    for (int ch = 0; ch < 3; ++ch) pre[ch] = s.rgbu[ch] > 0.0 ? d_rgb[ch] : 0.0;
    for (int k = 0; k < K; ++k)
      for (int ch = 0; ch < 3; ++ch) out->d_sh[(i * K + k) * 3 + ch] = s.basis[k] * pre[ch];
    if (f->sc.deg > 0) {
      double g[48], dd_[3] = {0, 0, 0};
      sh_basis_grad(s.vdir, f->sc.deg, g);
      for (int k = 0; k < K; ++k) {
        const double* c = f->sc.sh + (i * K + k) * 3;
        const double db = c[0] * pre[0] + c[1] * pre[1] + c[2] * pre[2];
        for (int d = 0; d < 3; ++d) dd_[d] += db * g[3 * k + d];
      }
      const double pr = dot3(dd_, s.vdir);
      for (int d = 0; d < 3; ++d) dmu[d] += (dd_[d] - pr * s.vdir[d]) / s.vdist;
    }
  }
  {
    double Mf[9], Ssym[9], dM[9], dR[9], ds[3] = {0, 0, 0};
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) Mf[3 * r + k] = s.R[3 * r + k] * s.s[k];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) Ssym[3 * a + b] = dS[3 * a + b] + dS[3 * b + a];
    mm(Ssym, Mf, dM);
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) {
        dR[3 * r + k] = dM[3 * r + k] * s.s[k];
        ds[k] += dM[3 * r + k] * s.R[3 * r + k];
      }
    for (int k = 0; k < 3; ++k) out->d_log_scale[3 * i + k] = ds[k] * s.s[k];
    const double w = s.qu[0], x = s.qu[1], y = s.qu[2], z = s.qu[3];
    const double D[4][9] = {{0, -z, y, z, 0, -x, -y, x, 0},
                            {0, y, z, y, -2 * x, -w, z, w, -2 * x},
                            {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
                            {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
    double dq[4];
    for (int j = 0; j < 4; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 9; ++k) acc += 2 * D[j][k] * dR[k];
      dq[j] = acc;
    }
    const double pr = dq[0] * w + dq[1] * x + dq[2] * y + dq[3] * z;
    for (int j = 0; j < 4; ++j) out->d_rotation[4 * i + j] = (dq[j] - pr * s.qu[j]) / s.qnorm;
  }
  {
    const double pr = dot3(dnu, s.nu);
    for (int k = 0; k < 3; ++k) out->d_normal[3 * i + k] = (dnu[k] - pr * s.nu[k]) / s.nnorm;
  }
  for (int k = 0; k < 3; ++k) out->d_mu[3 * i + k] = dmu[k];
  out->pos_grad_norm[i] = sqrt(d_muhat[0] * d_muhat[0] + d_muhat[1] * d_muhat[1]);
  out->touch[i] = 1;
}

/* render_backward (rasterizer.py:386-421).  Outputs are zero-filled by the caller. */
void oracle_backward(const oracle_frame* f, const double* bg, const double* d_color,
                     const double* trans, const int32_t* terminal, double* d_mu,
                     double* d_log_scale, double* d_rotation, double* d_sh, double* d_normal,
                     double* d_ra, double* d_rb, double* pos_grad_norm, int64_t* touch,
                     double* merged_out, int threads) {
  threads = resolve_threads(threads);
  const int64_t p = f->p, m = f->m;
  double* rows = (double*)calloc((size_t)(p > 0 ? p : 1) * 12, sizeof(double));
  oracle_backward_tiles(f->packed, f->mode, f->pair_splat, f->tile_starts, f->cam.height,
                        f->cam.width, f->tiles_x, bg, d_color, trans, terminal, rows, 0,
                        f->tiles_x * f->tiles_y, threads);
  /* np.add.at(merged, pair_splat, pair_grads): per splat, in increasing k */
  int64_t* start = (int64_t*)calloc(m + 1, sizeof(int64_t));
  for (int64_t k = 0; k < p; ++k) start[f->pair_splat[k] + 1]++;
  for (int64_t j = 0; j < m; ++j) start[j + 1] += start[j];
  int64_t* byk = (int64_t*)malloc(sizeof(int64_t) * (p > 0 ? p : 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (m > 0 ? m : 1));
  memcpy(fill, start, sizeof(int64_t) * m);
  for (int64_t k = 0; k < p; ++k) byk[fill[f->pair_splat[k]]++] = k;
  double* merged = (double*)calloc((size_t)(m > 0 ? m : 1) * 12, sizeof(double));
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t j = 0; j < m; ++j)
    for (int64_t q = start[j]; q < start[j + 1]; ++q)
      for (int c = 0; c < 12; ++c) merged[12 * j + c] += rows[12 * byk[q] + c];
  grads_t out = {d_mu, d_log_scale, d_rotation, d_sh, d_normal, d_ra, d_rb, pos_grad_norm, touch};
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t j = 0; j < m; ++j) geometry_backward_one(f, f->valid[j], merged + 12 * j, &out);
  if (merged_out) memcpy(merged_out, merged, sizeof(double) * 12 * m);
  free(merged);
  free(fill);
  free(byk);
  free(start);
  free(rows);
}

/* ---- training loss, loss.py:1-106 ------------------------------------------
 * compute_loss / ssim_with_grad restated in plain C on float64 (H,W,C) images.
 * The blur is scipy.ndimage.correlate1d (scipy, the reference's dependency;
 * its NI_Correlate1D symmetric-kernel branch: centre tap, then the pairs
 * (i-r, i+r) ... (i-1, i+1) summed before scaling) with mode="constant",
 * cval 0, along axis 0 and then axis 1 (loss.py:29-32). */
static void loss_window(double w[11]) { /* loss.py:19-23 */
  for (int k = 0; k < 11; ++k) {
    const double t = (double)(k - 5) / 1.5;
    w[k] = exp(-0.5 * (t * t));
  }
  /* numpy pairwise-sum order for 11 elements */
  double s = ((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7]));
  s += w[8];
  s += w[9];
  s += w[10];
  for (int k = 0; k < 11; ++k) w[k] /= s;
}

static void corr1d(const double* in, double* out, int h, int wd, int axis, const double w[11]) {
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < wd; ++x) {
      const int64_t stride = axis == 0 ? wd : 1;
      const int pos = axis == 0 ? y : x, len = axis == 0 ? h : wd;
      const double* c = in + (int64_t)y * wd + x;
      double s = c[0] * w[5];
      for (int j = 5; j >= 1; --j) {
        const double lo = pos - j >= 0 ? c[-j * stride] : 0.0;
        const double hi = pos + j < len ? c[j * stride] : 0.0;
        s += (lo + hi) * w[5 - j];
      }
      out[(int64_t)y * wd + x] = s;
    }
}

static void filt(const double* in, double* out, double* tmp, int h, int wd, const double w[11]) {
  corr1d(in, tmp, h, wd, 0, w);
  corr1d(tmp, out, h, wd, 1, w);
}

/* out3 = [loss, l1, mean ssim]; grad = d loss / d a.  lambda 0 skips SSIM
 * (loss.py:97-99). */
void oracle_loss(const double* a, const double* b, int h, int wd, int ch, double lam,
                 double* out3, double* grad) {
  const int64_t hw = (int64_t)h * wd, n = hw * ch;
  double win[11];
  loss_window(win);
  double l1 = 0.0;
  for (int64_t i = 0; i < n; ++i) l1 += fabs(a[i] - b[i]);
  l1 /= (double)n;
  for (int64_t i = 0; i < n; ++i) grad[i] = (1.0 - lam) * (sgn(a[i] - b[i]) / (double)n);
  out3[1] = l1;
  out3[2] = 0.0;
  out3[0] = l1;
  if (lam == 0.0) return;
  double* buf = (double*)malloc(sizeof(double) * hw * 14);
  double *x = buf, *y = buf + hw, *t = buf + 2 * hw, *m1 = buf + 3 * hw, *m2 = buf + 4 * hw,
         *fxx = buf + 5 * hw, *fyy = buf + 6 * hw, *fxy = buf + 7 * hw, *p = buf + 8 * hw,
         *q = buf + 9 * hw, *r = buf + 10 * hw, *g1 = buf + 11 * hw, *g2 = buf + 12 * hw,
         *g3 = buf + 13 * hw;
  double total = 0.0;
  for (int c = 0; c < ch; ++c) {
    for (int64_t i = 0; i < hw; ++i) {
      x[i] = a[i * ch + c];
      y[i] = b[i * ch + c];
    }
    filt(x, m1, t, h, wd, win);
    filt(y, m2, t, h, wd, win);
    for (int64_t i = 0; i < hw; ++i) p[i] = x[i] * x[i];
    filt(p, fxx, t, h, wd, win);
    for (int64_t i = 0; i < hw; ++i) p[i] = y[i] * y[i];
    filt(p, fyy, t, h, wd, win);
    for (int64_t i = 0; i < hw; ++i) p[i] = x[i] * y[i];
    filt(p, fxy, t, h, wd, win);
    for (int64_t i = 0; i < hw; ++i) { /* loss.py:62-75 */
      const double s1 = fxx[i] - m1[i] * m1[i], s2 = fyy[i] - m2[i] * m2[i];
      const double s12 = fxy[i] - m1[i] * m2[i];
      const double a1 = 2.0 * m1[i] * m2[i] + 0.01 * 0.01, a2 = 2.0 * s12 + 0.03 * 0.03;
      const double b1 = m1[i] * m1[i] + m2[i] * m2[i] + 0.01 * 0.01, b2 = s1 + s2 + 0.03 * 0.03;
      total += (a1 * a2) / (b1 * b2);
      const double d_m1 =
          (2.0 * m2[i] * a2 / (b1 * b2) - 2.0 * m1[i] * a1 * a2 / (b1 * b1 * b2)) / (double)n;
      const double d_s1 = (-a1 * a2 / (b1 * b2 * b2)) / (double)n;
      const double d_s12 = (2.0 * a1 / (b1 * b2)) / (double)n;
      p[i] = d_m1 - 2.0 * m1[i] * d_s1 - m2[i] * d_s12;
      q[i] = d_s1;
      r[i] = d_s12;
    }
    filt(p, g1, t, h, wd, win);
    filt(q, g2, t, h, wd, win);
    filt(r, g3, t, h, wd, win);
    for (int64_t i = 0; i < hw; ++i) { /* loss.py:74-78, 103 */
      const double s_grad = g1[i] + 2.0 * x[i] * g2[i] + y[i] * g3[i];
      grad[i * ch + c] = grad[i * ch + c] - lam * s_grad;
    }
  }
  free(buf);
  const double s_val = total / (double)n;
  out3[2] = s_val;
  out3[0] = (1.0 - lam) * l1 + lam * (1.0 - s_val);
}
