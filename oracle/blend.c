/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Plain-C fp64 restatement of the
 * reference's two pixel loops, used as the parity checker for the CUDA
 * rasterizer and as the CPU baseline timed by bench.py (cpu_baseline /
 * --impl reference).  Nothing in the product path links or calls this.
 *
 * Follows /root/reference/pkg/src/splatstream/_kernels.py:
 *   blend_forward   _kernels.py:20-53   (front-to-back, global depth order,
 *                                         per-splat bbox test, maha > 64 skip,
 *                                         alpha clamp 0.999, break when T < 1e-4)
 *   blend_backward  _kernels.py:56-130  (replay + back-to-front suffix sweep)
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math) so
 * the arithmetic is the same IEEE sequence numba emits for the reference
 * (numba njit, fastmath off); exp() is glibc's, as numba links it.
 *
 * Threading: rows of the image are split into `nthreads` contiguous bands.
 * With nthreads == 1 the accumulation order is exactly the reference's
 * (row-major pixels, back-to-front per pixel).  With nthreads > 1 every
 * band accumulates into its own gradient buffers, reduced in band order
 * afterwards (deterministic for a fixed thread count).
 *
 * The "tiled" variants walk per-16x16-tile lists (the a-4 binning restated
 * in oracle/splat_oracle.py) instead of the global order.  They produce the
 * same per-pixel contributor sequence by construction and
 * are checked equal to the global-order loops in tests; they exist so the
 * oracle finishes in seconds at DyNeRF resolution.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ALPHA_MAX 0.999
#define T_MIN 1e-4
#define MAHA_MAX 64.0

static void forward_rows(int64_t iy0, int64_t iy1, const int64_t* order, int64_t nord,
                         const double* mean2d, const double* inv2d, const double* alpha,
                         const double* color, const int64_t* x0, const int64_t* x1,
                         const int64_t* y0, const int64_t* y1, int64_t width, double* img) {
  for (int64_t iy = iy0; iy < iy1; ++iy) {
    for (int64_t ix = 0; ix < width; ++ix) {
      double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
      for (int64_t k = 0; k < nord; ++k) {
        if (trans < T_MIN) break;
        int64_t s = order[k];
        if (ix < x0[s] || ix >= x1[s] || iy < y0[s] || iy >= y1[s]) continue;
        double dx = (double)ix - mean2d[2 * s];
        double dy = (double)iy - mean2d[2 * s + 1];
        double m = inv2d[3 * s] * dx * dx + 2.0 * inv2d[3 * s + 1] * dx * dy +
                   inv2d[3 * s + 2] * dy * dy;
        if (m > MAHA_MAX) continue;
        double ap = alpha[s] * exp(-0.5 * m);
        if (ap > ALPHA_MAX) ap = ALPHA_MAX;
        double w = ap * trans;
        c0 += color[3 * s] * w;
        c1 += color[3 * s + 1] * w;
        c2 += color[3 * s + 2] * w;
        trans *= 1.0 - ap;
      }
      double* o = img + 3 * (iy * width + ix);
      o[0] = c0;
      o[1] = c1;
      o[2] = c2;
    }
  }
}

void oracle_blend_forward(const int64_t* order, int64_t nord, const double* mean2d,
                          const double* inv2d, const double* alpha, const double* color,
                          const int64_t* x0, const int64_t* x1, const int64_t* y0,
                          const int64_t* y1, int64_t height, int64_t width, double* img,
                          int nthreads) {
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
  for (int64_t iy = 0; iy < height; ++iy)
    forward_rows(iy, iy + 1, order, nord, mean2d, inv2d, alpha, color, x0, x1, y0, y1, width,
                 img);
}

typedef struct {
  int64_t* idx;
  double* ap;
  double* t;
  double* g;
} pix_scratch;

/* One pixel of blend_backward (_kernels.py:70-130), walking `list` (global
 * order or a tile list) of length nlist. */
static inline void backward_pixel(int64_t ix, int64_t iy, const int64_t* list, int64_t nlist,
                                  const double* mean2d, const double* inv2d,
                                  const double* alpha, const double* color, const int64_t* x0,
                                  const int64_t* x1, const int64_t* y0, const int64_t* y1,
                                  const double* gp, pix_scratch* sc, double* g_mean2d,
                                  double* g_inv2d, double* g_alpha, double* g_color) {
  double gp0 = gp[0], gp1 = gp[1], gp2 = gp[2];
  double trans = 1.0;
  int64_t cnt = 0;
  for (int64_t k = 0; k < nlist; ++k) {
    if (trans < T_MIN) break;
    int64_t s = list[k];
    if (ix < x0[s] || ix >= x1[s] || iy < y0[s] || iy >= y1[s]) continue;
    double dx = (double)ix - mean2d[2 * s];
    double dy = (double)iy - mean2d[2 * s + 1];
    double m = inv2d[3 * s] * dx * dx + 2.0 * inv2d[3 * s + 1] * dx * dy +
               inv2d[3 * s + 2] * dy * dy;
    if (m > MAHA_MAX) continue;
    double gauss = exp(-0.5 * m);
    double ap = alpha[s] * gauss;
    if (ap > ALPHA_MAX) ap = ALPHA_MAX;
    sc->idx[cnt] = s;
    sc->ap[cnt] = ap;
    sc->t[cnt] = trans;
    sc->g[cnt] = gauss;
    cnt++;
    trans *= 1.0 - ap;
  }
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t j = cnt - 1; j >= 0; --j) {
    int64_t s = sc->idx[j];
    double ap = sc->ap[j], tj = sc->t[j], gauss = sc->g[j];
    double w = ap * tj;
    g_color[3 * s] += gp0 * w;
    g_color[3 * s + 1] += gp1 * w;
    g_color[3 * s + 2] += gp2 * w;
    double inv_rest = 1.0 / (1.0 - ap);
    double d_ap = gp0 * (color[3 * s] * tj - s0 * inv_rest) +
                  gp1 * (color[3 * s + 1] * tj - s1 * inv_rest) +
                  gp2 * (color[3 * s + 2] * tj - s2 * inv_rest);
    s0 += color[3 * s] * w;
    s1 += color[3 * s + 1] * w;
    s2 += color[3 * s + 2] * w;
    if (alpha[s] * gauss > ALPHA_MAX) continue;
    g_alpha[s] += d_ap * gauss;
    double d_m = -0.5 * gauss * alpha[s] * d_ap;
    double dx = (double)ix - mean2d[2 * s];
    double dy = (double)iy - mean2d[2 * s + 1];
    g_inv2d[3 * s] += d_m * dx * dx;
    g_inv2d[3 * s + 1] += d_m * 2.0 * dx * dy;
    g_inv2d[3 * s + 2] += d_m * dy * dy;
    g_mean2d[2 * s] -= d_m * 2.0 * (inv2d[3 * s] * dx + inv2d[3 * s + 1] * dy);
    g_mean2d[2 * s + 1] -= d_m * 2.0 * (inv2d[3 * s + 1] * dx + inv2d[3 * s + 2] * dy);
  }
}

/* Shared driver for the global-order and tiled backward: bands of rows,
 * per-band gradient buffers, fixed-order reduction. */
static void backward_driver(int tiled, const int64_t* order, int64_t nord,
                            const int64_t* tile_ranges, const int64_t* tile_vals,
                            int64_t tiles_x, const double* mean2d, const double* inv2d,
                            const double* alpha, const double* color, const int64_t* x0,
                            const int64_t* x1, const int64_t* y0, const int64_t* y1,
                            int64_t height, int64_t width, const double* grad_img,
                            double* g_mean2d, double* g_inv2d, double* g_alpha,
                            double* g_color, int64_t npts, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > height) nthreads = (int)(height > 0 ? height : 1);
  size_t per = (size_t)npts * 9;
  double* bufs = NULL;
  if (nthreads > 1) bufs = (double*)calloc(per * (size_t)(nthreads - 1), sizeof(double));
#pragma omp parallel num_threads(nthreads)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double *gm, *gi, *ga, *gc;
    if (tid == 0) {
      gm = g_mean2d; gi = g_inv2d; ga = g_alpha; gc = g_color;
    } else {
      double* b = bufs + per * (size_t)(tid - 1);
      gm = b; gi = b + 2 * npts; ga = b + 5 * npts; gc = b + 6 * npts;
    }
    int64_t cap = tiled ? 0 : nord;
    if (tiled) {
      int64_t ntiles = tiles_x * ((height + 15) / 16);
      for (int64_t t = 0; t < ntiles; ++t) {
        int64_t len = tile_ranges[2 * t + 1] - tile_ranges[2 * t];
        if (len > cap) cap = len;
      }
    }
    if (cap < 1) cap = 1;
    pix_scratch sc;
    sc.idx = (int64_t*)malloc(sizeof(int64_t) * cap);
    sc.ap = (double*)malloc(sizeof(double) * cap);
    sc.t = (double*)malloc(sizeof(double) * cap);
    sc.g = (double*)malloc(sizeof(double) * cap);
    int team = 1;
#ifdef _OPENMP
    team = omp_get_num_threads();
#endif
    int64_t band = (height + team - 1) / team;
    int64_t r0 = band * tid, r1 = r0 + band < height ? r0 + band : height;
    for (int64_t iy = r0; iy < r1; ++iy) {
      for (int64_t ix = 0; ix < width; ++ix) {
        const int64_t* list = order;
        int64_t nlist = nord;
        if (tiled) {
          int64_t t = (iy / 16) * tiles_x + ix / 16;
          list = tile_vals + tile_ranges[2 * t];
          nlist = tile_ranges[2 * t + 1] - tile_ranges[2 * t];
        }
        backward_pixel(ix, iy, list, nlist, mean2d, inv2d, alpha, color, x0, x1, y0, y1,
                       grad_img + 3 * (iy * width + ix), &sc, gm, gi, ga, gc);
      }
    }
    free(sc.idx); free(sc.ap); free(sc.t); free(sc.g);
  }
  for (int t = 1; t < nthreads; ++t) {
    double* b = bufs + per * (size_t)(t - 1);
    for (int64_t i = 0; i < 2 * npts; ++i) g_mean2d[i] += b[i];
    for (int64_t i = 0; i < 3 * npts; ++i) g_inv2d[i] += b[2 * npts + i];
    for (int64_t i = 0; i < npts; ++i) g_alpha[i] += b[5 * npts + i];
    for (int64_t i = 0; i < 3 * npts; ++i) g_color[i] += b[6 * npts + i];
  }
  free(bufs);
}

void oracle_blend_backward(const int64_t* order, int64_t nord, const double* mean2d,
                           const double* inv2d, const double* alpha, const double* color,
                           const int64_t* x0, const int64_t* x1, const int64_t* y0,
                           const int64_t* y1, int64_t height, int64_t width,
                           const double* grad_img, double* g_mean2d, double* g_inv2d,
                           double* g_alpha, double* g_color, int64_t npts, int nthreads) {
  backward_driver(0, order, nord, NULL, NULL, 0, mean2d, inv2d, alpha, color, x0, x1, y0, y1,
                  height, width, grad_img, g_mean2d, g_inv2d, g_alpha, g_color, npts,
                  nthreads);
}

/* Tiled forward: pixel (ix, iy) walks the list of its 16x16 tile.  Also
 * reports, per pixel, how many list entries it walked before its break
 * (or the whole list), the number of contributors, and the final T. */
void oracle_blend_forward_tiled(const int64_t* tile_ranges, const int64_t* tile_vals,
                                int64_t tiles_x, const double* mean2d, const double* inv2d,
                                const double* alpha, const double* color, const int64_t* x0,
                                const int64_t* x1, const int64_t* y0, const int64_t* y1,
                                int64_t height, int64_t width, double* img, int64_t* walked,
                                int64_t* contrib, double* t_final, int nthreads) {
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
  for (int64_t iy = 0; iy < height; ++iy) {
    for (int64_t ix = 0; ix < width; ++ix) {
      int64_t t = (iy / 16) * tiles_x + ix / 16;
      const int64_t* list = tile_vals + tile_ranges[2 * t];
      int64_t nlist = tile_ranges[2 * t + 1] - tile_ranges[2 * t];
      double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
      int64_t k = 0, nc = 0;
      for (; k < nlist; ++k) {
        if (trans < T_MIN) break;
        int64_t s = list[k];
        if (ix < x0[s] || ix >= x1[s] || iy < y0[s] || iy >= y1[s]) continue;
        double dx = (double)ix - mean2d[2 * s];
        double dy = (double)iy - mean2d[2 * s + 1];
        double m = inv2d[3 * s] * dx * dx + 2.0 * inv2d[3 * s + 1] * dx * dy +
                   inv2d[3 * s + 2] * dy * dy;
        if (m > MAHA_MAX) continue;
        double ap = alpha[s] * exp(-0.5 * m);
        if (ap > ALPHA_MAX) ap = ALPHA_MAX;
        double w = ap * trans;
        c0 += color[3 * s] * w;
        c1 += color[3 * s + 1] * w;
        c2 += color[3 * s + 2] * w;
        trans *= 1.0 - ap;
        nc++;
      }
      int64_t p = iy * width + ix;
      img[3 * p] = c0;
      img[3 * p + 1] = c1;
      img[3 * p + 2] = c2;
      if (walked) walked[p] = k;
      if (contrib) contrib[p] = nc;
      if (t_final) t_final[p] = trans;
    }
  }
}

void oracle_blend_backward_tiled(const int64_t* tile_ranges, const int64_t* tile_vals,
                                 int64_t tiles_x, const double* mean2d, const double* inv2d,
                                 const double* alpha, const double* color, const int64_t* x0,
                                 const int64_t* x1, const int64_t* y0, const int64_t* y1,
                                 int64_t height, int64_t width, const double* grad_img,
                                 double* g_mean2d, double* g_inv2d, double* g_alpha,
                                 double* g_color, int64_t npts, int nthreads) {
  backward_driver(1, NULL, 0, tile_ranges, tile_vals, tiles_x, mean2d, inv2d, alpha, color, x0,
                  x1, y0, y1, height, width, grad_img, g_mean2d, g_inv2d, g_alpha, g_color,
                  npts, nthreads);
}
