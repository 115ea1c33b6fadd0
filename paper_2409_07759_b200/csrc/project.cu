// a-3 EWA projection (raster.py:76-173) and a-7 its backward chain
// (raster.py:249-348).  One thread per active Gaussian, fp64 throughout so
// the structural outputs (cull set, bbox, depth order) match the reference;
// the rasterizer record is rounded to fp32 once.
#include "ss_common.cuh"

#ifndef SS_PBWD_PDL
#define SS_PBWD_PDL 1
#endif

namespace ss {

struct CamK {
  int32_t width, height;
  double fx, fy, cx, cy;
  double R[3][3];
  double T[3];
};

static CamK to_camk(const ss_camera* c) {
  CamK k;
  k.width = c->width;
  k.height = c->height;
  k.fx = c->fx;
  k.fy = c->fy;
  k.cx = c->cx;
  k.cy = c->cy;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) k.R[i][j] = c->rot[3 * i + j];
    k.T[i] = c->trans[i];
  }
  return k;
}

// Everything the forward computes and the backward re-derives.
struct Proj {
  double t[3];
  double z, ux, uy;
  double qnorm, qn[4], rq[3][3], m3[3][3], sigma[3][3], mproj[2][3];
  double a, b, c;  // raw cov2d
  bool keep;
};

__device__ __forceinline__ void project_one(const CamK& cam, const Gauss64& g, Proj& p) {
  // raster.py:86  t = mean R^T + T
#pragma unroll
  for (int j = 0; j < 3; ++j)
    p.t[j] = dadd(dadd(dadd(dmul(g.mean[0], cam.R[j][0]), dmul(g.mean[1], cam.R[j][1])),
                       dmul(g.mean[2], cam.R[j][2])),
                  cam.T[j]);
  p.z = p.t[2];
  const bool in_front = p.z > kNearPlane;  // raster.py:88
  // raster.py:91-92
  p.ux = dadd(ddiv(dmul(cam.fx, p.t[0]), p.z), cam.cx);
  p.uy = dadd(ddiv(dmul(cam.fy, p.t[1]), p.z), cam.cy);
  // raster.py:94-98
  const double* q = g.quat;
  p.qnorm = sqrt(dadd(dadd(dadd(dmul(q[0], q[0]), dmul(q[1], q[1])), dmul(q[2], q[2])),
                      dmul(q[3], q[3])));
  const double qd = fmax(p.qnorm, 1e-12);
#pragma unroll
  for (int k = 0; k < 4; ++k) p.qn[k] = ddiv(q[k], qd);
  quat_to_rot(p.qn, p.rq);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) p.m3[a][b] = dmul(p.rq[a][b], g.scale[b]);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      p.sigma[a][c] = dadd(dadd(dmul(p.m3[a][0], p.m3[c][0]), dmul(p.m3[a][1], p.m3[c][1])),
                           dmul(p.m3[a][2], p.m3[c][2]));
  // raster.py:101-107  J (2x3) and M = J W
  const double z2 = dmul(p.z, p.z);
  double J[2][3] = {{ddiv(cam.fx, p.z), 0.0, ddiv(dmul(-cam.fx, p.t[0]), z2)},
                    {0.0, ddiv(cam.fy, p.z), ddiv(dmul(-cam.fy, p.t[1]), z2)}};
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      p.mproj[a][c] = dadd(dadd(dmul(J[a][0], cam.R[0][c]), dmul(J[a][1], cam.R[1][c])),
                           dmul(J[a][2], cam.R[2][c]));
  // raster.py:108  cov2d = M Sigma M^T
  double cov[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          acc = dadd(acc, dmul(dmul(p.mproj[a][b], p.sigma[b][c]), p.mproj[d][c]));
      cov[a][d] = acc;
    }
  p.a = cov[0][0];
  p.b = cov[0][1];
  p.c = cov[1][1];
  // raster.py:114-124  3-sigma cull on the raw covariance
  const double mid = dmul(0.5, dadd(p.a, p.c));
  const double disc =
      sqrt(fmax(dsub(dmul(mid, mid), dsub(dmul(p.a, p.c), dmul(p.b, p.b))), 0.0));
  const double r3 = dmul(3.0, sqrt(fmax(dadd(mid, disc), 0.0)));
  const bool on_image = (dadd(p.ux, r3) >= 0.0) && (dsub(p.ux, r3) <= cam.width - 1.0) &&
                        (dadd(p.uy, r3) >= 0.0) && (dsub(p.uy, r3) <= cam.height - 1.0);
  p.keep = in_front && on_image;
}

// The backward's re-derivation of the projection quantities (raster.py:
// 86-111): the same formulas as project_one with ordinary (contractible)
// fp64 arithmetic and shared reciprocals in place of the IEEE-sequenced
// operations -- the gradient chain needs fp64 accuracy, not numpy's exact
// rounding (parity is 1e-3 of the max per group), and the exact divides
// with their slow-path branches dominated this kernel.
__device__ __forceinline__ void project_basis_fast(const CamK& cam, const Gauss64& g, Proj& p) {
#pragma unroll
  for (int j = 0; j < 3; ++j)
    p.t[j] = g.mean[0] * cam.R[j][0] + g.mean[1] * cam.R[j][1] + g.mean[2] * cam.R[j][2] + cam.T[j];
  p.z = p.t[2];
  const double* q = g.quat;
  p.qnorm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double iqd = 1.0 / fmax(p.qnorm, 1e-12);
#pragma unroll
  for (int k = 0; k < 4; ++k) p.qn[k] = q[k] * iqd;
  {
    const double w = p.qn[0], x = p.qn[1], y = p.qn[2], z = p.qn[3];
    p.rq[0][0] = 1.0 - 2.0 * (y * y + z * z);
    p.rq[0][1] = 2.0 * (x * y - w * z);
    p.rq[0][2] = 2.0 * (x * z + w * y);
    p.rq[1][0] = 2.0 * (x * y + w * z);
    p.rq[1][1] = 1.0 - 2.0 * (x * x + z * z);
    p.rq[1][2] = 2.0 * (y * z - w * x);
    p.rq[2][0] = 2.0 * (x * z - w * y);
    p.rq[2][1] = 2.0 * (y * z + w * x);
    p.rq[2][2] = 1.0 - 2.0 * (x * x + y * y);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) p.m3[a][b] = p.rq[a][b] * g.scale[b];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      p.sigma[a][c] = p.m3[a][0] * p.m3[c][0] + p.m3[a][1] * p.m3[c][1] + p.m3[a][2] * p.m3[c][2];
  const double iz = 1.0 / p.z, iz2 = iz * iz;
  const double J[2][3] = {{cam.fx * iz, 0.0, -cam.fx * p.t[0] * iz2},
                          {0.0, cam.fy * iz, -cam.fy * p.t[1] * iz2}};
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      p.mproj[a][c] = J[a][0] * cam.R[0][c] + J[a][1] * cam.R[1][c] + J[a][2] * cam.R[2][c];
  double ms[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      ms[a][c] = p.mproj[a][0] * p.sigma[0][c] + p.mproj[a][1] * p.sigma[1][c] +
                 p.mproj[a][2] * p.sigma[2][c];
  p.a = ms[0][0] * p.mproj[0][0] + ms[0][1] * p.mproj[0][1] + ms[0][2] * p.mproj[0][2];
  p.b = ms[0][0] * p.mproj[1][0] + ms[0][1] * p.mproj[1][1] + ms[0][2] * p.mproj[1][2];
  p.c = ms[1][0] * p.mproj[1][0] + ms[1][1] * p.mproj[1][1] + ms[1][2] * p.mproj[1][2];
}

// Everything a-4 / a-5 need from one kept splat: the fp32 binning geometry,
// the exact kept-tile count and mask of its bbox, the depth key and the
// rasterizer record (raster.cu: conic pre-scaled by kappa = -log2(e)/2 so
// alpha G = 2^(kappa m + log2 alpha); alpha floored at 2^-100).
__device__ __forceinline__ int write_record(int i, double ux, double uy, double i0, double i1,
                                             double i2, int x0, int x1, int y0, int y1,
                                             double opacity, const double* color, uint64_t key,
                                             float4* __restrict__ rec_a, float4* __restrict__ rec_b,
                                             float* __restrict__ rec_c,
                                             uint64_t* __restrict__ depth_key,
                                             int4* __restrict__ bbox, int32_t* __restrict__ n_tiles,
                                             float* __restrict__ geom,
                                             uint64_t* __restrict__ tile_mask, int lf) {
  bbox[i] = make_int4(x0, x1, y0, y1);
  // per-splat margin: maha <= 64 and, with the alpha floor, alpha G >= 2^lf
  const double M = cull_margin(opacity, lf);
  float gl[kGeom];
  make_geom(ux, uy, i0, i1, i2, fmax(M, 0.0), gl);
  float* gm = geom + (int64_t)i * kGeom;
#pragma unroll
  for (int c = 0; c < kGeom; ++c) gm[c] = gl[c];
  int nt = 0;
  uint64_t mask = 0;
  if (x1 > x0 && y1 > y0 && M > 0.0) {
    // tiles of the bbox that the m <= M ellipse actually reaches (one
    // x-interval per tile row); the first 64 (row-major in the bbox tile
    // rectangle) are also recorded as a bit mask for the binning
    const int4 bb = make_int4(x0, x1, y0, y1);
    const int tx0 = x0 / kTile, tx1 = (x1 - 1) / kTile + 1;
    const int ty0 = y0 / kTile, ty1 = (y1 - 1) / kTile + 1;
    const int w = tx1 - tx0;
    for (int ty = ty0; ty < ty1; ++ty) {
      float L, R;
      if (!row_span(gl, ty, bb, L, R)) continue;
      // col_meets(tx) = (bx(tx) >= L) && (ax(tx) <= R) with the tile's
      // clipped pixel-centre columns ax <= bx, both non-decreasing in tx
      // (rounded subtraction of a fixed u is monotone): the kept tiles of
      // the row are one run [a, b].  Its ends are estimated from L and R and
      // settled with the exact tests -- the same decisions as testing every
      // tile, without the per-tile loop.
      const float u = gl[0];
      const auto left_ok = [&](int tx) {  // bx(tx) >= L
        return fsr((float)min(tx * kTile + kTile - 1, bb.y - 1), u) >= L;
      };
      const auto right_ok = [&](int tx) {  // ax(tx) <= R
        return fsr((float)max(tx * kTile, bb.x), u) <= R;
      };
      int a = min(max((int)floorf((L + u - (float)(kTile - 1)) * (1.f / kTile)), tx0), tx1 - 1);
      while (a > tx0 && left_ok(a - 1)) --a;
      while (a < tx1 && !left_ok(a)) ++a;
      int b = min(max((int)floorf((R + u) * (1.f / kTile)), tx0), tx1 - 1);
      while (b < tx1 - 1 && right_ok(b + 1)) ++b;
      while (b >= tx0 && !right_ok(b)) --b;
      if (a > b) continue;
      nt += b - a + 1;
      const int ja = (ty - ty0) * w + (a - tx0);
      if (ja < 64) {
        const int nb = min(b - a + 1, 64 - ja);
        mask |= (nb >= 64 ? ~0ull : ((1ull << nb) - 1ull)) << ja;
      }
    }
  }
  tile_mask[i] = mask;
  n_tiles[i] = nt;
  depth_key[i] = key;
  const double kappa = -0.72134752044448170368;
  const double l2a = fmax(log2(opacity), -100.0);
  rec_a[i] = make_float4((float)ux, (float)uy, (float)(kappa * i0), (float)(kappa * i1));
  rec_b[i] = make_float4((float)(kappa * i2), (float)l2a, (float)color[0], (float)color[1]);
  rec_c[i] = (float)color[2];
  return nt;
}

__device__ __forceinline__ void write_culled(int i, float4* rec_a, float4* rec_b, float* rec_c,
                                             uint64_t* depth_key, int4* bbox, int32_t* n_tiles,
                                             uint64_t* tile_mask) {
  depth_key[i] = ~0ull;
  n_tiles[i] = 0;
  tile_mask[i] = 0;
  bbox[i] = make_int4(0, 0, 0, 0);
  rec_a[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  rec_b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  rec_c[i] = 0.f;
}

// One splat of the projection; returns its kept-tile count (0 when culled).
__device__ __forceinline__ int project_splat(const StoreView& store, const int32_t* __restrict__ rows,
                                             int i, const CamK& cam, float4* __restrict__ rec_a,
                                             float4* __restrict__ rec_b, float* __restrict__ rec_c,
                                             uint64_t* __restrict__ depth_key, int4* __restrict__ bbox,
                                             int32_t* __restrict__ n_tiles, float* __restrict__ geom,
                                             uint64_t* __restrict__ tile_mask, int lf) {
  const int32_t row = rows ? rows[i] : i;
  Gauss64 g;
  load_row(store, row, g);
  Proj p;
  project_one(cam, g, p);
  if (!p.keep) {
    write_culled(i, rec_a, rec_b, rec_c, depth_key, bbox, n_tiles, tile_mask);
    return 0;
  }
  // raster.py:139-150  dilation, conic, 8-sigma bbox of the dilated covariance
  const double ad = dadd(p.a, kDilation), cd = dadd(p.c, kDilation);
  const double det = dsub(dmul(ad, cd), dmul(p.b, p.b));
  const double i0 = ddiv(cd, det), i1 = ddiv(-p.b, det), i2 = ddiv(ad, det);
  const double mid_d = dmul(0.5, dadd(ad, cd));
  const double disc_d = sqrt(fmax(dsub(dmul(mid_d, mid_d), det), 0.0));
  const double r8 = dmul(8.0, sqrt(dadd(mid_d, disc_d)));
  const int x0 = (int)fmax(ceil(dsub(p.ux, r8)), 0.0);
  const int x1 = (int)fmin(dadd(floor(dadd(p.ux, r8)), 1.0), (double)cam.width);
  const int y0 = (int)fmax(ceil(dsub(p.uy, r8)), 0.0);
  const int y1 = (int)fmin(dadd(floor(dadd(p.uy, r8)), 1.0), (double)cam.height);
  // z > 0.01: the fp64 bits are monotone
  return write_record(i, p.ux, p.uy, i0, i1, i2, x0, x1, y0, y1, g.opacity, g.color,
                      (uint64_t)__double_as_longlong(p.z), rec_a, rec_b, rec_c, depth_key, bbox,
                      n_tiles, geom, tile_mask, lf);
}

// kp.out != nullptr: the kernel also sums the kept-tile counts -- per-CTA
// partial, one atomic add per CTA, and the last CTA (done counter) writes
// K = sum to kp.out and, with a system-scope store, (seq, K) to the host
// word the view driver polls (what a separate sum kernel did; integer sums,
// so the result does not depend on the CTA order), then re-arms both words.
__global__ void __launch_bounds__(128) project_fwd_kernel(StoreView store, const int32_t* __restrict__ rows, int32_t n,
                                   CamK cam, float4* __restrict__ rec_a,
                                   float4* __restrict__ rec_b, float* __restrict__ rec_c,
                                   uint64_t* __restrict__ depth_key, int4* __restrict__ bbox,
                                   int32_t* __restrict__ n_tiles, float* __restrict__ geom,
                                   uint64_t* __restrict__ tile_mask, int lf, KPublish kp) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int nt = 0;
  if (i < n)
    nt = project_splat(store, rows, i, cam, rec_a, rec_b, rec_c, depth_key, bbox, n_tiles, geom,
                       tile_mask, lf);
  if (!kp.out) return;
  __shared__ int s_part[4];
  __shared__ bool s_last;
  const int wsum = __reduce_add_sync(0xffffffffu, nt);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int bsum = s_part[0] + s_part[1] + s_part[2] + s_part[3];
    atomicAdd(&kp.acc_done[0], (unsigned int)bsum);
    __threadfence();
    s_last = atomicAdd(&kp.acc_done[1], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    const int32_t K = (int32_t)atomicAdd(&kp.acc_done[0], 0u);
    *kp.out = K;
    kp.acc_done[0] = 0u;  // re-armed before the host can see K and launch the next view
    kp.acc_done[1] = 0u;
    __threadfence();
    *(volatile unsigned long long*)kp.host =
        ((unsigned long long)kp.seq << 32) | (unsigned long long)(uint32_t)K;
    __threadfence_system();
  }
}

// _kernels.blend_forward's inputs (already projected 2D splats, the blend
// order given as a rank per splat, -1 = not blended): same records, bbox
// clipped to the image, depth key = rank.
__global__ void records2d_kernel(const double* __restrict__ mean2d, const double* __restrict__ inv2d,
                                 const double* __restrict__ alpha, const double* __restrict__ color,
                                 const int4* __restrict__ bbox_in, const int32_t* __restrict__ rank,
                                 int32_t n, int32_t width, int32_t height, float4* __restrict__ rec_a,
                                 float4* __restrict__ rec_b, float* __restrict__ rec_c,
                                 uint64_t* __restrict__ depth_key, int4* __restrict__ bbox,
                                 int32_t* __restrict__ n_tiles, float* __restrict__ geom,
                                 uint64_t* __restrict__ tile_mask, int lf) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (rank[i] < 0) {
    write_culled(i, rec_a, rec_b, rec_c, depth_key, bbox, n_tiles, tile_mask);
    return;
  }
  const int4 b = bbox_in[i];
  const int x0 = max(b.x, 0), x1 = min(b.y, width), y0 = max(b.z, 0), y1 = min(b.w, height);
  (void)write_record(i, mean2d[2 * i], mean2d[2 * i + 1], inv2d[3 * i], inv2d[3 * i + 1], inv2d[3 * i + 2],
               x0, max(x0, x1), y0, max(y0, y1), alpha[i], color + 3 * i,
               // rank as a positive double key (same form as fp64 z bits)
               (uint64_t)__double_as_longlong(1.0 + (double)rank[i] * 0x1p-22), rec_a,
               rec_b, rec_c, depth_key, bbox, n_tiles, geom, tile_mask, lf);
}

// Basis sums (raster.cu) -> _kernels.blend_backward's 2D gradients, added
// into the caller's arrays.  t = alpha' G d alpha' with alpha' the record's
// alpha (floored at 2^-100), so d alpha = W5 / alpha' (finite for alpha = 0).
__global__ void basis_to_2d_kernel(const float* __restrict__ g2d, const double* __restrict__ inv2d,
                                   const float4* __restrict__ rec_b, const uint64_t* __restrict__ key,
                                   int32_t n, double* __restrict__ g_mean2d,
                                   double* __restrict__ g_inv2d, double* __restrict__ g_alpha,
                                   double* __restrict__ g_color) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || key[i] == ~0ull) return;
  const float* w = g2d + (int64_t)i * SS_G2D_ROW;
  const double i0 = inv2d[3 * i], i1 = inv2d[3 * i + 1], i2 = inv2d[3 * i + 2];
  const double W0 = w[0], W1 = w[1];
  g_mean2d[2 * i] += i0 * W0 + i1 * W1;
  g_mean2d[2 * i + 1] += i1 * W0 + i2 * W1;
  g_inv2d[3 * i] += -0.5 * (double)w[2];
  g_inv2d[3 * i + 1] += -(double)w[3];
  g_inv2d[3 * i + 2] += -0.5 * (double)w[4];
  g_alpha[i] += (double)w[5] * exp2(-(double)rec_b[i].y);
  g_color[3 * i] += w[6];
  g_color[3 * i + 1] += w[7];
  g_color[3 * i + 2] += w[8];
}

#ifndef SS_PROJ_BWD_MINB
#define SS_PROJ_BWD_MINB 4  // 128 registers (146 uncapped): 33.7 -> 30.6 us at config 3
#endif
__global__ void __launch_bounds__(128, SS_PROJ_BWD_MINB) project_bwd_kernel(StoreView store, const int32_t* __restrict__ rows, int32_t n,
                                   CamK cam, const float* __restrict__ g2d,
                                   const uint64_t* __restrict__ depth_key,
                                   const uint8_t* __restrict__ mask, int64_t trainable_rows,
                                   float* __restrict__ grads) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (mask && !mask[i]) return;
  const int32_t row = rows ? rows[i] : i;
  if (row >= trainable_rows) return;
  static_assert(SS_G2D_ROW == 12, "three float4 per basis-sum row");
  // this splat's basis sums, loaded up front (48-B rows: three float4) so
  // their latency overlaps the parameter row's
  const float4* g4 = reinterpret_cast<const float4*>(g2d + (int64_t)i * SS_G2D_ROW);
  const float4 ga = g4[0], gb4 = g4[1], gc4 = g4[2];
  if (depth_key[i] == ~0ull) {  // culled: a zero gradient row (the step needs no pre-zeroed buffer)
    float2* out2 = reinterpret_cast<float2*>(grads + (int64_t)row * SS_GRAD_ROW);
#pragma unroll
    for (int c = 0; c < SS_GRAD_ROW / 2; ++c) out2[c] = make_float2(0.f, 0.f);
    return;
  }
  Gauss64 g;
  load_row(store, row, g);
  Proj p;
  project_basis_fast(cam, g, p);
  // g2d holds the rasterizer's basis sums over every (pixel, entry) of this
  // splat (raster.cu): W = (t dx, t dy, t dx^2, t dx dy, t dy^2, t, colour[3])
  // with t = alpha G d alpha'.  With dm = -t/2 and the conic (i0, i1, i2):
  //   d mean2d = (i0 W0 + i1 W1, i1 W0 + i2 W1),  d inv2d = -(W2/2, W3, W4/2),
  //   d alpha = W5 / alpha, so d logit = W5 (1 - alpha)   (raster.py:231-246)
  const float gg[9] = {ga.x, ga.y, ga.z, ga.w, gb4.x, gb4.y, gb4.z, gb4.w, gc4.x};
  const double ad = p.a + kDilation, cd = p.c + kDilation, b = p.b;
  const double det = ad * cd - b * b;
  const double idet = 1.0 / det;
  const double ci0 = cd * idet, ci1 = -b * idet, ci2 = ad * idet;
  const double W0 = gg[0], W1 = gg[1];
  const double gm2x = ci0 * W0 + ci1 * W1, gm2y = ci1 * W0 + ci2 * W1;
  const double gia = -0.5 * gg[2], gib = -(double)gg[3], gic = -0.5 * gg[4];
  const double g_alpha_x_alpha = gg[5];  // d alpha times alpha
  const double idet2 = idet * idet;
  // raster.py:262-266
  const double g_a = (gia * (-cd * cd) + gib * (b * cd) + gic * (-b * b)) * idet2;
  const double g_b = (gia * (2.0 * b * cd) + gib * (-det - 2.0 * b * b) + gic * (2.0 * ad * b)) * idet2;
  const double g_c = (gia * (-b * b) + gib * (ad * b) + gic * (-ad * ad)) * idet2;
  // raster.py:269-280
  double sm0[3], sm1[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    sm0[r] = p.sigma[r][0] * p.mproj[0][0] + p.sigma[r][1] * p.mproj[0][1] + p.sigma[r][2] * p.mproj[0][2];
    sm1[r] = p.sigma[r][0] * p.mproj[1][0] + p.sigma[r][1] * p.mproj[1][1] + p.sigma[r][2] * p.mproj[1][2];
  }
  double gm[2][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gm[0][k] = 2.0 * g_a * sm0[k] + g_b * sm1[k];
    gm[1][k] = g_b * sm0[k] + 2.0 * g_c * sm1[k];
  }
  double gs[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      gs[r][c] = g_a * p.mproj[0][r] * p.mproj[0][c] + g_b * p.mproj[0][r] * p.mproj[1][c] +
                 g_c * p.mproj[1][r] * p.mproj[1][c];
  // raster.py:283-300  through J entries and the projected centre to camera t
  double gj[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      gj[r][c] = gm[r][0] * cam.R[c][0] + gm[r][1] * cam.R[c][1] + gm[r][2] * cam.R[c][2];
  const double iz = 1.0 / p.z, iz2 = iz * iz, iz3 = iz2 * iz;
  const double xc = p.t[0], yc = p.t[1];
  double gt[3];
  gt[0] = gj[0][2] * (-cam.fx * iz2);
  gt[1] = gj[1][2] * (-cam.fy * iz2);
  gt[2] = gj[0][0] * (-cam.fx * iz2) + gj[1][1] * (-cam.fy * iz2) +
          gj[0][2] * (2.0 * cam.fx * xc * iz3) + gj[1][2] * (2.0 * cam.fy * yc * iz3);
  gt[0] += gm2x * cam.fx * iz;
  gt[1] += gm2y * cam.fy * iz;
  gt[2] += -gm2x * cam.fx * xc * iz2 - gm2y * cam.fy * yc * iz2;
  float* out = grads + (int64_t)row * SS_GRAD_ROW;
#pragma unroll
  for (int c = 0; c < 3; ++c)
    out[c] = (float)(gt[0] * cam.R[0][c] + gt[1] * cam.R[1][c] + gt[2] * cam.R[2][c]);
  // raster.py:303-306  Sigma = M3 M3^T, M3 = R diag(s)
  double gm3[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      gm3[r][k] = (gs[r][0] + gs[0][r]) * p.m3[0][k] + (gs[r][1] + gs[1][r]) * p.m3[1][k] +
                  (gs[r][2] + gs[2][r]) * p.m3[2][k];
  double gr[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double g_scale = gm3[0][k] * p.rq[0][k] + gm3[1][k] * p.rq[1][k] + gm3[2][k] * p.rq[2][k];
    out[7 + k] = (float)(g_scale * g.scale[k]);
#pragma unroll
    for (int r = 0; r < 3; ++r) gr[r][k] = gm3[r][k] * g.scale[k];
  }
  // raster.py:308-334  dR/dq, then through the normalization
  const double w = p.qn[0], x = p.qn[1], y = p.qn[2], zz = p.qn[3];
  const double dr[4][3][3] = {
      {{0.0, -zz, y}, {zz, 0.0, -x}, {-y, x, 0.0}},
      {{0.0, y, zz}, {y, -2 * x, -w}, {zz, w, -2 * x}},
      {{-2 * y, x, w}, {x, 0.0, zz}, {-w, zz, -2 * y}},
      {{-2 * zz, -w, x}, {w, -2 * zz, y}, {x, y, 0.0}}};
  double gqn[4];
#pragma unroll
  for (int qi = 0; qi < 4; ++qi) {
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k) acc += gr[r][k] * (2.0 * dr[qi][r][k]);
    gqn[qi] = acc;
  }
  const double dot = p.qn[0] * gqn[0] + p.qn[1] * gqn[1] + p.qn[2] * gqn[2] + p.qn[3] * gqn[3];
  const double iqn = 1.0 / p.qnorm;
#pragma unroll
  for (int qi = 0; qi < 4; ++qi) out[3 + qi] = (float)((gqn[qi] - p.qn[qi] * dot) * iqn);
  // raster.py:336-343
  out[10] = (float)(g_alpha_x_alpha * (1.0 - g.opacity));  // d alpha * alpha (1 - alpha)
  out[11] = gg[6];
  out[12] = gg[7];
  out[13] = gg[8];
}

__global__ void project_splats_kernel(StoreView store, const int32_t* __restrict__ rows,
                                      int32_t n, CamK cam, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Gauss64 g;
  load_row(store, rows ? rows[i] : i, g);
  Proj p;
  project_one(cam, g, p);
  double* o = out + (int64_t)i * 7;
  o[0] = p.ux;
  o[1] = p.uy;
  o[2] = p.a;
  o[3] = p.b;
  o[4] = p.c;
  o[5] = p.z;
  o[6] = p.keep ? 1.0 : 0.0;
}

__global__ void to_direct_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                 int64_t n) {
  pdl_wait();
  pdl_trigger();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* s = src + i * SS_ROW;
  double* d = dst + i * SS_ROW;
#pragma unroll
  for (int k = 0; k < 7; ++k) d[k] = s[k];
#pragma unroll
  for (int k = 7; k < 10; ++k) d[k] = exp(s[k]);
  d[10] = 1.0 / (1.0 + exp(-s[10]));
#pragma unroll
  for (int k = 11; k < 14; ++k) d[k] = s[k];
}

}  // namespace ss

using namespace ss;

int project_fwd_publish(const ss_store* store, const int32_t* rows, int32_t n,
                        const ss_camera* cam, void* rec_a, void* rec_b, float* rec_c,
                        uint64_t* depth_key, int32_t* bbox, int32_t* n_tiles, float* geom,
                        uint64_t* tile_mask, const KPublish* kp, cudaStream_t stream) {
  if (!store || !cam || n < 0) return set_error(SS_ERR_INVALID, "ss_project_fwd: bad arguments");
  if (cam->width <= 0 || cam->height <= 0 || !(cam->fx > 0) || !(cam->fy > 0))
    return set_error(SS_ERR_INVALID, "ss_project_fwd: bad camera");
  if (n == 0) return SS_OK;
  StoreView sv{store->opt, store->n_opt, store->mat};
  const KPublish none{nullptr, nullptr, nullptr, 0u};
  launch_k(project_fwd_kernel, grid_for(n, 128), 128, 0, stream,
      sv, rows, n, to_camk(cam), (float4*)rec_a, (float4*)rec_b, rec_c, depth_key, (int4*)bbox,
      n_tiles, geom, tile_mask, (int)alpha_floor_log2(), kp ? *kp : none);
  return check_launch("ss_project_fwd");
}

extern "C" int ss_project_fwd(const ss_store* store, const int32_t* rows, int32_t n,
                              const ss_camera* cam, void* rec_a, void* rec_b, float* rec_c,
                              uint64_t* depth_key, int32_t* bbox, int32_t* n_tiles,
                              float* geom, uint64_t* tile_mask, cudaStream_t stream) {
  return project_fwd_publish(store, rows, n, cam, rec_a, rec_b, rec_c, depth_key, bbox, n_tiles,
                             geom, tile_mask, nullptr, stream);
}

extern "C" int ss_records_2d(const ss_splats2d* sp, int32_t width, int32_t height, void* rec_a,
                             void* rec_b, float* rec_c, uint64_t* depth_key, int32_t* bbox,
                             int32_t* n_tiles, float* geom, uint64_t* tile_mask,
                             cudaStream_t stream) {
  if (!sp || sp->n < 0 || width <= 0 || height <= 0)
    return set_error(SS_ERR_INVALID, "ss_records_2d: bad arguments");
  if (sp->n == 0) return SS_OK;
  launch_k(records2d_kernel, grid_for(sp->n, 128), 128, 0, stream, 
      sp->mean2d, sp->inv2d, sp->alpha, sp->color, (const int4*)sp->bbox, sp->rank, sp->n, width,
      height, (float4*)rec_a, (float4*)rec_b, rec_c, depth_key, (int4*)bbox, n_tiles, geom,
      tile_mask, (int)alpha_floor_log2());
  return check_launch("ss_records_2d");
}

extern "C" int ss_basis_to_2d(const float* g2d, const ss_splats2d* sp, const void* rec_b,
                              const uint64_t* depth_key, double* g_mean2d, double* g_inv2d,
                              double* g_alpha, double* g_color, cudaStream_t stream) {
  if (!sp || sp->n < 0) return set_error(SS_ERR_INVALID, "ss_basis_to_2d: bad arguments");
  if (sp->n == 0) return SS_OK;
  launch_k(basis_to_2d_kernel, grid_for(sp->n, 128), 128, 0, stream, 
      g2d, sp->inv2d, (const float4*)rec_b, depth_key, sp->n, g_mean2d, g_inv2d, g_alpha, g_color);
  return check_launch("ss_basis_to_2d");
}

extern "C" int ss_project_bwd(const ss_store* store, const int32_t* rows, int32_t n,
                              const ss_camera* cam, const float* g2d, const uint64_t* depth_key,
                              const uint8_t* trainable_mask, int64_t trainable_rows,
                              float* grads, cudaStream_t stream) {
  if (!store || !cam || n < 0) return set_error(SS_ERR_INVALID, "ss_project_bwd: bad arguments");
  if (n == 0) return SS_OK;
  StoreView sv{store->opt, store->n_opt, store->mat};
  launch_kx(SS_PBWD_PDL, project_bwd_kernel, grid_for(n, 128), 128, 0, stream, sv, rows, n, to_camk(cam), g2d,
                                                            depth_key, trainable_mask,
                                                            trainable_rows, grads);
  return check_launch("ss_project_bwd");
}

extern "C" int ss_project_splats(const ss_store* store, const int32_t* rows, int32_t n,
                                 const ss_camera* cam, double* out, cudaStream_t stream) {
  if (!store || !cam || n < 0 || (n > 0 && !out))
    return set_error(SS_ERR_INVALID, "ss_project_splats: bad arguments");
  if (n == 0) return SS_OK;
  StoreView sv{store->opt, store->n_opt, store->mat};
  launch_k(project_splats_kernel, grid_for(n, 128), 128, 0, stream, sv, rows, n, to_camk(cam), out);
  return check_launch("ss_project_splats");
}

extern "C" int ss_to_direct(const double* src, double* dst, int64_t n, cudaStream_t stream) {
  if (n < 0) return set_error(SS_ERR_INVALID, "ss_to_direct: n < 0");
  if (n == 0) return SS_OK;
  launch_k(to_direct_kernel, grid_for(n, 256), 256, 0, stream, src, dst, n);
  return check_launch("ss_to_direct");
}
