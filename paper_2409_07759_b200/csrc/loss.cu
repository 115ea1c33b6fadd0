// a-8 photometric loss: (1-w) L1 + w (1 - SSIM) with its exact image
// gradient (loss.py:29-60, 73-96).
//
// Two shared-memory tiled passes over 32x32 pixel tiles, one CTA per tile and
// channel:
//   pass 1: load x (prediction) and y (ground truth, u8 sRGB through the
//           256-entry linearisation LUT, raster.py:428-432) with a 5-px halo,
//           separable 11-tap blur of x, y, xx, xy, yy (zero padding), SSIM
//           map and its partials ds/dmu, ds/dmxx, ds/dmxy -> global scratch;
//           per-block fp64 sums of |x - y| and of the SSIM map.
//   pass 2: separable blur of the three partial maps, combine into
//           dL/dx = (1-w) sign(x-y)/N - w (B(ds_dmu) + 2x B(ds_dmxx) + y B(ds_dmxy))/N.
//   pass 3 (pass 2's first CTA): the per-block sums reduced in a fixed order.
//
// The blurs are register-blocked: a thread produces 8 consecutive outputs of
// a column (vertical pass) or 4 of a row (horizontal pass) from a sliding
// window held in registers, so each shared-memory value is loaded once per
// thread instead of once per tap; the 11 taps are compile-time immediates
// (full-rate FFMA with an immediate operand).
#include "ss_common.cuh"

#ifndef SS_SSIM_PDL
#define SS_SSIM_PDL 1
#endif

namespace ss {

constexpr int kLT = 32;               // output tile edge
constexpr int kHalo = 5;              // 11 taps
constexpr int kLR = kLT + 2 * kHalo;  // 42: loaded region edge
constexpr int kLP = kLR + 1;          // padded row pitch
constexpr int kLossThreads = 256;
constexpr int kVR = 8;                // vertical pass: outputs per thread
constexpr int kHC = 4;                // horizontal pass: outputs per thread

// loss.py:20-26 normalized 11-tap Gaussian, sigma 1.5 (fp64, rounded to fp32)
__device__ __forceinline__ constexpr float win(int t) {
  return t == 0 || t == 10 ? 0.001028380123898387f
       : t == 1 || t == 9  ? 0.0075987582094967365f
       : t == 2 || t == 8  ? 0.036000773310661316f
       : t == 3 || t == 7  ? 0.10936068743467331f
       : t == 4 || t == 6  ? 0.21300554275512695f
                           : 0.26601171493530273f;
}

struct LossArgs {
  const float* pred;
  const uint8_t* gt_u8;
  const float* lut;
  const float* gt_f32;
  int width, height;
  float* maps;        // 3 quantities x 3 channels x H x W
  double* partials;   // 2 per block
};

constexpr int kWarpsL = kLossThreads / 32;


// Separable 11-tap blur of one packed pair (A) and one scalar (B) quantity.
// Vertical pass: task = (column c of the 42-wide region, 8 output rows);
// out rows [r0, r0 + 8) from input rows [r0, r0 + 18).
template <typename Load>
__device__ __forceinline__ void vblur_pair(f2 (*outA)[kLP], float (*outB)[kLP], Load load) {
  for (int task = threadIdx.x; task < kLR * (kLT / kVR); task += kLossThreads) {
    const int c = task % kLR, r0 = (task / kLR) * kVR;
    f2 accA[kVR];
    float accB[kVR];
#pragma unroll
    for (int i = 0; i < kVR; ++i) {
      accA[i] = bc(0.f);
      accB[i] = 0.f;
    }
#pragma unroll
    for (int sidx = 0; sidx < kVR + 10; ++sidx) {
      f2 va;
      float vb;
      load(r0 + sidx, c, va, vb);
#pragma unroll
      for (int i = 0; i < kVR; ++i) {
        const int t = sidx - i;
        if (t >= 0 && t <= 10) {
          accA[i] = fma2(bc(win(t)), va, accA[i]);
          accB[i] = fmaf(win(t), vb, accB[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kVR; ++i) {
      outA[r0 + i][c] = accA[i];
      outB[r0 + i][c] = accB[i];
    }
  }
}

// Horizontal pass: res[i] = sum_t w_t v[r][c0 + i + t], i in [0, kHC)
__device__ __forceinline__ void hblur_pair(const f2 (*vA)[kLP], const float (*vB)[kLP], int r,
                                           int c0, f2 resA[kHC], float resB[kHC]) {
#pragma unroll
  for (int i = 0; i < kHC; ++i) {
    resA[i] = bc(0.f);
    resB[i] = 0.f;
  }
#pragma unroll
  for (int sidx = 0; sidx < kHC + 10; ++sidx) {
    const f2 a = vA[r][c0 + sidx];
    const float b = vB[r][c0 + sidx];
#pragma unroll
    for (int i = 0; i < kHC; ++i) {
      const int t = sidx - i;
      if (t >= 0 && t <= 10) {
        resA[i] = fma2(bc(win(t)), a, resA[i]);
        resB[i] = fmaf(win(t), b, resB[i]);
      }
    }
  }
}

// grid (tiles_x, tiles_y, 3): one CTA per 32x32 tile and channel.  The five
// blurred moments run as two packed pairs, (x, y) and (xx, yy), plus xy.
__global__ void __launch_bounds__(kLossThreads) ssim_fwd_kernel(LossArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ f2 s_xy[kLR][kLP];        // (x, y) with the 5-px halo
  __shared__ f2 s_v2[2][kLT][kLP];     // vertical pass: (mu_x, mu_y), (m_xx, m_yy)
  __shared__ float s_v1[kLT][kLP];     // vertical pass: m_xy
  __shared__ float s_lut[256];
  __shared__ double s_red[2][kWarpsL];
  const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT, ch = blockIdx.z;
  const int W = a.width, H = a.height;
  const int plane = W * H;  // 9 W H < 2^31 (checked on the host): 32-bit offsets
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (a.gt_u8)
    for (int i = threadIdx.x; i < 256; i += kLossThreads) s_lut[i] = a.lut[i];
  __syncthreads();
  // region rows by warp, columns by lane; every load of the thread is issued
  // before the first use (one memory round trip instead of one per row).
  // Offsets are hoisted: row k adds k * 8 rows to one base offset.
  constexpr int kRW = (kLR + kWarpsL - 1) / kWarpsL;  // rows per warp
  const int gx0 = x0 - kHalo + lane;
  const bool col_in[2] = {(unsigned)gx0 < (unsigned)W,
                          lane + 32 < kLR && (unsigned)(gx0 + 32) < (unsigned)W};
  const int gy0 = y0 - kHalo + warp;
  const int base = (gy0 * W + gx0) * 3 + ch;
  const int row_step = kWarpsL * 3 * W;
  float xv[kRW][2];
  uint32_t yv[kRW][2];  // u8: the byte or ~0u (outside); f32: the bits
#pragma unroll
  for (int k = 0; k < kRW; ++k) {
    const bool row_in = warp + kWarpsL * k < kLR && (unsigned)(gy0 + kWarpsL * k) < (unsigned)H;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const bool in = row_in && col_in[m];
      const int e = base + k * row_step + 96 * m;
      xv[k][m] = in ? a.pred[e] : 0.f;
      if (a.gt_u8)
        yv[k][m] = in ? (uint32_t)a.gt_u8[e] : ~0u;
      else
        yv[k][m] = in ? __float_as_uint(a.gt_f32[e]) : 0u;
    }
  }
#pragma unroll
  for (int k = 0; k < kRW; ++k) {
    const int r = warp + kWarpsL * k;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int q = lane + 32 * m;
      if (r < kLR && q < kLR) {
        const uint32_t yr = yv[k][m];
        const float y = a.gt_u8 ? (yr != ~0u ? s_lut[yr] : 0.f) : __uint_as_float(yr);
        s_xy[r][q] = pk2(xv[k][m], y);
      }
    }
  }
  __syncthreads();
  // vertical pass (axis 0, loss.py:31) of (x, y), xy and (xx, yy) in one
  // sweep over the region's columns
  for (int task = threadIdx.x; task < kLR * (kLT / kVR); task += kLossThreads) {
    const int c = task % kLR, r0 = (task / kLR) * kVR;
    f2 accA[kVR], accC[kVR];
    float accB[kVR];
#pragma unroll
    for (int i = 0; i < kVR; ++i) {
      accA[i] = accC[i] = bc(0.f);
      accB[i] = 0.f;
    }
#pragma unroll
    for (int sidx = 0; sidx < kVR + 10; ++sidx) {
      const f2 p = s_xy[r0 + sidx][c];
      const float xy = lo2(p) * hi2(p);
      const f2 sq = mul2(p, p);
#pragma unroll
      for (int i = 0; i < kVR; ++i) {
        const int t = sidx - i;
        if (t >= 0 && t <= 10) {
          accA[i] = fma2(bc(win(t)), p, accA[i]);
          accB[i] = fmaf(win(t), xy, accB[i]);
          accC[i] = fma2(bc(win(t)), sq, accC[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kVR; ++i) {
      s_v2[0][r0 + i][c] = accA[i];
      s_v1[r0 + i][c] = accB[i];
      s_v2[1][r0 + i][c] = accC[i];
    }
  }
  __syncthreads();
  // horizontal pass (axis 1, loss.py:32) + SSIM terms (loss.py:39-59)
  double l1 = 0.0, ss = 0.0;
  {
    const int r = threadIdx.x / (kLT / kHC), c0 = (threadIdx.x % (kLT / kHC)) * kHC;
    f2 mu[kHC], sq[kHC];
    float mxy[kHC];
    hblur_pair(s_v2[0], s_v1, r, c0, mu, mxy);
#pragma unroll
    for (int i = 0; i < kHC; ++i) sq[i] = bc(0.f);
#pragma unroll
    for (int sidx = 0; sidx < kHC + 10; ++sidx) {
      const f2 v = s_v2[1][r][c0 + sidx];
#pragma unroll
      for (int i = 0; i < kHC; ++i) {
        const int t = sidx - i;
        if (t >= 0 && t <= 10) sq[i] = fma2(bc(win(t)), v, sq[i]);
      }
    }
    const int gy = y0 + r;
#pragma unroll
    for (int i = 0; i < kHC; ++i) {
      const int gx = x0 + c0 + i;
      if (gy >= H || gx >= W) continue;
      const float mu_x = lo2(mu[i]), mu_y = hi2(mu[i]), mxx = lo2(sq[i]), myy = hi2(sq[i]);
      const float mxyv = mxy[i];
      const float C1 = 1e-4f, C2 = 9e-4f;
      const float sig_x = mxx - mu_x * mu_x;
      const float sig_y = myy - mu_y * mu_y;
      const float sig_xy = mxyv - mu_x * mu_y;
      const float a1 = 2.f * mu_x * mu_y + C1;
      const float a2 = 2.f * sig_xy + C2;
      const float b1 = mu_x * mu_x + mu_y * mu_y + C1;
      const float b2 = sig_x + sig_y + C2;
      const float inv_b2 = 1.f / b2;
      const float inv_den = inv_b2 / b1;  // 1 / (b1 b2)
      const float sv = (a1 * a2) * inv_den;
      const float ds_dmu = (2.f * mu_y * (a2 - a1) - 2.f * mu_x * sv * (b2 - b1)) * inv_den;
      const float ds_dmxx = -sv * inv_b2;
      const float ds_dmxy = 2.f * a1 * inv_den;
      const int pix = gy * W + gx;
      a.maps[(0 * 3 + ch) * plane + pix] = ds_dmu;
      a.maps[(1 * 3 + ch) * plane + pix] = ds_dmxx;
      a.maps[(2 * 3 + ch) * plane + pix] = ds_dmxy;
      ss += (double)sv;
      const f2 p = s_xy[r + kHalo][c0 + i + kHalo];
      l1 += (double)fabsf(lo2(p) - hi2(p));
    }
  }
  // block reduction of the two sums (fixed order -> deterministic)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if (lane == 0) {
    s_red[0][warp] = l1;
    s_red[1][warp] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int i = 0; i < kWarpsL; ++i) {
      t0 += s_red[0][i];
      t1 += s_red[1][i];
    }
    const int b = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    a.partials[2 * b] = t0;
    a.partials[2 * b + 1] = t1;
  }
}

// pass 2: blur of the partial maps as the pair (ds/dmu, ds/dmxx) + ds/dmxy
// Fixed-order sums of the forward's per-block (L1, SSIM) partials into out
// (one CTA; deterministic).
__device__ __forceinline__ void reduce_partials(const double* __restrict__ partials, int n_blocks,
                                                double* __restrict__ out) {
  __shared__ double s[2][kLossThreads / 32];
  double t0 = 0.0, t1 = 0.0;
  for (int i = threadIdx.x; i < n_blocks; i += blockDim.x) {
    t0 += partials[2 * i];
    t1 += partials[2 * i + 1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t0 += __shfl_xor_sync(0xffffffffu, t0, o);
    t1 += __shfl_xor_sync(0xffffffffu, t1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = t0;
    s[1][threadIdx.x >> 5] = t1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      x += s[0][i];
      y += s[1][i];
    }
    out[0] = x;
    out[1] = y;
  }
}

// pass 2 also holds pass 3: its first CTA reduces the forward's partials
// (complete once pdl_wait returns) before its own tile -- no separate
// one-CTA launch at the end of the loss.
__global__ void __launch_bounds__(kLossThreads) ssim_bwd_kernel(LossArgs a, float w_ssim,
                                                                 float* __restrict__ dimg,
                                                                 double* __restrict__ out_sums) {
  pdl_wait();
  pdl_trigger();
  if (out_sums && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
    reduce_partials(a.partials, gridDim.x * gridDim.y * gridDim.z, out_sums);
  __shared__ f2 s_m2[kLR][kLP];
  __shared__ float s_m1[kLR][kLP];
  __shared__ f2 s_v2[kLT][kLP];
  __shared__ float s_v1[kLT][kLP];
  __shared__ float s_lut[256];
  if (a.gt_u8)
    for (int i = threadIdx.x; i < 256; i += kLossThreads) s_lut[i] = a.lut[i];
  const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT, ch = blockIdx.z;
  const int W = a.width, H = a.height;
  const int plane = W * H;  // 9 W H < 2^31 (checked on the host)
  const float inv_n = 1.0f / (float)((double)plane * 3.0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* m0 = a.maps + (0 * 3 + ch) * plane;
  const float* m1 = a.maps + (1 * 3 + ch) * plane;
  const float* m2 = a.maps + (2 * 3 + ch) * plane;
  const int r = threadIdx.x / (kLT / kHC), c0 = (threadIdx.x % (kLT / kHC)) * kHC;
  const int gy = y0 + r;
  const int eo = (gy * W + x0 + c0) * 3 + ch;
  if ((W & 3) == 0) {
    // rows of 48 floats from x0 - 8 as 12 float4 (W % 4 == 0: a float4 is
    // wholly inside or outside the image; tile origins are multiples of 32),
    // every load of the thread issued before the first store.  Region
    // column j (x0 - 5 + j) is float 3 + j of the row.  The scalar path's
    // per-element address and bounds arithmetic was half the kernel.
    constexpr int kQ = 12, kItems = kLR * kQ;  // 504 float4 per map
    constexpr int kPer = (kItems + kLossThreads - 1) / kLossThreads;
    float4 u[kPer][3];
#pragma unroll
    for (int it = 0; it < kPer; ++it) {
      const int idx = threadIdx.x + it * kLossThreads;
      const int rr = idx / kQ, qq = idx - rr * kQ;
      const int gyy = y0 - kHalo + rr, gxx = x0 - 8 + 4 * qq;
      const bool in = idx < kItems && (unsigned)gyy < (unsigned)H && (unsigned)gxx < (unsigned)W;
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      const int e = gyy * W + gxx;
      u[it][0] = in ? *reinterpret_cast<const float4*>(m0 + e) : z;
      u[it][1] = in ? *reinterpret_cast<const float4*>(m1 + e) : z;
      u[it][2] = in ? *reinterpret_cast<const float4*>(m2 + e) : z;
    }
#pragma unroll
    for (int it = 0; it < kPer; ++it) {
      const int idx = threadIdx.x + it * kLossThreads;
      if (idx >= kItems) continue;
      const int rr = idx / kQ, qq = idx - rr * kQ;
      const float a0[4] = {u[it][0].x, u[it][0].y, u[it][0].z, u[it][0].w};
      const float a1[4] = {u[it][1].x, u[it][1].y, u[it][1].z, u[it][1].w};
      const float a2[4] = {u[it][2].x, u[it][2].y, u[it][2].z, u[it][2].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = 4 * qq + j - 3;
        if (col >= 0 && col < kLR) {
          s_m2[rr][col] = pk2(a0[j], a1[j]);
          s_m1[rr][col] = a2[j];
        }
      }
    }
  } else {
    constexpr int kRW = (kLR + kWarpsL - 1) / kWarpsL;  // rows per warp
    const int gx0 = x0 - kHalo + lane;
    const bool col_in[2] = {(unsigned)gx0 < (unsigned)W,
                            lane + 32 < kLR && (unsigned)(gx0 + 32) < (unsigned)W};
    const int gy0 = y0 - kHalo + warp;
    const int base = gy0 * W + gx0;
    float u[kRW][2][3];
#pragma unroll
    for (int k = 0; k < kRW; ++k) {
      const bool row_in = warp + kWarpsL * k < kLR && (unsigned)(gy0 + kWarpsL * k) < (unsigned)H;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const bool in = row_in && col_in[m];
        const int e = base + k * kWarpsL * W + 32 * m;
        u[k][m][0] = in ? m0[e] : 0.f;
        u[k][m][1] = in ? m1[e] : 0.f;
        u[k][m][2] = in ? m2[e] : 0.f;
      }
    }
#pragma unroll
    for (int k = 0; k < kRW; ++k) {
      const int rr = warp + kWarpsL * k;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int q = lane + 32 * m;
        if (rr < kLR && q < kLR) {
          s_m2[rr][q] = pk2(u[k][m][0], u[k][m][1]);
          s_m1[rr][q] = u[k][m][2];
        }
      }
    }
  }
  __syncthreads();
  vblur_pair(s_v2, s_v1, [&](int r, int c, f2& va, float& vb) {
    va = s_m2[r][c];
    vb = s_m1[r][c];
  });
  __syncthreads();
  f2 bl2[kHC];
  float bl1[kHC];
  // the outputs' x and y are loaded only now (loading them with the maps
  // costs 18 registers and one resident CTA per SM: measured slower)
  float xo[kHC];
  uint32_t yo[kHC];
#pragma unroll
  for (int i = 0; i < kHC; ++i) {
    const bool in = gy < H && x0 + c0 + i < W;
    xo[i] = in ? a.pred[eo + 3 * i] : 0.f;
    if (a.gt_u8)
      yo[i] = in ? (uint32_t)a.gt_u8[eo + 3 * i] : 0u;
    else
      yo[i] = in ? __float_as_uint(a.gt_f32[eo + 3 * i]) : 0u;
  }
  hblur_pair(s_v2, s_v1, r, c0, bl2, bl1);
#pragma unroll
  for (int i = 0; i < kHC; ++i) {
    if (gy >= H || x0 + c0 + i >= W) continue;
    const float x = xo[i];
    const float y = a.gt_u8 ? s_lut[yo[i]] : __uint_as_float(yo[i]);
    const float grad = (lo2(bl2[i]) + 2.f * x * hi2(bl2[i]) + y * bl1[i]) * inv_n;
    const float d = x - y;
    const float sgn = (d > 0.f) ? 1.f : ((d < 0.f) ? -1.f : 0.f);
    dimg[eo + 3 * i] = (1.f - w_ssim) * sgn * inv_n - w_ssim * grad;
  }
}

// loss.py:105-111 regularizer gradients and terms; one CTA, fixed-order sums
__global__ void __launch_bounds__(1024) reg_grads_kernel(const double* __restrict__ alpha,
                                                         const double* __restrict__ scales, int n,
                                                         double w_op, double w_sc,
                                                         double* __restrict__ reg_logit,
                                                         double* __restrict__ reg_log_scale,
                                                         double* __restrict__ terms) {
  pdl_wait();
  pdl_trigger();
  __shared__ double s[2][32];
  double ta = 0.0, ts = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = alpha[i];
    const double s0 = scales[3 * i], s1 = scales[3 * i + 1], s2 = scales[3 * i + 2];
    reg_logit[i] = w_op * a * (1.0 - a) / n;
    reg_log_scale[3 * i] = w_sc * s0 / n;
    reg_log_scale[3 * i + 1] = w_sc * s1 / n;
    reg_log_scale[3 * i + 2] = w_sc * s2 / n;
    ta += a;
    ts += (s0 + s1) + s2;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ta += __shfl_xor_sync(0xffffffffu, ta, o);
    ts += __shfl_xor_sync(0xffffffffu, ts, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = ta;
    s[1][threadIdx.x >> 5] = ts;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += s[0][w];
      b += s[1][w];
    }
    terms[0] = w_op * (a / n);
    terms[1] = w_sc * (b / n);
  }
}

}  // namespace ss

using namespace ss;

extern "C" int ss_reg_grads(const double* alpha, const double* scales, int32_t n, double w_op,
                            double w_sc, double* reg_logit, double* reg_log_scale, double* terms,
                            cudaStream_t stream) {
  if (n < 0 || !terms) return set_error(SS_ERR_INVALID, "ss_reg_grads: bad arguments");
  if (n == 0) {
    memzero(terms, 2 * sizeof(double), stream);
    return check_launch("ss_reg_grads");
  }
  launch_k(reg_grads_kernel, 1, 1024, 0, stream, alpha, scales, n, w_op, w_sc, reg_logit,
           reg_log_scale, terms);
  return check_launch("ss_reg_grads");
}

extern "C" size_t ss_loss_workspace_bytes(int32_t width, int32_t height) {
  size_t plane = (size_t)width * height;
  size_t nb = 3 * (size_t)((width + kLT - 1) / kLT) * ((height + kLT - 1) / kLT);
  return 9 * plane * sizeof(float) + 2 * nb * sizeof(double) + 256;
}

extern "C" int ss_loss_l1_ssim(const float* pred, const uint8_t* gt_u8, const float* lut,
                               const float* gt_f32, int32_t width, int32_t height,
                               double ssim_weight, float* dimg, double* out_sums, void* ws,
                               size_t ws_bytes, cudaStream_t stream) {
  if (width <= 0 || height <= 0) return set_error(SS_ERR_INVALID, "ss_loss: bad size");
  if (!gt_u8 && !gt_f32) return set_error(SS_ERR_INVALID, "ss_loss: no ground truth");
  if (9 * (int64_t)width * height >= ((int64_t)1 << 31))
    return set_error(SS_ERR_INVALID, "ss_loss: frame too large (9 W H must fit 31 bits)");
  if (gt_u8 && !lut) return set_error(SS_ERR_INVALID, "ss_loss: u8 ground truth needs a LUT");
  if (ws_bytes < ss_loss_workspace_bytes(width, height))
    return set_error(SS_ERR_WORKSPACE, "ss_loss: workspace too small");
  dim3 grid((width + kLT - 1) / kLT, (height + kLT - 1) / kLT, 3);
  const size_t plane = (size_t)width * height;
  LossArgs a{pred, gt_u8, lut, gt_f32, width, height, (float*)ws,
             (double*)((char*)ws + ((9 * plane * sizeof(float) + 255) & ~(size_t)255))};
  launch_kx(SS_SSIM_PDL, ssim_fwd_kernel, grid, kLossThreads, 0, stream, a);
  launch_kx(SS_SSIM_PDL, ssim_bwd_kernel, grid, kLossThreads, 0, stream, a, (float)ssim_weight, dimg,
            out_sums);
  return check_launch("ss_loss_l1_ssim");
}
