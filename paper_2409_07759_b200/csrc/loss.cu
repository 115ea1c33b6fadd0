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
//   pass 3: one block reduces the per-block sums in a fixed order.
//
// The blurs are register-blocked: a thread produces 8 consecutive outputs of
// a column (vertical pass) or 4 of a row (horizontal pass) from a sliding
// window held in registers, so each shared-memory value is loaded once per
// thread instead of once per tap; the 11 taps are compile-time immediates
// (full-rate FFMA with an immediate operand).
#include "ss_common.cuh"

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

__device__ __forceinline__ float gt_value(const uint8_t* gt_u8, const float* lut,
                                          const float* gt_f32, int64_t idx) {
  return gt_u8 ? lut[gt_u8[idx]] : gt_f32[idx];
}

// Loads the (42 x 42) halo region of channel ch of x and y (zero outside
// the image) into padded (42 x kLP) tiles.
__device__ __forceinline__ void load_region(const float* __restrict__ pred,
                                            const uint8_t* __restrict__ gt_u8,
                                            const float* s_lut, const float* __restrict__ gt_f32,
                                            int W, int H, int x0, int y0, int ch, float* s_x,
                                            float* s_y) {
  for (int idx = threadIdx.x; idx < kLR * kLR; idx += blockDim.x) {
    const int r = idx / kLR, q = idx % kLR;
    const int gy = y0 - kHalo + r, gx = x0 - kHalo + q;
    float xv = 0.f, yv = 0.f;
    if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
      const int64_t e = ((int64_t)gy * W + gx) * 3 + ch;
      xv = pred[e];
      yv = gt_u8 ? s_lut[gt_u8[e]] : gt_f32[e];
    }
    s_x[r * kLP + q] = xv;
    s_y[r * kLP + q] = yv;
  }
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

// Vertical blur of NQ quantities: out[q][r][c] = sum_t w_t src_q(r + t, c) for
// r in [0, 32), c in [0, 42), from a (42 x kLP) source; quantities are
// derived from the loaded sources by `load` (e.g. x, y, x*x, x*y, y*y).
template <int NQ, typename Load>
__device__ __forceinline__ void vblur(float (*out)[kLT][kLP], Load load) {
  for (int task = threadIdx.x; task < kLR * (kLT / kVR); task += kLossThreads) {
    const int c = task % kLR, r0 = (task / kLR) * kVR;
    float acc[NQ][kVR];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int i = 0; i < kVR; ++i) acc[q][i] = 0.f;
#pragma unroll
    for (int s = 0; s < kVR + 10; ++s) {
      float v[NQ];
      load(r0 + s, c, v);
#pragma unroll
      for (int i = 0; i < kVR; ++i) {
        const int t = s - i;
        if (t >= 0 && t <= 10) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) acc[q][i] = fmaf(win(t), v[q], acc[q][i]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int i = 0; i < kVR; ++i) out[q][r0 + i][c] = acc[q][i];
  }
}

// Horizontal blur: res[q][i] = sum_t w_t v[q][r][c0 + i + t], i in [0, kHC)
template <int NQ>
__device__ __forceinline__ void hblur(const float (*v)[kLT][kLP], int r, int c0,
                                      float res[NQ][kHC]) {
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int i = 0; i < kHC; ++i) res[q][i] = 0.f;
#pragma unroll
  for (int s = 0; s < kHC + 10; ++s) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float x = v[q][r][c0 + s];
#pragma unroll
      for (int i = 0; i < kHC; ++i) {
        const int t = s - i;
        if (t >= 0 && t <= 10) res[q][i] = fmaf(win(t), x, res[q][i]);
      }
    }
  }
}

// grid (tiles_x, tiles_y, 3): one CTA per 32x32 tile and channel
__global__ void __launch_bounds__(kLossThreads) ssim_fwd_kernel(LossArgs a) {
  __shared__ float s_x[kLR * kLP];
  __shared__ float s_y[kLR * kLP];
  __shared__ float s_v[5][kLT][kLP];
  __shared__ float s_lut[256];
  __shared__ double s_red[2][kLossThreads / 32];
  const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT, ch = blockIdx.z;
  const int W = a.width, H = a.height;
  const int64_t plane = (int64_t)W * H;
  if (a.gt_u8)
    for (int i = threadIdx.x; i < 256; i += kLossThreads) s_lut[i] = a.lut[i];
  __syncthreads();
  load_region(a.pred, a.gt_u8, s_lut, a.gt_f32, W, H, x0, y0, ch, s_x, s_y);
  __syncthreads();
  // vertical pass (axis 0, loss.py:31) of x, y, xx, xy, yy
  vblur<5>(s_v, [&](int r, int c, float* v) {
    const float xv = s_x[r * kLP + c], yv = s_y[r * kLP + c];
    v[0] = xv;
    v[1] = yv;
    v[2] = xv * xv;
    v[3] = xv * yv;
    v[4] = yv * yv;
  });
  __syncthreads();
  // horizontal pass (axis 1, loss.py:32) + SSIM terms (loss.py:39-59)
  double l1 = 0.0, ss = 0.0;
  {
    const int r = threadIdx.x / (kLT / kHC), c0 = (threadIdx.x % (kLT / kHC)) * kHC;
    float m[5][kHC];
    hblur<5>(s_v, r, c0, m);
    const int gy = y0 + r;
#pragma unroll
    for (int i = 0; i < kHC; ++i) {
      const int gx = x0 + c0 + i;
      if (gy >= H || gx >= W) continue;
      const float mu_x = m[0][i], mu_y = m[1][i], mxx = m[2][i], mxy = m[3][i], myy = m[4][i];
      const float C1 = 1e-4f, C2 = 9e-4f;
      const float sig_x = mxx - mu_x * mu_x;
      const float sig_y = myy - mu_y * mu_y;
      const float sig_xy = mxy - mu_x * mu_y;
      const float a1 = 2.f * mu_x * mu_y + C1;
      const float a2 = 2.f * sig_xy + C2;
      const float b1 = mu_x * mu_x + mu_y * mu_y + C1;
      const float b2 = sig_x + sig_y + C2;
      const float inv_b2 = 1.f / b2;
      const float inv_den = inv_b2 / b1;  // 1 / (b1 b2)
      const float s = (a1 * a2) * inv_den;
      const float ds_dmu = (2.f * mu_y * (a2 - a1) - 2.f * mu_x * s * (b2 - b1)) * inv_den;
      const float ds_dmxx = -s * inv_b2;
      const float ds_dmxy = 2.f * a1 * inv_den;
      const int64_t pix = (int64_t)gy * W + gx;
      a.maps[(0 * 3 + ch) * plane + pix] = ds_dmu;
      a.maps[(1 * 3 + ch) * plane + pix] = ds_dmxx;
      a.maps[(2 * 3 + ch) * plane + pix] = ds_dmxy;
      ss += (double)s;
      const int off = (r + kHalo) * kLP + (c0 + i + kHalo);
      l1 += (double)fabsf(s_x[off] - s_y[off]);
    }
  }
  // block reduction of the two sums (fixed order -> deterministic)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_red[0][threadIdx.x >> 5] = l1;
    s_red[1][threadIdx.x >> 5] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int i = 0; i < kLossThreads / 32; ++i) {
      t0 += s_red[0][i];
      t1 += s_red[1][i];
    }
    const int b = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    a.partials[2 * b] = t0;
    a.partials[2 * b + 1] = t1;
  }
}

__global__ void __launch_bounds__(kLossThreads) ssim_bwd_kernel(LossArgs a, float w_ssim,
                                                                 float* __restrict__ dimg) {
  __shared__ float s_m[3][kLR][kLP];
  __shared__ float s_v[3][kLT][kLP];
  __shared__ float s_lut[256];
  if (a.gt_u8)
    for (int i = threadIdx.x; i < 256; i += kLossThreads) s_lut[i] = a.lut[i];
  const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT, ch = blockIdx.z;
  const int W = a.width, H = a.height;
  const int64_t plane = (int64_t)W * H;
  const float inv_n = 1.0f / (float)((double)plane * 3.0);
  for (int idx = threadIdx.x; idx < kLR * kLR; idx += kLossThreads) {
    const int r = idx / kLR, q = idx % kLR;
    const int gy = y0 - kHalo + r, gx = x0 - kHalo + q;
    const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
    const int64_t pix = (int64_t)gy * W + gx;
#pragma unroll
    for (int k = 0; k < 3; ++k) s_m[k][r][q] = in ? a.maps[(k * 3 + ch) * plane + pix] : 0.f;
  }
  __syncthreads();
  vblur<3>(s_v, [&](int r, int c, float* v) {
    v[0] = s_m[0][r][c];
    v[1] = s_m[1][r][c];
    v[2] = s_m[2][r][c];
  });
  __syncthreads();
  const int r = threadIdx.x / (kLT / kHC), c0 = (threadIdx.x % (kLT / kHC)) * kHC;
  float bl[3][kHC];
  hblur<3>(s_v, r, c0, bl);
  const int gy = y0 + r;
#pragma unroll
  for (int i = 0; i < kHC; ++i) {
    const int gx = x0 + c0 + i;
    if (gy >= H || gx >= W) continue;
    const int64_t e = ((int64_t)gy * W + gx) * 3 + ch;
    const float x = a.pred[e];
    const float y = gt_value(a.gt_u8, s_lut, a.gt_f32, e);
    const float grad = (bl[0][i] + 2.f * x * bl[1][i] + y * bl[2][i]) * inv_n;
    const float d = x - y;
    const float sgn = (d > 0.f) ? 1.f : ((d < 0.f) ? -1.f : 0.f);
    dimg[e] = (1.f - w_ssim) * sgn * inv_n - w_ssim * grad;
  }
}

__global__ void loss_reduce_kernel(const double* __restrict__ partials, int n_blocks,
                                   double* __restrict__ out) {
  __shared__ double s[2][32];
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
    double a = 0.0, b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      a += s[0][i];
      b += s[1][i];
    }
    out[0] = a;
    out[1] = b;
  }
}

}  // namespace ss

using namespace ss;

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
  if (gt_u8 && !lut) return set_error(SS_ERR_INVALID, "ss_loss: u8 ground truth needs a LUT");
  if (ws_bytes < ss_loss_workspace_bytes(width, height))
    return set_error(SS_ERR_WORKSPACE, "ss_loss: workspace too small");
  dim3 grid((width + kLT - 1) / kLT, (height + kLT - 1) / kLT, 3);
  const size_t plane = (size_t)width * height;
  LossArgs a{pred, gt_u8, lut, gt_f32, width, height, (float*)ws,
             (double*)((char*)ws + ((9 * plane * sizeof(float) + 255) & ~(size_t)255))};
  ssim_fwd_kernel<<<grid, kLossThreads, 0, stream>>>(a);
  ssim_bwd_kernel<<<grid, kLossThreads, 0, stream>>>(a, (float)ssim_weight, dimg);
  loss_reduce_kernel<<<1, 1024, 0, stream>>>(a.partials, grid.x * grid.y * grid.z, out_sums);
  return check_launch("ss_loss_l1_ssim");
}
