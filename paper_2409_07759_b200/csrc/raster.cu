// a-5 blend forward (_kernels.py:20-53) and a-6 blend backward
// (_kernels.py:56-130) as 16x16-tile rasterizers.
//
// One CTA per tile, one thread per pixel.  The tile's list (already in the
// reference's global (z, src) order, see binning.cu) is staged through
// shared memory 256 records at a time; each record is 36 B (rec_a float4,
// rec_b float4, rec_c float).  Per pixel the reference rules are kept:
// maha > 64 skips, alpha' = min(alpha G, 0.999), accumulation stops once
// T < 1e-4 (the crossing splat included), no background.  The bbox test of
// _kernels.py:35-36 is implied by maha <= 64 (the 8-sigma bbox encloses the
// maha = 64 ellipse), so it is not repeated per pixel.
#include "ss_common.cuh"

namespace ss {

constexpr int kBatch = 256;
// exp(-m/2) = exp2(-m/2 * log2(e))
constexpr float kNegHalfLog2e = -0.72134752044448170368f;

__global__ void __launch_bounds__(256)
    raster_fwd_kernel(const int2* __restrict__ ranges, const int32_t* __restrict__ vals,
                      const float4* __restrict__ rec_a, const float4* __restrict__ rec_b,
                      const float* __restrict__ rec_c, int width, int height, int tiles_x,
                      float* __restrict__ img, float* __restrict__ t_final,
                      int32_t* __restrict__ n_contrib) {
  __shared__ float4 s_a[kBatch];
  __shared__ float4 s_b[kBatch];
  __shared__ float s_c[kBatch];
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * kTile + (threadIdx.x & (kTile - 1));
  const int py = ty * kTile + (threadIdx.x / kTile);
  const bool inside = px < width && py < height;
  const float fx = (float)px, fy = (float)py;
  const int2 rg = ranges[tile];
  bool done = !inside;
  float T = 1.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
  int last = 0;
  for (int base = rg.x; base < rg.y; base += kBatch) {
    if (__syncthreads_and(done)) break;
    const int idx = base + threadIdx.x;
    if (idx < rg.y) {
      const int g = vals[idx];
      s_a[threadIdx.x] = rec_a[g];
      s_b[threadIdx.x] = rec_b[g];
      s_c[threadIdx.x] = rec_c[g];
    }
    __syncthreads();
    const int cnt = min(kBatch, rg.y - base);
    if (!done) {
      for (int j = 0; j < cnt; ++j) {
        const float4 a = s_a[j];
        const float dx = fx - a.x, dy = fy - a.y;
        const float4 b = s_b[j];
        const float m = a.z * dx * dx + 2.f * a.w * dx * dy + b.x * dy * dy;
        if (m > kMahaMax) continue;
        const float G = exp2f(m * kNegHalfLog2e);
        const float ap = fminf(b.y * G, kAlphaMax);
        const float w = ap * T;
        c0 += b.z * w;
        c1 += b.w * w;
        c2 += s_c[j] * w;
        T *= 1.f - ap;
        last = base - rg.x + j + 1;
        if (T < kTMin) {
          done = true;
          break;
        }
      }
    }
  }
  if (inside) {
    const int64_t p = (int64_t)py * width + px;
    img[3 * p] = c0;
    img[3 * p + 1] = c1;
    img[3 * p + 2] = c2;
    t_final[p] = T;
    n_contrib[p] = last;
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256)
    raster_bwd_kernel(const int2* __restrict__ ranges, const int32_t* __restrict__ vals,
                      const float4* __restrict__ rec_a, const float4* __restrict__ rec_b,
                      const float* __restrict__ rec_c, int width, int height, int tiles_x,
                      const float* __restrict__ dimg, const float* __restrict__ t_final,
                      const int32_t* __restrict__ n_contrib, float4* __restrict__ g2d) {
  __shared__ float4 s_a[kBatch];
  __shared__ float4 s_b[kBatch];
  __shared__ float s_c[kBatch];
  __shared__ int32_t s_g[kBatch];
  __shared__ int s_max_last;
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * kTile + (threadIdx.x & (kTile - 1));
  const int py = ty * kTile + (threadIdx.x / kTile);
  const bool inside = px < width && py < height;
  const float fx = (float)px, fy = (float)py;
  const int2 rg = ranges[tile];
  float T = 1.f, d0 = 0.f, d1 = 0.f, d2 = 0.f;
  int last = 0;
  if (inside) {
    const int64_t p = (int64_t)py * width + px;
    T = t_final[p];
    last = n_contrib[p];
    d0 = dimg[3 * p];
    d1 = dimg[3 * p + 1];
    d2 = dimg[3 * p + 2];
  }
  if (threadIdx.x == 0) s_max_last = 0;
  __syncthreads();
  const int wmax = __reduce_max_sync(0xffffffffu, last);
  if ((threadIdx.x & 31) == 0) atomicMax(&s_max_last, wmax);
  __syncthreads();
  const int walk_end = rg.x + s_max_last;
  float S0 = 0.f, S1 = 0.f, S2 = 0.f;  // colour already blended behind (suffix)
  const int lane = threadIdx.x & 31;
  for (int end = walk_end; end > rg.x; end -= kBatch) {
    const int start = max(rg.x, end - kBatch);
    __syncthreads();
    const int idx = start + threadIdx.x;
    if (idx < end) {
      const int g = vals[idx];
      s_g[threadIdx.x] = g;
      s_a[threadIdx.x] = rec_a[g];
      s_b[threadIdx.x] = rec_b[g];
      s_c[threadIdx.x] = rec_c[g];
    }
    __syncthreads();
    for (int j = end - 1; j >= start; --j) {
      const int jj = j - start;
      const bool mine = (j - rg.x) < last;
      float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, v4 = 0.f, v5 = 0.f, v6 = 0.f, v7 = 0.f,
            v8 = 0.f;
      bool has = false;
      if (mine) {
        const float4 a = s_a[jj];
        const float dx = fx - a.x, dy = fy - a.y;
        const float4 b = s_b[jj];
        const float m = a.z * dx * dx + 2.f * a.w * dx * dy + b.x * dy * dy;
        if (m <= kMahaMax) {
          has = true;
          const float G = exp2f(m * kNegHalfLog2e);
          const float aG = b.y * G;
          const float ap = fminf(aG, kAlphaMax);
          const float one_m = 1.f - ap;
          const float inv_rest = __frcp_rn(one_m);
          T *= inv_rest;  // T before this splat
          const float w = ap * T;
          const float cr = b.z, cg = b.w, cb = s_c[jj];
          v6 = d0 * w;
          v7 = d1 * w;
          v8 = d2 * w;
          const float d_ap = d0 * (cr * T - S0 * inv_rest) + d1 * (cg * T - S1 * inv_rest) +
                             d2 * (cb * T - S2 * inv_rest);
          S0 += cr * w;
          S1 += cg * w;
          S2 += cb * w;
          if (aG <= kAlphaMax) {
            v5 = d_ap * G;                          // g_alpha
            const float dm = -0.5f * G * b.y * d_ap;
            v2 = dm * dx * dx;                      // g_inv2d
            v3 = dm * 2.f * dx * dy;
            v4 = dm * dy * dy;
            v0 = -dm * 2.f * (a.z * dx + a.w * dy);  // g_mean2d
            v1 = -dm * 2.f * (a.w * dx + b.x * dy);
          }
        }
      }
      if (__any_sync(0xffffffffu, has)) {
        v0 = warp_sum(v0);
        v1 = warp_sum(v1);
        v2 = warp_sum(v2);
        v3 = warp_sum(v3);
        v4 = warp_sum(v4);
        v5 = warp_sum(v5);
        v6 = warp_sum(v6);
        v7 = warp_sum(v7);
        v8 = warp_sum(v8);
        if (lane == 0) {
          float4* dst = g2d + (int64_t)s_g[jj] * 3;
          atomicAdd(dst, make_float4(v0, v1, v2, v3));
          atomicAdd(dst + 1, make_float4(v4, v5, v6, v7));
          atomicAdd(&dst[2].x, v8);
        }
      }
    }
  }
}

}  // namespace ss

using namespace ss;

extern "C" int ss_raster_fwd(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                             const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                             float* img, float* t_final, int32_t* n_contrib, cudaStream_t stream) {
  if (width <= 0 || height <= 0) return set_error(SS_ERR_INVALID, "ss_raster_fwd: bad size");
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  raster_fwd_kernel<<<tiles_x * tiles_y, kTilePix, 0, stream>>>(
      (const int2*)ranges, vals, (const float4*)rec_a, (const float4*)rec_b, rec_c, width, height,
      tiles_x, img, t_final, n_contrib);
  return check_launch("ss_raster_fwd");
}

extern "C" int ss_raster_bwd(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                             const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                             const float* dimg, const float* t_final, const int32_t* n_contrib,
                             float* g2d, cudaStream_t stream) {
  if (width <= 0 || height <= 0) return set_error(SS_ERR_INVALID, "ss_raster_bwd: bad size");
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  raster_bwd_kernel<<<tiles_x * tiles_y, kTilePix, 0, stream>>>(
      (const int2*)ranges, vals, (const float4*)rec_a, (const float4*)rec_b, rec_c, width, height,
      tiles_x, dimg, t_final, n_contrib, (float4*)g2d);
  return check_launch("ss_raster_bwd");
}
