// a-5 blend forward (_kernels.py:20-53) and a-6 blend backward
// (_kernels.py:56-130) as 16x16-tile rasterizers.
//
// Work mapping: one warp per tile (4 tiles per 128-thread CTA, warps are
// independent).  Lane l owns the 8-pixel column strip x = l % 16,
// y = 8 (l / 16) + 0..7 of the tile, so per list entry a lane evaluates 8
// pixels that share dx: the Mahalanobis term is A + dy (B + c dy) with
// A = a dx^2, B = 2 b dx computed once per entry (2 FMAs per pixel).  The
// tile's list (already in the reference's global (z, src) order, see
// binning.cu) is staged 32 records at a time through a warp-private shared
// buffer; each record is 36 B (rec_a float4, rec_b float4, rec_c float).
//
// Per pixel the reference rules are kept: maha > 64 skips, alpha' =
// min(alpha G, 0.999), accumulation stops once T < 1e-4 (the crossing splat
// included), no background.  The bbox test of _kernels.py:35-36 is implied
// by maha <= 64 (the 8-sigma bbox encloses the maha = 64 ellipse).
//
// Backward: back to front from each pixel's last contributor, T recovered
// by division by (1 - alpha'), suffix colour S accumulated as in
// _kernels.py:100-130.  Per entry a lane folds its 8 pixels into 7 partial
// sums (sum dm, sum dm dy, sum dm dy^2, sum dap G, colour x3) from which the
// 9 gradient components follow; one transposed warp reduction and one
// 9-lane float atomic per (tile, entry).
#include "ss_common.cuh"

namespace ss {

constexpr int kWarps = 4;        // tiles per CTA
constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // exp(-m/2) = 2^(m * this)

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct WarpStage {
  float4 a[32];
  float4 b[32];
  float c[32];
  int g[32];
};

__device__ __forceinline__ void stage_load(WarpStage& st, int lane, int idx, int end,
                                           const int32_t* __restrict__ vals,
                                           const float4* __restrict__ rec_a,
                                           const float4* __restrict__ rec_b,
                                           const float* __restrict__ rec_c) {
  if (idx < end) {
    const int g = __ldg(vals + idx);
    st.g[lane] = g;
    st.a[lane] = __ldg(rec_a + g);
    st.b[lane] = __ldg(rec_b + g);
    st.c[lane] = __ldg(rec_c + g);
  }
}

template <int STRIP>
__global__ void __launch_bounds__(kWarps * 32)
    raster_fwd_kernel(const int2* __restrict__ ranges, const int32_t* __restrict__ vals,
                      const float4* __restrict__ rec_a, const float4* __restrict__ rec_b,
                      const float* __restrict__ rec_c, int width, int height, int tiles_x,
                      int n_tiles, const int32_t* __restrict__ tile_order,
                      float* __restrict__ img, float* __restrict__ t_final,
                      int32_t* __restrict__ n_contrib) {
  __shared__ WarpStage s_stage[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int WPT = kTile / (2 * STRIP);  // warps per tile
  const int gwarp = blockIdx.x * kWarps + warp;
  const int slot_id = gwarp / WPT, sub = gwarp % WPT;
  if (slot_id >= n_tiles) return;
  const int tile = tile_order ? tile_order[slot_id] : slot_id;
  WarpStage& st = s_stage[warp];
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * kTile + (lane & 15);
  const int py0 = ty * kTile + sub * 2 * STRIP + (lane >> 4) * STRIP;
  const float fx = (float)px, fy0 = (float)py0;
  unsigned live = 0;
#pragma unroll
  for (int k = 0; k < STRIP; ++k)
    if (px < width && py0 + k < height) live |= 1u << k;
  float T[STRIP], c0[STRIP], c1[STRIP], c2[STRIP];
  int last[STRIP];
#pragma unroll
  for (int k = 0; k < STRIP; ++k) {
    T[k] = 1.f;
    c0[k] = c1[k] = c2[k] = 0.f;
    last[k] = 0;
  }
  const int2 rg = ranges[tile];
  for (int base = rg.x; base < rg.y; base += 32) {
    if (!__any_sync(0xffffffffu, live)) break;
    __syncwarp();
    stage_load(st, lane, base + lane, rg.y, vals, rec_a, rec_b, rec_c);
    __syncwarp();
    if (live) {
      const int cnt = min(32, rg.y - base);
      for (int j = 0; j < cnt; ++j) {
        const float4 a = st.a[j];
        const float4 b = st.b[j];
        const float cb = st.c[j];
        const float dx = fx - a.x, dy0 = fy0 - a.y;
        const float A = a.z * dx * dx, B = 2.f * a.w * dx, cc = b.x;
        const int pos = base - rg.x + j + 1;
        // branch-free over the strip: invalid pixels get alpha' = 0, which
        // leaves C and T untouched, so the 8 chains interleave freely
#pragma unroll
        for (int k = 0; k < STRIP; ++k) {
          const float dy = dy0 + (float)k;
          const float m = fmaf(dy, fmaf(cc, dy, B), A);
          const bool valid = ((live >> k) & 1u) && (m <= kMahaMax);
          const float G = ex2(m * kNegHalfLog2e);
          const float ap = valid ? fminf(b.y * G, kAlphaMax) : 0.f;
          const float w = ap * T[k];
          c0[k] = fmaf(b.z, w, c0[k]);
          c1[k] = fmaf(b.w, w, c1[k]);
          c2[k] = fmaf(cb, w, c2[k]);
          T[k] *= 1.f - ap;
          last[k] = valid ? pos : last[k];
          live &= ~((unsigned)(T[k] < kTMin) << k);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < STRIP; ++k) {
    const int py = py0 + k;
    if (px < width && py < height) {
      const int64_t p = (int64_t)py * width + px;
      img[3 * p] = c0[k];
      img[3 * p + 1] = c1[k];
      img[3 * p + 2] = c2[k];
      t_final[p] = T[k];
      n_contrib[p] = last[k];
    }
  }
}

// Transposed warp reduction of 16 slots: afterwards lane L holds the warp
// total of slot 8 b4 + 4 b3 + 2 b2 + b1 (b_i = bit i of L); lanes L, L^1 agree.
__device__ __forceinline__ float reduce16(float v[16], int lane) {
#pragma unroll
  for (int half = 8, off = 16; half >= 1; half >>= 1, off >>= 1) {
    const bool up = lane & off;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? v[i] : v[i + half];
      const float keep = up ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

template <int STRIP>
__global__ void __launch_bounds__(kWarps * 32)
    raster_bwd_kernel(const int2* __restrict__ ranges, const int32_t* __restrict__ vals,
                      const float4* __restrict__ rec_a, const float4* __restrict__ rec_b,
                      const float* __restrict__ rec_c, int width, int height, int tiles_x,
                      int n_tiles, const int32_t* __restrict__ tile_order,
                      const float* __restrict__ dimg, const float* __restrict__ t_final,
                      const int32_t* __restrict__ n_contrib, float* __restrict__ g2d) {
  __shared__ WarpStage s_stage[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int WPT = kTile / (2 * STRIP);  // warps per tile
  const int gwarp = blockIdx.x * kWarps + warp;
  const int slot_id = gwarp / WPT, sub = gwarp % WPT;
  if (slot_id >= n_tiles) return;
  const int tile = tile_order ? tile_order[slot_id] : slot_id;
  WarpStage& st = s_stage[warp];
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * kTile + (lane & 15);
  const int py0 = ty * kTile + sub * 2 * STRIP + (lane >> 4) * STRIP;
  const float fx = (float)px, fy0 = (float)py0;
  float T[STRIP], d0[STRIP], d1[STRIP], d2[STRIP], S0[STRIP], S1[STRIP], S2[STRIP];
  int last[STRIP];
  int my_max = 0;
#pragma unroll
  for (int k = 0; k < STRIP; ++k) {
    const int py = py0 + k;
    S0[k] = S1[k] = S2[k] = 0.f;
    if (px < width && py < height) {
      const int64_t p = (int64_t)py * width + px;
      T[k] = t_final[p];
      last[k] = n_contrib[p];
      d0[k] = dimg[3 * p];
      d1[k] = dimg[3 * p + 1];
      d2[k] = dimg[3 * p + 2];
    } else {
      T[k] = 1.f;
      last[k] = 0;
      d0[k] = d1[k] = d2[k] = 0.f;
    }
    my_max = max(my_max, last[k]);
  }
  const int2 rg = ranges[tile];
  const int walk_end = rg.x + __reduce_max_sync(0xffffffffu, my_max);
  const int slot = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                   ((lane >> 1) & 1);
  for (int end = walk_end; end > rg.x; end -= 32) {
    const int start = max(rg.x, end - 32);
    __syncwarp();
    stage_load(st, lane, start + lane, end, vals, rec_a, rec_b, rec_c);
    __syncwarp();
    for (int j = end - start - 1; j >= 0; --j) {
      const int pos = start - rg.x + j;  // 0-based position in the tile list
      const float4 a = st.a[j];
      const float4 b = st.b[j];
      const float cb = st.c[j];
      const float dx = fx - a.x, dy0 = fy0 - a.y;
      const float A = a.z * dx * dx, B = 2.f * a.w * dx, cc = b.x;
      const float alpha = b.y;
      float sdm = 0.f, sdmy = 0.f, sdmyy = 0.f, sal = 0.f, sc0 = 0.f, sc1 = 0.f, sc2 = 0.f;
      bool touched = false;
#pragma unroll
      for (int k = 0; k < STRIP; ++k) {
        // branch-free: an invalid pixel has alpha' = 0 (T and S unchanged) and
        // its d alpha' is zeroed, so it contributes nothing
        const float dy = dy0 + (float)k;
        const float m = fmaf(dy, fmaf(cc, dy, B), A);
        const bool valid = (pos < last[k]) && (m <= kMahaMax);
        touched |= valid;
        const float G = ex2(m * kNegHalfLog2e);
        const float aG = alpha * G;
        const float ap = valid ? fminf(aG, kAlphaMax) : 0.f;
        const float inv = __frcp_rn(1.f - ap);
        T[k] *= inv;  // T before this splat
        const float w = ap * T[k];
        sc0 = fmaf(d0[k], w, sc0);
        sc1 = fmaf(d1[k], w, sc1);
        sc2 = fmaf(d2[k], w, sc2);
        const float dap_raw = d0[k] * (b.z * T[k] - S0[k] * inv) +
                              d1[k] * (b.w * T[k] - S1[k] * inv) +
                              d2[k] * (cb * T[k] - S2[k] * inv);
        S0[k] = fmaf(b.z, w, S0[k]);
        S1[k] = fmaf(b.w, w, S1[k]);
        S2[k] = fmaf(cb, w, S2[k]);
        // clamped splats pass no alpha/footprint gradient (_kernels.py:120-121)
        const float dap = (valid && aG <= kAlphaMax) ? dap_raw : 0.f;
        sal = fmaf(dap, G, sal);
        const float dm = -0.5f * G * alpha * dap;
        sdm += dm;
        sdmy = fmaf(dm, dy, sdmy);
        sdmyy = fmaf(dm * dy, dy, sdmyy);
      }
      if (!__any_sync(0xffffffffu, touched)) continue;
      // g_mean2d = -2 dm (conic d), g_inv2d = dm (dx^2, 2 dx dy, dy^2) summed over the strip
      float v[16];
      v[0] = -2.f * (a.z * dx * sdm + a.w * sdmy);
      v[1] = -2.f * (a.w * dx * sdm + cc * sdmy);
      v[2] = dx * dx * sdm;
      v[3] = 2.f * dx * sdmy;
      v[4] = sdmyy;
      v[5] = sal;
      v[6] = sc0;
      v[7] = sc1;
      v[8] = sc2;
#pragma unroll
      for (int i = 9; i < 16; ++i) v[i] = 0.f;
      const float tot = reduce16(v, lane);
      if (!(lane & 1) && slot < 9) atomicAdd(g2d + (int64_t)st.g[j] * SS_G2D_ROW + slot, tot);
    }
  }
}

static int g_strip = 4;

}  // namespace ss

using namespace ss;

extern "C" int ss_set_raster_strip(int32_t strip) {
  if (strip != 2 && strip != 4 && strip != 8)
    return set_error(SS_ERR_INVALID, "ss_set_raster_strip: strip must be 2, 4 or 8");
  g_strip = strip;
  return SS_OK;
}

extern "C" int ss_raster_fwd(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                             const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                             const int32_t* tile_order, float* img, float* t_final,
                             int32_t* n_contrib, cudaStream_t stream) {
  if (width <= 0 || height <= 0) return set_error(SS_ERR_INVALID, "ss_raster_fwd: bad size");
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int n_tiles = tiles_x * tiles_y;
  const int wpt = kTile / (2 * g_strip);
  const int blocks = (n_tiles * wpt + kWarps - 1) / kWarps;
#define SS_FWD(S)                                                                             \
  raster_fwd_kernel<S><<<blocks, kWarps * 32, 0, stream>>>(                                   \
      (const int2*)ranges, vals, (const float4*)rec_a, (const float4*)rec_b, rec_c, width,  \
      height, tiles_x, n_tiles, tile_order, img, t_final, n_contrib)
  if (g_strip == 8) SS_FWD(8);
  else if (g_strip == 4) SS_FWD(4);
  else SS_FWD(2);
#undef SS_FWD
  return check_launch("ss_raster_fwd");
}

extern "C" int ss_raster_bwd(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                             const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                             const int32_t* tile_order, const float* dimg, const float* t_final,
                             const int32_t* n_contrib, float* g2d, cudaStream_t stream) {
  if (width <= 0 || height <= 0) return set_error(SS_ERR_INVALID, "ss_raster_bwd: bad size");
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int n_tiles = tiles_x * tiles_y;
  const int wpt = kTile / (2 * g_strip);
  const int blocks = (n_tiles * wpt + kWarps - 1) / kWarps;
#define SS_BWD(S)                                                                             \
  raster_bwd_kernel<S><<<blocks, kWarps * 32, 0, stream>>>(                                   \
      (const int2*)ranges, vals, (const float4*)rec_a, (const float4*)rec_b, rec_c, width,  \
      height, tiles_x, n_tiles, tile_order, dimg, t_final, n_contrib, g2d)
  if (g_strip == 8) SS_BWD(8);
  else if (g_strip == 4) SS_BWD(4);
  else SS_BWD(2);
#undef SS_BWD
  return check_launch("ss_raster_bwd");
}
