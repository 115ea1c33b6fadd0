// a-5 blend forward (_kernels.py:20-53) and a-6 blend backward
// (_kernels.py:56-130) as 16x16-tile rasterizers.
//
// Work mapping: a warp covers 16 x (2 STRIP) pixels of a tile (8 / STRIP
// warps per tile, 4 warps per CTA in both passes, warps independent).  Lane l owns the
// STRIP-pixel column strip x = l % 16, y = y0 + STRIP (l / 16) + k.  The
// tile's list (already in the reference's global (z, src) order, see
// binning.cu) is staged 32 records at a time through a warp-private shared
// buffer; a record is 36 B: rec_a = (u, v, kappa i0, kappa i1), rec_b =
// (kappa i2, log2 alpha, r, g), rec_c = b with kappa = -log2(e) / 2, so that
//
//     alpha G = alpha exp(-m/2) = 2^(kappa m + log2 alpha) = 2^(q0 + k (lin + k quad))
//
// per strip pixel k with q0, lin, quad computed once per (lane, entry): two
// FMAs with immediate k per pixel, no separate multiply by alpha.  On
// Blackwell 3-register FFMA/FMUL issue at half rate, so the per-pixel bodies
// are written to minimise them.
//
// Per pixel the reference rules are kept: maha > 64 skips (kappa m + log2 a
// >= 64 kappa + log2 a), alpha' = min(alpha G, 0.999), accumulation stops once
// T < 1e-4 (the crossing splat included), no background.  The bbox test of
// _kernels.py:35-36 is implied by maha <= 64 (the 8-sigma bbox encloses the
// maha = 64 ellipse).  Bodies are branch-free: an invalid pixel gets
// alpha' = 0, which leaves C and T unchanged.
//
// Backward: back to front from each pixel's last contributor, T recovered
// by multiplication with 1 / (1 - alpha').  The reference's suffix colour S
// (_kernels.py:100-130) only enters through sum_ch dC_ch S_ch, so a pixel
// carries the scalar Q = dC . S (Q += w dC . c) and d alpha' = T dC.c - Q/(1-a').
// With t = alpha G d alpha' (zero when clamped), g_alpha = sum t / alpha and
// dm = -t/2, and the strip sums sum t, sum t k, sum t k^2 give every
// footprint gradient.  g2d receives the 9 linear basis sums (see the strip
// epilogue) that ss_project_bwd turns into mean2d / conic / alpha gradients:
// a warp parks each entry's 32 x 9 lane values in shared memory and every
// 3 entries sums them (one lane per (entry, component)) into one float
// atomic per (warp, entry, component); the deterministic mode instead
// reduces each entry in registers (12-shuffle transposed reduction) into
// fixed-order partials.
#include "ss_common.cuh"

namespace ss {

// 4 warps (2 tiles) per forward CTA: a CTA's slot frees as soon as its two
// tiles are done (8 warps: fwd 0.239 ms, 4: 0.234, 2: 0.234; config 3)
#ifndef SS_RASTER_WARPS_FWD
#define SS_RASTER_WARPS_FWD 4
#endif
#ifndef SS_RASTER_WARPS_BWD
#define SS_RASTER_WARPS_BWD 4
#endif
#ifndef SS_RASTER_EARLY_TRIGGER
#define SS_RASTER_EARLY_TRIGGER 1
#endif
// The raster kernels are launched WITHOUT programmatic dependent launch:
// early-launched raster CTAs parked in griddepcontrol.wait held SM resources
// while their predecessors (the binning scatter, the loss) still ran --
// measured on one box: step 1.097 ms with PDL on the raster launches, 1.019 ms
// without (every other kernel keeps PDL; turning it off for the SSIM,
// projection-backward or Adam launches as well gained nothing).
#ifndef SS_RASTER_PDL
#define SS_RASTER_PDL 0
#endif
constexpr int kWarps = SS_RASTER_WARPS_BWD;     // warps per CTA, backward
constexpr int kWarpsF = SS_RASTER_WARPS_FWD;    // warps per CTA, forward
#ifndef SS_BWD_MINB
#define SS_BWD_MINB (32 / SS_RASTER_WARPS_BWD)  // 64 registers
#endif
constexpr float kKappa = -0.72134752044448170368f;  // -log2(e) / 2
constexpr float kMahaKappa = kMahaMax * kKappa;       // 64 kappa

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct WarpStage {
  float4 a[32];
  float4 b[32];
  float c[32];
  int g[32];
};

// Whether a record can pass the per-pixel test (kappa m + log2 alpha >=
// thr, thr = max(64 kappa + log2 alpha, lfloor)) anywhere in the warp's
// pixel-centre rectangle [x0, x0 + 15] x [y0, y1]: with Q = |kappa| m =
// A dx^2 + 2 B dx dy + C dy^2 the test is Q <= R, R = min(64 |kappa|,
// log2 alpha - lfloor), an ellipse; as in the binning's row_span, its
// x-interval over the rectangle's rows is [L, R] with the extreme points at
// dy = -+sy clamped into the rows.  Conservative (R inflated by 2^-8
// relative + 2^-6, ill-conditioned conics always pass): it only decides which
// entries a warp visits; the per-pixel test decides every contribution.
// One lane evaluates one staged entry, so a 32-entry batch costs each lane
// one evaluation (~1 instruction per entry) and the warp then walks only the
// entries its 128 pixels can use.
__device__ __forceinline__ bool touches_rect(const float4& a, const float4& b, float x0, float y0,
                                             float y1, float lfloor) {
  const float A = -a.z, B = -a.w, C = -b.x;  // kappa < 0: |kappa| conic
  float R = fminf(-kMahaKappa, b.y - lfloor);
  if (!(R > 0.f)) return false;
  R = fmaf(R, 1.00390625f, 0.015625f);
  const float det = fmaf(A, C, -B * B);
  if (!(det > 1e-3f * A * C)) return true;  // near-degenerate: no cheap exact test
  const float rdet = 1.f / det;
  const float ymax = sqrtf(A * R * rdet);
  const float lo = fmaxf(y0 - a.y, -ymax), hi = fminf(y1 - a.y, ymax);
  if (lo > hi) return false;
  const float sy = B * sqrtf(R * rdet / C);
  const float cR = clampf(-sy, lo, hi), cL = clampf(sy, lo, hi);
  const float AR = A * R;
  const float sR = sqrtf(fmaxf(fmaf(-det * cR, cR, AR), 0.f));
  const float sL = sqrtf(fmaxf(fmaf(-det * cL, cL, AR), 0.f));
  const float rA = 1.f / A;
  const float right = (fmaf(-B, cR, sR)) * rA, left = (fmaf(-B, cL, -sL)) * rA;
  return (x0 - a.x) <= right && (x0 + (kTile - 1) - a.x) >= left;
}

// Entry-use masks (view driver, strips equal): the forward records, per
// (tile, 32-entry batch, warp), which batch entries contributed to at least
// one of the warp's pixels; the backward walks exactly those (its per-pixel
// validity equals the forward's: a position before a pixel's last
// contributor was reached with T >= 1e-4).  Batch b of tile t's list
// (positions rg.x + 32 b ...) has slot floor(rg.x / 32) + t + b: lists lie in
// tile order, so slots never collide; ss_raster_used_words(K, tiles) words.
__device__ __forceinline__ int64_t used_slot(int list_start, int tile, int batch) {
  return (int64_t)(list_start >> 5) + tile + batch;
}

// Per (lane, entry) coefficients of kappa m + log2 alpha over the strip.
struct StripQuad {
  float q0, lin, quad, thr, dx, dy0;
};

__device__ __forceinline__ StripQuad strip_quad(const float4& a, const float4& b, float fx,
                                                float fy0, float lfloor) {
  StripQuad s;
  s.dx = fx - a.x;
  s.dy0 = fy0 - a.y;
  // kappa m(dy) = A + dy (B + C dy), A = ka dx^2, B = 2 kb dx, C = kc
  const float A = a.z * s.dx * s.dx;
  const float B = 2.f * a.w * s.dx;
  const float C = b.x;
  s.q0 = fmaf(s.dy0, fmaf(C, s.dy0, B), A) + b.y;
  s.lin = fmaf(2.f * C, s.dy0, B);
  s.quad = C;
  s.thr = fmaxf(kMahaKappa + b.y, lfloor);  // maha <= 64 and alpha G >= 2^lfloor
  return s;
}

// The strip's exponents as packed pairs, by forward differences:
// e_{k+1} = e_k + d_k, d_k = lin + (2k + 1) quad.  Plain two-register FADDs
// (no (k, k^2) constant pairs to keep in registers or rematerialise per
// entry); the rounding differs from the direct form by a few ulp of e.
template <int NP>
__device__ __forceinline__ void strip_exps(const StripQuad& s, f2 e[NP]) {
  float ev[2 * NP];
  const float q2 = s.quad + s.quad;
  float d = s.lin + s.quad;
  ev[0] = s.q0;
#pragma unroll
  for (int k = 1; k < 2 * NP; ++k) {
    ev[k] = ev[k - 1] + d;
    if (k + 1 < 2 * NP) d += q2;
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) e[p] = pk2(ev[2 * p], ev[2 * p + 1]);
}

// BB: also apply an explicit per-splat pixel bbox (pbox, x0 x1 y0 y1 half
// open) -- _kernels.blend_forward's bbox test for 2D input whose bbox need
// not enclose the maha <= 64 ellipse.  Off for the training path, where the
// 8-sigma bbox is implied by the maha cut.
template <int STRIP, bool BB = false>
__global__ void __launch_bounds__(kWarpsF * 32)
    raster_fwd_kernel(const int2* __restrict__ ranges, const int32_t* __restrict__ vals,
                      const float4* __restrict__ rec_a, const float4* __restrict__ rec_b,
                      const float* __restrict__ rec_c, int width, int height, int tiles_x,
                      int n_tiles, const int32_t* __restrict__ tile_order,
                      float* __restrict__ img, float* __restrict__ t_final,
                      int32_t* __restrict__ n_contrib, float lfloor,
                      const int4* __restrict__ pbox = nullptr,
                      uint32_t* __restrict__ used = nullptr,
                      int32_t* __restrict__ tile_work = nullptr) {
  pdl_wait();
  if (SS_RASTER_EARLY_TRIGGER) pdl_trigger();
  __shared__ WarpStage s_stage[kWarpsF];
  constexpr int WPT = kTile / (2 * STRIP);  // warps per tile
  constexpr int NP = STRIP / 2;             // pixel pairs per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gwarp = blockIdx.x * kWarpsF + warp;
  const int slot_id = gwarp / WPT, sub = gwarp % WPT;
  if (slot_id >= n_tiles) return;
  const int tile = tile_order ? tile_order[slot_id] : slot_id;
  WarpStage& st = s_stage[warp];
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * kTile + (lane & 15);
  const int py0 = ty * kTile + sub * 2 * STRIP + (lane >> 4) * STRIP;
  const float fx = (float)px, fy0 = (float)py0;
  // the warp's pixel-centre rectangle (for the per-entry region test)
  const float rx0 = (float)(tx * kTile), ry0 = (float)(ty * kTile + sub * 2 * STRIP);
  const float ry1 = ry0 + (float)(2 * STRIP - 1);
  f2 T[NP], c0[NP], c1[NP], c2[NP];
  int last[STRIP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    // pixels outside the image start "saturated" (T = 0) and never contribute
    const float tl = (px < width && py0 + 2 * p < height) ? 1.f : 0.f;
    const float th = (px < width && py0 + 2 * p + 1 < height) ? 1.f : 0.f;
    T[p] = pk2(tl, th);
    c0[p] = c1[p] = c2[p] = bc(0.f);
  }
#pragma unroll
  for (int k = 0; k < STRIP; ++k) last[k] = 0;
  const int2 rg = ranges[tile];
  SS_DCHECK(rg.x >= 0 && rg.x <= rg.y);
  for (int base = rg.x; base < rg.y; base += 32) {
    bool live = false;
#pragma unroll
    for (int p = 0; p < NP; ++p) live |= (lo2(T[p]) >= kTMin) | (hi2(T[p]) >= kTMin);
    if (!__any_sync(0xffffffffu, live)) break;
    __syncwarp();
    bool touch = false;
    if (base + lane < rg.y) {
      const int g = __ldg(vals + base + lane);
      const float4 a = __ldg(rec_a + g), b = __ldg(rec_b + g);
      st.g[lane] = g;
      st.a[lane] = a;
      st.b[lane] = b;
      st.c[lane] = __ldg(rec_c + g);
      touch = touches_rect(a, b, rx0, ry0, ry1, lfloor);
    }
    // only the entries that can reach this warp's pixels are walked
    uint32_t todo = __ballot_sync(0xffffffffu, touch);
    uint32_t used_bits = 0;  // entries that contributed to one of the warp's pixels
    __syncwarp();
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const float4 a = st.a[j];
      const float4 b = st.b[j];
      const float cb = st.c[j];
      const StripQuad s = strip_quad(a, b, fx, fy0, lfloor);
      const int pos = base - rg.x + j + 1;
      // exponents and validity of the whole strip first: a warp skips the
      // entry when none of its pixels is live and passes the per-pixel test
      f2 e[NP];
      strip_exps<NP>(s, e);
      bool valid[STRIP];
      bool any = false;
      int4 q = make_int4(0, 0, 0, 0);
      if (BB) q = __ldg(pbox + st.g[j]);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        valid[2 * p] = (lo2(T[p]) >= kTMin) && (lo2(e[p]) >= s.thr);
        valid[2 * p + 1] = (hi2(T[p]) >= kTMin) && (hi2(e[p]) >= s.thr);
        if (BB) {
          const bool xin = px >= q.x && px < q.y;
          valid[2 * p] &= xin && py0 + 2 * p >= q.z && py0 + 2 * p < q.w;
          valid[2 * p + 1] &= xin && py0 + 2 * p + 1 >= q.z && py0 + 2 * p + 1 < q.w;
        }
        any |= valid[2 * p] | valid[2 * p + 1];
      }
      if (!__any_sync(0xffffffffu, any)) continue;
      used_bits |= 1u << j;
      // branch-free over the strip: invalid pixels get alpha' = 0, which
      // leaves C and T untouched
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float al = valid[2 * p] ? fminf(ex2(lo2(e[p])), kAlphaMax) : 0.f;
        const float ah = valid[2 * p + 1] ? fminf(ex2(hi2(e[p])), kAlphaMax) : 0.f;
        const f2 w = mul2(pk2(al, ah), T[p]);
        fma2_acc(c0[p], bc(b.z), w);
        fma2_acc(c1[p], bc(b.w), w);
        fma2_acc(c2[p], bc(cb), w);
        sub2_acc(T[p], w);
        last[2 * p] = valid[2 * p] ? pos : last[2 * p];
        last[2 * p + 1] = valid[2 * p + 1] ? pos : last[2 * p + 1];
      }
    }
    if (used && lane == 0) used[used_slot(rg.x, tile, (base - rg.x) >> 5) * WPT + sub] = used_bits;
  }
#pragma unroll
  for (int k = 0; k < STRIP; ++k) {
    const int py = py0 + k;
    const int p = k >> 1;
    const bool h = k & 1;
    if (px < width && py < height) {
      const int64_t q = (int64_t)py * width + px;
      img[3 * q] = h ? hi2(c0[p]) : lo2(c0[p]);
      img[3 * q + 1] = h ? hi2(c1[p]) : lo2(c1[p]);
      img[3 * q + 2] = h ? hi2(c2[p]) : lo2(c2[p]);
      t_final[q] = h ? hi2(T[p]) : lo2(T[p]);
      n_contrib[q] = last[k];
    }
  }
  if (tile_work) {
    // the entries this warp's backward will walk (its pixels' longest
    // contributor prefix), summed per tile: the backward's launch order
    int mx = 0;
#pragma unroll
    for (int k = 0; k < STRIP; ++k) mx = max(mx, last[k]);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0 && mx > 0) atomicAdd(&tile_work[tile], mx);
  }
}

// Transposed warp reduction of 9 values in 12 shuffles: each round halves
// (unevenly) the slots a lane keeps -- 9 -> 5 (xor 16) -> 3 (xor 8) -> 2 (xor 4)
// -> 1 (xor 2) -> +xor 1.  Afterwards lane L (bits b4..b0) holds the warp total
// of value 5 b4 + 3 b3 + 2 b2 + b1 when red9_slot marks it valid (L and L^1 agree).
__device__ __forceinline__ float red_round(float lo, float hi, bool up, int off) {
  const float send = up ? lo : hi;
  const float keep = up ? hi : lo;
  return keep + __shfl_xor_sync(0xffffffffu, send, off);
}

__device__ __forceinline__ float reduce9(const float v[9], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  float w[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) w[i] = red_round(v[i], i + 5 < 9 ? v[i + 5] : 0.f, b4, 16);
  float x[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) x[i] = red_round(w[i], i + 3 < 5 ? w[i + 3] : 0.f, b3, 8);
  float y[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) y[i] = red_round(x[i], i + 2 < 3 ? x[i + 2] : 0.f, b2, 4);
  const float z = red_round(y[0], y[1], b1, 2);
  return z + __shfl_xor_sync(0xffffffffu, z, 1);
}

__device__ __forceinline__ int red9_slot(int lane, bool& valid) {
  const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1;
  const int p = 3 * b3 + 2 * b2 + b1;
  valid = !(lane & 1) && !(b2 && (b1 || b3)) && (b4 == 0 ? p < 5 : p < 4);
  return 5 * b4 + p;
}

// Batched per-entry reduction (the default, non-deterministic backward): a
// warp parks each blended entry's 32 x 9 lane values in shared memory,
// component-major (value c of lane l at [entry][c][l]: 9 STS.32 per lane),
// and every kRedE = 3 entries reduces them at once: lane L < 27 owns the sum
// (entry L / 9, component L % 9), reads its 32 contiguous lane values with
// 8 LDS.128, adds them (4 running sums) and issues one float atomic into
// g2d.  ~22 instructions per entry instead of the 12-shuffle transposed warp
// reduction's ~50 (and of the earlier lane-major rows + shuffle rounds'
// ~35).  Component rows are padded to 36 floats and entries are 324 floats
// apart (= 4 mod 32), so a quarter-warp's LDS.128 hit 8 distinct 4-bank
// groups.
constexpr int kRedE = 3;
constexpr int kRedCompPitch = 36;                  // floats per component row (32 used)
constexpr int kRedStride = 9 * kRedCompPitch;      // floats per entry
constexpr int kRedWarpFloats = kRedE * kRedStride;
static_assert(kRedE * 9 <= 32, "one sum per lane");
constexpr int kRedWarpTotal = kRedWarpFloats + 4;  // + entry ids; keeps 16-B alignment
static_assert(kRedWarpFloats % 4 == 0 && kRedE <= 4, "16-B aligned per-warp buffers");

__device__ __forceinline__ void red_flush(const float* buf, const int* gid, int nacc, int lane,
                                          float* __restrict__ g2d) {
  __syncwarp();
  if (lane < 9 * nacc) {
    const int e = lane / 9, c = lane - 9 * e;
    const float4* row = reinterpret_cast<const float4*>(buf + e * kRedStride + c * kRedCompPitch);
    // the 32 values as 8 float4, summed as packed pairs (FADD2)
    float4 q = row[0];
    f2 sa = pk2(q.x, q.y), sb = pk2(q.z, q.w);
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      q = row[k];
      sa = add2(sa, pk2(q.x, q.y));
      sb = add2(sb, pk2(q.z, q.w));
    }
    sa = add2(sa, sb);
    SS_DCHECK(gid[e] >= 0);
    atomicAdd(g2d + (int64_t)gid[e] * SS_G2D_ROW + c, lo2(sa) + hi2(sa));
  }
  __syncwarp();
}

// Deterministic mode (DET): instead of float atomics into g2d, a warp writes
// its 9 reduced values for an entry to partial[(e * WPT + sub) * 9 + c], where
// e is the entry's position in emit order (rank-ordered runs per splat, see
// binning.cu) -- recovered from the splat's rank, its kept-tile mask and a
// popcount -- and g2d_reduce_kernel sums each splat's run in a fixed order.
struct DetArgs {
  float* partial;
  const int32_t* rank;
  const int32_t* offsets;
  const int4* bbox;
  const uint64_t* tile_mask;
  const float* geom;
};

__device__ __forceinline__ int64_t emit_position(const DetArgs& d, int g, int tx, int ty) {
  const int4 bb = d.bbox[g];
  const int tx0 = bb.x / kTile, tx1 = (bb.y - 1) / kTile + 1, ty0 = bb.z / kTile;
  const int w = tx1 - tx0;
  const int local = (ty - ty0) * w + (tx - tx0);
  const uint64_t mask = d.tile_mask[g];
  int j;
  if (local < 64) {
    j = __popcll(mask & ((1ull << local) - 1ull));
  } else {
    j = __popcll(mask);
    float gl[kGeom];
#pragma unroll
    for (int c = 0; c < kGeom; ++c) gl[c] = d.geom[(int64_t)g * kGeom + c];
    for (int q = 64; q < local; ++q) j += tile_keeps(gl, tx0 + q % w, ty0 + q / w, bb);
  }
  return (int64_t)d.offsets[d.rank[g]] + j;
}

template <int STRIP, bool DET, bool BB = false>
__global__ void __launch_bounds__(kWarps * 32, SS_BWD_MINB)
    raster_bwd_kernel(const int2* __restrict__ ranges, const int32_t* __restrict__ vals,
                      const float4* __restrict__ rec_a, const float4* __restrict__ rec_b,
                      const float* __restrict__ rec_c, int width, int height, int tiles_x,
                      int n_tiles, const int32_t* __restrict__ tile_order,
                      const float* __restrict__ dimg, const float* __restrict__ t_final,
                      const int32_t* __restrict__ n_contrib, float* __restrict__ g2d,
                      DetArgs det, float lfloor, const int4* __restrict__ pbox = nullptr,
                      const uint32_t* __restrict__ used = nullptr) {
  pdl_wait();
  if (SS_RASTER_EARLY_TRIGGER) pdl_trigger();
  __shared__ int64_t s_epos[kWarps][DET ? 32 : 1];
  __shared__ WarpStage s_stage[kWarps];
  extern __shared__ __align__(16) float s_red[];  // !DET: kWarps x (entry rows + ids)
  constexpr int WPT = kTile / (2 * STRIP);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gwarp = blockIdx.x * kWarps + warp;
  const int slot_id = gwarp / WPT, sub = gwarp % WPT;
  if (slot_id >= n_tiles) return;
  const int tile = tile_order ? tile_order[slot_id] : slot_id;
  WarpStage& st = s_stage[warp];
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * kTile + (lane & 15);
  const int py0 = ty * kTile + sub * 2 * STRIP + (lane >> 4) * STRIP;
  const float fx = (float)px, fy0 = (float)py0;
  const float rx0 = (float)(tx * kTile), ry0 = (float)(ty * kTile + sub * 2 * STRIP);
  const float ry1 = ry0 + (float)(2 * STRIP - 1);
  constexpr int NP = STRIP / 2;
  // T: transmittance (after the current entry, walking back to front);
  // nQ = -(suffix colour Q); dimg channels per pixel pair
  f2 T[NP], d0[NP], d1[NP], d2[NP], nQ[NP];
  int last[STRIP];
  int my_max = 0;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    float tv[2], dv0[2], dv1[2], dv2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 2 * p + h, py = py0 + k;
      if (px < width && py < height) {
        const int64_t q = (int64_t)py * width + px;
        tv[h] = t_final[q];
        last[k] = n_contrib[q];
        dv0[h] = dimg[3 * q];
        dv1[h] = dimg[3 * q + 1];
        dv2[h] = dimg[3 * q + 2];
      } else {
        tv[h] = 1.f;
        last[k] = 0;
        dv0[h] = dv1[h] = dv2[h] = 0.f;
      }
      my_max = max(my_max, last[k]);
    }
    T[p] = pk2(tv[0], tv[1]);
    d0[p] = pk2(dv0[0], dv0[1]);
    d1[p] = pk2(dv1[0], dv1[1]);
    d2[p] = pk2(dv2[0], dv2[1]);
    nQ[p] = bc(0.f);
  }
  const int2 rg = ranges[tile];
  const int walk_end = rg.x + __reduce_max_sync(0xffffffffu, my_max);
  SS_DCHECK(rg.x >= 0 && rg.x <= rg.y && walk_end <= rg.y);
  bool slot_ok;
  const int slot = red9_slot(lane, slot_ok);
  float* rbuf = s_red + warp * kRedWarpTotal;
  int* rgid = reinterpret_cast<int*>(rbuf + kRedWarpFloats);
  int nacc = 0;  // entries parked in rbuf (warp-uniform)
  float* park = rbuf + lane;  // this lane's column of the next parked entry
  int* gidp = rgid;           // and the next entry's splat id
  const bool lane0 = lane == 0;
  if (DET) {
    // entries this warp never visits contribute zero partials
    for (int idx = walk_end + lane; idx < rg.y; idx += 32) {
      const int64_t e = emit_position(det, vals[idx], tx, ty);
      float* dst = det.partial + (e * WPT + sub) * 9;
#pragma unroll
      for (int c = 0; c < 9; ++c) dst[c] = 0.f;
    }
  }
  // batches aligned with the forward's (list positions rg.x + 32 b ...),
  // walked back to front from the one holding walk_end - 1
  for (int bt = (walk_end - rg.x - 1) >> 5; bt >= 0; --bt) {
    const int start = rg.x + 32 * bt;
    const int end = min(start + 32, walk_end);
    __syncwarp();
    bool touch = false;
    const bool mine = start + lane < end;
    // the forward's entry-use mask, else the per-entry region test
    const uint32_t umask = used ? used[used_slot(rg.x, tile, bt) * WPT + sub] : ~0u;
    const bool want = mine && ((umask >> lane) & 1u);
    if (DET ? mine : want) {
      const int g = __ldg(vals + start + lane);
      const float4 a = __ldg(rec_a + g), b = __ldg(rec_b + g);
      st.g[lane] = g;
      st.a[lane] = a;
      st.b[lane] = b;
      st.c[lane] = __ldg(rec_c + g);
      touch = want && (used || touches_rect(a, b, rx0, ry0, ry1, lfloor));
      if (DET) {
        const int64_t ep = emit_position(det, g, tx, ty);
        s_epos[warp][lane] = ep;
        if (!touch) {  // an entry the warp does not walk: zero partials
          float* dst = det.partial + (ep * WPT + sub) * 9;
#pragma unroll
          for (int c = 0; c < 9; ++c) dst[c] = 0.f;
        }
      }
    }
    uint32_t todo = __ballot_sync(0xffffffffu, touch);
    __syncwarp();
    while (todo) {
      const int j = 31 - __clz(todo);  // back to front
      todo &= ~(1u << j);
      const int pos = start - rg.x + j;  // 0-based position in the tile list
      const float4 a = st.a[j];
      const float4 b = st.b[j];
      const float cb = st.c[j];
      const StripQuad s = strip_quad(a, b, fx, fy0, lfloor);
      f2 e[NP];
      strip_exps<NP>(s, e);
      bool valid[STRIP];
      bool any = false;
      int4 q = make_int4(0, 0, 0, 0);
      if (BB) q = __ldg(pbox + st.g[j]);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        valid[2 * p] = (pos < last[2 * p]) && (lo2(e[p]) >= s.thr);
        valid[2 * p + 1] = (pos < last[2 * p + 1]) && (hi2(e[p]) >= s.thr);
        if (BB) {
          const bool xin = px >= q.x && px < q.y;
          valid[2 * p] &= xin && py0 + 2 * p >= q.z && py0 + 2 * p < q.w;
          valid[2 * p + 1] &= xin && py0 + 2 * p + 1 >= q.z && py0 + 2 * p + 1 < q.w;
        }
        any |= valid[2 * p] | valid[2 * p + 1];
      }
      // an entry the forward marked used has a valid pixel here (same
      // exponents, pos < last of the pixel that used it): no vote needed
      if ((DET || !used) && !__any_sync(0xffffffffu, any)) {
        if (DET && slot_ok) det.partial[(s_epos[warp][j] * WPT + sub) * 9 + slot] = 0.f;
        continue;
      }
      f2 nsc0, nsc1, nsc2, tp[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        // branch-free: an invalid pixel has alpha' = 0 (T and Q unchanged)
        // and a zero gradient weight g
        const float gl = ex2(lo2(e[p])), gh = ex2(hi2(e[p]));
        const bool vl = valid[2 * p], vh = valid[2 * p + 1];
        const f2 nap = pk2(vl ? fmaxf(-gl, -kAlphaMax) : 0.f, vh ? fmaxf(-gh, -kAlphaMax) : 0.f);
        // clamped splats pass no alpha/footprint gradient (_kernels.py:120-121);
        // -nap is alpha' = alpha G for a valid unclamped pixel and 0 when invalid
        const f2 g = pk2(gl <= kAlphaMax ? -lo2(nap) : 0.f, gh <= kAlphaMax ? -hi2(nap) : 0.f);
        const f2 om = add2(bc(1.f), nap);  // 1 - alpha'
        const f2 inv = pk2(rcp(lo2(om)), rcp(hi2(om)));
        const f2 Ta = T[p];
        mul2_acc(T[p], inv);                  // T before this splat
        const f2 nw = mul2(nap, T[p]);        // -w
        const f2 dc = fma2(d2[p], bc(cb), fma2(d1[p], bc(b.w), mul2(d0[p], bc(b.z))));
        const f2 dap = mul2(inv, fma2(Ta, dc, nQ[p]));  // T dc - Q / (1 - alpha')
        fma2_acc(nQ[p], nw, dc);
        tp[p] = mul2(g, dap);
        if (p == 0) {
          nsc0 = mul2(d0[p], nw);
          nsc1 = mul2(d1[p], nw);
          nsc2 = mul2(d2[p], nw);
        } else {
          nsc0 = fma2(d0[p], nw, nsc0);
          nsc1 = fma2(d1[p], nw, nsc1);
          nsc2 = fma2(d2[p], nw, nsc2);
        }
      }
      // strip moments sum t, sum t k, sum t k^2 with immediate k, k^2
      f2 st0 = tp[0];
#pragma unroll
      for (int p = 1; p < NP; ++p) st0 = add2(st0, tp[p]);
      float s_tk = hi2(tp[0]), s_tkk = hi2(tp[0]);
#pragma unroll
      for (int k = 2; k < STRIP; ++k) {
        const float tk = (k & 1) ? hi2(tp[k >> 1]) : lo2(tp[k >> 1]);
        s_tk = fmaf((float)k, tk, s_tk);
        s_tkk = fmaf((float)(k * k), tk, s_tkk);
      }
      // strip sums -> the 9 basis sums of the footprint gradient (with
      // dy = dy0 + k):  t dx, t dy, t dx^2, t dx dy, t dy^2, t, colour.  The
      // per-splat constants (the conic, 1/alpha) are applied once per splat
      // in ss_project_bwd, so only lane-dependent factors are formed here.
      const float s_t = lo2(st0) + hi2(st0);
      const float dx = s.dx, dy0 = s.dy0;
      const float s_dy = fmaf(dy0, s_t, s_tk);                               // sum t dy
      const float s_dyy = fmaf(dy0, fmaf(dy0, s_t, s_tk + s_tk), s_tkk);     // sum t dy^2
      float v[9];
      v[0] = dx * s_t;
      v[1] = s_dy;
      v[2] = dx * v[0];
      v[3] = dx * s_dy;
      v[4] = s_dyy;
      v[5] = s_t;
      // -(a + b) written as (-a) - b: one FADD with both operands negated
      // (the compiler may not fold the negation itself: the two differ only
      // in the sign of a zero sum, which no gradient sees)
      v[6] = -lo2(nsc0) - hi2(nsc0);
      v[7] = -lo2(nsc1) - hi2(nsc1);
      v[8] = -lo2(nsc2) - hi2(nsc2);
      if (DET) {
        const float tot = reduce9(v, lane);
        if (slot_ok) det.partial[(s_epos[warp][j] * WPT + sub) * 9 + slot] = tot;
      } else {
        // park through a running pointer (one add per entry instead of the
        // entry-index multiply-add)
#pragma unroll
        for (int c = 0; c < 9; ++c) park[c * kRedCompPitch] = v[c];
        park += kRedStride;
        if (lane0) *gidp = st.g[j];
        ++gidp;
        if (++nacc == kRedE) {
          red_flush(rbuf, rgid, nacc, lane, g2d);
          nacc = 0;
          park = rbuf + lane;
          gidp = rgid;
        }
      }
    }
  }
  if (!DET && nacc > 0) red_flush(rbuf, rgid, nacc, lane, g2d);
}

__global__ void rank_kernel(const int32_t* __restrict__ order, int n, int32_t* __restrict__ rank) {
  pdl_wait();
  pdl_trigger();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) rank[order[k]] = k;
}

// Fixed-order sum of each splat's partials (emit order, then warp sub-tile).
__global__ void g2d_reduce_kernel(const float* __restrict__ partial,
                                  const int32_t* __restrict__ order,
                                  const int32_t* __restrict__ offsets, int n, int wpt,
                                  float* __restrict__ g2d) {
  pdl_wait();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  float acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0.f;
  const int64_t e0 = offsets[k], e1 = offsets[k + 1];
  for (int64_t e = e0 * wpt; e < e1 * wpt; ++e) {
#pragma unroll
    for (int c = 0; c < 9; ++c) acc[c] += partial[e * 9 + c];
  }
  float* dst = g2d + (int64_t)order[k] * SS_G2D_ROW;
#pragma unroll
  for (int c = 0; c < 9; ++c) dst[c] = acc[c];
}

// log2 of the alpha floor as the kernels' threshold (-inf: off)
static float floor_threshold() {
  const int lf = alpha_floor_log2();
  return lf ? (float)lf : -INFINITY;
}

// dynamic shared memory of the non-deterministic backward (reduction rows)
constexpr size_t kBwdSmem = sizeof(float) * kWarps * kRedWarpTotal;

static int g_strip = 4;       // backward strip
static int g_strip_fwd = 4;   // forward strip

}  // namespace ss

using namespace ss;

extern "C" int ss_set_raster_strip(int32_t strip) {
  if (strip != 2 && strip != 4 && strip != 8)
    return set_error(SS_ERR_INVALID, "ss_set_raster_strip: strip must be 2, 4 or 8");
  g_strip = strip;
  g_strip_fwd = strip;
  return SS_OK;
}

extern "C" int ss_set_raster_strips(int32_t strip_fwd, int32_t strip_bwd) {
  const auto ok = [](int s) { return s == 2 || s == 4 || s == 8; };
  if (!ok(strip_fwd) || !ok(strip_bwd))
    return set_error(SS_ERR_INVALID, "ss_set_raster_strips: strips must be 2, 4 or 8");
  g_strip_fwd = strip_fwd;
  g_strip = strip_bwd;
  return SS_OK;
}

// Forward launch; pbox != nullptr selects the explicit per-pixel bbox test
// (strip 4); used != nullptr records the entry-use masks.
int raster_fwd_ex(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                  const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                  const int32_t* tile_order, float* img, float* t_final, int32_t* n_contrib,
                  const int32_t* pbox, uint32_t* used, int32_t* tile_work, cudaStream_t stream) {
  if (width <= 0 || height <= 0) return set_error(SS_ERR_INVALID, "ss_raster_fwd: bad size");
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int n_tiles = tiles_x * tiles_y;
  const int strip = pbox ? 4 : g_strip_fwd;
  const int wpt = kTile / (2 * strip);
  const int blocks = (n_tiles * wpt + kWarpsF - 1) / kWarpsF;
#define SS_FWD(S, B)                                                                          \
  launch_kx(SS_RASTER_PDL, raster_fwd_kernel<S, B>, blocks, kWarpsF * 32, 0, stream,         \
      (const int2*)ranges, vals, (const float4*)rec_a, (const float4*)rec_b, rec_c, width,  \
      height, tiles_x, n_tiles, tile_order, img, t_final, n_contrib, floor_threshold(),     \
      (const int4*)pbox, used, tile_work)
  if (pbox) SS_FWD(4, true);
  else if (strip == 8) SS_FWD(8, false);
  else if (strip == 4) SS_FWD(4, false);
  else SS_FWD(2, false);
#undef SS_FWD
  return check_launch("ss_raster_fwd");
}

extern "C" int ss_raster_fwd(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                             const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                             const int32_t* tile_order, float* img, float* t_final,
                             int32_t* n_contrib, cudaStream_t stream) {
  return raster_fwd_ex(ranges, vals, rec_a, rec_b, rec_c, width, height, tile_order, img, t_final,
                       n_contrib, nullptr, nullptr, nullptr, stream);
}

// Backward launch; det selects the deterministic partials, pbox the bbox
// test (strip 4), used the forward's entry-use masks (else the region test).
int raster_bwd_ex(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                  const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                  const int32_t* tile_order, const float* dimg, const float* t_final,
                  const int32_t* n_contrib, float* g2d, const DetArgs* det, const int32_t* pbox,
                  const uint32_t* used, cudaStream_t stream) {
  if (width <= 0 || height <= 0) return set_error(SS_ERR_INVALID, "ss_raster_bwd: bad size");
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int n_tiles = tiles_x * tiles_y;
  const int strip = pbox ? 4 : g_strip;
  const int wpt = kTile / (2 * strip);
  const int blocks = (n_tiles * wpt + kWarps - 1) / kWarps;
  DetArgs d = det ? *det : DetArgs{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int rc = 0;
#define SS_BWD(S, D, B)                                                                       \
  do {                                                                                        \
    if (!D && (rc = ensure_smem((const void*)raster_bwd_kernel<S, D, B>, kBwdSmem))) return rc; \
    launch_kx(SS_RASTER_PDL, raster_bwd_kernel<S, D, B>, blocks, kWarps * 32, D ? 0 : kBwdSmem, \
              stream,                                                                         \
        (const int2*)ranges, vals, (const float4*)rec_a, (const float4*)rec_b, rec_c, width, \
        height, tiles_x, n_tiles, tile_order, dimg, t_final, n_contrib, g2d, d,              \
        floor_threshold(), (const int4*)pbox, used);                                          \
  } while (0)
  if (pbox) {
    SS_BWD(4, false, true);
  } else if (det) {
    if (strip == 8) SS_BWD(8, true, false);
    else if (strip == 4) SS_BWD(4, true, false);
    else SS_BWD(2, true, false);
  } else {
    if (strip == 8) SS_BWD(8, false, false);
    else if (strip == 4) SS_BWD(4, false, false);
    else SS_BWD(2, false, false);
  }
#undef SS_BWD
  return check_launch("ss_raster_bwd");
}

extern "C" int ss_raster_bwd(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                             const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                             const int32_t* tile_order, const float* dimg, const float* t_final,
                             const int32_t* n_contrib, float* g2d, cudaStream_t stream) {
  return raster_bwd_ex(ranges, vals, rec_a, rec_b, rec_c, width, height, tile_order, dimg,
                       t_final, n_contrib, g2d, nullptr, nullptr, nullptr, stream);
}

// Words of entry-use mask storage for K pairs over n_tiles tiles (every
// strip: up to 4 warps per tile).
extern "C" int64_t ss_raster_used_words(int64_t n_pairs, int32_t n_tiles) {
  return 4 * (n_pairs / 32 + (int64_t)n_tiles + 2);
}

// masks are shared by the forward and backward warp mappings only when their
// strips are equal
bool raster_masks_usable() { return g_strip == g_strip_fwd; }

extern "C" int64_t ss_raster_partial_floats(int64_t n_pairs) {
  return n_pairs * (kTile / (2 * g_strip)) * 9;
}

int raster_bwd_det_ex(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                      const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                      const int32_t* tile_order, const float* dimg, const float* t_final,
                      const int32_t* n_contrib, const int32_t* order, const int32_t* offsets,
                      const int32_t* bbox, const uint64_t* tile_mask, const float* geom, int32_t n,
                      int32_t* rank, float* partial, float* g2d, const uint32_t* used,
                      cudaStream_t stream) {
  if (n <= 0) return SS_OK;
  launch_k(rank_kernel, grid_for(n, 256), 256, 0, stream, order, n, rank);
  DetArgs d{partial, rank, offsets, (const int4*)bbox, tile_mask, geom};
  int rc = raster_bwd_ex(ranges, vals, rec_a, rec_b, rec_c, width, height, tile_order, dimg,
                         t_final, n_contrib, g2d, &d, nullptr, used, stream);
  if (rc) return rc;
  launch_k(g2d_reduce_kernel, grid_for(n, 128), 128, 0, stream, partial, order, offsets, n,
                                                           kTile / (2 * g_strip), g2d);
  return check_launch("ss_raster_bwd_deterministic");
}

int raster_bwd_plain_ex(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                        const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                        const int32_t* tile_order, const float* dimg, const float* t_final,
                        const int32_t* n_contrib, float* g2d, const int32_t* pbox,
                        const uint32_t* used, cudaStream_t stream) {
  return raster_bwd_ex(ranges, vals, rec_a, rec_b, rec_c, width, height, tile_order, dimg,
                       t_final, n_contrib, g2d, nullptr, pbox, used, stream);
}

extern "C" int ss_raster_bwd_deterministic(
    const int32_t* ranges, const int32_t* vals, const void* rec_a, const void* rec_b,
    const float* rec_c, int32_t width, int32_t height, const int32_t* tile_order,
    const float* dimg, const float* t_final, const int32_t* n_contrib, const int32_t* order,
    const int32_t* offsets, const int32_t* bbox, const uint64_t* tile_mask, const float* geom,
    int32_t n, int32_t* rank, float* partial, float* g2d, cudaStream_t stream) {
  return raster_bwd_det_ex(ranges, vals, rec_a, rec_b, rec_c, width, height, tile_order, dimg,
                           t_final, n_contrib, order, offsets, bbox, tile_mask, geom, n, rank,
                           partial, g2d, nullptr, stream);
}
