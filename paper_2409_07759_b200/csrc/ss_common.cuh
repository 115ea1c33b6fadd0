// Shared helpers for the libswings.so kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/swings.h"

// Device-side invariant / bounds checks of the checked build (-DSS_CHECKED,
// lib/libswings_checked.so): a violation prints its site and traps.
#ifdef SS_CHECKED
#include <cstdio>
#define SS_DCHECK(cond)                                                                   \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("SS_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,    \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                \
      asm volatile("trap;");                                                              \
    }                                                                                     \
  } while (0)
#else
#define SS_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace ss {

constexpr float kAlphaMax = 0.999f;       // _kernels.py:15
constexpr float kTMin = 1e-4f;            // _kernels.py:16
constexpr float kMahaMax = 64.0f;         // _kernels.py:17
constexpr double kNearPlane = 0.01;       // raster.py:31
constexpr double kDilation = 0.3;         // raster.py:34
constexpr int kTile = SS_TILE;
constexpr int kTilePix = kTile * kTile;

int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  return (int)g;
}

// Row accessor: r < n_opt -> optimizable row (log-scale, logit); else matured.
struct StoreView {
  const double* opt;
  int64_t n_opt;
  const double* mat;
};

// Gaussian in direct space, fp64 (core.py:153-176).
struct Gauss64 {
  double mean[3];
  double quat[4];
  double scale[3];
  double opacity;
  double color[3];
};

__device__ __forceinline__ void load_row(const StoreView& s, int32_t row, Gauss64& g) {
  const bool opt = row < s.n_opt;
  const double* p = opt ? s.opt + (int64_t)row * SS_ROW : s.mat + (int64_t)(row - s.n_opt) * SS_ROW;
#pragma unroll
  for (int k = 0; k < 3; ++k) g.mean[k] = p[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) g.quat[k] = p[3 + k];
#pragma unroll
  for (int k = 0; k < 3; ++k) g.scale[k] = p[7 + k];
  g.opacity = p[10];
#pragma unroll
  for (int k = 0; k < 3; ++k) g.color[k] = p[11 + k];
  if (opt) {
    // train.py:155-161: exp(log_scale), 1 / (1 + exp(-logit))
#pragma unroll
    for (int k = 0; k < 3; ++k) g.scale[k] = exp(g.scale[k]);
    g.opacity = 1.0 / (1.0 + exp(-g.opacity));
  }
}

// Non-contracted fp64 helpers: structural quantities (z, cull, bbox) follow
// numpy's separate multiply/add roundings rather than fused FMAs.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// core.py:231-251 rotation matrix of a unit (w, x, y, z) quaternion, with
// numpy's rounding sequence (no FMA contraction).
__device__ __forceinline__ void quat_to_rot(const double q[4], double r[3][3]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  r[0][0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(z, z))));
  r[0][1] = dmul(2.0, dsub(dmul(x, y), dmul(w, z)));
  r[0][2] = dmul(2.0, dadd(dmul(x, z), dmul(w, y)));
  r[1][0] = dmul(2.0, dadd(dmul(x, y), dmul(w, z)));
  r[1][1] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(z, z))));
  r[1][2] = dmul(2.0, dsub(dmul(y, z), dmul(w, x)));
  r[2][0] = dmul(2.0, dsub(dmul(x, z), dmul(w, y)));
  r[2][1] = dmul(2.0, dadd(dmul(y, z), dmul(w, x)));
  r[2][2] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
}

// Exact ellipse-vs-tile test (a-4 refinement).  A tile row (pixel-centre
// rows [Y0, Y1], clipped to the bbox) meets the ellipse m <= M (m = i0 dx^2
// + 2 i1 dx dy + i2 dy^2, M = the splat's cull_margin) in an x-interval [L, R]: the right
// end is max over the row of (-i1 dy + sqrt(i0 M - det dy^2)) / i0, reached at
// dy = -sy clamped into the row (sy = i1 sqrt(M / (i2 det)), the ellipse's
// rightmost point), the left end symmetric at +sy; rows beyond |dy| <= ymax =
// sqrt(M i0 / det) miss it.  A tile is kept iff its pixel-centre columns
// [X0, X1] meet [L, R].  Per-splat constants come from fp64 (rounded once);
// the row/tile arithmetic is fp32 with every operation explicitly rounded (no
// FMA contraction), the sequence of oracle/splat_oracle.py tile_row_span in
// numpy float32, so keep / drop decisions (and tile keys) are bit-identical
// to it.  M = 64.0625 keeps a 1e-3 relative margin over the maha <= 64 cut
// (pixels beyond it blend nothing), far above the fp32 rounding.
constexpr float kCullMargin = 64.0625f;
constexpr double kCullMarginD = 64.0625;
constexpr int kGeom = 8;  // floats per splat: u, v, i0 M, i1, det, sy, ymax, 1/i0
constexpr double kTwoLn2 = 1.3862943611198906;

int32_t alpha_floor_log2();  // ss_api.cu: 0 (off) or the floor's log2 (ss_set_alpha_floor)

// Per-splat maha margin M of the tile test: the reference's m <= 64 cut
// (kCullMarginD, 1e-3 margin) or, with the alpha floor 2^lf, also
// alpha G >= 2^lf, i.e. m <= 2 ln(alpha / 2^lf).  With alpha = f 2^e
// (frexp, f in [0.5, 1)) and ln f <= f - 1, the bound
// (2 (f - 1) + 2 ln2 (e - lf)) (1 + 2^-10) + 2^-4 uses IEEE-rounded fp64
// operations only, so oracle/splat_oracle.py cull_margin reproduces it bit
// for bit.  M <= 0: the splat reaches no pixel.
__device__ __forceinline__ double cull_margin(double alpha, int lf) {
  if (lf == 0) return kCullMarginD;
  if (!(alpha > 0.0)) return -1.0;
  int e;
  const double f = frexp(alpha, &e);
  double m = dadd(dmul(2.0, dsub(f, 1.0)), dmul(kTwoLn2, (double)(e - lf)));
  m = dadd(dmul(m, 1.0009765625), 0.0625);
  return fmin(m, kCullMarginD);
}

__device__ __forceinline__ float fmr(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float far_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsr(float a, float b) { return __fsub_rn(a, b); }

__device__ __forceinline__ float clampf(float x, float lo, float hi) {
  return fminf(fmaxf(x, lo), hi);
}

// geom of a splat from its fp64 centre, conic and margin M (> 0)
__device__ __forceinline__ void make_geom(double ux, double uy, double i0, double i1, double i2,
                                          double M, float* g) {
  const double det = __dsub_rn(__dmul_rn(i0, i2), __dmul_rn(i1, i1));
  const double sy = __dmul_rn(i1, __dsqrt_rn(__ddiv_rn(M, __dmul_rn(i2, det))));
  const double ymax = __dsqrt_rn(__ddiv_rn(__dmul_rn(M, i0), det));
  const float fi0 = __double2float_rn(i0);
  g[0] = __double2float_rn(ux);
  g[1] = __double2float_rn(uy);
  g[2] = __double2float_rn(__dmul_rn(i0, M));
  g[3] = __double2float_rn(i1);
  g[4] = __double2float_rn(det);
  g[5] = __double2float_rn(sy);
  g[6] = __double2float_rn(ymax);
  g[7] = __frcp_rn(fi0);
}

// x-interval [L, R] (relative to u) of the ellipse within tile row ty;
// false when the row misses the ellipse.  bb = pixel bbox (x0, x1, y0, y1).
__device__ __forceinline__ bool row_span(const float* g, int ty, int4 bb, float& L, float& R) {
  const float v = g[1], m0 = g[2], i1 = g[3], det = g[4], sy = g[5], ymax = g[6], r0 = g[7];
  const float lo = fmaxf(fsr((float)max(ty * SS_TILE, bb.z), v), -ymax);
  const float hi = fminf(fsr((float)min(ty * SS_TILE + SS_TILE - 1, bb.w - 1), v), ymax);
  if (lo > hi) return false;
  const float cR = clampf(-sy, lo, hi), cL = clampf(sy, lo, hi);
  const float sR = __fsqrt_rn(fmaxf(fsr(m0, fmr(fmr(det, cR), cR)), 0.0f));
  const float sL = __fsqrt_rn(fmaxf(fsr(m0, fmr(fmr(det, cL), cL)), 0.0f));
  R = fmr(far_(fmr(-i1, cR), sR), r0);
  L = fmr(fsr(fmr(-i1, cL), sL), r0);
  return true;
}

__device__ __forceinline__ bool col_meets(const float* g, int tx, int4 bb, float L, float R) {
  const float ax = fsr((float)max(tx * SS_TILE, bb.x), g[0]);
  const float bx = fsr((float)min(tx * SS_TILE + SS_TILE - 1, bb.y - 1), g[0]);
  return ax <= R && bx >= L;
}

__device__ __forceinline__ bool tile_keeps(const float* g, int tx, int ty, int4 bb) {
  float L, R;
  return row_span(g, ty, bb, L, R) && col_meets(g, tx, bb, L, R);
}

// Packed fp32 pairs (Blackwell FFMA2 / FMUL2 / FADD2, PTX *.f32x2): two fp32
// values share one 64-bit register pair and one instruction issue (raster:
// a lane's pixels 2p / 2p + 1; SSIM: two blurred quantities).  A scalar
// operand broadcast with bc() folds into the instruction.
typedef float2 f2;

// CUDA's sm_100 float2 intrinsics (FFMA2 / FMUL2 / FADD2); values stay in
// ordinary register pairs, so the compiler allocates them in place.
__device__ __forceinline__ f2 pk2(float lo, float hi) { return make_float2(lo, hi); }
__device__ __forceinline__ float lo2(f2 r) { return r.x; }
__device__ __forceinline__ float hi2(f2 r) { return r.y; }
__device__ __forceinline__ f2 bc(float s) { return make_float2(s, s); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ f2 add2(f2 a, f2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ f2 sub2(f2 a, f2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// in-place accumulator forms
__device__ __forceinline__ void fma2_acc(f2& c, f2 a, f2 b) { c = __ffma2_rn(a, b, c); }
__device__ __forceinline__ void sub2_acc(f2& c, f2 a) { c = sub2(c, a); }
__device__ __forceinline__ void mul2_acc(f2& c, f2 a) { c = __fmul2_rn(c, a); }


// Programmatic dependent launch (sm_90+): every kernel of the library is
// launched with programmatic stream serialisation, so its CTAs may be
// scheduled while the previous kernel in the stream is finishing; each kernel
// begins with pdl_wait() (griddepcontrol.wait: the previous grid has completed
// and its writes are visible), so the data dependence is unchanged -- only
// the launch gap between consecutive kernels is hidden.  pdl_trigger()
// (griddepcontrol.launch_dependents) lets the next kernel be scheduled early;
// multi-wave kernels leave it to their exit so waiting dependents do not take
// SM slots from their later waves.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // ss_api.cu: false when SS_NO_PDL=1 (diagnostics: true kernel spans)

// pdl = false: an ordinary launch (the kernel starts only after its
// predecessor completes; its griddepcontrol.wait returns at once)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kx(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                             size_t smem, cudaStream_t stream, Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = pdl && pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t stream, Args&&... args) {
  return launch_kx(true, kernel, grid, block, smem, stream, static_cast<Args&&>(args)...);
}

// Philox4x32-10 counter-based generator (Salmon et al., SC'11).
struct Philox4 {
  uint32_t v[4];
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                  uint32_t c3, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0; k1 += W1;
  }
  Philox4 r;
  r.v[0] = c0; r.v[1] = c1; r.v[2] = c2; r.v[3] = c3;
  return r;
}

// Uniform in (0, 1] from 32 random bits, fp64 (53-bit from two words).
__device__ __forceinline__ double u01_53(uint32_t a, uint32_t b) {
  uint64_t x = ((uint64_t)(a >> 5) << 26) | (uint64_t)(b >> 6);   // 27 + 26 = 53 bits
  return ((double)x + 1.0) * (1.0 / 9007199254740992.0);
}

}  // namespace ss

// raster.cu: launches used by the view driver (csrc/view.cu).  pbox !=
// nullptr selects the explicit per-pixel bbox test (2D-input path); used !=
// nullptr records (forward) / consumes (backward) the entry-use masks
// (ss_raster_used_words words; only when raster_masks_usable()).
int raster_fwd_ex(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                  const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                  const int32_t* tile_order, float* img, float* t_final, int32_t* n_contrib,
                  const int32_t* pbox, uint32_t* used, int32_t* tile_work, cudaStream_t stream);
// binning.cu: longest-first tile order from per-tile work counts (one CTA)
int tile_order_from_work(const int32_t* work, int32_t n_tiles, int32_t* tile_order,
                         cudaStream_t stream);
int raster_bwd_plain_ex(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                        const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                        const int32_t* tile_order, const float* dimg, const float* t_final,
                        const int32_t* n_contrib, float* g2d, const int32_t* pbox,
                        const uint32_t* used, cudaStream_t stream);
int raster_bwd_det_ex(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                      const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                      const int32_t* tile_order, const float* dimg, const float* t_final,
                      const int32_t* n_contrib, const int32_t* order, const int32_t* offsets,
                      const int32_t* bbox, const uint64_t* tile_mask, const float* geom, int32_t n,
                      int32_t* rank, float* partial, float* g2d, const uint32_t* used,
                      cudaStream_t stream);
bool raster_masks_usable();
// project.cu: ss_project_fwd that also publishes K = sum of the kept-tile
// counts (kp: K's device slot, the host-mapped (seq, K) word, two re-armed
// device counters) -- the view driver's pair-count readback without a
// separate sum kernel
struct KPublish {
  int32_t* out;
  unsigned long long* host;
  unsigned int* acc_done;
  uint32_t seq;
};
int project_fwd_publish(const ss_store* store, const int32_t* rows, int32_t n,
                        const ss_camera* cam, void* rec_a, void* rec_b, float* rec_c,
                        uint64_t* depth_key, int32_t* bbox, int32_t* n_tiles, float* geom,
                        uint64_t* tile_mask, const KPublish* kp, cudaStream_t stream);
// binning.cu: ss_bin_tiles + the raster launch order from the same tile scan
int bin_tiles_with_order(const int32_t* order, const int32_t* offsets, const int32_t* bbox,
                         const float* geom, const uint64_t* tile_mask, int32_t n,
                         int64_t n_pairs, int32_t tiles_x, int32_t tiles_y, uint16_t* keys,
                         int32_t* vals, int32_t* vals_out, int32_t* ranges, int32_t* tile_order,
                         void* ws, size_t ws_bytes, cudaStream_t stream);
namespace ss {
int memzero(void* p, size_t bytes, cudaStream_t stream);  // ss_api.cu: PDL zero fill
// ss_api.cu: raise `kernel`'s dynamic shared-memory limit to at least `bytes`
// on the CURRENT device (the attribute is per device); thread-safe, one
// driver call per (device, kernel, larger size).
int ensure_smem(const void* kernel, size_t bytes);
}
