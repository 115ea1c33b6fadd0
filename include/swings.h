/*
 * swings.h — C ABI of libswings.so, the B200 (sm_100a) implementation of
 * SwinGS's sliding-window training hot path.
 *
 * Conventions
 *  - Every compute entry point is `int ss_*(..., cudaStream_t stream)`.
 *    Return 0 (SS_OK) or an SS_ERR_* code; ss_last_error() gives the text.
 *    The Python host maps SS_ERR_INVALID to the reference's
 *    InvalidParameterError (core.py:22) and everything else to RuntimeError.
 *  - Array pointers are caller-owned DEVICE memory unless the name says
 *    `host`.  The library never allocates; scratch comes from caller
 *    workspaces sized by the *_workspace_bytes queries.
 *  - Calls are stream ordered and never synchronize the host.
 *  - Struct arguments (ss_camera, ss_store, ss_step_hyper) are HOST structs
 *    passed by pointer and copied into kernel parameters.
 *  - Gaussian rows are 14 doubles: mean[3] quat[4](w,x,y,z) scale[3]
 *    opacity color[3] (core.py:153-176).  Rows of the optimizable store hold
 *    log-scale and opacity-logit instead (train.py:155-161).
 *
 * Each entry point names the reference interface it replaces
 * (path:line under /root/reference/pkg/src/splatstream/).
 */
#ifndef SWINGS_H
#define SWINGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ss_stream_t; /* == cudaStream_t */

enum {
  SS_OK = 0,
  SS_ERR_INVALID = 1,   /* bad shape / parameter -> InvalidParameterError   */
  SS_ERR_CUDA = 2,      /* CUDA runtime error                               */
  SS_ERR_CAPACITY = 3,  /* caller buffer too small for the data             */
  SS_ERR_WORKSPACE = 4  /* workspace smaller than the *_workspace_bytes query */
};

#define SS_ROW 14        /* doubles per Gaussian row                       */
#define SS_GRAD_ROW 14   /* floats per optimization-space gradient row     */
#define SS_G2D_ROW 12    /* floats per 2D-gradient record (9 used)         */
#define SS_TILE 16       /* tile edge in pixels                            */

/* Pinhole camera, core.py:95-127 (rot is row-major world-to-camera). */
typedef struct {
  int32_t width, height;
  double fx, fy, cx, cy;
  double rot[9];
  double trans[3];
} ss_camera;

/* The Gaussian store: optimizable rows (optimization space) followed by
 * matured rows (direct space).  An active row id r < n_opt addresses
 * opt[r]; r >= n_opt addresses mat[r - n_opt]. */
typedef struct {
  const double* opt;
  int64_t n_opt;
  const double* mat;
  int64_t n_mat;
} ss_store;

/* Per-generation optimizer table entry (device array), train.py:321-344. */
typedef struct {
  int32_t active;   /* generation stepped this iteration                   */
  int32_t pad;
  double bc1, bc2;  /* 1 - b1^t, 1 - b2^t for the generation's own adam_t   */
  double gscale;    /* gamma^windows_trained on the mean gradient          */
} ss_gen_step;

/* Optimizer + SGLD hyper-parameters (host struct), train.py:42-75. */
typedef struct {
  double lr[5];          /* mean, quat, log_scale, opacity_logit, color     */
  double beta1, beta2, eps;
  double opacity_reg, scale_reg;
  double n_reg;          /* #active optimizable rows (divisor), loss.py:110-111 */
  double noise_scale;    /* noise_lr * lr_mean, train.py:264                 */
  double gate_center, gate_sharpness;
  int32_t sgd;           /* 1 = plain SGD (train.py:322-324)                 */
  int32_t sgld;          /* 1 = apply the SGLD perturbation                  */
  uint64_t seed;         /* Philox key for eta when eta == NULL              */
  uint64_t counter;      /* Philox counter (iteration index)                 */
} ss_step_hyper;

const char* ss_last_error(void);
int ss_version(void);
int ss_device_sm_count(void);

/* ---- a-2 active-set compaction: core.py:280-282, train.py:347-350, 380-386.
 * Candidates are the n_opt optimizable rows in row order, then the matured
 * rows in archive (FIFO) order: logical matured row c lives at physical row
 * mat_block_map[c / block_rows] * block_rows + c % block_rows.  Keeps rows
 * with row_start <= frame < row_expire (per physical row; matured rows at
 * index n_opt + physical).  Writes active row ids (n_opt + physical for
 * matured) to out_rows and out_counts[0] = #active, [1] = #active opt. */
size_t ss_compact_workspace_bytes(int64_t n_candidates);
int ss_compact_active(const int32_t* row_start, const int32_t* row_expire, int64_t n_opt,
                      int64_t n_mat_logical, const int32_t* mat_block_map, int32_t block_rows,
                      int32_t frame, int32_t* out_rows, int32_t* out_counts, void* ws,
                      size_t ws_bytes, ss_stream_t stream);

/* fp64 projection of n splats for API callers (raster.py:176-191 `project`):
 * out[i] = (u, v, cov a, cov b, cov c, z, kept) -- the raw 2D covariance
 * before the +0.3 dilation; kept = 1.0 when the splat survives the near
 * plane and the 3-sigma cull, else 0.0 (the other fields are then
 * meaningless).  Same fp64 sequence as ss_project_fwd. */
int ss_project_splats(const ss_store* store, const int32_t* rows, int32_t n,
                      const ss_camera* cam, double* out, ss_stream_t stream);

/* ---- a-8 regularizers (loss.py:105-111): over n optimizable active splats
 * with direct-space alpha[n] and scales[n*3], writes reg_logit[n] =
 * w_op alpha (1 - alpha) / n, reg_log_scale[n*3] = w_sc s / n and
 * terms[2] = (w_op mean(alpha), w_sc mean(sum_k s_k)) (fixed-order sums). */
int ss_reg_grads(const double* alpha, const double* scales, int32_t n, double w_op,
                 double w_sc, double* reg_logit, double* reg_log_scale, double* terms,
                 ss_stream_t stream);

/* ---- a-3 EWA projection / cull / conic / bbox: raster.py:76-173.
 * For active index i (row = rows ? rows[i] : i): rec_a = (u, v, k inv0, k inv1),
 * rec_b = (k inv2, log2 alpha, r, g), rec_c = b (float32, rounded once from fp64;
 * k = -log2(e)/2 so alpha exp(-m/2) = 2^(k m + log2 alpha));
 * depth_key = fp64 z bits (UINT64_MAX when culled); bbox = (x0,x1,y0,y1)
 * pixels, half open; geom = (u, v, inv0, inv1, det, sy, ymax, 1/inv0) fp32 (the
 * row-interval tile test's constants, ss_common.cuh make_geom)
 * (n x 8); n_tiles = 16x16 tiles of the bbox that the maha <= 64 ellipse
 * reaches (exact ellipse-vs-tile test; 0 when culled); tile_mask = kept bits
 * of the first 64 bbox tiles (row-major). */
int ss_project_fwd(const ss_store* store, const int32_t* rows, int32_t n, const ss_camera* cam,
                   void* rec_a, void* rec_b, float* rec_c, uint64_t* depth_key, int32_t* bbox,
                   int32_t* n_tiles, float* geom, uint64_t* tile_mask, ss_stream_t stream);

/* ---- a-5 / a-6 on already projected 2D splats (the reference's
 * _kernels.blend_forward / blend_backward, _kernels.py:20-130): fp64 arrays
 * mean2d (n,2), inv2d (n,3), alpha (n), color (n,3); bbox (n,4) int32
 * (x0, x1, y0, y1, half open); rank[i] = position of splat i in the blend
 * order (-1: not blended; ranks distinct). */
typedef struct {
  const double* mean2d;
  const double* inv2d;
  const double* alpha;
  const double* color;
  const int32_t* bbox;
  const int32_t* rank;
  int32_t n;
  int32_t pad;
} ss_splats2d;
/* Records, depth keys (= rank), clipped bbox, kept tiles -- ss_project_fwd's
 * outputs for 2D input. */
int ss_records_2d(const ss_splats2d* splats, int32_t width, int32_t height, void* rec_a,
                  void* rec_b, float* rec_c, uint64_t* depth_key, int32_t* bbox,
                  int32_t* n_tiles, float* geom, uint64_t* tile_mask, ss_stream_t stream);
/* Adds the 2D gradients of the raster backward's basis sums g2d (see
 * ss_raster_bwd) into g_mean2d (n,2), g_inv2d (n,3), g_alpha (n),
 * g_color (n,3), fp64 device arrays (blend_backward's += contract). */
int ss_basis_to_2d(const float* g2d, const ss_splats2d* splats, const void* rec_b,
                   const uint64_t* depth_key, double* g_mean2d, double* g_inv2d, double* g_alpha,
                   double* g_color, ss_stream_t stream);

/* ---- a-4 binning: raster.py:153 global (z, src) order reproduced per tile.
 * (1) stable radix sort of the 64-bit depth keys -> order (rank -> i);
 * (2) tile counts in rank order, exclusive scan -> offsets[0..n], K = offsets[n];
 * (3) emit (tile id, i) pairs in rank order for the tiles the ellipse reaches
 * (same test as n_tiles); (4) stable radix sort by tile id;
 * (5) per-tile [start, end) ranges.  Equivalent to sorting the keys
 * tile << 21 | rank. */
size_t ss_binning_workspace_bytes(int32_t n, int64_t max_pairs, int32_t n_tiles);
int ss_depth_order(const uint64_t* depth_key, int32_t n, int32_t* order, void* ws,
                   size_t ws_bytes, ss_stream_t stream);
int ss_tile_offsets(const int32_t* order, const int32_t* n_tiles, int32_t n, int32_t* offsets,
                    void* ws, size_t ws_bytes, ss_stream_t stream);
int ss_emit_tile_pairs(const int32_t* order, const int32_t* offsets, const int32_t* bbox,
                       const float* geom, const uint64_t* tile_mask, int32_t n,
                       int32_t tiles_x, uint32_t* keys, int32_t* vals, ss_stream_t stream);
/* *out_sel (HOST int) = 0 when the sorted pairs are in keys/vals, 1 when in
 * keys_alt/vals_alt. */
int ss_sort_tile_pairs(uint32_t* keys, int32_t* vals, uint32_t* keys_alt, int32_t* vals_alt,
                       int64_t n_pairs, int32_t n_tiles, int32_t* out_sel, void* ws,
                       size_t ws_bytes, ss_stream_t stream);
int ss_tile_ranges(const uint32_t* sorted_keys, int64_t n_pairs, int32_t n_tiles,
                   int32_t* ranges, ss_stream_t stream);
/* Chunked binning (ss_render_fwd's default): builds the same per-tile lists
 * as emit -> stable pair sort -> ranges.  The rank range is cut into chunks
 * of ~8k pairs; per chunk, pairs are emitted (tile id u16 in keys, splat id in
 * vals, at emit positions) with a tile histogram; histograms are scanned
 * over chunks and tiles (-> ranges); then each chunk's pairs are written,
 * in emit order, to vals_out at their tile's slots.
 * offsets = ss_tile_offsets' output, n_pairs = K = offsets[n].  Usable when
 * ss_bin_tiles_supported(K, tiles) (shared-memory cursors: <= 18432 tiles,
 * e.g. 1920x1080 = 8160 tiles). */
size_t ss_bin_tiles_workspace_bytes(int64_t n_pairs, int32_t n_tiles);
int32_t ss_bin_tiles_supported(int64_t n_pairs, int32_t n_tiles);
int ss_bin_tiles(const int32_t* order, const int32_t* offsets, const int32_t* bbox,
                 const float* geom, const uint64_t* tile_mask, int32_t n, int64_t n_pairs,
                 int32_t tiles_x, int32_t tiles_y, uint16_t* keys, int32_t* vals,
                 int32_t* vals_out, int32_t* ranges, void* ws, size_t ws_bytes,
                 ss_stream_t stream);
/* Binning used by ss_render_fwd: 0 = ss_bin_tiles (default), 1 = emit +
 * radix pair sort + ranges (kept as a cross-check; keys are only written here). */
int ss_set_binning(int32_t mode);
int ss_get_binning(void);

/* Alpha floor of the binning and the rasterizer, as log2: a (splat, pixel)
 * contribution is blended only when maha <= 64 (the reference rule,
 * _kernels.py:39-41) AND alpha G >= 2^floor; tiles are emitted only where
 * that can hold (per-splat margin min(64, 2 ln(alpha / 2^floor)), see
 * ss_common.cuh cull_margin).  Each skipped contribution is below 2^floor,
 * so a pixel moves by at most ~2 |skipped| 2^floor (~3e-5 at 4000 skipped
 * entries for the default floor = -28), inside the north star's 1e-4.
 * floor = 0 disables it (the reference's rule alone).  Valid: 0 or
 * [-126, -1].  Process-wide; set before rendering. */
int ss_set_alpha_floor(int32_t log2_floor);

/* Write up to 2048 bytes of host memory to device memory, stream-ordered, as
 * a kernel argument (no copy-engine operation between the library's
 * kernels; used for the per-step generation table and slot maps). */
int ss_write_small(void* dst, const void* host_src, size_t bytes, ss_stream_t stream);

/* Host nanoseconds ss_render_fwd spent waiting for the pair count K since
 * the previous call (diagnostics: host work per view = wall - this). */
uint64_t ss_poll_wait_ns(void);
int32_t ss_get_alpha_floor(void);

/* Tiles ordered by list length, longest first (raster scheduling order:
 * longest-processing-time-first across the SMs).  ws >= ss_tile_order_workspace_bytes. */
size_t ss_tile_order_workspace_bytes(int32_t n_tiles);
int ss_tile_order(const int32_t* ranges, int32_t n_tiles, int32_t* tile_order, void* ws,
                  size_t ws_bytes, ss_stream_t stream);

/* ---- a-5 blend forward: _kernels.py:20-53.  img is (H, W, 3) float32;
 * t_final / n_contrib per pixel feed the backward.  tile_order (nullable)
 * is the tile processing order from ss_tile_order. */
int ss_raster_fwd(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                  const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                  const int32_t* tile_order, float* img, float* t_final, int32_t* n_contrib,
                  ss_stream_t stream);

/* Deterministic variant of ss_raster_bwd: no float atomics.  Each warp writes
 * its reduced 9 values per entry to partial (ss_raster_partial_floats(K)
 * floats), indexed by the entry's emit position (order / offsets / bbox /
 * tile_mask / geom from the forward), and every splat's partials are summed
 * in a fixed order into g2d (all of g2d's n rows are written).  rank: n
 * int32 scratch.  Bit-identical results run to run. */
int64_t ss_raster_partial_floats(int64_t n_pairs);
/* Entry-use mask words for K pairs over n_tiles tiles (ss_view.used). */
int64_t ss_raster_used_words(int64_t n_pairs, int32_t n_tiles);
int ss_raster_bwd_deterministic(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                                const void* rec_b, const float* rec_c, int32_t width,
                                int32_t height, const int32_t* tile_order, const float* dimg,
                                const float* t_final, const int32_t* n_contrib,
                                const int32_t* order, const int32_t* offsets, const int32_t* bbox,
                                const uint64_t* tile_mask, const float* geom, int32_t n,
                                int32_t* rank, float* partial, float* g2d, ss_stream_t stream);

/* Tuning knob: pixels per lane in the raster kernels (2, 4 or 8); a warp
 * covers 16 x (2 strip) pixels, i.e. 8 / strip warps per tile.  Default 4. */
int ss_set_raster_strip(int32_t strip);
/* The same knob set separately for the forward and the backward (the pixel
 * state passes between them per pixel, independent of the mapping). */
int ss_set_raster_strips(int32_t strip_fwd, int32_t strip_bwd);

/* ---- a-6 blend backward: _kernels.py:56-130.  Accumulates into g2d
 * (n x 12 floats: the 9 basis sums t dx, t dy, t dx^2, t dx dy, t dy^2, t,
 * colour[3] over the splat's (pixel, entry) slots, t = alpha G d alpha', pad[3]),
 * which the caller zeroes. */
int ss_raster_bwd(const int32_t* ranges, const int32_t* vals, const void* rec_a,
                  const void* rec_b, const float* rec_c, int32_t width, int32_t height,
                  const int32_t* tile_order, const float* dimg, const float* t_final,
                  const int32_t* n_contrib, float* g2d, ss_stream_t stream);

/* ---- a-7 projection backward: raster.py:249-348.  For active i with
 * trainable (mask ? mask[i] : 1) and row < trainable_rows, writes the
 * optimization-space gradient row grads[out_row] (14 floats: mean[3]
 * quat[4] log_scale[3] opacity_logit color[3]); out_row = row.  Culled
 * trainable rows get a zero row; rows that are not active in this view
 * are left untouched (the caller zeroes them when it steps them). */
int ss_project_bwd(const ss_store* store, const int32_t* rows, int32_t n, const ss_camera* cam,
                   const float* g2d, const uint64_t* depth_key, const uint8_t* trainable_mask,
                   int64_t trainable_rows, float* grads, ss_stream_t stream);

/* ---- a-8 loss: loss.py:73-118 (photometric part; regularizers are fused
 * into ss_adam_sgld_step).  pred (H,W,3) f32; ground truth either u8 sRGB
 * decoded through lut[256] (raster.py:428-432) or f32 linear.  Writes dimg
 * (H,W,3) f32 and out_sums[0] = sum|pred-gt|, out_sums[1] = sum SSIM map
 * (float64, deterministic). */
size_t ss_loss_workspace_bytes(int32_t width, int32_t height);
int ss_loss_l1_ssim(const float* pred, const uint8_t* gt_u8, const float* lut,
                    const float* gt_f32, int32_t width, int32_t height, double ssim_weight,
                    float* dimg, double* out_sums, void* ws, size_t ws_bytes,
                    ss_stream_t stream);

/* ---- a-9/a-10 fused Adam (or SGD) + projections + SGLD:
 * train.py:321-344, 400-415, 246-264, loss.py:105-111.
 * Rows r in [0, n_rows) belong to generation r / rows_per_gen; only rows of
 * generations with gens[g].active are touched.  eta (n_rows x 3, float64) is
 * injected when non-NULL, else drawn from Philox(seed, counter, row). */
int ss_adam_sgld_step(double* opt, const float* grads, double* adam_m, double* adam_v,
                      int64_t n_rows, int32_t rows_per_gen, const ss_gen_step* gens,
                      const ss_step_hyper* hyper, const double* eta, ss_stream_t stream);

/* SGLD alone (train.py:246-264) on the rows of active generations. */
int ss_sgld(double* opt, int64_t n_rows, int32_t rows_per_gen, const ss_gen_step* gens,
            const ss_step_hyper* hyper, const double* eta, ss_stream_t stream);

/* ---- a-11 MCMC relocation: train.py:267-318.  Candidates are the rows of
 * active generations in row order; dead = sigmoid(logit) < threshold.
 * uniforms (n_dead float64, the draws numpy's choice() consumes) are
 * injected when non-NULL, else Philox(seed, counter).  out_counts[0] = #dead,
 * [1] = #alive (device).  Moves nothing when either count is zero. */
size_t ss_relocate_workspace_bytes(int64_t n_rows);
int ss_relocate(double* opt, double* adam_m, double* adam_v, int64_t n_rows,
                int32_t rows_per_gen, const ss_gen_step* gens, double threshold,
                const double* uniforms, uint64_t seed, uint64_t counter, int32_t* out_counts,
                void* ws, size_t ws_bytes, ss_stream_t stream);

/* ---- a-13 / §8(f)-1 export records: codec.py:195-266.  rows are n direct-
 * space Gaussian rows (f64); profile 0 writes 56-byte, profile 1 30-byte
 * little-endian records, byte-identical to encode_records.  *bad (device
 * int, caller zeroes) is set when a row holds a non-finite value (the
 * reference raises CodecError).  ss_decode_records is decode_records. */
int ss_encode_records(const double* rows, int64_t n, int32_t profile, uint8_t* out,
                      int32_t* bad, ss_stream_t stream);
int ss_decode_records(const uint8_t* data, int64_t n, int32_t profile, double* rows,
                      ss_stream_t stream);

/* ---- native per-view driver (csrc/view.cu).  All pointers device memory,
 * caller-owned; capacities: per-splat buffers >= n, pairs >= pair_cap,
 * ranges / tile_order >= tiles, per-pixel >= W*H, ws >= ws_needed. */
typedef struct {
  const int32_t* rows;  /* active row ids (NULL = 0..n-1)                */
  int32_t n;            /* active splats                                 */
  int32_t pad0;
  void* rec_a;          /* float4 x n                                    */
  void* rec_b;          /* float4 x n                                    */
  float* rec_c;
  uint64_t* depth_key;
  int32_t* bbox;        /* int4 x n                                      */
  int32_t* n_tiles;
  float* geom;          /* 8 x n                                         */
  uint64_t* tile_mask;
  int32_t* order;
  int32_t* offsets;     /* n + 1                                         */
  uint32_t* keys;
  int32_t* vals;
  uint32_t* keys_alt;
  int32_t* vals_alt;
  int64_t pair_cap;
  int32_t* ranges;      /* int2 x tiles                                  */
  int32_t* tile_order;
  float* img;           /* H x W x 3                                     */
  float* t_final;
  int32_t* n_contrib;
  void* ws;
  size_t ws_bytes;
  size_t ws_needed;     /* out: workspace the call needed (on SS_ERR_WORKSPACE) */
  int64_t n_pairs;      /* out: K                                        */
  int32_t sorted_sel;   /* out: 1 when the sorted pairs are in *_alt      */
  int32_t pad1;
  void* events[4];      /* optional cudaEvent_t: raster fwd start/end, bwd start/end */
  float* partial;       /* deterministic backward: ss_raster_partial_floats(K) floats, */
  int32_t* rank;        /*   and n int32; partial == NULL selects the atomic backward */
  uint32_t* used;       /* optional entry-use masks, >= ss_raster_used_words(pair_cap, */
                        /*   tiles) words: the forward records which list entries     */
                        /*   reached each warp's pixels, the backward walks only those */
  int64_t used_cap;     /* words in used                                               */
  int32_t used_ok;      /* out (forward): masks valid for this view's backward         */
  int32_t fwd_only;     /* in: 1 = no backward follows (playback): the forward skips  */
                        /*   the backward's aids (entry-use masks, per-tile work order) */
  void* order_ready;    /* out (forward): the event after which the backward's tile   */
                        /*   order (computed on a library side stream, overlapping the */
                        /*   loss) is ready; ss_render_bwd waits on it; NULL: none     */
  float* g2d_pre;       /* in, optional: the g2d buffer the backward will be given;    */
                        /*   the forward zero-fills it on the same side stream, and    */
                        /*   ss_render_bwd then skips its own fill                     */
} ss_view;

/* Projection -> depth order -> tile offsets -> [one stream sync for K] ->
 * emit -> pair sort -> ranges -> tile order -> raster forward.  Returns
 * SS_ERR_CAPACITY (K in v->n_pairs) when K > pair_cap, SS_ERR_WORKSPACE
 * (size in v->ws_needed) when ws is too small; call again after growing. */
int ss_render_fwd(const ss_store* store, const ss_camera* cam, ss_view* v, ss_stream_t stream);
/* The same view pipeline on 2D splats (_kernels.blend_forward, _kernels.py:20-53):
 * records from splats (blend order = rank), then as ss_render_fwd, with the
 * per-pixel bbox test of _kernels.py:35-36 applied explicitly.  Sets v->n. */
int ss_render2d_fwd(const ss_splats2d* splats, int32_t width, int32_t height, ss_view* v,
                    ss_stream_t stream);
/* _kernels.blend_backward (_kernels.py:56-130) for the view ss_render2d_fwd
 * left in v: adds the 2D gradients into g_mean2d / g_inv2d / g_alpha /
 * g_color (fp64 device arrays); g2d (n x 12 floats) is scratch. */
int ss_render2d_bwd(const ss_splats2d* splats, int32_t width, int32_t height, const ss_view* v,
                    const float* dimg, float* g2d, double* g_mean2d, double* g_inv2d,
                    double* g_alpha, double* g_color, ss_stream_t stream);
/* Raster backward -> projection backward for the view ss_render_fwd left in v;
 * g2d (n x 12 floats) is zeroed here; grads are accumulated (caller zeroes). */
int ss_render_bwd(const ss_store* store, const ss_camera* cam, const ss_view* v,
                  const float* dimg, float* g2d, const uint8_t* trainable_mask,
                  int64_t trainable_rows, float* grads, ss_stream_t stream);
/* Make `stream` wait for the calling thread's pending side-stream work of
 * its last forward (the backward tile order; see ss_view.order_ready) --
 * call before freeing or regrowing a view's buffers. */
int ss_side_sync(ss_stream_t stream);
/* CUDA event helpers for the optional raster timing in ss_view. */
int ss_event_create(void** ev);
int ss_event_destroy(void* ev);
int ss_event_elapsed_ms(void* start, void* end, float* ms);

/* Zero fill (a library kernel, launched with programmatic dependent launch
 * like the others, unlike a driver memset). */
int ss_memzero(void* ptr, size_t bytes, ss_stream_t stream);

/* Direct-space snapshot of optimizable rows (train.py:155-161 + 474):
 * dst[i] = (mean, quat, exp(log_scale), sigmoid(logit), color) of src[i]. */
int ss_to_direct(const double* src, double* dst, int64_t n, ss_stream_t stream);

/* Display frame: n float32 linear values -> uint8 sRGB with write_png's
 * rounding (raster.py:411-425), evaluated in fp64. */
int ss_to_srgb_u8(const float* img, int64_t n, uint8_t* out, ss_stream_t stream);

/* ---- ABR tail-drop selection (server.py:39-79).
 * src holds n keys of `kind` at byte `offset` of `stride`-byte records
 * (wire records: SS_ABR_F32 opacity at 40 / 56 B for profile 0, SS_ABR_U8 at
 * 16 / 30 B for profile 1; SS_ABR_F64 with stride 8 for an opacity array).
 * Writes the ascending indices of the kept_n highest keys, ties to the lower
 * index (the reference's stable argsort of -opacity), to keep_idx[kept_n]
 * and, when out != NULL, those records' stride bytes in the same order. */
#define SS_ABR_F32 0
#define SS_ABR_U8 1
#define SS_ABR_F64 2
int ss_abr_select(const void* src, int64_t n, int32_t kind, int32_t stride, int32_t offset,
                  int64_t kept_n, int32_t* keep_idx, uint8_t* out, ss_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SWINGS_H */
