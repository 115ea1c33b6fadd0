// a-9 / a-10 fused optimizer step + SGLD (train.py:321-344, 400-415,
// 246-264; regularizer gradients loss.py:105-111) and a-11 MCMC relocation
// (train.py:267-318).  All parameter math in fp64; one thread per row.  No
// library kernels: the relocation partition and scan are this file's own.
#include "ss_common.cuh"

#ifndef SS_ADAM_TMA
#define SS_ADAM_TMA 1
#endif
#ifndef SS_ADAM_PDL
#define SS_ADAM_PDL 1
#endif

namespace ss {

struct HyperK {
  double lr[5];
  double b1, b2, eps, opacity_reg, scale_reg, n_reg, noise_scale, gate_center, gate_sharp;
  int sgd, sgld;
  uint32_t k0, k1, c0, c1;
};

static HyperK to_hyper(const ss_step_hyper* h) {
  HyperK k;
  for (int i = 0; i < 5; ++i) k.lr[i] = h->lr[i];
  k.b1 = h->beta1;
  k.b2 = h->beta2;
  k.eps = h->eps;
  k.opacity_reg = h->opacity_reg;
  k.scale_reg = h->scale_reg;
  k.n_reg = h->n_reg;
  k.noise_scale = h->noise_scale;
  k.gate_center = h->gate_center;
  k.gate_sharp = h->gate_sharpness;
  k.sgd = h->sgd;
  k.sgld = h->sgld;
  k.k0 = (uint32_t)h->seed;
  k.k1 = (uint32_t)(h->seed >> 32);
  k.c0 = (uint32_t)h->counter;
  k.c1 = (uint32_t)(h->counter >> 32);
  return k;
}

// Standard normal triple for `row` from Philox (Box-Muller on 32-bit
// uniforms, evaluated in fp32: the noise sample needs no fp64 precision).
__device__ __forceinline__ void philox_normal3(const HyperK& h, int64_t row, double out[3]) {
  Philox4 r = philox4x32_10((uint32_t)row, (uint32_t)(row >> 32), h.c0, h.c1, h.k0, h.k1);
  const float inv32 = 2.3283064365386963e-10f;  // 2^-32
  const float u1 = ((float)(r.v[0] >> 8) + 1.0f) * 5.9604644775390625e-08f;  // (0, 1], 24 bits
  const float u2 = (float)r.v[1] * inv32;
  const float u3 = ((float)(r.v[2] >> 8) + 1.0f) * 5.9604644775390625e-08f;
  const float u4 = (float)r.v[3] * inv32;
  const float rad1 = sqrtf(-2.0f * logf(u1)), rad2 = sqrtf(-2.0f * logf(u3));
  float s1, c1, s2, c2;
  sincospif(2.0f * u2, &s1, &c1);
  sincospif(2.0f * u4, &s2, &c2);
  out[0] = (double)(rad1 * c1);
  out[1] = (double)(rad1 * s1);
  out[2] = (double)(rad2 * c2);
}

__device__ __forceinline__ double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

// train.py:246-264 on one row (mean += noise_lr lr gate(alpha) R diag(s) eta)
__device__ __forceinline__ void sgld_row(double* p, const HyperK& h, const double eta[3]) {
  const double alpha = sigmoid(p[10]);
  const double gate = sigmoid(-h.gate_sharp * (alpha - h.gate_center));
  double R[3][3];
  quat_to_rot(p + 3, R);
  double s[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) s[k] = exp(p[7 + k]);
  const double gain = dmul(h.noise_scale, gate);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double step = dadd(dadd(dmul(dmul(R[i][0], s[0]), eta[0]), dmul(dmul(R[i][1], s[1]), eta[1])),
                             dmul(dmul(R[i][2], s[2]), eta[2]));
    p[i] = dadd(p[i], dmul(gain, step));
  }
}

// One row of the fused step (train.py:321-344, 400-415): parameters,
// gradients and moments read through p_in / g_in / m_in / v_in (global
// memory, or the TMA kernel's shared-memory copy), results to the global
// rows p_out / m_out / v_out.
__device__ __forceinline__ void adam_sgld_row(int64_t r, const double* __restrict__ p_in,
                                              const float* __restrict__ g_in,
                                              const double* __restrict__ m_in,
                                              const double* __restrict__ v_in,
                                              double* __restrict__ p_out,
                                              double* __restrict__ m_out,
                                              double* __restrict__ v_out, const ss_gen_step& gs,
                                              const HyperK& h, const double* __restrict__ eta) {
  double g[SS_ROW], pv[SS_ROW];
  // rows are 112 B (params, moments) / 56 B (gradients): 16 B / 8 B vector loads
#pragma unroll
  for (int k = 0; k < SS_ROW / 2; ++k) {
    const double2 d = reinterpret_cast<const double2*>(p_in)[k];
    pv[2 * k] = d.x;
    pv[2 * k + 1] = d.y;
    const float2 f = reinterpret_cast<const float2*>(g_in)[k];
    g[2 * k] = (double)f.x;
    g[2 * k + 1] = (double)f.y;
  }
  // loss.py:110-111 regularizer gradients (train.py:397-398)
  const double alpha = sigmoid(pv[10]);
  g[10] = dadd(g[10], ddiv(dmul(dmul(h.opacity_reg, alpha), dsub(1.0, alpha)), h.n_reg));
#pragma unroll
  for (int k = 0; k < 3; ++k) g[7 + k] = dadd(g[7 + k], ddiv(dmul(h.scale_reg, exp(pv[7 + k])), h.n_reg));
  // train.py:404-407  gamma^w on the mean gradient
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = dmul(g[k], gs.gscale);
  // group of each column: mean 0-2, quat 3-6, log_scale 7-9, logit 10, color 11-13
  const int group[SS_ROW] = {0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 3, 4, 4, 4};
  if (h.sgd) {
#pragma unroll
    for (int k = 0; k < SS_ROW; ++k) pv[k] = dsub(pv[k], dmul(h.lr[group[k]], g[k]));
  } else {
    const double2* mr = reinterpret_cast<const double2*>(m_in);
    const double2* vr = reinterpret_cast<const double2*>(v_in);
    double2* mw = reinterpret_cast<double2*>(m_out);
    double2* vw = reinterpret_cast<double2*>(v_out);
    // moments in two halves, each half's loads issued together (one memory
    // round trip per half instead of one per column pair).  The bias
    // corrections divide every column by the same two constants: products
    // with their reciprocals (one more rounding than numpy's x / c, ~1e-16
    // relative, inside the optimizer's 1e-8 / 1e-6 parity).
    const double ibc1 = 1.0 / gs.bc1, ibc2 = 1.0 / gs.bc2;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      constexpr int kH = 4;  // column pairs of the first half (7 = 4 + 3)
      const int b0 = half ? kH : 0, nb = half ? SS_ROW / 2 - kH : kH;
      double2 mm[kH], vv[kH];
#pragma unroll
      for (int q = 0; q < kH; ++q)
        if (q < nb) {
          mm[q] = mr[b0 + q];
          vv[q] = vr[b0 + q];
        }
#pragma unroll
      for (int q = 0; q < kH; ++q) {
        if (q >= nb) continue;
        double mk[2] = {mm[q].x, mm[q].y}, vk[2] = {vv[q].x, vv[q].y};
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int k = 2 * (b0 + q) + h2;
          mk[h2] = __dadd_rn(__dmul_rn(mk[h2], h.b1), __dmul_rn(1.0 - h.b1, g[k]));
          vk[h2] = __dadd_rn(__dmul_rn(vk[h2], h.b2), __dmul_rn(__dmul_rn(1.0 - h.b2, g[k]), g[k]));
          const double step = ddiv(dmul(mk[h2], ibc1), dadd(sqrt(dmul(vk[h2], ibc2)), h.eps));
          pv[k] = dsub(pv[k], dmul(h.lr[group[k]], step));
        }
        mw[b0 + q] = make_double2(mk[0], mk[1]);
        vw[b0 + q] = make_double2(vk[0], vk[1]);
      }
    }
  }
  // train.py:341-344 projections
  const double qn = sqrt(dadd(dadd(dadd(dmul(pv[3], pv[3]), dmul(pv[4], pv[4])), dmul(pv[5], pv[5])),
                             dmul(pv[6], pv[6])));
  const double qd = fmax(qn, 1e-12);
#pragma unroll
  for (int k = 3; k < 7; ++k) pv[k] = ddiv(pv[k], qd);
#pragma unroll
  for (int k = 11; k < 14; ++k) pv[k] = fmin(fmax(pv[k], 0.0), 1.0);
  const double ls_floor = -13.815510557964274;  // log(1e-6)
#pragma unroll
  for (int k = 7; k < 10; ++k) pv[k] = fmax(pv[k], ls_floor);
  if (h.sgld) {
    double e[3];
    if (eta) {
      e[0] = eta[3 * r];
      e[1] = eta[3 * r + 1];
      e[2] = eta[3 * r + 2];
    } else {
      philox_normal3(h, r, e);
    }
    sgld_row(pv, h, e);
  }
#pragma unroll
  for (int k = 0; k < SS_ROW / 2; ++k)
    reinterpret_cast<double2*>(p_out)[k] = make_double2(pv[2 * k], pv[2 * k + 1]);
}

__global__ void __launch_bounds__(128, 4) adam_sgld_kernel(double* __restrict__ opt, const float* __restrict__ grads,
                                 double* __restrict__ m, double* __restrict__ v, int64_t n_rows,
                                 int32_t rows_per_gen, const ss_gen_step* __restrict__ gens,
                                 HyperK h, const double* __restrict__ eta) {
  pdl_wait();
  pdl_trigger();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const ss_gen_step gs = gens[r / rows_per_gen];
  if (!gs.active) return;
  double* p = opt + r * SS_ROW;
  adam_sgld_row(r, p, grads + r * SS_GRAD_ROW, m + r * SS_ROW, v + r * SS_ROW, p, m + r * SS_ROW,
                v + r * SS_ROW, gs, h, eta);
}

// The same step with the CTA's rows brought into shared memory by TMA bulk
// copies (cp.async.bulk, one mbarrier): 64 rows of parameters, moments and
// gradients (25 KB) are in flight at once without holding registers, where
// the per-thread loads left the kernel waiting on three dependent memory
// round trips per row at a quarter occupancy (long-scoreboard stalls).
constexpr int kAdamTmaRows = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(kAdamTmaRows) adam_sgld_tma_kernel(
    double* __restrict__ opt, const float* __restrict__ grads, double* __restrict__ m,
    double* __restrict__ v, int64_t n_rows, int32_t rows_per_gen,
    const ss_gen_step* __restrict__ gens, HyperK h, const double* __restrict__ eta) {
  __shared__ __align__(128) double s_p[kAdamTmaRows * SS_ROW];
  __shared__ __align__(128) double s_m[kAdamTmaRows * SS_ROW];
  __shared__ __align__(128) double s_v[kAdamTmaRows * SS_ROW];
  __shared__ __align__(128) float s_g[kAdamTmaRows * SS_GRAD_ROW];
  __shared__ __align__(8) unsigned long long s_bar;
  pdl_wait();
  pdl_trigger();
  const int64_t r0 = (int64_t)blockIdx.x * kAdamTmaRows;
  const int rows = (int)min((int64_t)kAdamTmaRows, n_rows - r0);
  // a CTA spans at most two generations (rows_per_gen >= 64, checked by the
  // launcher): skip it when both are frozen this step
  if (!gens[r0 / rows_per_gen].active && !gens[(r0 + rows - 1) / rows_per_gen].active) return;
  const bool sgd = h.sgd != 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t pb = (uint32_t)rows * SS_ROW * 8, gb = (uint32_t)rows * SS_GRAD_ROW * 4;
    const uint32_t total = pb + gb + (sgd ? 0u : 2u * pb);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar)),
                 "r"(total)
                 : "memory");
    const auto bulk = [&](void* dst, const void* src, uint32_t bytes) {
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(&s_bar))
          : "memory");
    };
    bulk(s_p, opt + r0 * SS_ROW, pb);
    bulk(s_g, grads + r0 * SS_GRAD_ROW, gb);
    if (!sgd) {
      bulk(s_m, m + r0 * SS_ROW, pb);
      bulk(s_v, v + r0 * SS_ROW, pb);
    }
  }
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra W_%=;\n}" ::"r"(smem_u32(&s_bar))
      : "memory");
  const int t = threadIdx.x;
  if (t >= rows) return;
  const int64_t r = r0 + t;
  const ss_gen_step gs = gens[r / rows_per_gen];
  if (!gs.active) return;
  // results straight to the global rows (TMA bulk stores from shared memory
  // measured slower: 29 -> 31 us at config 3)
  adam_sgld_row(r, s_p + t * SS_ROW, s_g + t * SS_GRAD_ROW, s_m + t * SS_ROW, s_v + t * SS_ROW,
                opt + r * SS_ROW, m + r * SS_ROW, v + r * SS_ROW, gs, h, eta);
}

__global__ void sgld_kernel(double* __restrict__ opt, int64_t n_rows, int32_t rows_per_gen,
                            const ss_gen_step* __restrict__ gens, HyperK h,
                            const double* __restrict__ eta) {
  pdl_wait();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  if (!gens[r / rows_per_gen].active) return;
  double* p = opt + r * SS_ROW;
  double pv[SS_ROW];
#pragma unroll
  for (int k = 0; k < SS_ROW; ++k) pv[k] = p[k];
  double e[3];
  if (eta) {
    e[0] = eta[3 * r];
    e[1] = eta[3 * r + 1];
    e[2] = eta[3 * r + 2];
  } else {
    philox_normal3(h, r, e);
  }
  sgld_row(pv, h, e);
#pragma unroll
  for (int k = 0; k < 3; ++k) p[k] = pv[k];
}

// ---------------------------------------------------------------- relocation
// flags: 1 = dead, 2 = alive, 0 = row of an inactive generation
// Relocation bookkeeping in the library's own kernels (no CUB): a stable
// partition of the active optimizable rows into dead (alpha < threshold) and
// alive rows, in row order (train.py:279-292), and the fp64 inclusive scan
// of the alive rows' alphas -- the unnormalised cdf; reloc_targets_kernel
// compares cdf[i] / cdf[last] with u, numpy's choice(p=alpha / sum) up to
// rounding (train.py:293-294).  Fixed-order block sums: deterministic.
constexpr int kRelThreads = 256;
constexpr int kRelItems = 4;
constexpr int kRelTile = kRelThreads * kRelItems;

template <typename T>
__device__ __forceinline__ T block_exclusive_t(T v, T* s_warp, T& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T w = lane < nw ? s_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) s_warp[lane] = w;
  }
  __syncthreads();
  total = s_warp[nw - 1];
  const T ex = x - v + (wid > 0 ? s_warp[wid - 1] : T(0));
  __syncthreads();  // s_warp reusable by the caller
  return ex;
}

// 0: row of an inactive generation, 1: dead, 2: alive
__device__ __forceinline__ int reloc_flag(const double* __restrict__ opt, int64_t r, int64_t n_rows,
                                          int32_t rows_per_gen, const ss_gen_step* __restrict__ gens,
                                          double threshold) {
  if (r >= n_rows || !gens[r / rows_per_gen].active) return 0;
  return sigmoid(opt[r * SS_ROW + 10]) < threshold ? 1 : 2;
}

// per block of kRelTile rows: (dead << 32) | alive; zeroes the hit counts
__global__ void __launch_bounds__(kRelThreads) reloc_count_kernel(
    const double* __restrict__ opt, int64_t n_rows, int32_t rows_per_gen,
    const ss_gen_step* __restrict__ gens, double threshold, int32_t* __restrict__ hits,
    unsigned long long* __restrict__ block_counts) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned long long s_warp[32];
  const int64_t r0 = (int64_t)blockIdx.x * kRelTile;
  unsigned long long c = 0;
#pragma unroll
  for (int k = 0; k < kRelItems; ++k) {
    const int64_t r = r0 + k * kRelThreads + threadIdx.x;
    if (r < n_rows) hits[r] = 0;
    const int f = reloc_flag(opt, r, n_rows, rows_per_gen, gens, threshold);
    c += f == 1 ? (1ull << 32) : f == 2 ? 1ull : 0ull;
  }
  unsigned long long total;
  block_exclusive_t(c, s_warp, total);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = total;
}

// one CTA: exclusive scan of the packed per-block counts; totals -> counts
__global__ void __launch_bounds__(kRelThreads) reloc_count_scan_kernel(
    unsigned long long* __restrict__ block_counts, int nblocks, int32_t* __restrict__ counts) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned long long s_warp[32];
  unsigned long long carry = 0;
  for (int base = 0; base < nblocks; base += kRelThreads) {
    const int i = base + threadIdx.x;
    const unsigned long long v = i < nblocks ? block_counts[i] : 0ull;
    unsigned long long total;
    const unsigned long long ex = block_exclusive_t(v, s_warp, total);
    if (i < nblocks) block_counts[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) {
    counts[0] = (int32_t)(carry >> 32);
    counts[1] = (int32_t)(carry & 0xffffffffull);
  }
}

// stable partition: dead / alive row ids in row order, alive alphas
__global__ void __launch_bounds__(kRelThreads) reloc_scatter_kernel(
    const double* __restrict__ opt, int64_t n_rows, int32_t rows_per_gen,
    const ss_gen_step* __restrict__ gens, double threshold,
    const unsigned long long* __restrict__ block_counts, int32_t* __restrict__ dead_rows,
    int32_t* __restrict__ alive_rows, double* __restrict__ alpha_alive) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned long long s_warp[32];
  const int64_t r0 = (int64_t)blockIdx.x * kRelTile;
  unsigned long long run = block_counts[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kRelItems; ++k) {
    const int64_t r = r0 + k * kRelThreads + threadIdx.x;
    const int f = reloc_flag(opt, r, n_rows, rows_per_gen, gens, threshold);
    const unsigned long long c = f == 1 ? (1ull << 32) : f == 2 ? 1ull : 0ull;
    unsigned long long total;
    const unsigned long long pos = run + block_exclusive_t(c, s_warp, total);
    if (f == 1) dead_rows[pos >> 32] = (int32_t)r;
    if (f == 2) {
      const uint32_t a = (uint32_t)(pos & 0xffffffffull);
      alive_rows[a] = (int32_t)r;
      alpha_alive[a] = sigmoid(opt[r * SS_ROW + 10]);
    }
    run += total;
  }
}

// fp64 inclusive scan of alpha_alive[0, counts[1]) in three launches
__global__ void __launch_bounds__(kRelThreads) reloc_dsum_kernel(
    const double* __restrict__ a, const int32_t* __restrict__ counts, double* __restrict__ sums) {
  pdl_wait();
  pdl_trigger();
  __shared__ double s_warp[32];
  const int n = counts[1];
  const int64_t e0 = (int64_t)blockIdx.x * kRelTile + (int64_t)threadIdx.x * kRelItems;
  if ((int64_t)blockIdx.x * kRelTile >= n) return;
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < kRelItems; ++k)
    if (e0 + k < n) v += a[e0 + k];
  double total;
  block_exclusive_t(v, s_warp, total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kRelThreads) reloc_dtop_kernel(double* __restrict__ sums,
                                                                const int32_t* __restrict__ counts) {
  pdl_wait();
  pdl_trigger();
  __shared__ double s_warp[32];
  const int nblocks = (counts[1] + kRelTile - 1) / kRelTile;
  double carry = 0.0;
  for (int base = 0; base < nblocks; base += kRelThreads) {
    const int i = base + threadIdx.x;
    const double v = i < nblocks ? sums[i] : 0.0;
    double total;
    const double ex = block_exclusive_t(v, s_warp, total);
    if (i < nblocks) sums[i] = carry + ex;
    carry += total;
  }
}

__global__ void __launch_bounds__(kRelThreads) reloc_dscan_kernel(
    const double* __restrict__ a, const int32_t* __restrict__ counts,
    const double* __restrict__ sums, double* __restrict__ cdf) {
  pdl_wait();
  pdl_trigger();
  __shared__ double s_warp[32];
  const int n = counts[1];
  if ((int64_t)blockIdx.x * kRelTile >= n) return;
  const int64_t e0 = (int64_t)blockIdx.x * kRelTile + (int64_t)threadIdx.x * kRelItems;
  double x[kRelItems];
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < kRelItems; ++k) {
    x[k] = e0 + k < n ? a[e0 + k] : 0.0;
    v += x[k];
  }
  double total;
  double run = sums[blockIdx.x] + block_exclusive_t(v, s_warp, total);
#pragma unroll
  for (int k = 0; k < kRelItems; ++k) {
    run += x[k];
    if (e0 + k < n) cdf[e0 + k] = run;
  }
}

// numpy Generator.choice(p=...): cdf = cumsum(p); cdf /= cdf[-1];
// idx = searchsorted(cdf, u, side='right')  (see oracle relocation_targets)
__global__ void reloc_targets_kernel(const double* __restrict__ cdf,
                                     const int32_t* __restrict__ alive_rows,
                                     const int32_t* __restrict__ counts,
                                     const double* __restrict__ uniforms, uint32_t k0,
                                     uint32_t k1, uint32_t c0, uint32_t c1,
                                     int32_t* __restrict__ target, int32_t* __restrict__ hits,
                                     int64_t n_rows) {
  pdl_wait();
  pdl_trigger();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n_dead = counts[0], n_alive = counts[1];
  if (k >= n_dead || n_alive == 0) return;
  double u;
  if (uniforms) {
    u = uniforms[k];
  } else {
    Philox4 r = philox4x32_10((uint32_t)k, (uint32_t)(k >> 32), c0, c1 ^ 0x5bd1e995u, k0, k1);
    u = (double)(((uint64_t)(r.v[0] >> 5) << 26) | (r.v[1] >> 6)) * (1.0 / 9007199254740992.0);
  }
  const double last = cdf[n_alive - 1];
  // upper bound over normalized cdf values cdf[i] / last
  int lo = 0, hi = n_alive;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cdf[mid] / last <= u) lo = mid + 1;
    else hi = mid;
  }
  if (lo >= n_alive) lo = n_alive - 1;
  const int32_t t = alive_rows[lo];
  target[k] = t;
  atomicAdd(&hits[t], 1);
}

__device__ __forceinline__ double logit_clip(double p) {
  p = fmin(fmax(p, 1e-9), 1.0 - 1e-9);  // train.py:129-131
  return log(p / (1.0 - p));
}

__global__ void reloc_clones_kernel(double* __restrict__ opt, double* __restrict__ m,
                                    double* __restrict__ v, const int32_t* __restrict__ dead_rows,
                                    const int32_t* __restrict__ target,
                                    const int32_t* __restrict__ hits,
                                    const int32_t* __restrict__ counts) {
  pdl_wait();
  pdl_trigger();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= counts[0] || counts[1] == 0) return;
  const int32_t d = dead_rows[k], t = target[k];
  const int n = hits[t];
  const double* tp = opt + (int64_t)t * SS_ROW;
  double* dp = opt + (int64_t)d * SS_ROW;
  const double o_t = sigmoid(tp[10]);
  const double o_new = 1.0 - pow(1.0 - o_t, 1.0 / (n + 1));
  const double nl = logit_clip(o_new);
  const double shrink = 0.5 * log((double)(n + 1));
#pragma unroll
  for (int c = 0; c < 7; ++c) dp[c] = tp[c];                 // mean, quat
#pragma unroll
  for (int c = 7; c < 10; ++c) dp[c] = tp[c] - shrink;       // log_scale
  dp[10] = nl;
#pragma unroll
  for (int c = 11; c < 14; ++c) dp[c] = tp[c];               // color
#pragma unroll
  for (int c = 0; c < SS_ROW; ++c) {
    m[(int64_t)d * SS_ROW + c] = 0.0;
    v[(int64_t)d * SS_ROW + c] = 0.0;
  }
}

__global__ void reloc_targets_update_kernel(double* __restrict__ opt, double* __restrict__ m,
                                            double* __restrict__ v,
                                            const int32_t* __restrict__ hits, int64_t n_rows) {
  pdl_wait();
  pdl_trigger();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int n = hits[r];
  if (n == 0) return;
  double* tp = opt + r * SS_ROW;
  const double o_t = sigmoid(tp[10]);
  tp[10] = logit_clip(1.0 - pow(1.0 - o_t, 1.0 / (n + 1)));
#pragma unroll
  for (int c = 0; c < SS_ROW; ++c) {
    m[r * SS_ROW + c] = 0.0;
    v[r * SS_ROW + c] = 0.0;
  }
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct RelocWs {
  int32_t* dead_rows;
  int32_t* alive_rows;
  int32_t* target;
  int32_t* hits;
  double* alpha;               // alive rows' alphas (unnormalised probabilities)
  double* cdf;
  double* dsums;               // per-block sums of the scan
  unsigned long long* bcounts;  // per-block packed (dead, alive) counts
  size_t total_bytes;
};

static RelocWs carve(void* base, int64_t n) {
  RelocWs w;
  size_t nn = (size_t)(n > 0 ? n : 1);
  size_t nb = (nn + kRelTile - 1) / kRelTile;
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = p + off;
    off += align256(bytes);
    return r;
  };
  w.dead_rows = (int32_t*)take(nn * 4);
  w.alive_rows = (int32_t*)take(nn * 4);
  w.target = (int32_t*)take(nn * 4);
  w.hits = (int32_t*)take(nn * 4);
  w.alpha = (double*)take(nn * 8);
  w.cdf = (double*)take(nn * 8);
  w.dsums = (double*)take(nb * 8);
  w.bcounts = (unsigned long long*)take(nb * 8);
  w.total_bytes = off;
  return w;
}

}  // namespace ss

using namespace ss;

extern "C" int ss_adam_sgld_step(double* opt, const float* grads, double* adam_m,
                                 double* adam_v, int64_t n_rows, int32_t rows_per_gen,
                                 const ss_gen_step* gens, const ss_step_hyper* hyper,
                                 const double* eta, cudaStream_t stream) {
  if (n_rows < 0 || rows_per_gen <= 0 || !hyper)
    return set_error(SS_ERR_INVALID, "ss_adam_sgld_step: bad arguments");
  if (n_rows == 0) return SS_OK;
  // the TMA path needs 16-B aligned row blocks (grads: an even row count per
  // copy) and at most two generations per CTA
  const bool tma = SS_ADAM_TMA && rows_per_gen >= kAdamTmaRows && (n_rows % 2 == 0) &&
                   ((uintptr_t)opt % 16 == 0) && ((uintptr_t)grads % 16 == 0) &&
                   ((uintptr_t)adam_m % 16 == 0) && ((uintptr_t)adam_v % 16 == 0);
  if (tma)
    launch_kx(SS_ADAM_PDL, adam_sgld_tma_kernel, grid_for(n_rows, kAdamTmaRows), kAdamTmaRows, 0,
              stream, opt, grads, adam_m, adam_v, n_rows, rows_per_gen, gens, to_hyper(hyper), eta);
  else
    launch_kx(SS_ADAM_PDL, adam_sgld_kernel, grid_for(n_rows, 128), 128, 0, stream,
        opt, grads, adam_m, adam_v, n_rows, rows_per_gen, gens, to_hyper(hyper), eta);
  return check_launch("ss_adam_sgld_step");
}

extern "C" int ss_sgld(double* opt, int64_t n_rows, int32_t rows_per_gen, const ss_gen_step* gens,
                       const ss_step_hyper* hyper, const double* eta, cudaStream_t stream) {
  if (n_rows < 0 || rows_per_gen <= 0 || !hyper)
    return set_error(SS_ERR_INVALID, "ss_sgld: bad arguments");
  if (n_rows == 0) return SS_OK;
  launch_k(sgld_kernel, grid_for(n_rows, 128), 128, 0, stream, opt, n_rows, rows_per_gen, gens,
                                                          to_hyper(hyper), eta);
  return check_launch("ss_sgld");
}

extern "C" size_t ss_relocate_workspace_bytes(int64_t n_rows) {
  return carve(nullptr, n_rows).total_bytes + 256;
}

extern "C" int ss_relocate(double* opt, double* adam_m, double* adam_v, int64_t n_rows,
                           int32_t rows_per_gen, const ss_gen_step* gens, double threshold,
                           const double* uniforms, uint64_t seed, uint64_t counter,
                           int32_t* out_counts, void* ws, size_t ws_bytes,
                           cudaStream_t stream) {
  if (n_rows < 0 || rows_per_gen <= 0 || n_rows > 0x7fffffffll)
    return set_error(SS_ERR_INVALID, "ss_relocate: bad arguments");
  if (ws_bytes < ss_relocate_workspace_bytes(n_rows))
    return set_error(SS_ERR_WORKSPACE, "ss_relocate: workspace too small");
  if (n_rows == 0) return cudaMemsetAsync(out_counts, 0, 8, stream) == cudaSuccess ? SS_OK : SS_ERR_CUDA;
  void* base = (void*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  RelocWs w = carve(base, n_rows);
  const int nb = grid_for(n_rows, 256);
  const int nbt = grid_for(n_rows, kRelTile);
  // dead / alive partition (row order) + alive alphas; counts = (n_dead, n_alive)
  launch_k(reloc_count_kernel, nbt, kRelThreads, 0, stream, (const double*)opt, n_rows,
           rows_per_gen, gens, threshold, w.hits, w.bcounts);
  launch_k(reloc_count_scan_kernel, 1, kRelThreads, 0, stream, w.bcounts, nbt, out_counts);
  launch_k(reloc_scatter_kernel, nbt, kRelThreads, 0, stream, (const double*)opt, n_rows,
           rows_per_gen, gens, threshold, (const unsigned long long*)w.bcounts, w.dead_rows,
           w.alive_rows, w.alpha);
  // cdf = inclusive scan of the alive alphas (train.py:293-294, unnormalised)
  launch_k(reloc_dsum_kernel, nbt, kRelThreads, 0, stream, (const double*)w.alpha,
           (const int32_t*)out_counts, w.dsums);
  launch_k(reloc_dtop_kernel, 1, kRelThreads, 0, stream, w.dsums, (const int32_t*)out_counts);
  launch_k(reloc_dscan_kernel, nbt, kRelThreads, 0, stream, (const double*)w.alpha,
           (const int32_t*)out_counts, (const double*)w.dsums, w.cdf);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const uint32_t c0 = (uint32_t)counter, c1 = (uint32_t)(counter >> 32);
  launch_k(reloc_targets_kernel, nb, 256, 0, stream, w.cdf, w.alive_rows, out_counts, uniforms, k0, k1,
                                               c0, c1, w.target, w.hits, n_rows);
  launch_k(reloc_clones_kernel, nb, 256, 0, stream, opt, adam_m, adam_v, w.dead_rows, w.target, w.hits,
                                              out_counts);
  launch_k(reloc_targets_update_kernel, nb, 256, 0, stream, opt, adam_m, adam_v, w.hits, n_rows);
  return check_launch("ss_relocate");
}
