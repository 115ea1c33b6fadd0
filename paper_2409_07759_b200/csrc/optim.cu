// a-9 / a-10 fused optimizer step + SGLD (train.py:321-344, 400-415,
// 246-264; regularizer gradients loss.py:105-111) and a-11 MCMC relocation
// (train.py:267-318).  All parameter math in fp64; one thread per row.
#include <cub/cub.cuh>

#include "ss_common.cuh"

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
  const float* gf = grads + r * SS_GRAD_ROW;
  double g[SS_ROW], pv[SS_ROW];
  // rows are 112 B (params, moments) / 56 B (gradients): 16 B / 8 B vector loads
#pragma unroll
  for (int k = 0; k < SS_ROW / 2; ++k) {
    const double2 d = reinterpret_cast<const double2*>(p)[k];
    pv[2 * k] = d.x;
    pv[2 * k + 1] = d.y;
    const float2 f = reinterpret_cast<const float2*>(gf)[k];
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
    double2* mr = reinterpret_cast<double2*>(m + r * SS_ROW);
    double2* vr = reinterpret_cast<double2*>(v + r * SS_ROW);
    // moments in two halves, each half's loads issued together (one memory
    // round trip per half instead of one per column pair)
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
          const double step = ddiv(ddiv(mk[h2], gs.bc1), dadd(sqrt(ddiv(vk[h2], gs.bc2)), h.eps));
          pv[k] = dsub(pv[k], dmul(h.lr[group[k]], step));
        }
        mr[b0 + q] = make_double2(mk[0], mk[1]);
        vr[b0 + q] = make_double2(vk[0], vk[1]);
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
    reinterpret_cast<double2*>(p)[k] = make_double2(pv[2 * k], pv[2 * k + 1]);
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
__global__ void reloc_flags_kernel(const double* __restrict__ opt, int64_t n_rows,
                                   int32_t rows_per_gen, const ss_gen_step* __restrict__ gens,
                                   double threshold, uint8_t* __restrict__ dead,
                                   uint8_t* __restrict__ alive, int32_t* __restrict__ hits) {
  pdl_wait();
  pdl_trigger();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  hits[r] = 0;
  if (!gens[r / rows_per_gen].active) {
    dead[r] = 0;
    alive[r] = 0;
    return;
  }
  const double a = sigmoid(opt[r * SS_ROW + 10]);
  dead[r] = a < threshold;
  alive[r] = !(a < threshold);
}

__global__ void reloc_probs_kernel(const double* __restrict__ opt,
                                   const int32_t* __restrict__ alive_rows,
                                   const int32_t* __restrict__ counts, int64_t n_rows,
                                   double* __restrict__ alpha_alive) {
  pdl_wait();
  pdl_trigger();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_rows) return;
  const int n_alive = counts[1];
  alpha_alive[k] = k < n_alive ? sigmoid(opt[(int64_t)alive_rows[k] * SS_ROW + 10]) : 0.0;
}

__global__ void reloc_div_kernel(double* __restrict__ p, int64_t n_rows,
                                 const double* __restrict__ total) {
  pdl_wait();
  pdl_trigger();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_rows) return;
  p[k] = p[k] / *total;
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
  uint8_t* dead_flag;
  uint8_t* alive_flag;
  int32_t* dead_rows;
  int32_t* alive_rows;
  int32_t* target;
  int32_t* hits;
  double* p;
  double* cdf;
  double* total;
  int32_t* row_ids;
  void* cub;
  size_t cub_bytes;
  size_t total_bytes;
};

static size_t reloc_cub_bytes(int64_t n) {
  size_t a = 0, b = 0, c = 0;
  int nn = (int)(n > 0 ? n : 1);
  cub::DeviceSelect::Flagged(nullptr, a, (int32_t*)nullptr, (uint8_t*)nullptr, (int32_t*)nullptr,
                             (int32_t*)nullptr, nn);
  cub::DeviceReduce::Sum(nullptr, b, (double*)nullptr, (double*)nullptr, nn);
  cub::DeviceScan::InclusiveSum(nullptr, c, (double*)nullptr, (double*)nullptr, nn);
  size_t m = a > b ? a : b;
  return m > c ? m : c;
}

static RelocWs carve(void* base, int64_t n) {
  RelocWs w;
  size_t nn = (size_t)(n > 0 ? n : 1);
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = p + off;
    off += align256(bytes);
    return r;
  };
  w.dead_flag = (uint8_t*)take(nn);
  w.alive_flag = (uint8_t*)take(nn);
  w.dead_rows = (int32_t*)take(nn * 4);
  w.alive_rows = (int32_t*)take(nn * 4);
  w.target = (int32_t*)take(nn * 4);
  w.hits = (int32_t*)take(nn * 4);
  w.p = (double*)take(nn * 8);
  w.cdf = (double*)take(nn * 8);
  w.total = (double*)take(64);
  w.row_ids = (int32_t*)take(nn * 4);
  w.cub_bytes = reloc_cub_bytes(n);
  w.cub = take(w.cub_bytes);
  w.total_bytes = off;
  return w;
}

__global__ void iota32_kernel(int32_t* v, int64_t n) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
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
  launch_k(adam_sgld_kernel, grid_for(n_rows, 128), 128, 0, stream, 
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
  const int n = (int)n_rows;
  launch_k(reloc_flags_kernel, nb, 256, 0, stream, opt, n_rows, rows_per_gen, gens, threshold,
                                             w.dead_flag, w.alive_flag, w.hits);
  launch_k(iota32_kernel, nb, 256, 0, stream, w.row_ids, n_rows);
  size_t cb = w.cub_bytes;
  cudaError_t e = cub::DeviceSelect::Flagged(w.cub, cb, w.row_ids, w.dead_flag, w.dead_rows,
                                             out_counts, n, stream);
  cb = w.cub_bytes;
  if (e == cudaSuccess)
    e = cub::DeviceSelect::Flagged(w.cub, cb, w.row_ids, w.alive_flag, w.alive_rows,
                                   out_counts + 1, n, stream);
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "ss_relocate: %s", cudaGetErrorString(e));
  // p = alpha[alive] / sum(alpha[alive]); cdf = cumsum(p)  (train.py:293-294)
  launch_k(reloc_probs_kernel, nb, 256, 0, stream, opt, w.alive_rows, out_counts, n_rows, w.p);
  cb = w.cub_bytes;
  e = cub::DeviceReduce::Sum(w.cub, cb, w.p, w.total, n, stream);
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "ss_relocate: %s", cudaGetErrorString(e));
  launch_k(reloc_div_kernel, nb, 256, 0, stream, w.p, n_rows, w.total);
  cb = w.cub_bytes;
  e = cub::DeviceScan::InclusiveSum(w.cub, cb, w.p, w.cdf, n, stream);
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "ss_relocate: %s", cudaGetErrorString(e));
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const uint32_t c0 = (uint32_t)counter, c1 = (uint32_t)(counter >> 32);
  launch_k(reloc_targets_kernel, nb, 256, 0, stream, w.cdf, w.alive_rows, out_counts, uniforms, k0, k1,
                                               c0, c1, w.target, w.hits, n_rows);
  launch_k(reloc_clones_kernel, nb, 256, 0, stream, opt, adam_m, adam_v, w.dead_rows, w.target, w.hits,
                                              out_counts);
  launch_k(reloc_targets_update_kernel, nb, 256, 0, stream, opt, adam_m, adam_v, w.hits, n_rows);
  return check_launch("ss_relocate");
}
