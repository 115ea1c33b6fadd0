// Native per-view driver: the whole forward (projection -> binning -> raster
// forward) and backward (raster backward -> projection backward) of one view
// as single C-ABI calls, so the host issues two calls per view instead of ~25
// (the Python-side launch overhead left the GPU idle ~16 % of a step).
//
// The forward waits once for the number of (splat, tile) pairs K that sizes
// the binning (read back right after the projection, so the depth sort runs
// meanwhile); if K exceeds the caller's pair capacity it returns
// SS_ERR_CAPACITY with K in v->n_pairs and the caller grows the buffers and
// calls again.
#include <algorithm>
#include <atomic>
#include <chrono>

#include "ss_common.cuh"

using namespace ss;

// K = sum of v[0..n) (int32), grid-stride.  Every CTA parks its partial in
// partial[block]; the last CTA to finish (done counter) adds the partials in
// block order (deterministic), writes the total to out and, with a
// system-scope store, to the host-mapped pinned word the host is polling, and
// re-arms the counter.  No copy-engine node and no zero fill in the stream.
constexpr int kSumBlocks = 296;

__global__ void __launch_bounds__(256) sum_kernel(const int32_t* __restrict__ v, int32_t n,
                                                  int32_t* __restrict__ out,
                                                  unsigned long long* __restrict__ host_out,
                                                  uint32_t seq,
                                                  int32_t* __restrict__ partial,
                                                  unsigned int* __restrict__ done) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_part[8];
  __shared__ bool s_last;
  int32_t acc = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    acc += v[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) acc += s_part[w];
    partial[blockIdx.x] = acc;
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    int32_t t = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) t += ((volatile int32_t*)partial)[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) {
      *out = t;
      *done = 0u;  // re-armed before the host can see K and launch the next view
      __threadfence();
      // one 8-byte store: (view sequence number, K) arrive together
      *(volatile unsigned long long*)host_out =
          ((unsigned long long)seq << 32) | (unsigned long long)(uint32_t)t;
      __threadfence_system();
    }
  }
}

static std::atomic<uint64_t> g_poll_ns{0};

// Host nanoseconds spent waiting for the pair count K since the last call
// (diagnostics: the host's own per-view work is wall time minus this).
extern "C" uint64_t ss_poll_wait_ns(void) { return g_poll_ns.exchange(0); }

static void record(void* ev, cudaStream_t stream) {
  if (ev) cudaEventRecord((cudaEvent_t)ev, stream);
}

// The backward's tile order (tile_order_from_work, one CTA) runs on a side
// stream per host thread and device, overlapping the loss on the caller's
// stream instead of sitting between the forward and the loss.  The next
// forward from this thread and the view's backward wait for it (order_done).
struct SideOrder {
  cudaStream_t s = nullptr;
  cudaEvent_t fwd_done = nullptr, order_done = nullptr;
  bool pending = false;
};

static SideOrder* side_order() {
  constexpr int kMaxDev = 64;
  thread_local SideOrder tab[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  SideOrder& so = tab[dev];
  if (!so.s) {
    if (cudaStreamCreateWithFlags(&so.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&so.fwd_done, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&so.order_done, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      so.s = nullptr;
      return nullptr;
    }
  }
  return &so;
}

extern "C" int ss_event_create(void** ev) {
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return check_launch("ss_event_create");
  *ev = (void*)e;
  return SS_OK;
}

extern "C" int ss_event_destroy(void* ev) {
  cudaEventDestroy((cudaEvent_t)ev);
  return SS_OK;
}

extern "C" int ss_event_elapsed_ms(void* start, void* end, float* ms) {
  if (cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)end) != cudaSuccess)
    return check_launch("ss_event_elapsed_ms");
  return SS_OK;
}

// Make `stream` wait for this thread's pending side-stream tile order (the
// forward does it itself; callers that free or regrow a view's buffers call
// it first, so the side kernel never touches reused memory).
extern "C" int ss_side_sync(cudaStream_t stream) {
  SideOrder* so = side_order();
  if (so && so->pending) {
    if (cudaStreamWaitEvent(stream, so->order_done, 0) != cudaSuccess)
      return check_launch("ss_side_sync");
    so->pending = false;
  }
  return SS_OK;
}

// Shared by the 3D (store + camera) and 2D (_kernels) entries: workspace
// check, records (via `make_records`), depth order, offsets, K, binning,
// tile order, raster forward.  pbox != nullptr selects the per-pixel bbox test.
template <typename MakeRecords>
static int render_fwd_common(int W, int H, ss_view* v, const int32_t* pbox,
                             MakeRecords make_records, cudaStream_t stream) {
  if (W <= 0 || H <= 0) return set_error(SS_ERR_INVALID, "ss_render_fwd: bad image size");
  const int tiles_x = (W + kTile - 1) / kTile, tiles_y = (H + kTile - 1) / kTile;
  const int n_tiles = tiles_x * tiles_y;
  const int n = v->n;
  v->n_pairs = 0;
  v->sorted_sel = 0;
  v->order_ready = nullptr;
  int rc;
  if (SideOrder* so = side_order(); so && so->pending) {
    cudaStreamWaitEvent(stream, so->order_done, 0);
    so->pending = false;
  }
  if (n == 0) {
    memzero(v->img, sizeof(float) * 3 * (size_t)W * H, stream);
    memzero(v->n_contrib, sizeof(int32_t) * (size_t)W * H, stream);
    memzero(v->ranges, sizeof(int32_t) * 2 * (size_t)n_tiles, stream);
    return check_launch("ss_render_fwd");
  }
  size_t need_ws = ss_binning_workspace_bytes(n, v->pair_cap > 0 ? v->pair_cap : 1, n_tiles);
  const size_t need_order = ss_tile_order_workspace_bytes(n_tiles);
  if (need_order > need_ws) need_ws = need_order;
  if (v->ws_bytes < need_ws) {
    v->ws_needed = need_ws;
    return set_error(SS_ERR_WORKSPACE, "ss_render_fwd: workspace %zu < %zu", v->ws_bytes, need_ws);
  }
  // K = sum of the per-splat tile counts, read back early: the host waits on
  // it (to size the binning) while the GPU runs the depth sort and offsets.
  // It is parked in offsets[n], which ss_tile_offsets rewrites with K.
  // per host thread and device (views may render from several threads, e.g.
  // a trainer and a player; the partials and counter live on the device)
  constexpr int kMaxDev = 64;
  struct KRead {
    unsigned long long* host = nullptr;  // pinned, mapped: (seq, K) lands here
    uint32_t seq = 0;                    // views issued by this thread on this device
    int32_t* partial = nullptr;  // device: per-CTA partial sums
    unsigned int* done = nullptr;
  };
  thread_local KRead k_tab[kMaxDev] = {};
  int devid = 0;
  if (cudaGetDevice(&devid) != cudaSuccess || devid < 0 || devid >= kMaxDev)
    return check_launch("ss_render_fwd: device");
  KRead& kr = k_tab[devid];
  if (!kr.host) {
    if (cudaHostAlloc(&kr.host, sizeof(unsigned long long), cudaHostAllocMapped) != cudaSuccess ||
        cudaMalloc(&kr.partial, kSumBlocks * sizeof(int32_t) + 4 * sizeof(unsigned int)) !=
            cudaSuccess ||
        cudaMemsetAsync(kr.partial, 0, kSumBlocks * sizeof(int32_t) + 4 * sizeof(unsigned int),
                        stream) != cudaSuccess)
      return check_launch("ss_render_fwd: pair count readback");
    kr.done = reinterpret_cast<unsigned int*>(kr.partial + kSumBlocks);
    *(volatile unsigned long long*)kr.host = 0ull;  // no view has sequence number 0
  }
  // the word carries the view's sequence number, so a late write from an
  // earlier (abandoned) view can never be taken for this view's K
  volatile unsigned long long* k_poll = kr.host;
  const uint32_t seq = ++kr.seq;
  // records (+ K for the 3D path: the projection publishes it); the 2D path
  // sums the counts with sum_kernel
  const KPublish kp{v->offsets + n, kr.host, kr.done + 1, seq};
  bool published = false;
  if ((rc = make_records(&kp, published))) return rc;
  if (!published)
    launch_k(sum_kernel, std::max(1, std::min(kSumBlocks, (n + 255) / 256)), 256, 0, stream,
             (const int32_t*)v->n_tiles, n, v->offsets + n, kr.host, seq, kr.partial, kr.done);
  if ((rc = ss_depth_order(v->depth_key, n, v->order, v->ws, v->ws_bytes, stream))) return rc;
  if ((rc = ss_tile_offsets(v->order, v->n_tiles, n, v->offsets, v->ws, v->ws_bytes, stream)))
    return rc;
  // the host polls the mapped word (no event or copy node in the stream);
  // after 2 s of polling it falls back to draining the stream
  const auto arrived = [&]() { return (uint32_t)(*k_poll >> 32) == seq; };
  if (!arrived()) {
    const auto t0 = std::chrono::steady_clock::now();
    struct PollClock {  // host time spent waiting for K (ss_poll_wait_ns)
      std::chrono::steady_clock::time_point t0;
      ~PollClock() {
        g_poll_ns.fetch_add((uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                                std::chrono::steady_clock::now() - t0).count(),
                            std::memory_order_relaxed);
      }
    } poll_clock{t0};
    while (!arrived()) {
#if defined(__x86_64__) || defined(__i386__)
      __builtin_ia32_pause();  // spin politely (SMT sibling, power)
#endif
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
        if (cudaStreamSynchronize(stream) != cudaSuccess)
          return check_launch("ss_render_fwd: pair count");
        if (!arrived()) return set_error(SS_ERR_CUDA, "ss_render_fwd: pair count never arrived");
        break;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  const int32_t k_host = (int32_t)(uint32_t)*k_poll;
  v->n_pairs = k_host;
  if (k_host > v->pair_cap) return set_error(SS_ERR_CAPACITY, "ss_render_fwd: %d pairs > capacity", k_host);
  const int32_t* sv = v->vals;
  bool tile_order_done = false;  // the chunked binning's tile scan writes it
  if (ss_get_binning() == 0 && ss_bin_tiles_supported(k_host, n_tiles)) {
    const size_t need_bin = ss_bin_tiles_workspace_bytes(k_host, n_tiles);
    if (v->ws_bytes < need_bin) {
      v->ws_needed = need_bin;
      return set_error(SS_ERR_WORKSPACE, "ss_render_fwd: workspace %zu < %zu", v->ws_bytes, need_bin);
    }
    if ((rc = bin_tiles_with_order(v->order, v->offsets, v->bbox, v->geom, v->tile_mask, n,
                                   k_host, tiles_x, tiles_y, (uint16_t*)v->keys, v->vals,
                                   v->vals_alt, v->ranges, v->tile_order, v->ws, v->ws_bytes,
                                   stream)))
      return rc;
    tile_order_done = n > 0 && k_host > 0;  // (no pairs: the scan is skipped)
    v->sorted_sel = 1;
    sv = v->vals_alt;
  } else {
    if ((rc = ss_emit_tile_pairs(v->order, v->offsets, v->bbox, v->geom, v->tile_mask, n,
                                 tiles_x, v->keys, v->vals, stream)))
      return rc;
    int32_t sel = 0;
    if ((rc = ss_sort_tile_pairs(v->keys, v->vals, v->keys_alt, v->vals_alt, k_host, n_tiles,
                                 &sel, v->ws, v->ws_bytes, stream)))
      return rc;
    v->sorted_sel = sel;
    sv = sel ? v->vals_alt : v->vals;
    if ((rc = ss_tile_ranges(sel ? v->keys_alt : v->keys, k_host, n_tiles, v->ranges, stream)))
      return rc;
  }
  if (!tile_order_done &&
      (rc = ss_tile_order(v->ranges, n_tiles, v->tile_order, v->ws, v->ws_bytes, stream)))
    return rc;
  // entry-use masks for the backward when the caller gave room for them
#ifndef SS_USE_MASKS
#define SS_USE_MASKS 1
#endif
  const bool masks = SS_USE_MASKS && !v->fwd_only && v->used && raster_masks_usable() &&
                     v->used_cap >= ss_raster_used_words(k_host, n_tiles);
  v->used_ok = masks ? 1 : 0;
  // per-tile backward work (walked entries), accumulated by the forward into
  // the binning workspace (dead once the lists exist); the backward then
  // runs in that longest-first order (v->tile_order is rewritten after the
  // forward has used it)
  int32_t* tile_work = !v->fwd_only && n_tiles <= (1 << 20) &&
                               v->ws_bytes >= sizeof(int32_t) * (size_t)n_tiles
                           ? (int32_t*)v->ws
                           : nullptr;
  // the chunked binning's scatter leaves them zeroed (its chunk-0 base row)
  if (tile_work && !tile_order_done) memzero(tile_work, sizeof(int32_t) * (size_t)n_tiles, stream);
  record(v->events[0], stream);
  rc = raster_fwd_ex(v->ranges, sv, v->rec_a, v->rec_b, v->rec_c, W, H, v->tile_order, v->img,
                     v->t_final, v->n_contrib, pbox, masks ? v->used : nullptr, tile_work, stream);
  record(v->events[1], stream);
  if (!rc && tile_work) {
    SideOrder* so = side_order();
    if (so) {
      cudaEventRecord(so->fwd_done, stream);
      cudaStreamWaitEvent(so->s, so->fwd_done, 0);
      rc = tile_order_from_work(tile_work, n_tiles, v->tile_order, so->s);
      if (!rc && v->g2d_pre) rc = memzero(v->g2d_pre, sizeof(float) * SS_G2D_ROW * (size_t)n, so->s);
      cudaEventRecord(so->order_done, so->s);
      so->pending = true;
      v->order_ready = (void*)so->order_done;
    } else {
      rc = tile_order_from_work(tile_work, n_tiles, v->tile_order, stream);
    }
  }
  return rc;
}

extern "C" int ss_render_fwd(const ss_store* store, const ss_camera* cam, ss_view* v,
                             cudaStream_t stream) {
  if (!store || !cam || !v || v->n < 0) return set_error(SS_ERR_INVALID, "ss_render_fwd: bad args");
  return render_fwd_common(cam->width, cam->height, v, nullptr,
                           [&](const KPublish* kp, bool& published) {
    published = true;
    return project_fwd_publish(store, v->rows, v->n, cam, v->rec_a, v->rec_b, v->rec_c,
                               v->depth_key, v->bbox, v->n_tiles, v->geom, v->tile_mask, kp,
                               stream);
  }, stream);
}

extern "C" int ss_render2d_fwd(const ss_splats2d* sp, int32_t width, int32_t height, ss_view* v,
                               cudaStream_t stream) {
  if (!sp || !v || sp->n < 0) return set_error(SS_ERR_INVALID, "ss_render2d_fwd: bad args");
  v->n = sp->n;
  return render_fwd_common(width, height, v, v->bbox, [&](const KPublish*, bool& published) {
    published = false;
    return ss_records_2d(sp, width, height, v->rec_a, v->rec_b, v->rec_c, v->depth_key, v->bbox,
                         v->n_tiles, v->geom, v->tile_mask, stream);
  }, stream);
}

extern "C" int ss_render2d_bwd(const ss_splats2d* sp, int32_t width, int32_t height,
                               const ss_view* v, const float* dimg, float* g2d, double* g_mean2d,
                               double* g_inv2d, double* g_alpha, double* g_color,
                               cudaStream_t stream) {
  if (!sp || !v) return set_error(SS_ERR_INVALID, "ss_render2d_bwd: bad args");
  if (v->n == 0 || v->n_pairs == 0) return SS_OK;
  // zero-filled by the forward's side stream when it was given this buffer
  if (v->order_ready) cudaStreamWaitEvent(stream, (cudaEvent_t)v->order_ready, 0);
  if (!(v->order_ready && v->g2d_pre == g2d))
    memzero(g2d, sizeof(float) * SS_G2D_ROW * (size_t)v->n, stream);
  const int32_t* sv = v->sorted_sel ? v->vals_alt : v->vals;
  const uint32_t* used = v->used_ok && raster_masks_usable() ? v->used : nullptr;
  int rc = raster_bwd_plain_ex(v->ranges, sv, v->rec_a, v->rec_b, v->rec_c, width, height,
                               v->tile_order, dimg, v->t_final, v->n_contrib, g2d, v->bbox, used,
                               stream);
  if (rc) return rc;
  return ss_basis_to_2d(g2d, sp, v->rec_b, v->depth_key, g_mean2d, g_inv2d, g_alpha, g_color,
                        stream);
}

extern "C" int ss_render_bwd(const ss_store* store, const ss_camera* cam, const ss_view* v,
                             const float* dimg, float* g2d, const uint8_t* trainable_mask,
                             int64_t trainable_rows, float* grads, cudaStream_t stream) {
  if (!store || !cam || !v) return set_error(SS_ERR_INVALID, "ss_render_bwd: bad args");
  if (v->n == 0) return SS_OK;
  // zero-filled by the forward's side stream when it was given this buffer
  // (ordered by the wait on order_ready below)
  const bool pre = v->order_ready && v->g2d_pre == g2d;
  if (v->order_ready) cudaStreamWaitEvent(stream, (cudaEvent_t)v->order_ready, 0);
  if (!pre) memzero(g2d, sizeof(float) * SS_G2D_ROW * (size_t)v->n, stream);
  if (v->n_pairs == 0)  // nothing reached a pixel: zero gradients for every active row
    return ss_project_bwd(store, v->rows, v->n, cam, g2d, v->depth_key, trainable_mask,
                          trainable_rows, grads, stream);
  const int32_t* sv = v->sorted_sel ? v->vals_alt : v->vals;
  // the forward's entry-use masks, when it recorded them for this view
  const uint32_t* used = v->used_ok && raster_masks_usable() ? v->used : nullptr;
  record(v->events[2], stream);
  int rc;
  if (v->partial)
    rc = raster_bwd_det_ex(v->ranges, sv, v->rec_a, v->rec_b, v->rec_c, cam->width, cam->height,
                           v->tile_order, dimg, v->t_final, v->n_contrib, v->order, v->offsets,
                           v->bbox, v->tile_mask, v->geom, v->n, v->rank, v->partial, g2d, used,
                           stream);
  else
    rc = raster_bwd_plain_ex(v->ranges, sv, v->rec_a, v->rec_b, v->rec_c, cam->width,
                             cam->height, v->tile_order, dimg, v->t_final, v->n_contrib, g2d,
                             nullptr, used, stream);
  record(v->events[3], stream);
  if (rc) return rc;
  return ss_project_bwd(store, v->rows, v->n, cam, g2d, v->depth_key, trainable_mask,
                        trainable_rows, grads, stream);
}
