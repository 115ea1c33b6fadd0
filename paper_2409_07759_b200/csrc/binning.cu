// a-4 binning: the reference's global stable (z, src) order (raster.py:153)
// restricted per 16x16 tile.
//
//   depth order : stable LSD radix sort of 64-bit fp64-z keys (CUB onesweep)
//   offsets     : tile counts gathered in rank order, exclusive scan -> K
//   emit        : (tile id, i) pairs written in rank order (warp per splat)
//   pair sort   : stable radix sort on the tile-id bits only; stability keeps
//                 rank order inside a tile, so the result equals sorting the
//                 SURVEY's 34-bit keys tile << 21 | rank
//   ranges      : boundary detection over the sorted tile ids
#include <cub/cub.cuh>

#include "ss_common.cuh"

namespace ss {

__global__ void iota_kernel(int32_t* v, int32_t n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void high_keys_kernel(const uint64_t* __restrict__ key64, int32_t n,
                                 uint32_t* __restrict__ hi, int32_t* __restrict__ vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  hi[i] = (uint32_t)(key64[i] >> 32);
  vals[i] = i;
}

// After a stable sort on the high 32 bits, each run of equal high keys is
// re-sorted by (full 64-bit key, index).  Runs of <= 32 (the usual case: a
// few splats per 2^-20 relative depth) take a per-thread insertion sort; longer
// runs are queued for long_runs_kernel (one CTA per run, bitonic sort of
// (low 32 key bits, position in run) -- positions keep it stable).
constexpr int kShortRun = 32;
constexpr int kSmemRun = 8192;

__global__ void fix_runs_kernel(const uint32_t* __restrict__ hi_sorted,
                                const uint64_t* __restrict__ key64, int32_t n,
                                int32_t* __restrict__ order, int2* __restrict__ long_runs,
                                int32_t* __restrict__ n_long) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t h = hi_sorted[p];
  if (p > 0 && hi_sorted[p - 1] == h) return;          // not a run start
  if (p + 1 >= n || hi_sorted[p + 1] != h) return;      // singleton run
  int q = p + 1;
  while (q < n && hi_sorted[q] == h) ++q;
  if (q - p > kShortRun) {
    long_runs[atomicAdd(n_long, 1)] = make_int2(p, q);
    return;
  }
  for (int a = p + 1; a < q; ++a) {
    const int32_t v = order[a];
    const uint64_t kv = key64[v];
    int b = a - 1;
    while (b >= p) {
      const int32_t w = order[b];
      const uint64_t kw = key64[w];
      if (kw < kv || (kw == kv && w < v)) break;
      order[b + 1] = w;
      --b;
    }
    order[b + 1] = v;
  }
}

// Bitonic sort of n2 (power of two) 64-bit keys in `a` by one CTA.
__device__ void cta_bitonic(uint64_t* a, int n2) {
  for (int size = 2; size <= n2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const uint64_t x = a[lo], y = a[hi];
        if ((x > y) == asc) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) long_runs_kernel(const uint64_t* __restrict__ key64,
                                                         int32_t* __restrict__ order,
                                                         const int2* __restrict__ long_runs,
                                                         const int32_t* __restrict__ n_long,
                                                         uint64_t* __restrict__ scratch,
                                                         int32_t* __restrict__ tmp) {
  extern __shared__ uint64_t s_keys[];
  for (int r = blockIdx.x; r < *n_long; r += gridDim.x) {
    const int2 run = long_runs[r];
    const int L = run.y - run.x;
    int n2 = 1;
    while (n2 < L) n2 <<= 1;
    // long runs use a private slice of the scratch buffer at the run's offset
    uint64_t* a = n2 <= kSmemRun ? s_keys : scratch + 2 * (int64_t)run.x;
    for (int i = threadIdx.x; i < n2; i += blockDim.x)
      a[i] = i < L ? (((uint64_t)(uint32_t)key64[order[run.x + i]]) << 32) | (uint32_t)i : ~0ull;
    __syncthreads();
    cta_bitonic(a, n2);
    for (int i = threadIdx.x; i < L; i += blockDim.x) tmp[run.x + i] = order[run.x + (int)(a[i] & 0xffffffffu)];
    __syncthreads();
    for (int i = threadIdx.x; i < L; i += blockDim.x) order[run.x + i] = tmp[run.x + i];
    __syncthreads();
  }
}

__global__ void gather_counts_kernel(const int32_t* __restrict__ order,
                                     const int32_t* __restrict__ n_tiles, int32_t n,
                                     int32_t* __restrict__ out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = n_tiles[order[k]];
  if (k == n) out[k] = 0;
}

// One thread per splat in rank order: walk the kept-tile bits of its bbox
// tile rectangle (tile_mask for the first 64 tiles, the fp64 test beyond) and
// write its run [offsets[k], offsets[k+1]) of (tile id, splat) pairs.
__global__ void emit_pairs_kernel(const int32_t* __restrict__ order,
                                  const int32_t* __restrict__ offsets,
                                  const int4* __restrict__ bbox, const float* __restrict__ geom,
                                  const uint64_t* __restrict__ tile_mask, int32_t n,
                                  int32_t tiles_x, uint32_t* __restrict__ keys,
                                  int32_t* __restrict__ vals) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t off = offsets[k];
  const int32_t cnt = offsets[k + 1] - off;
  if (cnt == 0) return;
  const int32_t i = order[k];
  const int4 bb = bbox[i];
  const int tx0 = bb.x / kTile, tx1 = (bb.y - 1) / kTile + 1;
  const int ty0 = bb.z / kTile, ty1 = (bb.w - 1) / kTile + 1;
  const int w = tx1 - tx0;
  const int total = w * (ty1 - ty0);
  uint64_t mask = tile_mask[i];
  while (mask) {
    const int j = __ffsll((long long)mask) - 1;
    mask &= mask - 1;
    keys[off] = (uint32_t)((ty0 + j / w) * tiles_x + tx0 + j % w);
    vals[off] = i;
    ++off;
  }
  if (total > 64) {
    float gl[kGeom];
#pragma unroll
    for (int c = 0; c < kGeom; ++c) gl[c] = geom[(int64_t)i * kGeom + c];
    for (int j = 64; j < total; ++j) {
      const int ty = ty0 + j / w, tx = tx0 + j % w;
      if (tile_keeps(gl, tx, ty, bb)) {
        keys[off] = (uint32_t)(ty * tiles_x + tx);
        vals[off] = i;
        ++off;
      }
    }
  }
}

__global__ void tile_ranges_kernel(const uint32_t* __restrict__ keys, int64_t n_pairs,
                                   int2* __restrict__ ranges) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const uint32_t t = keys[p];
  if (p == 0 || keys[p - 1] != t) ranges[t].x = (int32_t)p;
  if (p == n_pairs - 1 || keys[p + 1] != t) ranges[t].y = (int32_t)(p + 1);
}

__global__ void tile_len_kernel(const int2* __restrict__ ranges, int n_tiles,
                                int32_t* __restrict__ len, int32_t* __restrict__ ids) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  const int2 r = ranges[t];
  len[t] = r.y - r.x;
  ids[t] = t;
}

static int bits_for(int64_t v) {
  int b = 1;
  while ((1ll << b) < v) ++b;
  return b;
}

}  // namespace ss

using namespace ss;

// Workspace layout: [cub temp | n+1 int32 scratch | n uint64 keys A | n uint64 keys B | n int32 vals]
static size_t cub_bytes(int32_t n, int64_t max_pairs) {
  size_t a = 0, b = 0, c = 0;
  cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, dk, dv, n > 0 ? n : 1, 0, 64);
  cub::DoubleBuffer<uint32_t> pk(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> pv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, b, pk, pv, (int)(max_pairs > 0 ? max_pairs : 1), 0, 16);
  cub::DeviceScan::ExclusiveSum(nullptr, c, (int32_t*)nullptr, (int32_t*)nullptr, n + 1);
  size_t m = a > b ? a : b;
  return m > c ? m : c;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" size_t ss_binning_workspace_bytes(int32_t n, int64_t max_pairs, int32_t n_tiles) {
  (void)n_tiles;
  size_t nn = (size_t)(n > 0 ? n : 1);
  // [cub temp | n+1 int32 | n u64 | n u64 | n int32 | 4n u64 (long-run bitonic scratch)]
  return align256(cub_bytes(n, max_pairs)) + align256((nn + 1) * 4) + 2 * align256(nn * 8) +
         align256(nn * 4) + align256(4 * nn * 8) + 1024;
}

extern "C" int ss_depth_order(const uint64_t* depth_key, int32_t n, int32_t* order, void* ws,
                              size_t ws_bytes, cudaStream_t stream) {
  if (n < 0) return set_error(SS_ERR_INVALID, "ss_depth_order: n < 0");
  if (n == 0) return SS_OK;
  if (ws_bytes < ss_binning_workspace_bytes(n, 1, 1))
    return set_error(SS_ERR_WORKSPACE, "ss_depth_order: workspace too small");
  // stable radix sort of the high 32 key bits (4 passes instead of 8), then a
  // fix-up of equal-high-key runs on the exact 64-bit keys: the result is the
  // stable 64-bit order, i.e. np.lexsort((src, z)) (raster.py:153)
  char* w = (char*)ws;
  const size_t nn = (size_t)n;
  const size_t tb = align256(cub_bytes(n, 1));
  // workspace regions (see ss_binning_workspace_bytes): [cub | n+1 int32 | 2 x n u64 | n int32 | ...]
  int32_t* scratch32 = (int32_t*)(w + tb);
  uint64_t* u64a = (uint64_t*)((char*)scratch32 + align256((nn + 1) * 4));
  uint64_t* u64b = (uint64_t*)((char*)u64a + align256(nn * 8));
  int32_t* vals_in = (int32_t*)((char*)u64b + align256(nn * 8));
  uint32_t* hi_a = (uint32_t*)u64a;
  uint32_t* hi_b = hi_a + nn;  // both high-key buffers fit in region u64a
  high_keys_kernel<<<grid_for(n, 256), 256, 0, stream>>>(depth_key, n, hi_a, vals_in);
  cub::DoubleBuffer<uint32_t> dk(hi_a, hi_b);
  cub::DoubleBuffer<int32_t> dv(vals_in, order);
  size_t tmp_bytes = tb;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(w, tmp_bytes, dk, dv, n, 0, 32, stream);
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "ss_depth_order: %s", cudaGetErrorString(e));
  if (dv.Current() != order)
    cudaMemcpyAsync(order, dv.Current(), nn * 4, cudaMemcpyDeviceToDevice, stream);
  // long-run list in region u64b (int2 per potential run start), its count in scratch32[0]
  int2* long_runs = (int2*)u64b;
  cudaMemsetAsync(scratch32, 0, sizeof(int32_t), stream);
  fix_runs_kernel<<<grid_for(n, 256), 256, 0, stream>>>(dk.Current(), depth_key, n, order,
                                                         long_runs, scratch32);
  // long runs: a run of length L >= 33 sorts in place via the vals_in region
  // (tmp) and, beyond kSmemRun, the u64 region after it (scratch, 2x run.x
  // offset keeps runs disjoint: next_pow2(L) <= 2 L)
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(long_runs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmemRun * 8);
    attr = true;
  }
  long_runs_kernel<<<64, 1024, kSmemRun * 8, stream>>>(depth_key, order, long_runs, scratch32,
                                                        (uint64_t*)((char*)vals_in + align256(nn * 4)),
                                                        vals_in);
  return check_launch("ss_depth_order");
}

extern "C" int ss_tile_offsets(const int32_t* order, const int32_t* n_tiles, int32_t n,
                               int32_t* offsets, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (n < 0) return set_error(SS_ERR_INVALID, "ss_tile_offsets: n < 0");
  size_t need = ss_binning_workspace_bytes(n, 1, 1);
  if (ws_bytes < need) return set_error(SS_ERR_WORKSPACE, "ss_tile_offsets: workspace too small");
  char* w = (char*)ws;
  size_t tb = align256(cub_bytes(n, 1));
  int32_t* cnt = (int32_t*)(w + tb);
  gather_counts_kernel<<<grid_for(n + 1, 256), 256, 0, stream>>>(order, n_tiles, n, cnt);
  size_t tmp_bytes = tb;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(w, tmp_bytes, cnt, offsets, n + 1, stream);
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "ss_tile_offsets: %s", cudaGetErrorString(e));
  return check_launch("ss_tile_offsets");
}

extern "C" int ss_emit_tile_pairs(const int32_t* order, const int32_t* offsets,
                                  const int32_t* bbox, const float* geom,
                                  const uint64_t* tile_mask, int32_t n, int32_t tiles_x,
                                  uint32_t* keys, int32_t* vals, cudaStream_t stream) {
  if (n < 0 || tiles_x <= 0) return set_error(SS_ERR_INVALID, "ss_emit_tile_pairs: bad sizes");
  if (n == 0) return SS_OK;
  emit_pairs_kernel<<<grid_for(n, 128), 128, 0, stream>>>(
      order, offsets, (const int4*)bbox, geom, tile_mask, n, tiles_x, keys, vals);
  return check_launch("ss_emit_tile_pairs");
}

extern "C" int ss_sort_tile_pairs(uint32_t* keys, int32_t* vals, uint32_t* keys_alt,
                                  int32_t* vals_alt, int64_t n_pairs, int32_t n_tiles,
                                  int32_t* out_sel, void* ws, size_t ws_bytes,
                                  cudaStream_t stream) {
  if (n_pairs < 0 || n_tiles <= 0 || n_pairs > 0x7fffffffll)
    return set_error(SS_ERR_INVALID, "ss_sort_tile_pairs: bad sizes");
  *out_sel = 0;
  if (n_pairs == 0) return SS_OK;
  cub::DoubleBuffer<uint32_t> dk(keys, keys_alt);
  cub::DoubleBuffer<int32_t> dv(vals, vals_alt);
  size_t tmp_bytes = 0;
  int bits = bits_for(n_tiles);
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, (int)n_pairs, 0, bits, stream);
  if (tmp_bytes > ws_bytes) return set_error(SS_ERR_WORKSPACE, "ss_sort_tile_pairs: workspace");
  cudaError_t e =
      cub::DeviceRadixSort::SortPairs(ws, tmp_bytes, dk, dv, (int)n_pairs, 0, bits, stream);
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "ss_sort_tile_pairs: %s", cudaGetErrorString(e));
  *out_sel = dk.selector;
  return check_launch("ss_sort_tile_pairs");
}

extern "C" int ss_tile_ranges(const uint32_t* sorted_keys, int64_t n_pairs, int32_t n_tiles,
                              int32_t* ranges, cudaStream_t stream) {
  if (n_pairs < 0 || n_tiles <= 0) return set_error(SS_ERR_INVALID, "ss_tile_ranges: bad sizes");
  cudaMemsetAsync(ranges, 0, sizeof(int32_t) * 2 * (size_t)n_tiles, stream);
  if (n_pairs > 0)
    tile_ranges_kernel<<<grid_for(n_pairs, 256), 256, 0, stream>>>(sorted_keys, n_pairs,
                                                                    (int2*)ranges);
  return check_launch("ss_tile_ranges");
}

// Longest-first tile order in one CTA: counting sort of the tiles by a
// length bucket (4 buckets per octave, longest first).  Only the launch
// order depends on it (each tile's work is independent), so ties within a
// bucket need no fixed order.
constexpr int kOrderMax = 1 << 20;
constexpr int kBuckets = 128;

__device__ __forceinline__ int len_bucket(int len) {
  // 4 * log2(len + 1) without a log: exponent and the top two mantissa bits
  const float f = (float)(len + 1);
  const int b = ((__float_as_int(f) >> 21) - (127 << 2));  // 4 * floor-ish(log2)
  return kBuckets - 1 - min(max(b, 0), kBuckets - 1);
}

__global__ void __launch_bounds__(1024) tile_order_bucket_kernel(const int2* __restrict__ ranges,
                                                                 int n_tiles,
                                                                 int32_t* __restrict__ out) {
  __shared__ int hist[kBuckets];
  __shared__ int cursor[kBuckets];
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int2 r = ranges[t];
    atomicAdd(&hist[len_bucket(r.y - r.x)], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int b = 0; b < kBuckets; ++b) {
      cursor[b] = acc;
      acc += hist[b];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int2 r = ranges[t];
    out[atomicAdd(&cursor[len_bucket(r.y - r.x)], 1)] = t;
  }
}

static size_t tile_order_cub_bytes(int32_t n_tiles) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr,
                                            (int32_t*)nullptr, (int32_t*)nullptr,
                                            n_tiles > 0 ? n_tiles : 1);
  return b;
}

extern "C" size_t ss_tile_order_workspace_bytes(int32_t n_tiles) {
  size_t nn = (size_t)(n_tiles > 0 ? n_tiles : 1);
  return align256(tile_order_cub_bytes(n_tiles)) + 3 * align256(nn * 4) + 256;
}

extern "C" int ss_tile_order(const int32_t* ranges, int32_t n_tiles, int32_t* tile_order,
                             void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (n_tiles <= 0) return set_error(SS_ERR_INVALID, "ss_tile_order: n_tiles <= 0");
  if (n_tiles <= kOrderMax) {
    tile_order_bucket_kernel<<<1, 1024, 0, stream>>>((const int2*)ranges, n_tiles, tile_order);
    return check_launch("ss_tile_order");
  }
  if (ws_bytes < ss_tile_order_workspace_bytes(n_tiles))
    return set_error(SS_ERR_WORKSPACE, "ss_tile_order: workspace too small");
  char* w = (char*)ws;
  const size_t nn = (size_t)n_tiles;
  const size_t tb = align256(tile_order_cub_bytes(n_tiles));
  int32_t* len = (int32_t*)(w + tb);
  int32_t* len_out = (int32_t*)((char*)len + align256(nn * 4));
  int32_t* ids = (int32_t*)((char*)len_out + align256(nn * 4));
  tile_len_kernel<<<grid_for(n_tiles, 256), 256, 0, stream>>>((const int2*)ranges, n_tiles, len,
                                                               ids);
  size_t tmp = tb;
  cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(w, tmp, len, len_out, ids, tile_order,
                                                            n_tiles, 0, 32, stream);
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "ss_tile_order: %s", cudaGetErrorString(e));
  return check_launch("ss_tile_order");
}
