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
#include <stdlib.h>

#include "ss_common.cuh"

namespace ss {

__global__ void iota_kernel(int32_t* v, int32_t n) {
  pdl_wait();
  pdl_trigger();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

// Depth order by buckets (no radix sort): the kept keys' range [kmin, kmax]
// is cut into NB = 4 n buckets, b(k) = floor((k - kmin) / (kmax - kmin) *
// (NB - 1)) in fp64 (monotone in k; a bucket holds ~0.25 keys on average);
// culled keys (UINT64_MAX) go to bucket NB.  Keys are scattered to their
// bucket's slots by atomics (order inside a bucket arbitrary), then every
// bucket with more than one key is sorted on (64-bit key, index) -- the
// result is np.lexsort((index, z)) (raster.py:153) on the kept prefix.
constexpr int kBucketsPerKey = 4;

__device__ __forceinline__ uint32_t depth_bucket(uint64_t k, uint64_t kmin, uint64_t kmax,
                                                 uint32_t nb) {
  if (k == ~0ull) return nb;
  const double span = (double)(kmax - kmin);
  const double f = span > 0.0 ? (double)(k - kmin) / span : 0.0;
  const uint32_t b = (uint32_t)(f * (double)(nb - 1));
  return b < nb - 1 ? b : nb - 1;
}

// zero the histogram and reduce the kept keys' range per CTA: partial[2b] =
// ~kmin, partial[2b + 1] = kmax of CTA b (max-reduced from 0); CTA 0 also
// clears the long-run count.  No pre-zeroed accumulator: depth_hist
// reduces the partials itself (a memset launch fewer per view).
constexpr int kRangeBlocks = 296;

__global__ void depth_range_kernel(const uint64_t* __restrict__ key64, int32_t n,
                                   unsigned long long* __restrict__ partial,
                                   int32_t* __restrict__ hist, int32_t nb_total,
                                   int32_t* __restrict__ n_long) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned long long s_r[2][8];
  const int stride = gridDim.x * blockDim.x;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) *n_long = 0;
  for (int i = tid; i < nb_total; i += stride) hist[i] = 0;
  unsigned long long inv_min = 0ull, mx = 0ull;
  for (int i = tid; i < n; i += stride) {
    const uint64_t k = key64[i];
    if (k != ~0ull) {
      inv_min = inv_min > ~k ? inv_min : ~k;
      mx = mx > k ? mx : k;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, inv_min, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, mx, o);
    inv_min = inv_min > a ? inv_min : a;
    mx = mx > b ? mx : b;
  }
  if ((threadIdx.x & 31) == 0) {
    s_r[0][threadIdx.x >> 5] = inv_min;
    s_r[1][threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0ull, b = 0ull;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a = a > s_r[0][w] ? a : s_r[0][w];
      b = b > s_r[1][w] ? b : s_r[1][w];
    }
    partial[2 * blockIdx.x] = a;
    partial[2 * blockIdx.x + 1] = b;
  }
}

// (~kmin, kmax) from depth_range's per-CTA partials, by every CTA of the
// histogram (a few KB of L2 reads each); CTA 0 stores it for the scatter.
__device__ __forceinline__ void reduce_range(const unsigned long long* __restrict__ partial,
                                             int n_part, unsigned long long* __restrict__ range,
                                             unsigned long long& kmin, unsigned long long& kmax) {
  __shared__ unsigned long long s_r[2][8];
  unsigned long long a = 0ull, b = 0ull;
  for (int i = threadIdx.x; i < n_part; i += blockDim.x) {
    const unsigned long long x = partial[2 * i], y = partial[2 * i + 1];
    a = a > x ? a : x;
    b = b > y ? b : y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, a, o);
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, b, o);
    a = a > x ? a : x;
    b = b > y ? b : y;
  }
  if ((threadIdx.x & 31) == 0) {
    s_r[0][threadIdx.x >> 5] = a;
    s_r[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  a = 0ull;
  b = 0ull;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    a = a > s_r[0][w] ? a : s_r[0][w];
    b = b > s_r[1][w] ? b : s_r[1][w];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    range[0] = a;
    range[1] = b;
  }
  kmin = ~a;
  kmax = b;
}

__global__ void depth_hist_kernel(const uint64_t* __restrict__ key64, int32_t n,
                                  const unsigned long long* __restrict__ partial, int n_part,
                                  unsigned long long* __restrict__ range, uint32_t nb,
                                  int32_t* __restrict__ hist) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_culled;
  if (threadIdx.x == 0) s_culled = 0;
  unsigned long long kmin, kmax;
  reduce_range(partial, n_part, range, kmin, kmax);  // (its barrier also covers s_culled)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t k = i < n ? key64[i] : 0ull;
  // culled keys all land in bucket nb: counted per CTA in shared memory and
  // added with one global atomic per CTA (off-view splats are most of a novel
  // view's store; a global atomic per warp on one address serialises), one
  // atomic per kept key otherwise
  const bool culled = i < n && k == ~0ull;
  const uint32_t cm = __ballot_sync(0xffffffffu, culled);
  if (culled && (threadIdx.x & 31) == __ffs(cm) - 1) atomicAdd(&s_culled, __popc(cm));
  if (i < n && !culled) atomicAdd(&hist[depth_bucket(k, kmin, kmax, nb)], 1);
  __syncthreads();
  if (threadIdx.x == 0 && s_culled) atomicAdd(&hist[nb], s_culled);
}

__global__ void depth_scatter_kernel(const uint64_t* __restrict__ key64, int32_t n,
                                     const unsigned long long* __restrict__ range, uint32_t nb,
                                     int32_t* __restrict__ cursor, int32_t* __restrict__ order,
                                     uint32_t* __restrict__ bucket_of) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t k = i < n ? key64[i] : 0ull;
  const bool culled = i < n && k == ~0ull;
  // culled keys: one warp-aggregated atomic on bucket nb (their order inside
  // the trailing culled run is free)
  // (per CTA: warps take offsets in shared memory, one global atomic per CTA)
  __shared__ int32_t s_culled, s_base;
  if (threadIdx.x == 0) s_culled = 0;
  __syncthreads();
  const uint32_t cm = __ballot_sync(0xffffffffu, culled);
  int32_t cbase = 0;
  const int lane = threadIdx.x & 31;
  if (cm && lane == __ffs(cm) - 1) cbase = atomicAdd(&s_culled, __popc(cm));
  __syncthreads();
  if (threadIdx.x == 0 && s_culled) s_base = atomicAdd(&cursor[nb], s_culled);
  __syncthreads();
  cbase = __shfl_sync(0xffffffffu, cbase, cm ? __ffs(cm) - 1 : 0) + (cm ? s_base : 0);
  if (i >= n) return;
  const uint32_t b = culled ? nb : depth_bucket(k, ~range[0], range[1], nb);
  const int32_t pos = culled ? cbase + __popc(cm & ((1u << lane) - 1u)) : atomicAdd(&cursor[b], 1);
  SS_DCHECK(pos >= 0 && pos < n);
  order[pos] = i;
  bucket_of[pos] = b;
}

// Each bucket (a run of equal bucket ids) is sorted by (full 64-bit key,
// index).  Runs of <= 32 (the usual case: a
// few splats per 2^-20 relative depth) take a per-thread insertion sort; longer
// runs are queued for long_runs_kernel (one CTA per run, bitonic sort of
// (64-bit key, index) pairs).
constexpr int kShortRun = 32;
constexpr int kSmemRun = 8192;

__global__ void fix_runs_kernel(const uint32_t* __restrict__ hi_sorted,
                                const uint64_t* __restrict__ key64, int32_t n,
                                int32_t* __restrict__ order, int2* __restrict__ long_runs,
                                int32_t* __restrict__ n_long, uint32_t culled) {
  pdl_wait();
  pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t h = hi_sorted[p];
  if (p > 0 && hi_sorted[p - 1] == h) return;          // not a run start
  if (p + 1 >= n || hi_sorted[p + 1] != h) return;      // singleton run
  if (h == culled) return;  // culled splats: no place in the blend order
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

// Bitonic sort of n2 (power of two) (64-bit depth key, element index) pairs
// by one CTA, lexicographic.
__device__ void cta_bitonic(ulonglong2* a, int n2) {
  for (int size = 2; size <= n2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const ulonglong2 x = a[lo], y = a[hi];
        const bool gt = x.x > y.x || (x.x == y.x && x.y > y.y);
        if (gt == asc) {
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
                                                         ulonglong2* __restrict__ scratch) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ ulonglong2 s_pairs[];
  for (int r = blockIdx.x; r < *n_long; r += gridDim.x) {
    const int2 run = long_runs[r];
    const int L = run.y - run.x;
    int n2 = 1;
    while (n2 < L) n2 <<= 1;
    // beyond shared memory: a private slice of the scratch buffer at the
    // run's offset (n2 <= 2 L, so slices of disjoint runs do not overlap)
    ulonglong2* a = n2 <= kSmemRun ? s_pairs : scratch + 2 * (int64_t)run.x;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
      const int32_t v = i < L ? order[run.x + i] : 0;
      a[i] = i < L ? make_ulonglong2(key64[v], (unsigned long long)v)
                   : make_ulonglong2(~0ull, ~0ull);
    }
    __syncthreads();
    cta_bitonic(a, n2);
    for (int i = threadIdx.x; i < L; i += blockDim.x) order[run.x + i] = (int32_t)a[i].y;
    __syncthreads();
  }
}

// Exclusive scan of N int32 in three library kernels (so the whole chain
// keeps programmatic dependent launch): per-block sums, one CTA over the
// block sums, per-block scan + offset.  GATHER: element e < n is
// in[order[e]] (tile counts in rank order), element n is 0; otherwise in[e].
// In place (in == out) is fine: each element is read and written by the same
// thread in the last pass.
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <bool GATHER>
__device__ __forceinline__ int32_t scan_in(const int32_t* in, const int32_t* order, int n,
                                           int64_t e) {
  if (GATHER) return e < n ? in[order[e]] : 0;
  return in[e];
}

__device__ __forceinline__ int32_t block_exclusive(int32_t v, int32_t* s_warp, int32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  total = s_warp[31];
  const int32_t before = warp > 0 ? s_warp[warp - 1] : 0;
  return before + inc - v;
}

template <bool GATHER>
__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(const int32_t* __restrict__ in,
                                                                 const int32_t* __restrict__ order,
                                                                 int32_t n, int64_t N,
                                                                 int32_t* __restrict__ sums) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_warp[32];
  const int64_t e0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t v = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (e0 + k < N) v += scan_in<GATHER>(in, order, n, e0 + k);
  int32_t total;
  block_exclusive(v, s_warp, total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) scan_top_kernel(int32_t* __restrict__ sums,
                                                                int32_t nblocks) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_warp[32];
  // sequential chunks of the block sums, carried across iterations
  int32_t carry = 0;
  for (int base = 0; base < nblocks; base += kScanThreads) {
    const int i = base + threadIdx.x;
    const int32_t v = i < nblocks ? sums[i] : 0;
    int32_t total;
    const int32_t ex = block_exclusive(v, s_warp, total);
    if (i < nblocks) sums[i] = carry + ex;
    carry += total;
    __syncthreads();
  }
}

template <bool GATHER>
__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const int32_t* in,
                                                                 const int32_t* __restrict__ order,
                                                                 int32_t n, int64_t N,
                                                                 const int32_t* __restrict__ sums,
                                                                 int32_t* out) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_warp[32];
  const int64_t e0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t x[kScanItems];
  int32_t v = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    x[k] = e0 + k < N ? scan_in<GATHER>(in, order, n, e0 + k) : 0;
    v += x[k];
  }
  int32_t total;
  int32_t run = sums[blockIdx.x] + block_exclusive(v, s_warp, total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (e0 + k < N) out[e0 + k] = run;
    run += x[k];
  }
}

template <bool GATHER>
static int exclusive_scan(const int32_t* in, const int32_t* order, int32_t n, int64_t N,
                          int32_t* out, int32_t* block_sums, cudaStream_t stream) {
  const int nblocks = (int)((N + kScanTile - 1) / kScanTile);
  launch_k(scan_sums_kernel<GATHER>, nblocks, kScanThreads, 0, stream, in, order, n, N, block_sums);
  launch_k(scan_top_kernel, 1, kScanThreads, 0, stream, block_sums, nblocks);
  launch_k(scan_down_kernel<GATHER>, nblocks, kScanThreads, 0, stream, in, order, n, N, block_sums,
           out);
  return check_launch("exclusive_scan");
}

__global__ void gather_counts_kernel(const int32_t* __restrict__ order,
                                     const int32_t* __restrict__ n_tiles, int32_t n,
                                     int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const uint32_t t = keys[p];
  if (p == 0 || keys[p - 1] != t) ranges[t].x = (int32_t)p;
  if (p == n_pairs - 1 || keys[p + 1] != t) ranges[t].y = (int32_t)(p + 1);
}

__global__ void tile_len_kernel(const int2* __restrict__ ranges, int n_tiles,
                                int32_t* __restrict__ len, int32_t* __restrict__ ids) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  const int2 r = ranges[t];
  len[t] = r.y - r.x;
  ids[t] = t;
}

// ---------------------------------------------------------------------------
// Chunked binning (default): the rank range [0, n) is cut into C chunks of
// about equal pair counts (bounds from the offsets prefix).
//   emit   : CTA per chunk; lane-per-pair waves write every pair's tile id
//            (u16) and splat id at its emit position offsets[k] + j, and a
//            shared-memory histogram of the chunk's tiles -> counts[c][t]
//   scan   : per tile, exclusive scan of counts[.][t] over the chunks (in
//            place -> base[c][t]) and the tile totals; one CTA scans the
//            totals into tile starts -> ranges
//   scatter: CTA per chunk; waves of 256 pairs in emit order go to their
//            tile's slot start[t] + base[c][t] + (earlier pairs of the chunk
//            in that tile), ranked stably inside the wave (see below).
// Chunks are rank ranges laid out in chunk order inside every tile list and
// each step is stable, so the lists equal the stable global pair sort's.
// equal-tile lanes by a ballot per tile-id bit instead of __match_any
// (whose result latency was the scatter's top short-scoreboard stall)
#ifndef SS_SCATTER_BALLOT_MATCH
#define SS_SCATTER_BALLOT_MATCH 1
#endif
constexpr int kBinThreads = 256;
constexpr int kBinWarps = kBinThreads / 32;

// Chunk c covers ranks [bounds[c], bounds[c+1]): equal shares of the K pairs
// (offsets is the exclusive per-rank pair prefix), so a chunk of near, large
// splats is as short as one of far, small splats.
__global__ void bin_bounds_kernel(const int32_t* __restrict__ offsets, int32_t n, int32_t n_chunks,
                                  int32_t* __restrict__ bounds) {
  pdl_wait();
  pdl_trigger();
  // warp per boundary, 32-ary search: first k with offsets[k] >= target
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c > n_chunks) return;
  if (c == 0) {
    if (lane == 0) bounds[c] = 0;
    return;
  }
  // c == n_chunks searches for K: the trailing ranks with no pair (the culled
  // splats, whose depth key sorts last) belong to no chunk -- as the last
  // chunk's tail they made one CTA walk up to ~25k empty ranks (config 5)
  const int64_t K = offsets[n];
  const int32_t target = (int32_t)(K * c / n_chunks);
  int lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) / 32;
    const int probe = min(hi, lo + (lane + 1) * step);
    const uint32_t below = __ballot_sync(0xffffffffu, offsets[probe] < target);
    const int nb = __popc(below);  // probes below target form a prefix
    const int nlo = lo + nb * step;
    hi = min(hi, lo + (nb + 1) * step);
    lo = nlo;
  }
  const int k = lo + lane;
  const uint32_t below = __ballot_sync(0xffffffffu, k < hi && offsets[k] < target);
  if (lane == 0) bounds[c] = lo + __popc(below);
}

// q = x / w for 0 <= x < 2^20, 1 <= w via the float reciprocal rw = 1/w:
// (x + 0.5) / w is at least 0.5 / w from an integer, far above the rounding.
__device__ __forceinline__ int div_small(int x, float rw) {
  return (int)(((float)x + 0.5f) * rw);
}

__device__ __forceinline__ bool kept_tile(uint64_t mask, int j, const float* gl, int tx, int ty,
                                          int4 bb) {
  return j < 64 ? (bool)((mask >> j) & 1ull) : tile_keeps(gl, tx, ty, bb);
}

// j-th (0-based) set bit of a 64-bit mask (j < popc(mask)).
__device__ __forceinline__ int nth_set_bit(uint64_t mask, int j) {
  const uint32_t lo = (uint32_t)mask;
  const int pl = __popc(lo);
  uint32_t m = j < pl ? lo : (uint32_t)(mask >> 32);
  int jj = j < pl ? j : j - pl;
  int pos = j < pl ? 0 : 32;
#pragma unroll
  for (int width = 16; width >= 1; width >>= 1) {
    const int c = __popc(m & ((1u << width) - 1u));
    if (jj >= c) {
      jj -= c;
      m >>= width;
      pos += width;
    }
  }
  return pos;
}

// pairs a warp stages per 32-splat batch in the emit's common path (at most;
// the launch picks `stage` <= this so that the grid fits one wave, below)
constexpr int kEmitStage = 512;

__global__ void __launch_bounds__(kBinThreads) bin_emit_kernel(
    const int32_t* __restrict__ order, const int32_t* __restrict__ offsets,
    const int4* __restrict__ bbox, const float* __restrict__ geom,
    const uint64_t* __restrict__ tile_mask, const int32_t* __restrict__ bounds, int32_t n_tiles,
    int32_t tiles_x, uint16_t* __restrict__ keys, int32_t* __restrict__ vals,
    int32_t* __restrict__ counts, int stage) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ int32_t s_hist[];  // n_tiles counts, then the warps' stages
  int32_t* stage_v = s_hist + ((n_tiles + 3) & ~3);
  uint16_t* stage_t = reinterpret_cast<uint16_t*>(stage_v + kBinWarps * stage);
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) s_hist[t] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k0 = bounds[blockIdx.x], k1 = bounds[blockIdx.x + 1];
  // the next batch's (offsets, order) are loaded while this batch is
  // walked: only the bbox / mask gathers stay on a batch's critical path
  int pk = k0 + warp * 32 + lane;
  int32_t p_o0 = pk < k1 ? offsets[pk] : 0, p_o1 = pk < k1 ? offsets[pk + 1] : 0;
  int32_t p_i = pk < k1 ? order[pk] : 0;
  for (int kb = k0 + warp * 32; kb < k1; kb += kBinWarps * 32) {
    const int k = kb + lane;
    int32_t i = 0, o0 = 0, cnt = 0, tx0 = 0, ty0 = 0, w = 1, total = 0;
    int4 bb = make_int4(0, 0, 0, 0);
    uint64_t mask = 0;
    const int32_t c_o0 = p_o0, c_o1 = p_o1, c_i = p_i;
    pk = k + kBinWarps * 32;
    p_o0 = pk < k1 ? offsets[pk] : 0;
    p_o1 = pk < k1 ? offsets[pk + 1] : 0;
    p_i = pk < k1 ? order[pk] : 0;
    if (k < k1) {
      o0 = c_o0;
      cnt = c_o1 - o0;
      if (cnt > 0) {
        i = c_i;
        bb = bbox[i];
        mask = tile_mask[i];
        tx0 = bb.x / kTile;
        ty0 = bb.z / kTile;
        w = (bb.y - 1) / kTile + 1 - tx0;
        total = w * ((bb.w - 1) / kTile + 1 - ty0);
      }
    }
    const float rw = 1.f / (float)w;
    const int nm = __popcll(mask);  // the first nm pairs of the splat
    // lane-per-pair waves over the batch's in-mask pairs
    int incl = nm;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - nm;
    const int P = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t far = __ballot_sync(0xffffffffu, total > 64);
    if (!far && P <= stage) {
      // common case: the batch's pairs are exactly its in-mask pairs, one
      // contiguous emit range.  Each lane walks its own splat's mask bits
      // (no per-pair search / shuffles) into the warp's shared stage, which
      // the warp then writes out coalesced.
      uint16_t* st_t = stage_t + warp * stage;
      int32_t* st_v = stage_v + warp * stage;
      // 32-bit halves of the mask; tile = t0 + bit + r (tiles_x - w) with
      // r = bit / w by the float reciprocal
      int pos = excl;
      uint32_t mlo = (uint32_t)mask, mhi = (uint32_t)(mask >> 32);
      const int t0 = ty0 * tiles_x + tx0, dt = tiles_x - w;
      while (mlo | mhi) {
        const bool in_lo = mlo != 0;
        const uint32_t cur = in_lo ? mlo : mhi;
        const int bit = (in_lo ? 0 : 32) + __ffs(cur) - 1;
        if (in_lo) mlo &= mlo - 1u; else mhi &= mhi - 1u;
        const int t = t0 + bit + div_small(bit, rw) * dt;
        SS_DCHECK(t >= 0 && t < n_tiles && pos < stage);
        st_t[pos] = (uint16_t)t;
        st_v[pos] = i;
        atomicAdd(&s_hist[t], 1);
        ++pos;
      }
      __syncwarp();
      const int obase = __shfl_sync(0xffffffffu, o0, 0);
      SS_DCHECK(obase + P <= offsets[bounds[gridDim.x]]);
      for (int p = lane; p < P; p += 32) {
        keys[obase + p] = st_t[p];
        vals[obase + p] = st_v[p];
      }
      __syncwarp();
      continue;
    }
    for (int q = 0; q < P; q += 32) {
      const int p = q + lane;
      int src = 0;  // last lane with excl <= p
#pragma unroll
      for (int b = 16; b >= 1; b >>= 1) {
        const int e = __shfl_sync(0xffffffffu, excl, src + b);
        if (e <= p) src += b;
      }
      const int j = p - __shfl_sync(0xffffffffu, excl, src);
      const int32_t si = __shfl_sync(0xffffffffu, i, src);
      const uint32_t mlo = __shfl_sync(0xffffffffu, (uint32_t)mask, src);
      const uint32_t mhi = __shfl_sync(0xffffffffu, (uint32_t)(mask >> 32), src);
      const int stx0 = __shfl_sync(0xffffffffu, tx0, src);
      const int sty0 = __shfl_sync(0xffffffffu, ty0, src);
      const int sw = __shfl_sync(0xffffffffu, w, src);
      const float srw = __shfl_sync(0xffffffffu, rw, src);
      const int so0 = __shfl_sync(0xffffffffu, o0, src);
      if (p < P) {
        const int bit = nth_set_bit(((uint64_t)mhi << 32) | mlo, j);
        const int r = div_small(bit, srw);
        const int t = (sty0 + r) * tiles_x + stx0 + bit - r * sw;
        SS_DCHECK(bit >= 0 && bit < 64 && t >= 0 && t < n_tiles && so0 + j < offsets[bounds[gridDim.x]]);
        keys[so0 + j] = (uint16_t)t;
        vals[so0 + j] = si;
        atomicAdd(&s_hist[t], 1);
      }
    }
    // tiles past the 64-bit mask of large splats: splat by splat, lanes over
    // the bbox tiles, emit positions by ballot prefix (bbox order)
    while (far) {
      const int src = __ffs(far) - 1;
      far &= far - 1;
      const int32_t si = __shfl_sync(0xffffffffu, i, src);
      const int4 sbb = make_int4(__shfl_sync(0xffffffffu, bb.x, src),
                                 __shfl_sync(0xffffffffu, bb.y, src),
                                 __shfl_sync(0xffffffffu, bb.z, src),
                                 __shfl_sync(0xffffffffu, bb.w, src));
      const int stx0 = __shfl_sync(0xffffffffu, tx0, src);
      const int sty0 = __shfl_sync(0xffffffffu, ty0, src);
      const int sw = __shfl_sync(0xffffffffu, w, src);
      const int stot = __shfl_sync(0xffffffffu, total, src);
      const float srw = __shfl_sync(0xffffffffu, rw, src);
      int e = __shfl_sync(0xffffffffu, o0 + nm, src);
      float gl[kGeom];
#pragma unroll
      for (int q = 0; q < kGeom; ++q) gl[q] = geom[(int64_t)si * kGeom + q];
      for (int j0 = 64; j0 < stot; j0 += 32) {
        const int j = j0 + lane;
        int t = 0;
        bool keep = false;
        if (j < stot) {
          const int r = div_small(j, srw);
          const int ty = sty0 + r, tx = stx0 + j - r * sw;
          keep = tile_keeps(gl, tx, ty, sbb);
          t = ty * tiles_x + tx;
        }
        const uint32_t kb2 = __ballot_sync(0xffffffffu, keep);
        if (keep) {
          const int q = e + __popc(kb2 & ((1u << lane) - 1u));
          SS_DCHECK(t >= 0 && t < n_tiles && q < offsets[bounds[gridDim.x]]);
          keys[q] = (uint16_t)t;
          vals[q] = si;
          atomicAdd(&s_hist[t], 1);
        }
        e += __popc(kb2);
      }
    }
  }
  __syncthreads();
  int32_t* row = counts + (int64_t)blockIdx.x * n_tiles;
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) row[t] = s_hist[t];
}

// Block (32 tiles) x (8 warps); warp w scans chunks [w C8, (w+1) C8).
__global__ void __launch_bounds__(kBinThreads) bin_col_scan_kernel(int32_t* __restrict__ counts,
                                                                   int32_t n_chunks,
                                                                   int32_t n_tiles,
                                                                   int32_t* __restrict__ totals) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_part[kBinWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  const int per = (n_chunks + kBinWarps - 1) / kBinWarps;
  const int c0 = warp * per, c1 = min(n_chunks, c0 + per);
  int32_t sum = 0;
  if (t < n_tiles) {
#pragma unroll 8
    for (int c = c0; c < c1; ++c) sum += counts[(int64_t)c * n_tiles + t];
  }
  s_part[warp][lane] = sum;
  __syncthreads();
  int32_t run = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kBinWarps; ++w) {
    run += w < warp ? s_part[w][lane] : 0;
    all += s_part[w][lane];
  }
  if (t >= n_tiles) return;
  if (warp == 0) totals[t] = all;
  for (int cb = c0; cb < c1; cb += 8) {
    int32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = cb + u < c1 ? counts[(int64_t)(cb + u) * n_tiles + t] : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (cb + u < c1) counts[(int64_t)(cb + u) * n_tiles + t] = run;
      run += v[u];
    }
  }
}

// One CTA: exclusive scan of the tile totals -> start[t], ranges[t].
constexpr int kOrderMax = 1 << 20;
constexpr int kBuckets = 128;
static_assert(kBuckets == 4 * 32, "scan_buckets: 4 buckets per lane of one warp");

__device__ __forceinline__ int len_bucket(int len) {
  // 4 * log2(len + 1) without a log: exponent and the top two mantissa bits
  const float f = (float)(len + 1);
  const int b = ((__float_as_int(f) >> 21) - (127 << 2));  // 4 * floor-ish(log2)
  return kBuckets - 1 - min(max(b, 0), kBuckets - 1);
}

// Exclusive scan of the kBuckets (= 128) length-bucket counts by warp 0
// (4 per lane + one warp scan) instead of a serial loop on thread 0.
__device__ __forceinline__ void scan_buckets(const int* hist, int* cursor) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int v[4], run = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = hist[4 * lane + k];
    run += v[k];
  }
  int incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int acc = incl - run;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    cursor[4 * lane + k] = acc;
    acc += v[k];
  }
}

__global__ void __launch_bounds__(1024) bin_tile_scan_kernel(const int32_t* __restrict__ totals,
                                                             int32_t n_tiles,
                                                             int32_t* __restrict__ start,
                                                             int2* __restrict__ ranges,
                                                             int32_t* __restrict__ tile_order) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_warp[32];
  __shared__ int s_hist[kBuckets];
  extern __shared__ int32_t s_tot[];  // totals staged by coalesced loads
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) s_tot[t] = totals[t];
  __syncthreads();
  const int per = (n_tiles + blockDim.x - 1) / blockDim.x;
  const int t0 = threadIdx.x * per, t1 = min(n_tiles, t0 + per);
  int32_t local = 0;
  for (int t = t0; t < t1; ++t) local += s_tot[t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t inc = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int32_t v = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    s_warp[lane] = v;  // inclusive over warps
  }
  __syncthreads();
  int32_t run = inc - local + (warp > 0 ? s_warp[warp - 1] : 0);
  for (int t = t0; t < t1; ++t) {
    const int32_t c = s_tot[t];
    s_tot[t] = run;
    run += c;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) s_hist[i] = 0;
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int32_t a = s_tot[t];
    const int32_t len = totals[t];
    start[t] = a;
    ranges[t] = make_int2(a, a + len);
    s_tot[t] = len;  // this thread's own entries only: no race with the scan reads above
  }
  if (!tile_order) return;
  // the raster launch order (ss_tile_order's counting sort by list-length
  // bucket, longest first) from the totals already in shared memory
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) atomicAdd(&s_hist[len_bucket(s_tot[t])], 1);
  __syncthreads();
  scan_buckets(s_hist, s_hist);  // in place: each lane reads its 4 before writing them
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
    tile_order[atomicAdd(&s_hist[len_bucket(s_tot[t])], 1)] = t;
}

// Stable scatter of one chunk: waves of 256 pairs in emit order, one per
// thread.  Equal tiles inside a warp are ranked by lane (__match_any); the
// warps' counts per tile sit in byte w of a 64-bit shared word per tile, so
// a pair's slot is cur[t] + (counts of lower warps) + (rank in its warp) --
// the wave's pairs land in emit order.  The highest warp holding a tile then
// advances cur[t] and clears the word.
__global__ void __launch_bounds__(kBinThreads) bin_scatter_kernel(
    const int32_t* __restrict__ offsets, const int32_t* __restrict__ bounds,
    const uint16_t* __restrict__ keys, const int32_t* __restrict__ vals, int32_t n_tiles,
    int32_t* __restrict__ base, const int32_t* __restrict__ start,
    int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char s_dyn[];
  unsigned long long* s_wc = reinterpret_cast<unsigned long long*>(s_dyn);  // n_tiles
  int32_t* s_cur = reinterpret_cast<int32_t*>(s_wc + n_tiles);              // n_tiles
  const int c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* brow = base + (int64_t)c * n_tiles;
  const int q0 = offsets[bounds[c]], q1 = offsets[bounds[c + 1]];
  // software pipelined: the pairs of the next kAhead waves are in flight
  // while this one is placed (one wave of lookahead left the loop waiting
  // on L2 latency: long_scoreboard was the top stall)
  constexpr int kAhead = 4;
  int tq[kAhead];
  int32_t vq[kAhead];
#pragma unroll
  for (int d = 0; d < kAhead; ++d) {
    const int q = q0 + d * kBinThreads + threadIdx.x;
    tq[d] = q < q1 ? keys[q] : n_tiles;  // n_tiles: no tile
    vq[d] = q < q1 ? vals[q] : 0;
  }
  // cursor init, 8 tiles per thread in flight (written as separate load
  // and store phases: ptxas otherwise serialised load -> add -> store)
  for (int t0 = threadIdx.x; t0 < n_tiles; t0 += 8 * kBinThreads) {
    int32_t a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u * kBinThreads;
      a[u] = t < n_tiles ? start[t] + brow[t] : 0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u * kBinThreads;
      if (t < n_tiles) {
        s_cur[t] = a[u];
        s_wc[t] = 0ull;
        // chunk 0's base row is dead once read: it becomes the zeroed
        // per-tile work counts of the raster forward (view.cu aliases them
        // to the workspace start), which then needs no memset launch
        if (c == 0) brow[t] = 0;
      }
    }
  }
  const uint32_t lt = (1u << lane) - 1u;
  const unsigned long long below_mask = (1ull << (8 * warp)) - 1ull;
  unsigned char* s_wc8 = reinterpret_cast<unsigned char*>(s_wc);
  const int tbits = 32 - __clz(n_tiles);  // t <= n_tiles (n_tiles: no tile)
  for (int qr = q0; qr < q1; qr += kAhead * kBinThreads) {
#pragma unroll
    for (int d = 0; d < kAhead; ++d) {
      const int qb = qr + d * kBinThreads;
      if (qb >= q1) break;  // uniform over the CTA
      const bool ok = qb + threadIdx.x < q1;
      const int t = tq[d];
      const int32_t v = vq[d];
#if SS_SCATTER_BALLOT_MATCH
      uint32_t peers = 0xffffffffu;  // lanes with the same t, by ballots over t's bits
      for (int b = 0; b < tbits; ++b) {
        const uint32_t ones = __ballot_sync(0xffffffffu, (t >> b) & 1);
        peers &= ((t >> b) & 1) ? ones : ~ones;
      }
#else
      const uint32_t peers = __match_any_sync(0xffffffffu, t);
#endif
      const int leader = __ffs(peers) - 1;
      const int cnt = __popc(peers), rin = __popc(peers & lt);
      __syncthreads();  // previous wave's cursor updates / clears are done
      if (ok && lane == leader) s_wc8[(size_t)t * 8 + warp] = (unsigned char)cnt;
      __syncthreads();
      int prefix = 0;
      bool last = false;
      if (ok) {
        const unsigned long long word = s_wc[t];
        // byte sum of the lower warps' counts (each <= 32, sum <= 224 < 256)
        prefix = (int)(((word & below_mask) * 0x0101010101010101ull) >> 56);
        last = warp == 7 || (word >> (8 * (warp + 1))) == 0ull;
        SS_DCHECK(t >= 0 && t < n_tiles && s_cur[t] + prefix + rin >= start[t] &&
                  s_cur[t] + prefix + rin < (t + 1 < n_tiles ? start[t + 1] : offsets[bounds[gridDim.x]]));
#ifdef SS_DIAG_SCATTER_NOSTORE
        if (v == -12345) out[s_cur[t] + prefix + rin] = v;
#else
        out[s_cur[t] + prefix + rin] = v;
#endif
      }
      __syncthreads();
      if (ok && lane == leader && last) {
        s_cur[t] += prefix + cnt;
        s_wc[t] = 0ull;
      }
      // refill this slot only now that t and v are dead: the load can then
      // target their registers (a refill at the top of the section made
      // ptxas load into a temporary and MOV it back at the end -- a MOV
      // that waited on the load, i.e. one wave of lookahead, not kAhead)
      const int qn = qb + kAhead * kBinThreads + threadIdx.x;
      tq[d] = qn < q1 ? keys[qn] : n_tiles;
      vq[d] = qn < q1 ? vals[qn] : 0;
    }
  }
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
  size_t d = 0;  // depth-order bucket scan (kBucketsPerKey n + 1 counts)
  cub::DeviceScan::ExclusiveSum(nullptr, d, (int32_t*)nullptr, (int32_t*)nullptr,
                                kBucketsPerKey * (n > 0 ? n : 1) + 1);
  size_t m = a > b ? a : b;
  m = m > c ? m : c;
  return m > d ? m : d;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" size_t ss_binning_workspace_bytes(int32_t n, int64_t max_pairs, int32_t n_tiles) {
  (void)n_tiles;
  size_t nn = (size_t)(n > 0 ? n : 1);
  // [cub temp | n+1 int32 | n u64 | n u64 | n int32 | 4n u64 (long-run bitonic scratch:
  //  16-byte pairs, a run of L at offset 2 run.x pairs, next_pow2(L) <= 2 L)]
  return align256(cub_bytes(n, max_pairs)) + align256((nn + 1) * 4) + 2 * align256(nn * 8) +
         align256(nn * 4) + align256(4 * nn * 8) + 1024;
}

extern "C" int ss_depth_order(const uint64_t* depth_key, int32_t n, int32_t* order, void* ws,
                              size_t ws_bytes, cudaStream_t stream) {
  if (n < 0) return set_error(SS_ERR_INVALID, "ss_depth_order: n < 0");
  if (n == 0) return SS_OK;
  if (ws_bytes < ss_binning_workspace_bytes(n, 1, 1))
    return set_error(SS_ERR_WORKSPACE, "ss_depth_order: workspace too small");
  // workspace regions (ss_binning_workspace_bytes): [cub | n+1 int32 | n u64 | n u64 | n int32 |
  // 4n u64]; here: scratch32 = [n_long, pad, range (2 u64)], u64a = bucket ids (n u32) + long
  // run list, the 4n u64 region = histogram / cursors (NB + 1 int32), later long-run scratch
  char* w = (char*)ws;
  const size_t nn = (size_t)n;
  const size_t tb = align256(cub_bytes(n, 1));
  int32_t* scratch32 = (int32_t*)(w + tb);
  unsigned long long* range = (unsigned long long*)(scratch32 + 2);
  uint64_t* u64a = (uint64_t*)((char*)scratch32 + align256((nn + 1) * 4));
  uint64_t* u64b = (uint64_t*)((char*)u64a + align256(nn * 8));
  int32_t* vals_in = (int32_t*)((char*)u64b + align256(nn * 8));
  int32_t* big = (int32_t*)((char*)vals_in + align256(nn * 4));
  uint32_t* bucket_of = (uint32_t*)u64a;
  int2* long_runs = (int2*)((char*)u64a + align256(nn * 4));
  const uint32_t nb = (uint32_t)(kBucketsPerKey * nn);
  int32_t* hist = big;  // nb + 1 counts, scanned in place into the bucket cursors
  // per-CTA range partials at the end of the scratch32 region (n + 1 int32;
  // its head holds n_long, range and the histogram scan's block sums:
  // ~n / 256 + 8 ints, the partials n / 16 + 16 bytes at most)
  const int n_range = min(kRangeBlocks, (n + 255) / 256);
  unsigned long long* partial =
      (unsigned long long*)((char*)scratch32 + align256((nn + 1) * 4) - (size_t)n_range * 16);
  launch_k(depth_range_kernel, n_range, 256, 0, stream, depth_key, n, partial, hist,
           (int32_t)nb + 1, scratch32);
  launch_k(depth_hist_kernel, grid_for(n, 256), 256, 0, stream, depth_key, n,
           (const unsigned long long*)partial, n_range, range, nb, hist);
  // block sums after n_long / pad / range in the scratch32 region
  int rc = exclusive_scan<false>(hist, nullptr, 0, (int64_t)nb + 1, hist, scratch32 + 8, stream);
  if (rc) return rc;
  launch_k(depth_scatter_kernel, grid_for(n, 256), 256, 0, stream, depth_key, n, range, nb, hist, order,
                                                             bucket_of);
  launch_k(fix_runs_kernel, grid_for(n, 256), 256, 0, stream, bucket_of, depth_key, n, order, long_runs,
                                                         scratch32, nb);
  // long runs: a run of length L >= 33 sorts in shared memory, or beyond
  // kSmemRun in the 4n u64 region (a run of L at offset 2 run.x pairs)
  if (int rc2 = ensure_smem((const void*)long_runs_kernel, kSmemRun * 16)) return rc2;
  launch_k(long_runs_kernel, 64, 1024, kSmemRun * 16, stream, depth_key, order, long_runs, scratch32,
                                                         (ulonglong2*)big);
  return check_launch("ss_depth_order");
}

extern "C" int ss_tile_offsets(const int32_t* order, const int32_t* n_tiles, int32_t n,
                               int32_t* offsets, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (n < 0) return set_error(SS_ERR_INVALID, "ss_tile_offsets: n < 0");
  size_t need = ss_binning_workspace_bytes(n, 1, 1);
  if (ws_bytes < need) return set_error(SS_ERR_WORKSPACE, "ss_tile_offsets: workspace too small");
  char* w = (char*)ws;
  size_t tb = align256(cub_bytes(n, 1));
  int32_t* block_sums = (int32_t*)(w + tb);  // the n+1 int32 scratch region
  // offsets[k] = sum of the kept-tile counts of ranks < k (gathered on the fly)
  return exclusive_scan<true>(n_tiles, order, n, (int64_t)n + 1, offsets, block_sums, stream);
}

extern "C" int ss_emit_tile_pairs(const int32_t* order, const int32_t* offsets,
                                  const int32_t* bbox, const float* geom,
                                  const uint64_t* tile_mask, int32_t n, int32_t tiles_x,
                                  uint32_t* keys, int32_t* vals, cudaStream_t stream) {
  if (n < 0 || tiles_x <= 0) return set_error(SS_ERR_INVALID, "ss_emit_tile_pairs: bad sizes");
  if (n == 0) return SS_OK;
  launch_k(emit_pairs_kernel, grid_for(n, 128), 128, 0, stream, 
      order, offsets, (const int4*)bbox, geom, tile_mask, n, tiles_x, keys, vals);
  return check_launch("ss_emit_tile_pairs");
}

static int g_binning = 0;  // 0 = counting sort, 1 = pair radix sort

extern "C" int ss_set_binning(int32_t mode) {
  if (mode != 0 && mode != 1) return set_error(SS_ERR_INVALID, "ss_set_binning: mode must be 0 or 1");
  g_binning = mode;
  return SS_OK;
}

extern "C" int ss_get_binning(void) { return g_binning; }

// Chunks: a whole number of scatter waves (resident CTAs on 148 SMs), each
// chunk at most ~32k pairs (bounds balance them by pairs), at most 4096.  At
// large K (config 5: 1M splats, 1920x1080) fewer, longer chunks keep the
// (chunks x tiles) histogram small: 32k measured best (16k / 64k slower).
#ifndef SS_BIN_PAIRS_PER_CHUNK
#define SS_BIN_PAIRS_PER_CHUNK 32768
#endif
constexpr int kBinPairsPerChunk = SS_BIN_PAIRS_PER_CHUNK;
constexpr int kBinChunksCap = 4096;
constexpr int kBinMaxTiles = 18 * 1024;  // 12 bytes of shared memory per tile in the scatter

static int bin_chunks(int64_t n_pairs, int n_tiles) {
  int per_sm = (int)(228 * 1024 / ((size_t)n_tiles * 12 + 1024));
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  const int64_t slots = 148ll * per_sm;
  const int64_t waves = (n_pairs + slots * kBinPairsPerChunk - 1) / (slots * kBinPairsPerChunk);
  const int64_t c = slots * (waves < 1 ? 1 : waves);
  return (int)(c > kBinChunksCap ? kBinChunksCap : c);
}

// Stage entries per emit warp: the largest multiple of 32 (<= kEmitStage)
// that lets the C emit CTAs run in ONE wave (a grid of 1.33 waves -- e.g. 592
// chunks at 3 CTAs per SM at 1920x1080 -- leaves a quarter of the SMs
// running a second chunk alone: 2x the kernel time).  Batches with more
// pairs than the stage take the lane-per-pair path.  Below 256 entries the
// full stage is kept (too many batches would fall off the fast path).
static int emit_stage(int C, int n_tiles) {
  const int per_sm = (C + 147) / 148;
  const size_t hist = (size_t)((n_tiles + 3) & ~3) * 4;
  if (per_sm > 4) return kEmitStage;  // the register limit (57 regs x 256 threads) is 4 CTAs/SM
  const size_t per_cta = (size_t)228 * 1024 / per_sm - 1024;  // 1 KB reserved per CTA
  if (per_cta <= hist) return kEmitStage;
  const size_t s = (per_cta - hist) / ((size_t)kBinWarps * 6) / 32 * 32;
  return s >= (size_t)kEmitStage ? kEmitStage : (s >= 256 ? (int)s : kEmitStage);
}

extern "C" size_t ss_bin_tiles_workspace_bytes(int64_t n_pairs, int32_t n_tiles) {
  const size_t nt = (size_t)(n_tiles > 0 ? n_tiles : 1);
  const size_t C = (size_t)bin_chunks(n_pairs, (int)nt);
  return align256(C * nt * 4) + 2 * align256(nt * 4) + align256((C + 1) * 4) + 256;
}

extern "C" int32_t ss_bin_tiles_supported(int64_t n_pairs, int32_t n_tiles) {
  return n_tiles > 0 && n_tiles <= kBinMaxTiles && n_pairs < (1ll << 31) ? 1 : 0;
}

extern "C" int ss_bin_tiles(const int32_t* order, const int32_t* offsets, const int32_t* bbox,
                            const float* geom, const uint64_t* tile_mask, int32_t n,
                            int64_t n_pairs, int32_t tiles_x, int32_t tiles_y, uint16_t* keys,
                            int32_t* vals, int32_t* vals_out, int32_t* ranges, void* ws,
                            size_t ws_bytes, cudaStream_t stream) {
  return bin_tiles_with_order(order, offsets, bbox, geom, tile_mask, n, n_pairs, tiles_x, tiles_y,
                              keys, vals, vals_out, ranges, nullptr, ws, ws_bytes, stream);
}

// ss_bin_tiles that also writes the raster launch order (ss_tile_order's
// result) from its tile scan when tile_order != NULL -- except with no pairs
// (n == 0 or n_pairs == 0), where only the empty ranges are written.
int bin_tiles_with_order(const int32_t* order, const int32_t* offsets, const int32_t* bbox,
                         const float* geom, const uint64_t* tile_mask, int32_t n,
                         int64_t n_pairs, int32_t tiles_x, int32_t tiles_y, uint16_t* keys,
                         int32_t* vals, int32_t* vals_out, int32_t* ranges, int32_t* tile_order,
                         void* ws, size_t ws_bytes, cudaStream_t stream) {
  const int n_tiles = tiles_x * tiles_y;
  if (n < 0 || tiles_x <= 0 || tiles_y <= 0 || n_pairs < 0)
    return set_error(SS_ERR_INVALID, "ss_bin_tiles: bad sizes");
  if (!ss_bin_tiles_supported(n_pairs, n_tiles))
    return set_error(SS_ERR_INVALID, "ss_bin_tiles: %d tiles / %lld pairs unsupported (use the pair sort)",
                     n_tiles, (long long)n_pairs);
  if (ws_bytes < ss_bin_tiles_workspace_bytes(n_pairs, n_tiles))
    return set_error(SS_ERR_WORKSPACE, "ss_bin_tiles: workspace too small");
  if (n == 0 || n_pairs == 0) {
    memzero(ranges, sizeof(int32_t) * 2 * (size_t)n_tiles, stream);
    return check_launch("ss_bin_tiles");
  }
  const int C = bin_chunks(n_pairs, n_tiles);
  char* w = (char*)ws;
  int32_t* counts = (int32_t*)w;
  int32_t* totals = (int32_t*)(w + align256((size_t)C * n_tiles * 4));
  int32_t* start = (int32_t*)((char*)totals + align256((size_t)n_tiles * 4));
  int32_t* bounds = (int32_t*)((char*)start + align256((size_t)n_tiles * 4));
  const size_t smem = (size_t)n_tiles * 4;  // tile scan
  const int stage = emit_stage(C, n_tiles);
  const size_t smem_emit = (size_t)((n_tiles + 3) & ~3) * 4 + (size_t)kBinWarps * stage * 6;
  const size_t smem_scatter = (size_t)n_tiles * 12;
  int rc;
  if ((rc = ensure_smem((const void*)bin_emit_kernel, smem_emit)) ||
      (rc = ensure_smem((const void*)bin_tile_scan_kernel, smem)) ||
      (rc = ensure_smem((const void*)bin_scatter_kernel, smem_scatter)))
    return rc;
  launch_k(bin_bounds_kernel, (32 * (C + 1) + 127) / 128, 128, 0, stream, offsets, n, C, bounds);
  launch_k(bin_emit_kernel, C, kBinThreads, smem_emit, stream, order, offsets, (const int4*)bbox, geom,
                                                    tile_mask, bounds, n_tiles, tiles_x, keys,
                                                    vals, counts, stage);
  launch_k(bin_col_scan_kernel, (n_tiles + 31) / 32, kBinThreads, 0, stream, counts, C, n_tiles, totals);
  launch_k(bin_tile_scan_kernel, 1, 1024, (size_t)n_tiles * 4, stream, totals, n_tiles, start,
           (int2*)ranges, tile_order);
  launch_k(bin_scatter_kernel, C, kBinThreads, smem_scatter, stream, offsets, bounds, keys, vals,
                                                               n_tiles, counts, start, vals_out);
  return check_launch("ss_bin_tiles");
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
  memzero(ranges, sizeof(int32_t) * 2 * (size_t)n_tiles, stream);
  if (n_pairs > 0)
    launch_k(tile_ranges_kernel, grid_for(n_pairs, 256), 256, 0, stream, sorted_keys, n_pairs,
                                                                    (int2*)ranges);
  return check_launch("ss_tile_ranges");
}

// Longest-first tile order in one CTA: counting sort of the tiles by a
// length bucket (4 buckets per octave, longest first).  Only the launch
// order depends on it (each tile's work is independent), so ties within a
// bucket need no fixed order.
__global__ void __launch_bounds__(1024) tile_order_bucket_kernel(const int2* __restrict__ ranges,
                                                                 int n_tiles,
                                                                 int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ int hist[kBuckets];
  __shared__ int cursor[kBuckets];
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int2 r = ranges[t];
    atomicAdd(&hist[len_bucket(r.y - r.x)], 1);
  }
  __syncthreads();
  scan_buckets(hist, cursor);
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int2 r = ranges[t];
    out[atomicAdd(&cursor[len_bucket(r.y - r.x)], 1)] = t;
  }
}

// The same counting sort keyed by a per-tile work count (the backward's
// walked entries, accumulated by the forward).
__global__ void __launch_bounds__(1024) tile_order_work_kernel(const int32_t* __restrict__ work,
                                                               int n_tiles,
                                                               int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ int hist[kBuckets];
  __shared__ int cursor[kBuckets];
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) atomicAdd(&hist[len_bucket(work[t])], 1);
  __syncthreads();
  scan_buckets(hist, cursor);
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
    out[atomicAdd(&cursor[len_bucket(work[t])], 1)] = t;
}

int tile_order_from_work(const int32_t* work, int32_t n_tiles, int32_t* tile_order,
                         cudaStream_t stream) {
  if (n_tiles <= 0 || n_tiles > kOrderMax)
    return set_error(SS_ERR_INVALID, "tile_order_from_work: %d tiles", n_tiles);
  launch_k(tile_order_work_kernel, 1, 1024, 0, stream, work, n_tiles, tile_order);
  return check_launch("tile_order_from_work");
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
    launch_k(tile_order_bucket_kernel, 1, 1024, 0, stream, (const int2*)ranges, n_tiles, tile_order);
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
  launch_k(tile_len_kernel, grid_for(n_tiles, 256), 256, 0, stream, (const int2*)ranges, n_tiles, len,
                                                               ids);
  size_t tmp = tb;
  cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(w, tmp, len, len_out, ids, tile_order,
                                                            n_tiles, 0, 32, stream);
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "ss_tile_order: %s", cudaGetErrorString(e));
  return check_launch("ss_tile_order");
}
