// §8(f)-4 ABR tail-drop selection (server.py:39-79): keep the
// ceil(fraction n) highest-opacity records of a slice, ties to the lower
// index (numpy's stable argsort of -opacity), in ascending index order, and
// gather their wire bytes unchanged.
//
// One CTA per call (a slice holds at most a few 10^5 records):
//   1. radix select, most significant byte first, of the kept_n-th largest
//      opacity key (order-preserving integer image of the opacity);
//   2. a record is kept when its key is above that threshold, or equal to it
//      and among the first (kept_n - #above) equal keys by index (block scans
//      in index order);
//   3. kept records are written in index order: their indices and, for wire
//      slices, their bytes.
#include <cub/block/block_scan.cuh>

#include "ss_common.cuh"

namespace ss {

constexpr int kAbrThreads = 1024;

// Order-preserving 64-bit key of the opacity of record i.  -0.0 is taken as
// +0.0 (numpy compares them equal, so they must tie).
__device__ __forceinline__ uint64_t abr_key(const uint8_t* src, int64_t i, int kind, int stride,
                                            int offset) {
  const uint8_t* p = src + i * stride + offset;
  if (kind == SS_ABR_U8) return (uint64_t)*p;
  if (kind == SS_ABR_F32) {
    uint32_t u = *reinterpret_cast<const uint32_t*>(p);  // 4-aligned (checked on the host)
    if ((u & 0x7fffffffu) == 0u) u = 0u;
    return (uint64_t)((u & 0x80000000u) ? ~u : (u | 0x80000000u));
  }
  uint64_t u = *reinterpret_cast<const uint64_t*>(p);  // 8-aligned (checked on the host)
  if ((u & 0x7fffffffffffffffull) == 0ull) u = 0ull;
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// One record's bytes in the widest words both ends' alignment allows.
__device__ __forceinline__ void copy_record(uint8_t* dst, const uint8_t* src, int stride,
                                            int word) {
  if (word == 8) {
    for (int b = 0; b < stride; b += 8)
      *reinterpret_cast<uint64_t*>(dst + b) = *reinterpret_cast<const uint64_t*>(src + b);
  } else if (word == 4) {
    for (int b = 0; b < stride; b += 4)
      *reinterpret_cast<uint32_t*>(dst + b) = *reinterpret_cast<const uint32_t*>(src + b);
  } else if (word == 2) {
    for (int b = 0; b < stride; b += 2)
      *reinterpret_cast<uint16_t*>(dst + b) = *reinterpret_cast<const uint16_t*>(src + b);
  } else {
    for (int b = 0; b < stride; ++b) dst[b] = src[b];
  }
}

__global__ void __launch_bounds__(kAbrThreads) abr_select_kernel(
    const uint8_t* __restrict__ src, int64_t n, int kind, int stride, int offset, int64_t kept_n,
    int32_t* __restrict__ keep_idx, uint8_t* __restrict__ out, int word) {
  pdl_wait();
  pdl_trigger();
  using Scan = cub::BlockScan<int, kAbrThreads>;
  __shared__ typename Scan::TempStorage s_scan;
  __shared__ int s_hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_need;
  const int tid = threadIdx.x;
  const int key_bytes = kind == SS_ABR_U8 ? 1 : (kind == SS_ABR_F32 ? 4 : 8);
  if (tid == 0) {
    s_prefix = 0ull;
    s_need = kept_n;
  }
  // 1. radix select of the kept_n-th largest key
  for (int byte = key_bytes - 1; byte >= 0; --byte) {
    const int shift = 8 * byte;
    for (int d = tid; d < 256; d += kAbrThreads) s_hist[d] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    const uint64_t hi_mask = byte == 7 ? 0ull : (~0ull << (shift + 8));
    for (int64_t i = tid; i < n; i += kAbrThreads) {
      const uint64_t k = abr_key(src, i, kind, stride, offset);
      if ((k & hi_mask) == prefix) atomicAdd(&s_hist[(k >> shift) & 255u], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int64_t need = s_need;
      int d = 255;
      for (; d > 0; --d) {
        if (s_hist[d] >= need) break;
        need -= s_hist[d];
      }
      s_need = need;
      s_prefix = prefix | ((uint64_t)d << shift);
    }
    __syncthreads();
  }
  const uint64_t thr = s_prefix;
  const int64_t need_eq = s_need;  // equal keys to keep, lowest indices first
  // 2./3. keep flags and index-order compaction, kAbrThreads records a round
  int64_t eq_before = 0, kept_before = 0;
  for (int64_t base = 0; base < n; base += kAbrThreads) {
    const int64_t i = base + tid;
    uint64_t k = 0;
    if (i < n) k = abr_key(src, i, kind, stride, offset);
    const int eq = (i < n && k == thr) ? 1 : 0;
    int eq_rank, eq_total;
    Scan(s_scan).ExclusiveSum(eq, eq_rank, eq_total);
    __syncthreads();
    const int keep = (i < n && (k > thr || (eq && eq_before + eq_rank < need_eq))) ? 1 : 0;
    int pos, kept_total;
    Scan(s_scan).ExclusiveSum(keep, pos, kept_total);
    __syncthreads();
    if (keep) {
      const int64_t o = kept_before + pos;
      keep_idx[o] = (int32_t)i;
      if (out) copy_record(out + o * stride, src + i * stride, stride, word);
    }
    eq_before += eq_total;
    kept_before += kept_total;
  }
}

}  // namespace ss

using namespace ss;

extern "C" int ss_abr_select(const void* src, int64_t n, int32_t kind, int32_t stride,
                             int32_t offset, int64_t kept_n, int32_t* keep_idx, uint8_t* out,
                             cudaStream_t stream) {
  const int key_bytes = kind == SS_ABR_U8 ? 1 : (kind == SS_ABR_F32 ? 4 : 8);
  if (n < 0 || n > 0x7fffffffll || kept_n < 0 || kept_n > n || !src ||
      (kind != SS_ABR_U8 && kind != SS_ABR_F32 && kind != SS_ABR_F64) || offset < 0 ||
      stride < offset + key_bytes || (kept_n > 0 && !keep_idx) ||
      (offset % key_bytes) || (stride % key_bytes) || ((uintptr_t)src % key_bytes))
    return set_error(SS_ERR_INVALID, "ss_abr_select: bad arguments");
  if (n == 0 || kept_n == 0) return SS_OK;
  // copy width: the largest of 8 / 4 / 2 / 1 dividing the stride and both base addresses
  int word = 8;
  while (word > 1 && ((stride % word) || ((uintptr_t)src % word) || (out && (uintptr_t)out % word)))
    word >>= 1;
  launch_k(abr_select_kernel, 1, kAbrThreads, 0, stream, (const uint8_t*)src, n, (int)kind,
           (int)stride, (int)offset, kept_n, keep_idx, out, word);
  return check_launch("ss_abr_select");
}
