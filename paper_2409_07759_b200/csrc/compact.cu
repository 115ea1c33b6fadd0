// a-2  Active-set compaction by lifespan (core.py:280-282; train.py:347-350, 380-386).
//
// Stream compaction over per-row int32 lifespans: ballot + warp/block
// prefix sums in two passes (per-block counts, then a single-block scan of
// the counts, then an order-preserving scatter).  Candidates: optimizable
// rows in row order, then matured rows in archive (FIFO) order.
#include "ss_common.cuh"

namespace ss {

constexpr int kCompactBlock = 256;
constexpr int kCompactItems = 4;  // items per thread
constexpr int kCompactTile = kCompactBlock * kCompactItems;

struct CandMap {
  const int32_t* start;
  const int32_t* expire;
  int64_t n_opt;
  int64_t n_cand;
  const int32_t* blk_map;
  int32_t block_rows;
  int32_t frame;
};

// Physical row of candidate c (optimizable rows in order, then matured rows
// through the block map), or -1 past the end.
__device__ __forceinline__ int64_t cand_phys(const CandMap& m, int64_t c) {
  if (c >= m.n_cand) return -1;
  if (c < m.n_opt) return c;
  const int64_t lc = c - m.n_opt;
  const int64_t pb = m.blk_map ? m.blk_map[lc / m.block_rows] : lc / m.block_rows;
  return m.n_opt + pb * m.block_rows + lc % m.block_rows;
}

// Active row ids of a thread's kCompactItems candidates (-1: inactive): the
// physical rows first, then every lifespan load in flight together (one
// memory round trip instead of one per candidate).
__device__ __forceinline__ void cand_rows(const CandMap& m, int64_t base, int32_t out[kCompactItems]) {
  int64_t phys[kCompactItems];
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k) phys[k] = cand_phys(m, base + k * kCompactBlock + threadIdx.x);
  int32_t s[kCompactItems], e[kCompactItems];
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k) {
    s[k] = phys[k] >= 0 ? m.start[phys[k]] : 1;
    e[k] = phys[k] >= 0 ? m.expire[phys[k]] : 0;
  }
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k)
    out[k] = (s[k] <= m.frame && m.frame < e[k]) ? (int32_t)phys[k] : -1;
}

__global__ void compact_count(CandMap m, int32_t* block_counts) {
  pdl_wait();
  pdl_trigger();
  int64_t base = (int64_t)blockIdx.x * kCompactTile;
  int32_t rowv[kCompactItems];
  cand_rows(m, base, rowv);
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k) cnt += rowv[k] >= 0;
  __shared__ int s_sum[kCompactBlock / 32];
  int w = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < kCompactBlock / 32; ++i) t += s_sum[i];
    block_counts[blockIdx.x] = t;
  }
}

// Single block: exclusive scan of block counts in place (n_blocks <= any).
__global__ void compact_scan(int32_t* block_counts, int n_blocks, int32_t* total) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_carry;
  __shared__ int s_warp[32];
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n_blocks; base += blockDim.x) {
    int i = base + threadIdx.x;
    int v = i < n_blocks ? block_counts[i] : 0;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int nw = blockDim.x >> 5;
      int wv = lane < nw ? s_warp[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, wv, o);
        if (lane >= o) wv += y;
      }
      if (lane < nw) s_warp[lane] = wv;
    }
    __syncthreads();
    int incl = x + (wid > 0 ? s_warp[wid - 1] : 0) + s_carry;
    if (i < n_blocks) block_counts[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = s_carry;
}

__global__ void compact_scatter(CandMap m, const int32_t* block_offsets, int32_t* out_rows,
                                int32_t* out_counts, const int32_t* total) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_warp[kCompactBlock / 32];
  __shared__ int s_base;
  int64_t base = (int64_t)blockIdx.x * kCompactTile;
  if (threadIdx.x == 0) s_base = block_offsets[blockIdx.x];
  __syncthreads();
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t rowv[kCompactItems];
  cand_rows(m, base, rowv);
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k) {
    int64_t c = base + k * kCompactBlock + threadIdx.x;
    int32_t row = rowv[k];
    unsigned ball = __ballot_sync(0xffffffffu, row >= 0);
    int wpre = __popc(ball & ((1u << lane) - 1));
    if (lane == 0) s_warp[wid] = __popc(ball);
    __syncthreads();
    int before = 0, chunk = 0;
    for (int i = 0; i < kCompactBlock / 32; ++i) {
      int v = s_warp[i];
      if (i < wid) before += v;
      chunk += v;
    }
    int pos = s_base + before + wpre;
    SS_DCHECK(row < 0 || (pos >= 0 && pos < *total));
    if (row >= 0) out_rows[pos] = row;
    // the thread owning candidate n_opt - 1 publishes #active optimizable
    if (c == m.n_opt - 1) out_counts[1] = pos + (row >= 0 ? 1 : 0);
    __syncthreads();
    if (threadIdx.x == 0) s_base += chunk;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out_counts[0] = *total;
    if (m.n_opt == 0) out_counts[1] = 0;
  }
}

}  // namespace ss

using namespace ss;

extern "C" size_t ss_compact_workspace_bytes(int64_t n_candidates) {
  int64_t nb = (n_candidates + kCompactTile - 1) / kCompactTile;
  if (nb < 1) nb = 1;
  return (size_t)(nb + 1) * sizeof(int32_t) + 256;
}

extern "C" int ss_compact_active(const int32_t* row_start, const int32_t* row_expire,
                                 int64_t n_opt, int64_t n_mat_logical,
                                 const int32_t* mat_block_map, int32_t block_rows, int32_t frame,
                                 int32_t* out_rows, int32_t* out_counts, void* ws,
                                 size_t ws_bytes, cudaStream_t stream) {
  if (n_opt < 0 || n_mat_logical < 0 || (n_mat_logical > 0 && block_rows <= 0))
    return set_error(SS_ERR_INVALID, "ss_compact_active: bad sizes");
  int64_t n_cand = n_opt + n_mat_logical;
  if (ws_bytes < ss_compact_workspace_bytes(n_cand))
    return set_error(SS_ERR_WORKSPACE, "ss_compact_active: workspace too small");
  CandMap m{row_start, row_expire, n_opt, n_cand, mat_block_map, block_rows > 0 ? block_rows : 1,
            frame};
  int nb = grid_for(n_cand, kCompactTile);
  int32_t* counts = (int32_t*)ws;
  int32_t* total = counts + nb;
  launch_k(compact_count, nb, kCompactBlock, 0, stream, m, counts);
  launch_k(compact_scan, 1, 1024, 0, stream, counts, nb, total);
  launch_k(compact_scatter, nb, kCompactBlock, 0, stream, m, counts, out_rows, out_counts, total);
  return check_launch("ss_compact_active");
}
