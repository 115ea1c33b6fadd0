// Error reporting and device queries for the libswings.so C ABI.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "ss_common.cuh"

namespace ss {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return SS_OK;
}

// Zero fill launched like every other library kernel (programmatic dependent
// launch), so it does not break the launch-gap hiding the way a driver
// memset between two kernels does.  16-byte stores where aligned.
__global__ void memzero_kernel(unsigned char* __restrict__ p, size_t bytes) {
  pdl_wait();
  pdl_trigger();
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t head = (16 - ((uintptr_t)p & 15)) & 15;
  const size_t h = head < bytes ? head : bytes;
  for (size_t i = tid; i < h; i += stride) p[i] = 0;
  const size_t nv = (bytes - h) / 16;
  uint4* v = reinterpret_cast<uint4*>(p + h);
  for (size_t i = tid; i < nv; i += stride) v[i] = make_uint4(0, 0, 0, 0);
  for (size_t i = h + nv * 16 + tid; i < bytes; i += stride) p[i] = 0;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SS_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

int memzero(void* p, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return SS_OK;
  size_t blocks = (bytes / 16 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_k(memzero_kernel, (unsigned)blocks, 256, 0, stream, (unsigned char*)p, bytes);
  return check_launch("memzero");
}

// Per (device, kernel) high-water mark of the dynamic shared-memory attribute.
constexpr int kAttrDevs = 64;
constexpr int kAttrKernels = 32;
struct SmemMark {
  const void* kernel;
  size_t bytes;
};
static SmemMark g_smem_attr[kAttrDevs][kAttrKernels];
static std::mutex g_smem_mu;

int ensure_smem(const void* kernel, size_t bytes) {
  if (bytes == 0) return SS_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kAttrDevs)
    return set_error(SS_ERR_CUDA, "ensure_smem: bad device");
  std::lock_guard<std::mutex> lock(g_smem_mu);
  SmemMark* marks = g_smem_attr[dev];
  int i = 0;
  while (i < kAttrKernels && marks[i].kernel && marks[i].kernel != kernel) ++i;
  if (i == kAttrKernels) return set_error(SS_ERR_CUDA, "ensure_smem: too many kernels");
  if (marks[i].kernel == kernel && bytes <= marks[i].bytes) return SS_OK;
  // the attribute and the mark only ever grow together (under the lock)
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
      cudaSuccess)
    return check_launch("ensure_smem");
  marks[i].kernel = kernel;
  marks[i].bytes = bytes;
  return SS_OK;
}

// Small host -> device writes (per-step tables: a few hundred bytes) as a
// kernel whose argument carries the bytes: no copy-engine operation in the
// stream, so the surrounding kernels keep their programmatic-dependent-launch
// overlap (a DMA memcpy between two kernels left a ~15 us bubble).
constexpr int kSmallMax = 2048;
struct SmallBlob {
  unsigned char b[kSmallMax];
};

__global__ void write_small_kernel(unsigned char* __restrict__ dst, SmallBlob blob, int n) {
  pdl_wait();
  pdl_trigger();
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = blob.b[i];
}

}  // namespace ss

extern "C" int ss_write_small(void* dst, const void* host_src, size_t bytes, cudaStream_t stream) {
  if (bytes > (size_t)ss::kSmallMax || (!dst && bytes) || (!host_src && bytes))
    return ss::set_error(SS_ERR_INVALID, "ss_write_small: %zu bytes (max %d)", bytes, ss::kSmallMax);
  if (bytes == 0) return SS_OK;
  ss::SmallBlob blob;
  memcpy(blob.b, host_src, bytes);
  ss::launch_k(ss::write_small_kernel, 1, 256, 0, stream, (unsigned char*)dst, blob, (int)bytes);
  return ss::check_launch("ss_write_small");
}

extern "C" int ss_memzero(void* ptr, size_t bytes, cudaStream_t stream) {
  if (!ptr && bytes) return ss::set_error(SS_ERR_INVALID, "ss_memzero: null pointer");
  return ss::memzero(ptr, bytes, stream);
}

// default alpha floor 2^-28 (swings.h ss_set_alpha_floor)
static std::atomic<int32_t> g_alpha_floor{-28};

namespace ss {
int32_t alpha_floor_log2() { return g_alpha_floor.load(std::memory_order_relaxed); }
}  // namespace ss

extern "C" int ss_set_alpha_floor(int32_t log2_floor) {
  if (log2_floor != 0 && (log2_floor < -126 || log2_floor > -1))
    return ss::set_error(SS_ERR_INVALID, "ss_set_alpha_floor: %d not in {0} U [-126, -1]",
                         log2_floor);
  g_alpha_floor.store(log2_floor, std::memory_order_relaxed);
  return SS_OK;
}

extern "C" int32_t ss_get_alpha_floor(void) { return ss::alpha_floor_log2(); }

extern "C" const char* ss_last_error(void) { return ss::g_err; }

extern "C" int ss_version(void) { return 1; }

extern "C" int ss_device_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return sms;
}
