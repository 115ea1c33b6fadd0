// Error reporting and device queries for the libswings.so C ABI.
#include <stdarg.h>
#include <stdio.h>

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

}  // namespace ss

extern "C" const char* ss_last_error(void) { return ss::g_err; }

extern "C" int ss_version(void) { return 1; }

extern "C" int ss_device_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return sms;
}
