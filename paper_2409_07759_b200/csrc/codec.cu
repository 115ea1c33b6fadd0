// a-13 / §8(f)-1 per-frame update export: fixed-size record encode and
// decode on the device (reference codec.py:195-266).
//
//   profile 0 (56 B): f32 mean[3] rot[4] scale[3] opacity color[3]
//   profile 1 (30 B): f16 mean[3] | u8 rot[4] (fixed-point, renormalisation-
//                     stable) | f16 scale[3] | u8 rint(255 a) | f32 color[3] | pad
//
// One thread per record; every rounding follows numpy's (round-to-nearest-
// even conversions, np.rint = rint, left-to-right quaternion norms), so the
// bytes equal the reference's encode_records on the same float64 input.
#include "ss_common.cuh"

namespace ss {

__device__ __forceinline__ void put_f32(uint8_t* p, float v) {
  const uint32_t u = __float_as_uint(v);
  p[0] = u & 0xff;
  p[1] = (u >> 8) & 0xff;
  p[2] = (u >> 16) & 0xff;
  p[3] = u >> 24;
}

__device__ __forceinline__ float get_f32(const uint8_t* p) {
  return __uint_as_float((uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
                         ((uint32_t)p[3] << 24));
}

// float64 -> binary16, round to nearest even, directly from the double (as
// numpy's astype('<f2')).  Integer implementation: the hardware F2F.F16.F64
// conversion did not reproduce numpy's bytes on sm_100a.
__device__ __forceinline__ unsigned short f64_to_f16_rn(double d) {
  const uint64_t x = (uint64_t)__double_as_longlong(d);
  const unsigned short sign = (unsigned short)((x >> 48) & 0x8000u);
  const int exp = (int)((x >> 52) & 0x7ff);
  uint64_t mant = x & 0xFFFFFFFFFFFFFull;
  if (exp == 0x7ff) return sign | 0x7c00u | (mant ? 0x200u : 0u);
  const int e = exp - 1023 + 15;
  if (e >= 31) return sign | 0x7c00u;
  if (e <= 0) {
    if (e < -10) return sign;
    mant |= 1ull << 52;
    const int shift = 43 - e;
    uint64_t m = mant >> shift;
    const uint64_t rem = mant & ((1ull << shift) - 1), half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (m & 1))) ++m;
    return sign | (unsigned short)m;
  }
  uint32_t h = ((uint32_t)e << 10) | (uint32_t)(mant >> 42);
  const uint64_t rem = mant & ((1ull << 42) - 1), half = 1ull << 41;
  if (rem > half || (rem == half && (h & 1))) ++h;
  return sign | (unsigned short)h;
}

__device__ __forceinline__ void put_f16(uint8_t* p, double v) {
  const unsigned short h = f64_to_f16_rn(v);
  p[0] = h & 0xff;
  p[1] = h >> 8;
}

// binary16 -> float64 (exact)
__device__ __forceinline__ double get_f16(const uint8_t* p) {
  const unsigned h = (unsigned)(p[0] | (p[1] << 8));
  const int e = (h >> 10) & 0x1f;
  const double m = (double)(h & 0x3ff);
  double v;
  if (e == 0) v = ldexp(m, -24);
  else if (e == 31) v = (h & 0x3ff) ? __longlong_as_double(0x7ff8000000000000ll)
                                   : __longlong_as_double(0x7ff0000000000000ll);
  else v = ldexp(1024.0 + m, e - 25);
  return (h & 0x8000) ? -v : v;
}

// codec.py:183-186 left-to-right sum of squares
__device__ __forceinline__ double quat_norm(const double q[4]) {
  return sqrt(dadd(dadd(dadd(dmul(q[0], q[0]), dmul(q[1], q[1])), dmul(q[2], q[2])),
                   dmul(q[3], q[3])));
}

__device__ __forceinline__ uint8_t u8_code(double x) {
  return (uint8_t)fmin(fmax(rint(x), 0.0), 255.0);
}

// codec.py:189-212: quantize(normalize(decode(b))) iterated to a fixed point
__device__ void quantize_rot_u8(const double q[4], uint8_t out[4]) {
  uint8_t b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = u8_code(dmul(dadd(q[k], 1.0), 127.5));
  for (int it = 0; it < 4; ++it) {
    double raw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) raw[k] = dsub(ddiv((double)b[k], 127.5), 1.0);
    const double nrm = fmax(quat_norm(raw), 1e-12);
    uint8_t b2[4];
    bool same = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      b2[k] = u8_code(dmul(dadd(ddiv(raw[k], nrm), 1.0), 127.5));
      same &= b2[k] == b[k];
    }
    if (same) break;
#pragma unroll
    for (int k = 0; k < 4; ++k) b[k] = b2[k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) out[k] = b[k];
}

__global__ void encode_kernel(const double* __restrict__ rows, int64_t n, int profile,
                              uint8_t* __restrict__ out, int32_t* __restrict__ bad) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* r = rows + i * SS_ROW;
  bool finite = true;
#pragma unroll
  for (int k = 0; k < SS_ROW; ++k) finite &= isfinite(r[k]);
  if (!finite) atomicExch(bad, 1);
  if (profile == 0) {
    uint8_t* o = out + i * 56;
#pragma unroll
    for (int k = 0; k < SS_ROW; ++k) put_f32(o + 4 * k, __double2float_rn(r[k]));
  } else {
    uint8_t* o = out + i * 30;
#pragma unroll
    for (int k = 0; k < 3; ++k) put_f16(o + 2 * k, r[k]);
    quantize_rot_u8(r + 3, o + 6);
#pragma unroll
    for (int k = 0; k < 3; ++k) put_f16(o + 10 + 2 * k, r[7 + k]);
    o[16] = u8_code(dmul(r[10], 255.0));
#pragma unroll
    for (int k = 0; k < 3; ++k) put_f32(o + 17 + 4 * k, __double2float_rn(r[11 + k]));
    o[29] = 0;
  }
}

// codec.py:235-266
__global__ void decode_kernel(const uint8_t* __restrict__ data, int64_t n, int profile,
                              double* __restrict__ rows) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* r = rows + i * SS_ROW;
  double q[4];
  if (profile == 0) {
    const uint8_t* p = data + i * 56;
#pragma unroll
    for (int k = 0; k < 3; ++k) r[k] = (double)get_f32(p + 4 * k);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = (double)get_f32(p + 12 + 4 * k);
#pragma unroll
    for (int k = 0; k < 3; ++k) r[7 + k] = (double)get_f32(p + 28 + 4 * k);
    r[10] = (double)get_f32(p + 40);
#pragma unroll
    for (int k = 0; k < 3; ++k) r[11 + k] = (double)get_f32(p + 44 + 4 * k);
  } else {
    const uint8_t* p = data + i * 30;
#pragma unroll
    for (int k = 0; k < 3; ++k) r[k] = get_f16(p + 2 * k);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = dsub(ddiv((double)p[6 + k], 127.5), 1.0);
#pragma unroll
    for (int k = 0; k < 3; ++k) r[7 + k] = get_f16(p + 10 + 2 * k);
    r[10] = ddiv((double)p[16], 255.0);
#pragma unroll
    for (int k = 0; k < 3; ++k) r[11 + k] = (double)get_f32(p + 17 + 4 * k);
  }
  const double nrm = quat_norm(q);
  const double safe = fabs(dsub(nrm, 1.0)) > 1e-6 ? fmax(nrm, 1e-12) : 1.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) r[3 + k] = ddiv(q[k], safe);
  if (nrm < 1e-12) {
    r[3] = 1.0;
    r[4] = r[5] = r[6] = 0.0;
  }
#pragma unroll
  for (int k = 7; k < 10; ++k) r[k] = fmax(r[k], 1e-6);  // SCALE_FLOOR
  r[10] = fmin(fmax(r[10], 0.0), 1.0);
}

}  // namespace ss

using namespace ss;

extern "C" int ss_encode_records(const double* rows, int64_t n, int32_t profile, uint8_t* out,
                                 int32_t* bad, cudaStream_t stream) {
  if (n < 0 || (profile != 0 && profile != 1))
    return set_error(SS_ERR_INVALID, "ss_encode_records: bad arguments");
  if (n == 0) return SS_OK;
  launch_k(encode_kernel, grid_for(n, 128), 128, 0, stream, rows, n, profile, out, bad);
  return check_launch("ss_encode_records");
}

extern "C" int ss_decode_records(const uint8_t* data, int64_t n, int32_t profile, double* rows,
                                 cudaStream_t stream) {
  if (n < 0 || (profile != 0 && profile != 1))
    return set_error(SS_ERR_INVALID, "ss_decode_records: bad arguments");
  if (n == 0) return SS_OK;
  launch_k(decode_kernel, grid_for(n, 128), 128, 0, stream, data, n, profile, rows);
  return check_launch("ss_decode_records");
}

// Display conversion of a rendered frame: write_png's quantisation
// (raster.py:411-425: clip, sRGB transfer, rint(255 v)) evaluated in fp64 per
// channel value, float32 linear in, uint8 out.
__global__ void srgb_u8_kernel(const float* __restrict__ img, int64_t n, uint8_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = (double)img[i];
  x = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
  const double y = x <= 0.0031308 ? 12.92 * x : 1.055 * pow(x, 1.0 / 2.4) - 0.055;
  out[i] = (uint8_t)rint(y * 255.0);
}

extern "C" int ss_to_srgb_u8(const float* img, int64_t n, uint8_t* out, cudaStream_t stream) {
  if (n < 0) return set_error(SS_ERR_INVALID, "ss_to_srgb_u8: n < 0");
  if (n == 0) return SS_OK;
  launch_k(srgb_u8_kernel, (unsigned)((n + 255) / 256), 256, 0, stream, img, n, out);
  return check_launch("ss_to_srgb_u8");
}
