// Microbenchmark: issue rate of 3-register FFMA vs packed FFMA2 (fma.rn.f32x2)
// on sm_100a.  8 independent chains per thread, 148*8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float sum2(unsigned long long r) {
  float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a + b; }
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(a), "f"(b));
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b, int iters) {
  unsigned long long x[8];
  const unsigned long long A = pk(a, a), B = pk(b, b);
  for (int i = 0; i < 8; ++i) x[i] = pk(threadIdx.x * 0.001f + i, i * 0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma2(x[i], A, B);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += sum2(x[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    float ms1, ms2;
    cudaEventRecord(e0); k_ffma<<<148 * 8, 256>>>(out, 0.999f, 0.001f, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0); k_ffma2<<<148 * 8, 256>>>(out, 0.999f, 0.001f, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms2, e0, e1);
    double ops = 148.0 * 8 * 256 * iters * 8;  // instructions (per thread) x threads
    printf("FFMA : %.3f ms  %.1f Ginstr/s (thread)  = %.1f TFLOP/s\n", ms1, ops / ms1 / 1e6, 2 * ops / ms1 / 1e9);
    printf("FFMA2: %.3f ms  %.1f Ginstr/s (thread)  = %.1f TFLOP/s\n", ms2, ops / ms2 / 1e6, 4 * ops / ms2 / 1e9);
  }
  return 0;
}
