// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__global__ void k1(float* out, int iters, float a, float b) {
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
  float s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* out, int iters, float a, float b) {
  unsigned long long acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = f2u(make_float2(threadIdx.x + i, i));
  unsigned long long A = f2u(make_float2(a, a)), B = f2u(make_float2(b, b));
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(A), "l"(B));
  float s = 0; for (int i = 0; i < 16; ++i) { float2 v = u2f(acc[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    float ms1, ms2;
    cudaEventRecord(e0); k1<<<148 * 8, 256>>>(out, iters, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0); k2<<<148 * 8, 256>>>(out, iters, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms2, e0, e1);
    double fma = 148.0 * 8 * 256 * iters * 16;
    printf("FFMA : %.3f ms  %.1f TFLOP/s\nFFMA2: %.3f ms  %.1f TFLOP/s (counting 2 FMA per lane)\n", ms1, 2 * fma / ms1 / 1e9,
           ms2, 2 * 2 * fma / ms2 / 1e9);
  }
  return 0;
}
