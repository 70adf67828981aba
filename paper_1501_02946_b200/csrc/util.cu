// Small elementwise kernels: float64 <-> float32 conversion for the host
// path, and a fill used to flush L2 between timed iterations.
#include <cuda_runtime.h>

#include "fft_smem.cuh"
#include "patfft_internal.h"

namespace patfft {
namespace {
__global__ void f64_to_f32_kernel(const double* __restrict__ s, float* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = (float)s[i];
}
__global__ void f32_to_f64_kernel(const float* __restrict__ s, double* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = (double)s[i];
}
// widening that also counts non-finite values (the ScalarField finiteness rule)
__global__ void f32_to_f64_count_kernel(const float* __restrict__ s, double* __restrict__ d, size_t n,
                                        unsigned long long* __restrict__ bad) {
  unsigned k = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float v = __ldcs(&s[i]);
    k += !isfinite(v);
    __stcs(&d[i], (double)v);
  }
  k = __reduce_add_sync(0xffffffffu, k);
  if (k && (threadIdx.x & 31) == 0) atomicAdd(bad, (unsigned long long)k);
}
// columns [tb, te) of an M x T row-major array
__global__ void f64_to_f32_cols_kernel(const double* __restrict__ s, float* __restrict__ d, int M, int T, int tb,
                                       int te) {
  const int w = te - tb;
  const size_t n = (size_t)M * w;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / w);
    const size_t o = (size_t)m * T + tb + (int)(i - (size_t)m * w);
    d[o] = (float)__ldcs(&s[o]);
  }
}
__global__ void fill_kernel(float* __restrict__ d, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = v;
}
// grid[gidx[m]][t] = samples[m][t] (full-grid cube, recon.py:327-333)
__global__ void gather_rows_kernel(const float2* __restrict__ s, const int* __restrict__ gidx, float2* __restrict__ g,
                                   int M, int Th) {
  const size_t n = (size_t)M * Th;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / Th);
    const int t = (int)(i - (size_t)m * Th);
    g[(size_t)__ldg(&gidx[m]) * Th + t] = __ldcs(&s[i]);
  }
}
unsigned grid_for(size_t n) {
  const size_t b = (n + 255) / 256;
  const size_t cap = 148 * 32;
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}
}  // namespace

cudaError_t launch_f32_to_f64_count(const float* src, double* dst, size_t n, unsigned long long* bad,
                                    cudaStream_t s) {
  f32_to_f64_count_kernel<<<grid_for(n), 256, 0, s>>>(src, dst, n, bad);
  return cudaGetLastError();
}
cudaError_t launch_f64_to_f32_cols(const double* src, float* dst, int M, int T, int tb, int te, cudaStream_t s) {
  f64_to_f32_cols_kernel<<<grid_for((size_t)M * (te - tb)), 256, 0, s>>>(src, dst, M, T, tb, te);
  return cudaGetLastError();
}

cudaError_t launch_f64_to_f32(const double* src, float* dst, size_t n, cudaStream_t s) {
  f64_to_f32_kernel<<<grid_for(n), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}
cudaError_t launch_f32_to_f64(const float* src, double* dst, size_t n, cudaStream_t s) {
  f32_to_f64_kernel<<<grid_for(n), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}
cudaError_t launch_gather_rows(const float* samples, const int* gidx, float* grid, int M, int T, cudaStream_t s) {
  const int Th = T / 2;  // T is even: move float2 pairs
  gather_rows_kernel<<<grid_for((size_t)M * Th), 256, 0, s>>>(reinterpret_cast<const float2*>(samples), gidx,
                                                              reinterpret_cast<float2*>(grid), M, Th);
  return cudaGetLastError();
}
cudaError_t launch_fill(float* dst, size_t n, float v, cudaStream_t s) {
  fill_kernel<<<grid_for(n), 256, 0, s>>>(dst, n, v);
  return cudaGetLastError();
}

}  // namespace patfft

namespace patfft {

std::vector<float2> make_twiddles() {
  std::vector<float2> tw(fft::kTwiddleTableLen);
  for (int k = 0; k < (1 << fft::kLogTwiddles); ++k) {
    const double a = -2.0 * M_PI * k / (1 << fft::kLogTwiddles);
    tw[k] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  for (int logh = 1; logh <= fft::kPassTwMaxLog; ++logh) {
    const int H = 1 << logh;
    for (int k = 0; k < H; ++k)
      for (int i = 0; i < 4; ++i) {
        const double a = -2.0 * M_PI * k / ((double)H * (2 << i));  // W_{H 2^(i+1)}^k
        tw[fft::kPassTwOffset(logh) + 4 * k + i] = make_float2((float)std::cos(a), (float)std::sin(a));
      }
  }
  return tw;
}

}  // namespace patfft
