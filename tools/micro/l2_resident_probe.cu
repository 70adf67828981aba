// L2 residency probe for producer -> consumer buffers (the lateral FFT's Y round trip).
// Kernel A writes a W-MB buffer while it streams S MB from another array (the way colfft reads
// the grid and writes Y); kernel B reads the W-MB buffer back.  B's bandwidth tells whether the
// buffer survived in L2 (>> HBM rate) or went to DRAM.  Variants: how the stream is loaded
// (.cs / evict_first policy / no_allocate) and how the buffer is stored / loaded (plain,
// evict_last policy), with and without a persisting-L2 set-aside.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2_resident_probe.cu -o l2_resident_probe
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ float4 ld_mode(const float4* a, int mode, uint64_t pol) {
  float4 v;
  if (mode == 0) asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a));
  else if (mode == 1) asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a));
  else if (mode == 2) asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol));
  else asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a));
  return v;
}
__device__ __forceinline__ void st_mode(float4* a, float4 v, int mode, uint64_t pol) {
  if (mode == 0) asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  else asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// A: every thread streams `ratio` float4 from src per float4 it writes to buf
__global__ void produce(const float4* __restrict__ src, float4* __restrict__ buf, size_t nbuf, int ratio, int ldm, int stm) {
  uint64_t pf, pl;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nbuf; i += (size_t)gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < ratio; ++r) {
      const float4 v = ld_mode(src + (size_t)r * nbuf + i, ldm, pf);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    st_mode(buf + i, acc, stm, pl);
  }
}
__global__ void consume(const float4* __restrict__ buf, size_t nbuf, float* out, int ldm) {
  uint64_t pl;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  float s = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nbuf; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = ld_mode(buf + i, ldm, pl);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.f) *out = s;
}

int main() {
  const size_t MB = 1 << 20;
  float4 *src, *buf, *flush;
  float* out;
  cudaMalloc(&src, 1024 * MB);
  cudaMalloc(&buf, 256 * MB);
  cudaMalloc(&flush, 512 * MB);
  cudaMalloc(&out, 4);
  cudaMemset(src, 0, 1024 * MB);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  int maxp = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
  printf("max persisting L2 %d MB\n", maxp >> 20);
  for (int persist = 0; persist < 2; ++persist) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist ? (size_t)maxp : 0);
    printf("== persisting L2 set-aside: %s\n", persist ? "max" : "0");
    // (stream load mode, buffer store mode, buffer load mode)
    const int variants[][3] = {{1, 0, 0}, {1, 0, 3}, {2, 0, 3}, {2, 1, 3}, {2, 1, 2}, {0, 0, 0}};
    for (auto& v : variants) {
      for (int W : {8, 17, 34, 51, 68, 100}) {
        for (int ratio : {0, 2, 4}) {
          const size_t nbuf = W * MB / 16;
          float best_b = 1e9f, best_a = 1e9f;
          for (int it = 0; it < 4; ++it) {
            cudaMemsetAsync(flush, it, 512 * MB);
            cudaEventRecord(e0);
            produce<<<148 * 8, 256>>>(src, buf, nbuf, ratio, v[0], v[1]);
            cudaEventRecord(e1);
            consume<<<148 * 8, 256>>>(buf, nbuf, out, v[2]);
            cudaEventRecord(e2);
            cudaEventSynchronize(e2);
            float a, b;
            cudaEventElapsedTime(&a, e0, e1);
            cudaEventElapsedTime(&b, e1, e2);
            if (it) { best_a = a < best_a ? a : best_a; best_b = b < best_b ? b : best_b; }
          }
          printf("ld %d st %d rd %d  W %3d MB stream %3d MB: produce %.1f us (%.0f GB/s)  consume %.1f us (%.0f GB/s)\n", v[0], v[1], v[2], W,
                 W * ratio, best_a * 1e3, (double)W * MB * (ratio + 1) / best_a / 1e6, best_b * 1e3, (double)W * MB / best_b / 1e6);
        }
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
