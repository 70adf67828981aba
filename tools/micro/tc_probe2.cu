// Probe single UMMAs (M=128, N=32): tf32 with B MN-major / K-major, and bf16 K-major.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46);
}
__device__ float Af(int p, int k) { return (float)((p % 7) + 1) * (k + 1); }
__device__ float Bf(int k, int n) { return (float)((n % 5) - 2) + 0.5f * k; }

__global__ void probe(float* out, int variant, int withmask) {
  __shared__ __align__(1024) uint8_t A[128 * 16 * 4];
  __shared__ __align__(1024) uint8_t B[16 * 32 * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  int tid = threadIdx.x, warp = tid / 32;
  int K = variant == 2 ? 16 : 8;
  for (int i = tid; i < 128 * K; i += 128) {
    int p = i / K, k = i % K;
    if (variant < 2) ((float*)A)[(k / 4) * 512 + p * 4 + (k % 4)] = Af(p, k);               // K-major, LBO 2048, SBO 128
    else ((__nv_bfloat16*)A)[(k / 8) * 1024 + p * 8 + (k % 8)] = __float2bfloat16(Af(p, k));  // K-major bf16, LBO 2048
  }
  for (int i = tid; i < K * 32; i += 128) {
    int k = i / 32, n = i % 32;
    if (variant == 0) ((float*)B)[(n / 4) * 32 + k * 4 + (n % 4)] = Bf(k, n);                 // MN-major, SBO 128 (n), LBO 1024 (k)
    else if (variant == 1) ((float*)B)[(k / 4) * 128 + n * 4 + (k % 4)] = Bf(k, n);           // K-major, LBO 512, SBO 128
    else ((__nv_bfloat16*)B)[(k / 8) * 256 + n * 8 + (k % 8)] = __float2bfloat16(Bf(k, n));  // K-major bf16, LBO 512
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tb)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem = tb;
  if (tid == 0) {
    uint32_t fmt = variant < 2 ? 2u : 1u;
    uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((variant == 0 ? 1u : 0u) << 16) | ((32u >> 3) << 17) |
                     ((128u >> 4) << 24);
    uint64_t ad = desc(su32(A), 2048, 128);
    uint64_t bd = variant == 0 ? desc(su32(B), 1024, 128) : desc(su32(B), 512, 128);
    uint32_t z = 0;
    if (variant < 2) {
      if (withmask)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(0u), "r"(z));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
    } else {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\nD:\n}\n" ::"r"(su32(&bar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int j0 = 0; j0 < 32; j0 += 4) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tmem + ((uint32_t)(warp * 32) << 16) + j0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 4; ++j) out[tid * 32 + j0 + j] = __uint_as_float(r[j]);
  }
  if (tid < 128) {
    float mx = 0;
    for (int n = 0; n < 32; ++n) {
      float w = 0;
      for (int k = 0; k < K; ++k) w += Af(tid, k) * Bf(k, n);
      mx = fmaxf(mx, fabsf(w - out[tid * 32 + n]));
    }
    out[128 * 32 + tid] = mx;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
  float* d;
  cudaMalloc(&d, 129 * 32 * 4 * 4);
  for (int v = 0; v < 4; ++v) {
    int var = v == 3 ? 0 : v, mask = v == 3;
    cudaMemset(d, 0, 129 * 32 * 4 * 4);
    probe<<<1, 128>>>(d, var, mask);
    cudaError_t e = cudaDeviceSynchronize();
    static float h[129 * 32 * 4];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    float mx = 0;
    for (int i = 0; i < 128; ++i) mx = fmaxf(mx, h[128 * 32 + i]);
    printf("variant %d mask %d: %s  D[0][0..3] %g %g %g %g  D[5][7] %g  maxerr %g\n", var, mask, cudaGetErrorString(e),
           h[0], h[1], h[2], h[3], h[5 * 32 + 7], mx);
  }
}
