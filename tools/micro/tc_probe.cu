// Probe tcgen05 basics: TMEM st/ld round trip and one tf32 UMMA (M=128, N=32, K=8)
// with no-swizzle K-major A and MN-major B.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, int ver) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         ((uint64_t)ver << 46);
}

__global__ void probe(float* out, int variant) {
  __shared__ __align__(1024) float A[128 * 8];
  __shared__ __align__(1024) float B[8 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  int tid = threadIdx.x, warp = tid / 32;
  // A[p][k] = p + 1 (k-independent), K-major no swizzle: (k/4)*LBO + p*16 + (k%4)*4, LBO = 2048
  for (int i = tid; i < 128 * 8; i += 128) {
    int p = i / 8, k = i % 8;
    A[(k / 4) * 512 + p * 4 + (k % 4)] = (float)(p + 1);
  }
  // B[k][n] = (k == 0) * (n + 1), MN-major: (n/4)*SBO + k*16 + (n%4)*4 with SBO = 128
  for (int i = tid; i < 8 * 32; i += 128) {
    int k = i / 32, n = i % 32;
    B[(n / 4) * 32 + k * 4 + (n % 4)] = k == 0 ? (float)(n + 1) : 0.f;
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
  if (variant == 0) {
    // st/ld round trip
    uint32_t v = 1000 * tid + 7;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + 3), "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else if (tid == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    uint64_t ad = desc(su32(A), 2048, 128, 1), bd = desc(su32(B), 1024, 128, 1);
    if (variant == 2) { ad = desc(su32(A), 128, 2048, 1); bd = desc(su32(B), 128, 1024, 1); }
    printf("tmem %08x A %08x B %08x ad %016llx bd %016llx idesc %08x\n", tmem, su32(A), su32(B),
           (unsigned long long)ad, (unsigned long long)bd, idesc);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  if (variant) {
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\nD:\n}\n" ::"r"(su32(&bar)), "r"(0) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 4; ++j) out[tid * 4 + j] = variant == 0 ? (float)r[j] : __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 4 * 4);
  for (int v = 0; v < 3; ++v) {
    cudaMemset(d, 0, 128 * 16);
    probe<<<1, 128>>>(d, v);
    cudaError_t e = cudaDeviceSynchronize();
    float h[512];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("variant %d: %s  p0: %g %g %g %g  p1: %g %g %g %g  p127: %g %g %g %g\n", v, cudaGetErrorString(e), h[0], h[1],
           h[2], h[3], h[4], h[5], h[6], h[7], h[508], h[509], h[510], h[511]);
  }
}
