// NED gridding on the 5th-generation tensor cores (tcgen05, TMEM).
//
// Same operator as spread.cu (reference nufft.py:373-404 with the weighting
// of recon.py:374): grid[p][t] = sum_m W[p][m] * S[m][t], W the separable
// Kaiser-Bessel row x column weights of sensor m at oversampled grid point p.
// Per tile of 8 grid rows x 16 grid columns (128 points = UMMA M) the
// contributing sensors (those whose 2K x 2K footprint meets the tile) form a
// dense K dimension, so the tile is a small GEMM
//
//     D[128 points][N time] = W_tile[128][K sensors] * S[K sensors][N time]
//
// with D accumulated in TMEM (fp32, N <= 256 columns).  Operands are fp32
// split into tf32 hi + lo parts and multiplied as hi*hi + hi*lo + lo*hi
// ("3xTF32", ~22-bit products, fp32 accumulation), which keeps the result at
// the fp32 SIMT kernel's accuracy.  Redundancy: a sensor meets (8+2K-1) x
// (16+2K-1) tile points on average, 3.6x the 4K^2 useful MACs at K = 6.
//
// CTA = (tile, N-sample time block), 128 threads, 2 shared-memory stages of
// 16 sensors.  Every thread builds its grid point's 16 weights (A) and 16
// sensors x N/128 time samples of the gathered sample rows (B), both in
// the K-major (sensor-contiguous) UMMA layout; thread 0 issues the 6 UMMAs of a stage (2 k-steps x 3 products)
// and commits them to the stage's mbarrier, so building stage s+1 overlaps
// the tensor cores working on stage s.  Epilogue: tcgen05.ld of the
// accumulator (thread = grid point, 32 time samples per load) straight to
// the [nrows][ncols][T] grid.  Layouts are the canonical no-swizzle UMMA
// layouts (8 x 16-byte core matrices), written conflict-free.
#include <cuda_runtime.h>

#include <cstdint>

#include "patfft_internal.h"

namespace patfft {
namespace {

constexpr int kTR = 8, kTC = 16, kTM = kTR * kTC;  // tile rows, cols, points (UMMA M)
constexpr int kKC = 16;                              // sensors per stage
constexpr int kThreadsTC = 128;
constexpr int kStages = 2;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init_tc(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait_tc(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TC_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra TC_DONE;\n\t"
      "bra TC_WAIT;\n"
      "TC_DONE:\n}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}

// UMMA shared-memory matrix descriptor, SWIZZLE_NONE: start, leading (K
// direction) and stride (M/N direction) byte offsets between 8x16B core
// matrices, version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N.
// (An MN-major tf32 B operand in the no-swizzle layout reads as zeros on
// sm_100a -- measured with tools/micro/tc_probe2.cu -- so B is K-major.)
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(kTM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ float4 split_hi(float4 v) {
  return make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
}
__device__ __forceinline__ float4 sub4(float4 a, float4 b) {
  return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}

template <int N>
__global__ void __launch_bounds__(kThreadsTC) spread_tc_kernel(const SpreadParams p) {
  constexpr int A_BYTES = kTM * kKC * 4;          // 8 KB: [kKC/4][128][4]
  constexpr int B_BYTES = kKC * N * 4;            // [kKC/4][N][4]
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  constexpr uint32_t A_LBO = kTM * 16, A_SBO = 128;       // K step of 4 / 8-row group
  constexpr uint32_t B_LBO = N * 16, B_SBO = 128;         // K step of 4 / 8-sample group
  constexpr uint32_t TCOLS = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  constexpr uint32_t IDESC = umma_idesc_tf32(N);

  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mma_bar[kStages];
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int4 tile = p.tc_tiles[blockIdx.x / p.tc_tblocks];  // {first record, records, row0, col0}
  const int tb = blockIdx.x % p.tc_tblocks;
  const int t0 = p.t_begin + tb * N;
  const int nch = tile.y / kKC;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base_s)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init_tc(&mma_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  // this thread's grid point (A rows) and its B-producer coordinates
  const int pr = tid / kTC, pc = tid % kTC;
  const float* __restrict__ recs = p.tc_recs + (size_t)tile.x * 32;

  for (int c = 0; c < nch; ++c) {
    const int s = c & 1;
    if (c >= kStages) mbar_wait_tc(&mma_bar[s], ((c >> 1) - 1) & 1);
    uint8_t* st = smem + s * STAGE;
    float* Ahi = reinterpret_cast<float*>(st);
    float* Alo = reinterpret_cast<float*>(st + A_BYTES);
    float* Bhi = reinterpret_cast<float*>(st + 2 * A_BYTES);
    float* Blo = reinterpret_cast<float*>(st + 2 * A_BYTES + B_BYTES);
    const float* rc = recs + (size_t)c * kKC * 32;
    // ---- A: W[p][k] = wrow[k][pr] * wcol[k][pc], k-quads of 16 bytes
#pragma unroll
    for (int g = 0; g < kKC / 4; ++g) {
      float w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float* r = rc + (g * 4 + j) * 32;
        w[j] = __ldg(r + 8 + pr) * __ldg(r + 16 + pc);
      }
      const float4 v = make_float4(w[0], w[1], w[2], w[3]);
      const float4 h = split_hi(v);
      *reinterpret_cast<float4*>(Ahi + g * (A_LBO / 4) + tid * 4) = h;
      *reinterpret_cast<float4*>(Alo + g * (A_LBO / 4) + tid * 4) = sub4(v, h);
    }
    // ---- B: gathered sample rows, K-major [k/4][n][4] (thread = time sample,
    // 4 sensors per 16-byte store; every load instruction is one 128-byte run)
#pragma unroll
    for (int kq = 0; kq < kKC / 4; ++kq) {
      const float* __restrict__ s0 = p.samples + (size_t)__float_as_int(__ldg(rc + (kq * 4 + 0) * 32)) * p.T + t0;
      const float* __restrict__ s1 = p.samples + (size_t)__float_as_int(__ldg(rc + (kq * 4 + 1) * 32)) * p.T + t0;
      const float* __restrict__ s2 = p.samples + (size_t)__float_as_int(__ldg(rc + (kq * 4 + 2) * 32)) * p.T + t0;
      const float* __restrict__ s3 = p.samples + (size_t)__float_as_int(__ldg(rc + (kq * 4 + 3) * 32)) * p.T + t0;
#pragma unroll
      for (int n = tid; n < N; n += kThreadsTC) {
        const float4 v = make_float4(__ldg(s0 + n), __ldg(s1 + n), __ldg(s2 + n), __ldg(s3 + n));
        const float4 h = split_hi(v);
        const int off = kq * (B_LBO / 4) + n * 4;
        *reinterpret_cast<float4*>(Bhi + off) = h;
        *reinterpret_cast<float4*>(Blo + off) = sub4(v, h);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_hi = su32(Ahi), a_lo = su32(Alo), b_hi = su32(Bhi), b_lo = su32(Blo);
#pragma unroll
      for (int ks = 0; ks < kKC / 8; ++ks) {
        const uint64_t dah = umma_desc(a_hi + ks * 2 * A_LBO, A_LBO, A_SBO);
        const uint64_t dal = umma_desc(a_lo + ks * 2 * A_LBO, A_LBO, A_SBO);
        const uint64_t dbh = umma_desc(b_hi + ks * 2 * B_LBO, B_LBO, B_SBO);
        const uint64_t dbl = umma_desc(b_lo + ks * 2 * B_LBO, B_LBO, B_SBO);
        umma_tf32(tmem, dah, dbh, IDESC, (c | ks) ? 1u : 0u);
        umma_tf32(tmem, dah, dbl, IDESC, 1u);
        umma_tf32(tmem, dal, dbh, IDESC, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       su32(&mma_bar[s]))
                   : "memory");
    }
  }

  // ---- epilogue: TMEM -> registers -> grid (thread = grid point)
  float* __restrict__ out =
      p.grid + ((size_t)(tile.z + pr) * p.ncols + (tile.w + pc)) * p.T + t0;
  if (nch > 0) {
    const int cl = nch - 1;
    mbar_wait_tc(&mma_bar[cl & 1], (cl >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
    for (int j = 0; j < N / 32; ++j) {
      uint32_t r[32];
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(j * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
          "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float4* o4 = reinterpret_cast<float4*>(out + j * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        o4[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                            __uint_as_float(r[4 * q + 3]));
    }
  } else {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < N / 4; ++j) reinterpret_cast<float4*>(out)[j] = z;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

template <int N>
cudaError_t go_tc(const SpreadParams& p, cudaStream_t s) {
  constexpr int STAGE = 2 * kTM * kKC * 4 + 2 * kKC * N * 4;
  const size_t smem = (size_t)kStages * STAGE;
  auto k = spread_tc_kernel<N>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err) return err;
  SpreadParams q = p;
  q.tc_tblocks = (p.t_end - p.t_begin) / N;
  const unsigned blocks = (unsigned)(q.tc_ntiles * q.tc_tblocks);
  if (blocks) k<<<blocks, kThreadsTC, smem, s>>>(q);
  return cudaGetLastError();
}

}  // namespace

bool spread_tc_supported(int n_lat, int nrows, int ncols, int T) {
  return n_lat == 2 && nrows % kTR == 0 && ncols % kTC == 0 && spread_tc_block(T) > 0;
}

int spread_tc_block(int T) {
  for (int n : {256, 128, 64, 32})
    if (T % n == 0) return n;
  return 0;
}

cudaError_t launch_spread_tc(const SpreadParams& p, cudaStream_t s) {
  const int n = p.tc_n;
  if ((p.t_end - p.t_begin) % n || p.t_begin % n) return cudaErrorInvalidValue;
  switch (n) {
    case 256: return go_tc<256>(p, s);
    case 128: return go_tc<128>(p, s);
    case 64: return go_tc<64>(p, s);
    case 32: return go_tc<32>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace patfft
