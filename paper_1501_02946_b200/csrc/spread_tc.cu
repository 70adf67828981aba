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
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "patfft_internal.h"

namespace patfft {
namespace {

constexpr int kTR = 8, kTC = 16, kTM = kTR * kTC;  // tile rows, cols, points (UMMA M)
constexpr int kKC = 16;                              // sensors per stage
constexpr int kThreadsTC = 256;
constexpr int kStages = 2;
constexpr int kRecSlots = 4;  // record ring (bulk copies three stages ahead)

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

// x = hi + lo with hi = x rounded to tf32 (10 explicit mantissa bits, ties
// away) and lo = x - hi exact in fp32; the tensor core truncates lo to tf32.
__device__ __forceinline__ void split_tf32(float4 v, float4& h, float4& l) {
  h.x = __uint_as_float((__float_as_uint(v.x) + 0x1000u) & 0xFFFFE000u);
  h.y = __uint_as_float((__float_as_uint(v.y) + 0x1000u) & 0xFFFFE000u);
  h.z = __uint_as_float((__float_as_uint(v.z) + 0x1000u) & 0xFFFFE000u);
  h.w = __uint_as_float((__float_as_uint(v.w) + 0x1000u) & 0xFFFFE000u);
  float2 l01, l23;
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tsub.rn.f32x2 d, a, b;\n\t"
      "mov.b64 {%0, %1}, d;\n}" : "=f"(l01.x), "=f"(l01.y) : "f"(v.x), "f"(v.y), "f"(h.x), "f"(h.y));
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tsub.rn.f32x2 d, a, b;\n\t"
      "mov.b64 {%0, %1}, d;\n}" : "=f"(l23.x), "=f"(l23.y) : "f"(v.z), "f"(v.w), "f"(h.z), "f"(h.w));
  l = make_float4(l01.x, l01.y, l23.x, l23.y);
}

// Position in a CTA's stage sequence.  Work items w = (tile w / tblocks,
// time block w % tblocks) are claimed dynamically (atomic counter, items in
// longest-tile-first order) by thread 0's record cursor, which runs three
// stages ahead and publishes each claimed item in a small shared ring; the
// sample cursor (two stages ahead) and the build cursor follow the ring.
constexpr int kRing = 8;
struct Cursor {
  int k, tb, c, nch, rec0, row0, col0;  // ring position, time block, chunk, chunks, first record, tile origin
  bool valid;
};
__device__ __forceinline__ void cursor_load(const SpreadParams& p, Cursor& u, int w) {
  u.valid = w < p.tc_nonempty * p.tc_tblocks;
  if (!u.valid) return;
  const int4 t = __ldg(&p.tc_tiles[w / p.tc_tblocks]);
  u.tb = w % p.tc_tblocks;
  u.c = 0;
  u.nch = t.y / kKC;
  u.rec0 = t.x;
  u.row0 = t.z;
  u.col0 = t.w;
}
__device__ __forceinline__ void cursor_next(const SpreadParams& p, Cursor& u, const int* ring) {
  if (!u.valid || ++u.c < u.nch) return;
  ++u.k;
  cursor_load(p, u, ring[u.k & (kRing - 1)]);
}
__device__ __forceinline__ void cursor_claim(const SpreadParams& p, Cursor& u, int* ring) {  // thread 0
  if (!u.valid || ++u.c < u.nch) return;
  ++u.k;
  const int w = atomicAdd(p.tc_counter, 1);
  ring[u.k & (kRing - 1)] = w;
  cursor_load(p, u, w);
}

template <int N>
__global__ void __launch_bounds__(kThreadsTC, 2) spread_tc_kernel(const SpreadParams p) {
  constexpr int A_BYTES = kTM * kKC * 4;          // 8 KB: [kKC/4][128][4]
  constexpr int B_BYTES = kKC * N * 4;            // [kKC/4][N][4]
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  constexpr uint32_t A_LBO = kTM * 16, A_SBO = 128;  // K step of 4 / 8-row group
  constexpr uint32_t B_LBO = N * 16, B_SBO = 128;    // K step of 4 / 8-sample group
  constexpr uint32_t TCOLS = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  constexpr uint32_t IDESC = umma_idesc_tf32(N);
  constexpr uint32_t REC_BYTES = kKC * 32 * 4;  // one stage of records (2 KB)
  constexpr int NI = (N + kThreadsTC - 1) / kThreadsTC;

  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mma_bar[kStages];
  __shared__ uint64_t rec_bar[kRecSlots];
  __shared__ __align__(16) float recbuf[kRecSlots * kKC * 32];
  __shared__ uint32_t tmem_base_s;
  __shared__ int ring[kRing];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q4 = warp & 3;

  // ---- empty tiles (no sensor meets them): zeros, one warp per point row
  for (int i = p.tc_nonempty + blockIdx.x; i < p.tc_ntiles; i += gridDim.x) {
    const int4 t = __ldg(&p.tc_tiles[i]);
    const int len = p.t_end - p.t_begin;
    for (int pt = warp; pt < kTM; pt += kThreadsTC / 32) {
      float* o = p.grid + ((size_t)(t.z + pt / kTC) * p.ncols + (t.w + pt % kTC)) * p.T + p.t_begin;
      for (int q = lane * 4; q < len; q += 128) *reinterpret_cast<float4*>(o + q) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  Cursor cur, cs, cr;  // stage being built, sample prefetch (+2), record prefetch (+3, thread 0)
  if (tid == 0) ring[0] = atomicAdd(p.tc_counter, 1);
  __syncthreads();
  cur.k = 0;
  cursor_load(p, cur, ring[0]);
  if (!cur.valid) return;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base_s)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init_tc(&mma_bar[s], 1);
    for (int s = 0; s < kRecSlots; ++s) mbar_init_tc(&rec_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  // A producer: grid point pa (row pr, column pc), k-quads ga0, ga0 + 1
  const int pa = tid & (kTM - 1), pr = pa / kTC, pc = pa % kTC, ga0 = (tid >> 7) * 2;
  // records: 4-slot ring filled by bulk (TMA) copies three stages ahead (thread 0 only)
  auto fetch_recs = [&](int g, const Cursor& u) {
    const int r = g % kRecSlots;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&rec_bar[r])), "r"(REC_BYTES)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(recbuf + r * kKC * 32)),
                 "l"(p.tc_recs + ((size_t)u.rec0 + (size_t)u.c * kKC) * 32), "r"(REC_BYTES), "r"(su32(&rec_bar[r]))
                 : "memory");
  };
  if (tid == 0) {
    cr = cur;
    for (int g = 0; g < kRecSlots - 1 && cr.valid; ++g) {
      fetch_recs(g, cr);
      cursor_claim(p, cr, ring);
    }
  }
  __syncthreads();  // ring entries of the first stages
  // B producer: samples prefetched into registers two stages ahead (two
  // register sets, the stage loop is unrolled by two so indices stay static):
  // sv[i][k] = S[sensor k][t0 + tid + 256 i]
  float sv0[NI][kKC], sv1[NI][kKC];
  auto load_samples = [&](int g, const Cursor& u, float (&sv)[NI][kKC]) {
    const int r = g % kRecSlots;
    mbar_wait_tc(&rec_bar[r], (g / kRecSlots) & 1);
    const float* rb = recbuf + r * kKC * 32;
    const int t0 = p.t_begin + u.tb * N;
    const uint32_t base = (uint32_t)(t0 + tid);
#pragma unroll
    for (int k = 0; k < kKC; ++k) {
      const uint32_t off = __float_as_uint(rb[k * 32]) + base;  // record word 0: sensor row offset m * T
#pragma unroll
      for (int i = 0; i < NI; ++i)
        if (tid + i * kThreadsTC < N) sv[i][k] = __ldg(p.samples + (off + i * kThreadsTC));
    }
  };
  cs = cur;
  load_samples(0, cs, sv0);
  cursor_next(p, cs, ring);
  if (cs.valid) load_samples(1, cs, sv1);
  cursor_next(p, cs, ring);

  auto epilogue = [&](int g) {
    const int t0 = p.t_begin + cur.tb * N;
    mbar_wait_tc(&mma_bar[g & 1], (g >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* stg = reinterpret_cast<float*>(smem) + warp * 32 * 36;
#pragma unroll 1
    for (int j = warp >> 2; j < N / 32; j += kThreadsTC / 128) {
      uint32_t r[32];
      const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(j * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
          "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint4*>(stg + lane * 36 + 4 * q) = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int pl = q * 4 + (lane >> 3), pt = q4 * 32 + pl;  // point within the tile
        const float4 v = *reinterpret_cast<const float4*>(stg + pl * 36 + (lane & 7) * 4);
        float* o = p.grid + ((size_t)(cur.row0 + pt / kTC) * p.ncols + (cur.col0 + pt % kTC)) * p.T + t0 + j * 32;
        *reinterpret_cast<float4*>(o + (lane & 7) * 4) = v;
      }
      __syncwarp();
    }
    // TMEM and the staging area (stage slot 0) are reused by the next stages
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
  };

  auto stage = [&](int g, float (&sv)[NI][kKC]) {
    const int s = g & 1;
    if (g >= kStages) mbar_wait_tc(&mma_bar[s], ((g >> 1) - 1) & 1);
    uint8_t* st = smem + s * STAGE;
    float* Ahi = reinterpret_cast<float*>(st);
    float* Alo = reinterpret_cast<float*>(st + A_BYTES);
    float* Bhi = reinterpret_cast<float*>(st + 2 * A_BYTES);
    float* Blo = reinterpret_cast<float*>(st + 2 * A_BYTES + B_BYTES);
    const float* rb = recbuf + (g % kRecSlots) * kKC * 32;
    // ---- A: W[p][k] = wrow[k][pr] * wcol[k][pc], K-major [k/4][p][4]
#pragma unroll
    for (int gq = ga0; gq < ga0 + 2; ++gq) {
      const float4 v = make_float4(rb[(gq * 4 + 0) * 32 + 8 + pr] * rb[(gq * 4 + 0) * 32 + 16 + pc],
                                   rb[(gq * 4 + 1) * 32 + 8 + pr] * rb[(gq * 4 + 1) * 32 + 16 + pc],
                                   rb[(gq * 4 + 2) * 32 + 8 + pr] * rb[(gq * 4 + 2) * 32 + 16 + pc],
                                   rb[(gq * 4 + 3) * 32 + 8 + pr] * rb[(gq * 4 + 3) * 32 + 16 + pc]);
      float4 h, l;
      split_tf32(v, h, l);
      *reinterpret_cast<float4*>(Ahi + gq * (A_LBO / 4) + pa * 4) = h;
      *reinterpret_cast<float4*>(Alo + gq * (A_LBO / 4) + pa * 4) = l;
    }
    // ---- B: K-major [k/4][n][4], thread = time sample, 4 sensors per 16-byte store
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int n = tid + i * kThreadsTC;
      if (n < N) {
#pragma unroll
        for (int kq = 0; kq < kKC / 4; ++kq) {
          float4 h, l;
          split_tf32(make_float4(sv[i][4 * kq], sv[i][4 * kq + 1], sv[i][4 * kq + 2], sv[i][4 * kq + 3]), h, l);
          const int off = kq * (B_LBO / 4) + n * 4;
          *reinterpret_cast<float4*>(Bhi + off) = h;
          *reinterpret_cast<float4*>(Blo + off) = l;
        }
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
        umma_tf32(tmem, dah, dbh, IDESC, (cur.c | ks) ? 1u : 0u);
        umma_tf32(tmem, dah, dbl, IDESC, 1u);
        umma_tf32(tmem, dal, dbh, IDESC, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       su32(&mma_bar[s]))
                   : "memory");
      // slot (g + 3) % 4 was last read in stage g - 1 (before this stage's barrier)
      if (cr.valid) {
        fetch_recs(g + kRecSlots - 1, cr);
        cursor_claim(p, cr, ring);
      }
    }
    if (cs.valid) load_samples(g + 2, cs, sv);
    cursor_next(p, cs, ring);
    const bool last = cur.c == cur.nch - 1;
    if (last) epilogue(g);
    cursor_next(p, cur, ring);
  };
  for (int g = 0; cur.valid; g += 2) {
    stage(g, sv0);
    if (cur.valid) stage(g + 1, sv1);
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

template <int N>
cudaError_t go_tc(const SpreadParams& p, cudaStream_t s) {
  constexpr int STAGE = 2 * kTM * kKC * 4 + 2 * kKC * N * 4;
  const size_t smem = (size_t)kStages * STAGE;
  auto k = spread_tc_kernel<N>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err) return err;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  SpreadParams q = p;
  q.tc_tblocks = (p.t_end - p.t_begin) / N;
  const int blocks = std::min(q.tc_ntiles * q.tc_tblocks, 2 * sms);
  if ((err = cudaMemsetAsync(q.tc_counter, 0, sizeof(int), s))) return err;
  if (blocks > 0 && q.tc_tblocks > 0) k<<<blocks, kThreadsTC, smem, s>>>(q);
  return cudaGetLastError();
}


// ===========================================================================
// fp16 two-term variant (default): kind::f16 UMMAs on hi/lo halves.
//
// x = hi + lo with hi = fp16(x), lo = fp16(x - hi) keeps 22 significant bits
// (as the tf32 split), provided |x| stays inside the fp16 range: the records
// are scaled by powers of two at plan time so every weight product is below
// 2^14, the samples by a power of two from their maximum per launch
// (absmax_kernel), and the epilogue undoes both exactly.  Half the operand
// bytes and MMA work of 3xTF32.
//
// The weights W[p][k] do not depend on the data, so the A operands (hi, lo)
// of every 16-sensor stage are built once per plan, in the UMMA layout
// (build_a16_kernel, 8 KB per stage), and each stage just bulk-copies them.
// The 16 gathered sample rows of a stage (N samples each, contiguous in HBM)
// are bulk-copied too, two stages ahead, into a staging ring, so no thread
// holds prefetched samples in registers or issues per-sample loads.
// ===========================================================================

__device__ __forceinline__ void split_f16x8(const float (&v)[8], uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __half2 a = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
    const float2 af = __half22float2(a);
    const __half2 b = __floats2half2_rn(v[2 * j] - af.x, v[2 * j + 1] - af.y);  // v - hi exact in fp32
    h[j] = *reinterpret_cast<const uint32_t*>(&a);
    l[j] = *reinterpret_cast<const uint32_t*>(&b);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Same split of s * v[0..7] with packed FP32 ops (FMUL2 / FADD2) and f16x2 conversions.
__device__ __forceinline__ void split_f16x8_scaled(const float (&v)[8], float sc, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    asm("{\n\t.reg .b64 x, s, hf, d;\n\t.reg .b32 x0, x1, h0f, h1f, d0, d1;\n\t.reg .b16 h0, h1;\n\t"
        "mov.b64 x, {%2, %3};\n\tmov.b64 s, {%4, %4};\n\tmul.rn.f32x2 x, x, s;\n\t"
        "mov.b64 {x0, x1}, x;\n\tcvt.rn.f16x2.f32 %0, x1, x0;\n\t"
        "mov.b32 {h0, h1}, %0;\n\tcvt.f32.f16 h0f, h0;\n\tcvt.f32.f16 h1f, h1;\n\t"
        "mov.b64 hf, {h0f, h1f};\n\tsub.rn.f32x2 d, x, hf;\n\tmov.b64 {d0, d1}, d;\n\t"
        "cvt.rn.f16x2.f32 %1, d1, d0;\n\t}"
        : "=r"(h[j]), "=r"(l[j])
        : "f"(v[2 * j]), "f"(v[2 * j + 1]), "f"(sc));
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// D f32, A/B f16, both K-major, M = 128, N.
__host__ __device__ constexpr uint32_t umma_idesc_f16(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}

// Plan time: per stage of 16 records, A hi/lo in the K-major no-swizzle UMMA
// layout [part][octet][128 points][8 halves] (8 KB) and the 16 sample row offsets.
__global__ void build_a16_kernel(const float* __restrict__ recs, int nstages, uint4* __restrict__ a16,
                                 uint32_t* __restrict__ offs) {
  const int tid = threadIdx.x, pa = tid & (kTM - 1), pr = pa / kTC, pc = pa % kTC, o = tid >> 7;
  for (int st = blockIdx.x; st < nstages; st += gridDim.x) {
    const float* rb = recs + (size_t)st * kKC * 32;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = rb[(o * 8 + j) * 32 + 8 + pr] * rb[(o * 8 + j) * 32 + 16 + pc];
    uint4 h, l;
    split_f16x8(v, h, l);
    uint4* d = a16 + (size_t)st * 512;  // 512 x 16 B
    d[o * kTM + pa] = h;
    d[256 + o * kTM + pa] = l;
    if (tid < kKC) offs[(size_t)st * kKC + tid] = __float_as_uint(rb[tid * 32]);
  }
}

// max |s| over rows [0, M), samples [tb, te), as float bits; one warp per row
__global__ void absmax_kernel(const float* __restrict__ s, int M, int T, int tb, int te, unsigned* __restrict__ out) {
  const int lane = threadIdx.x & 31, w4 = (te - tb) >> 2;
  unsigned m = 0;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < M; r += gridDim.x * (blockDim.x >> 5)) {
    const float4* row = reinterpret_cast<const float4*>(s + (size_t)r * T + tb);
#pragma unroll 4
    for (int c = lane; c < w4; c += 32) {
      const float4 v = __ldcs(row + c);
      m = max(m, max(max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu),
                     max(__float_as_uint(v.z) & 0x7fffffffu, __float_as_uint(v.w) & 0x7fffffffu)));
    }
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if (lane == 0 && m) atomicMax(out, m);
}

// p.tc_counter slots (ints): work-item counters of the two launches, max |sample| bits seen, redo flag
// (zeroed before every gridding) and the scale hint, which persists from call to call
constexpr int kCtrWork0 = 0, kCtrSeen = 1, kCtrWork1 = 2, kCtrRedo = 3;
constexpr int kCtrBatch = 5;  // max |sample| over a batch of frames (spread_tc16_batch_max), set by the caller
// scale hints: one per time block a launch may start at (launches over time chunks of one record --
// the host-buffer path uploads and grids in chunks -- see different maxima; each keeps its own hint)
constexpr int kCtrHint = 8, kHintSlots = 16;

// The sample scale is 2^(14 - 4 b) with b = ceil(e / 4) the 4-binade bucket of max |sample| in
// [2^(e-1), 2^e): the scaled maximum lies in [2^10, 2^14).  Quantising the exponent makes a scale
// hint from the previous call (go_tc16) valid for a 16x range of maxima instead of 2x.
__host__ __device__ __forceinline__ int scale_bucket(unsigned float_bits) {
  const int e = (int)((float_bits >> 23) & 0xffu) - 126;  // frexp exponent of a normal float
  return e >= 0 ? (e + 3) / 4 : -((-e) / 4);              // ceil(e / 4)
}

// Work items of the fp16 kernel, resolved by thread 0 into a shared ring:
// {tile's first record / 16, stages, row0, col0, time block}; stages == 0
// marks the end.  Thread 0 claims items two ahead (atomicAdd result and the
// tile-table load are consumed one item later), so neither latency stalls
// the stage loop.
struct Item16 {
  int st0, nch, row0, col0, tb;
};
struct Claimer16 {  // thread 0 only
  int wb, wc;       // claimed ids: B (tile loaded into tb_), C (atomic in flight)
  int4 tb_;
};
__device__ __forceinline__ Item16 item16_make(const SpreadParams& p, int w, int4 t) {
  Item16 it;
  if (w < p.tc_nonempty * p.tc_tblocks) {
    it.st0 = t.x / kKC;
    it.nch = t.y / kKC;
    it.row0 = t.z;
    it.col0 = t.w;
    it.tb = w % p.tc_tblocks;
  } else {
    it.st0 = it.nch = it.row0 = it.col0 = it.tb = 0;
  }
  return it;
}
__device__ __forceinline__ int4 item16_tile(const SpreadParams& p, int w) {
  return w < p.tc_nonempty * p.tc_tblocks ? __ldg(&p.tc_tiles[w / p.tc_tblocks]) : make_int4(0, 0, 0, 0);
}
// next item into ring slot k: B's resolved item; B <- C (issue its tile load); C <- new claim
__device__ __forceinline__ void claim16(const SpreadParams& p, Claimer16& q, Item16* ring, int k, int* counter) {
  ring[k & (kRing - 1)] = item16_make(p, q.wb, q.tb_);
  q.wb = q.wc;
  q.tb_ = item16_tile(p, q.wb);
  q.wc = atomicAdd(counter, 1);
}
struct Cursor16 {
  int k, c;  // ring position, stage within the item
  Item16 it;
};
__device__ __forceinline__ bool c16_valid(const Cursor16& u) { return u.it.nch > 0; }
__device__ __forceinline__ void c16_next(Cursor16& u, const Item16* ring) {
  if (!c16_valid(u) || ++u.c < u.it.nch) return;
  ++u.k;
  u.c = 0;
  u.it = ring[u.k & (kRing - 1)];
}

// experiment switches (tools/variants.sh): drop one part of the work to time the rest
#ifndef PATFFT_TC16_NOSTORE
#define PATFFT_TC16_NOSTORE 0
#endif
#ifndef PATFFT_TC16_NOBUILD
#define PATFFT_TC16_NOBUILD 0
#endif
#ifndef PATFFT_TC16_BUILD_WARP0
#define PATFFT_TC16_BUILD_WARP0 2  // first warp of the B build (0: all warps, tid < N; 2: spread 0.471 -> 0.461 ms; 1: 0.497, 3: 0.462)
#endif
#ifndef PATFFT_TC16_NOMMA
#define PATFFT_TC16_NOMMA 0
#endif
#ifndef PATFFT_TC16_NOEPI
#define PATFFT_TC16_NOEPI 0
#endif
#ifndef PATFFT_TC16_NOA
#define PATFFT_TC16_NOA 0  // diagnosis: skip the A operand copies (wrong results; DRAM traffic of the sample gathers alone)
#endif
#ifndef PATFFT_TC16_MBAR
#define PATFFT_TC16_MBAR 0  // B hand-off by an mbarrier only the MMA thread and load warp wait on (1): measured 0.504 vs 0.480 ms
#endif

template <int N>
__global__ void __launch_bounds__(kThreadsTC, 2) spread_tc16_kernel(const __grid_constant__ SpreadParams p) {
  constexpr int A_SLOT = 8192;                     // hi + lo, [part][octet][128][8] halves
  constexpr int A_SLOTS = 4;
  constexpr int B_HALF = kKC * N * 2;              // one part: [octet][N][8] halves
  constexpr int B_SLOT = 2 * B_HALF;
  constexpr int S_SLOT = kKC * N * 4;              // gathered rows [16][N] fp32
  constexpr uint32_t A_LBO = kTM * 16, A_SBO = 128;
  constexpr uint32_t B_LBO = N * 16, B_SBO = 128;
  constexpr uint32_t TCOLS = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  constexpr uint32_t IDESC = umma_idesc_f16(N);
  constexpr int NH = N / 2;

  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* const a_ring = smem;                               // A_SLOTS x 8 KB
  constexpr int BO_AREA = 2 * B_SLOT > 32768 ? 2 * B_SLOT : 32768;  // B slots, also the epilogue staging
  uint8_t* const b_ops = smem + A_SLOTS * A_SLOT;
  float* const s_ring = reinterpret_cast<float*>(b_ops + BO_AREA);  // 2 x S_SLOT
  constexpr int OFF_SLOTS = 8;  // sample row offsets of stage x: slot x % 8, fetched at stage x - 4
  __shared__ uint64_t mma_bar[2], ld_bar[2], off_bar[OFF_SLOTS], full_bar[2];
  __shared__ __align__(16) uint32_t offbuf[OFF_SLOTS * kKC];
  __shared__ uint32_t tmem_base_s;
  __shared__ Item16 ring[kRing];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q4 = warp & 3;
  // speculative sample scale (go_tc16): the second launch runs only when the check after the first
  // one found the scale hint in the wrong binade
  if (p.tc_pass == 1 && p.tc_counter[kCtrRedo] == 0) return;
  int* const work_counter = p.tc_counter + (p.tc_pass == 1 ? kCtrWork1 : kCtrWork0);

  // ---- empty tiles (no sensor meets them): zeros
  for (int i = p.tc_nonempty + blockIdx.x; i < p.tc_ntiles; i += gridDim.x) {
    const int4 t = __ldg(&p.tc_tiles[i]);
    const int len = p.t_end - p.t_begin;
    for (int pt = warp; pt < kTM; pt += kThreadsTC / 32) {
      float* o = p.grid + ((size_t)(t.z + pt / kTC) * p.ncols + (t.w + pt % kTC)) * p.T + p.t_begin;
      for (int q = lane * 4; q < len; q += 128) *reinterpret_cast<float4*>(o + q) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  Cursor16 cur, cs, cr;  // stage being built, loads (+2, warp 1), offsets (+3, thread 0)
  Claimer16 claim;
  if (tid == 0) {
    const int w0 = atomicAdd(work_counter, 1);
    claim.wb = atomicAdd(work_counter, 1);
    claim.wc = atomicAdd(work_counter, 1);
    ring[0] = item16_make(p, w0, item16_tile(p, w0));
    claim.tb_ = item16_tile(p, claim.wb);
  }
  __syncthreads();
  cur.k = 0;
  cur.c = 0;
  cur.it = ring[0];
  if (!c16_valid(cur)) return;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base_s)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  if (tid == 0) {
    for (int s2 = 0; s2 < 2; ++s2) {
      mbar_init_tc(&mma_bar[s2], 1);
      mbar_init_tc(&ld_bar[s2], 1);
      mbar_init_tc(&full_bar[s2], kThreadsTC);
    }
    for (int s2 = 0; s2 < OFF_SLOTS; ++s2) mbar_init_tc(&off_bar[s2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  // scales: samples by 2^es (max |s| * 2^es < 2^14), output by 2^-(wexp + es)
  float s_scale, o_scale;
  {
    const float mx = __uint_as_float(p.tc_counter[p.tc_scale_src]);
    int es = 0;
    if (mx > 0.f && mx <= 3.4e38f) es = 14 - 4 * scale_bucket(p.tc_counter[p.tc_scale_src]);
    es = min(es, 126 - p.tc_wexp);
    s_scale = ldexpf(1.f, es);
    o_scale = ldexpf(1.f, -(p.tc_wexp + es));
  }

  // thread 0: offsets of stage g (16 sample row offsets, 64 B) into slot g % OFF_SLOTS
  auto fetch_offs = [&](int g, const Cursor16& u) {
    const int r = g % OFF_SLOTS;
    mbar_expect(&off_bar[r], kKC * 4);
    bulk_g2s(offbuf + r * kKC, p.tc_off + ((size_t)u.it.st0 + u.c) * kKC, kKC * 4, &off_bar[r]);
  };
  // thread 0: advance the offsets cursor, resolving the next item at a crossing
  auto cr_next = [&]() {
    if (!c16_valid(cr) || ++cr.c < cr.it.nch) return;
    ++cr.k;
    cr.c = 0;
    claim16(p, claim, ring, cr.k, work_counter);
    cr.it = ring[cr.k & (kRing - 1)];
  };
  // warp 1 (all lanes, uniform cursor): A operands and the 16 sample rows of stage g,
  // one bulk copy per lane, while thread 0 issues the MMAs of the current stage
  auto issue_loads = [&](int g, const Cursor16& u) {
    const int r = g % OFF_SLOTS;
    mbar_wait_tc(&off_bar[r], (g / OFF_SLOTS) & 1);
    uint64_t* bar = &ld_bar[g & 1];
    if (lane == 0) mbar_expect(bar, (PATFFT_TC16_NOA ? 0 : A_SLOT) + S_SLOT);
    __syncwarp();
    if (lane < kKC) {
      const int t0 = p.t_begin + u.it.tb * N;
      bulk_g2s(s_ring + (g & 1) * (S_SLOT / 4) + lane * N, p.samples + ((size_t)offbuf[r * kKC + lane] + t0), N * 4,
               bar);
    } else if (lane == kKC && !PATFFT_TC16_NOA) {
      bulk_g2s(a_ring + (g % A_SLOTS) * A_SLOT, p.tc_a16 + ((size_t)u.it.st0 + u.c) * (A_SLOT / 16), A_SLOT, bar);
    }
  };
  if (tid == 0) {
    cr = cur;
    for (int g = 0; g < 4 && c16_valid(cr); ++g) {
      fetch_offs(g, cr);
      cr_next();
    }
  }
  __syncthreads();  // ring entries of the first stages
  if (warp == 1) {
    cs = cur;
    for (int g = 0; g < 2 && c16_valid(cs); ++g) {
      issue_loads(g, cs);
      c16_next(cs, ring);
    }
  }

  // B builder: thread = (time sample tq and tq + N/2, sensor octet ko)
  const int tq = tid % NH, ko = tid / NH;
  float seen_max = 0.f;

  auto epilogue = [&](int g) {
    const int t0 = p.t_begin + cur.it.tb * N;
    mbar_wait_tc(&mma_bar[g & 1], (g >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (PATFFT_TC16_NOEPI) {
      __syncthreads();
      return;
    }
    // staging: per warp 32 points x 32 floats, 16-byte chunks XOR-swizzled (conflict-free both ways)
    float* stg = reinterpret_cast<float*>(b_ops) + warp * 32 * 32;
#pragma unroll 1
    for (int j = warp >> 2; j < N / 32; j += kThreadsTC / 128) {
      uint32_t r[32];
      const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(j * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
          "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (p.tc_tma_store) {  // the previous chunk's tensor store must have read the staging
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(stg + lane * 32 + ((q ^ (lane & 7)) * 4)) =
            make_float4(__uint_as_float(r[4 * q]) * o_scale, __uint_as_float(r[4 * q + 1]) * o_scale,
                        __uint_as_float(r[4 * q + 2]) * o_scale, __uint_as_float(r[4 * q + 3]) * o_scale);
      if (p.tc_tma_store) {
        // the warp's 32 points are 2 grid rows x 16 columns: one 32 x 16 x 2 box; the staging's XOR
        // swizzle (16-byte chunk q of point row pl at q ^ (pl & 7)) is the 128B swizzle of the map
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && !PATFFT_TC16_NOSTORE) {
          asm volatile(
              "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                  reinterpret_cast<uint64_t>(&p.tc_gmap)),
              "r"(t0 + j * 32), "r"(cur.it.col0), "r"(cur.it.row0 + q4 * 2), "r"(su32(stg))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        continue;
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int pl = q * 4 + (lane >> 3), pt = q4 * 32 + pl, c = lane & 7;  // point within the tile
        const float4 v = *reinterpret_cast<const float4*>(stg + pl * 32 + ((c ^ (pl & 7)) * 4));
        float* o = p.grid + ((size_t)(cur.it.row0 + pt / kTC) * p.ncols + (cur.it.col0 + pt % kTC)) * p.T + t0 + j * 32;
        if (!PATFFT_TC16_NOSTORE || v.x == 12345.f) *reinterpret_cast<float4*>(o + c * 4) = v;
      }
      __syncwarp();
    }
    if (p.tc_tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
  };

  for (int g = 0; c16_valid(cur); ++g) {
    const int sb = g & 1;
    if (g >= 2) {
      mbar_wait_tc(&mma_bar[sb], ((g >> 1) - 1) & 1);  // B slot free (stage g - 2 done)
      // (acquire of everyone's stage g - 2 arrival: the ring entries thread 0 resolved before it)
      if (PATFFT_TC16_MBAR) mbar_wait_tc(&full_bar[sb], ((g >> 1) - 1) & 1);
    }
    mbar_wait_tc(&ld_bar[sb], (g >> 1) & 1);                      // A + samples of stage g landed
    uint8_t* bo = b_ops + sb * B_SLOT;
    const float* sr = s_ring + sb * (S_SLOT / 4);
#if PATFFT_TC16_BUILD_WARP0
    // B built by warps PATFFT_TC16_BUILD_WARP0.. only: warp 0 (MMA issue, offset fetches,
    // item claims) and warp 1 (bulk copies) reach the stage barrier without the build's latency
    if (warp >= PATFFT_TC16_BUILD_WARP0 && !PATFFT_TC16_NOBUILD) {
      constexpr int FT = 32 * PATFFT_TC16_BUILD_WARP0;
#pragma unroll 1
      for (int u = tid - FT; u < 2 * N; u += kThreadsTC - FT) {
        const int n = u % N, kb = u / N;
        float w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = sr[(8 * kb + j) * N + n];
        if (p.tc_track)  // max |sample| of everything this launch grids (checked against the scale hint)
          seen_max = fmaxf(seen_max, fmaxf(fmaxf(fmaxf(fabsf(w[0]), fabsf(w[1])), fmaxf(fabsf(w[2]), fabsf(w[3]))),
                                           fmaxf(fmaxf(fabsf(w[4]), fabsf(w[5])), fmaxf(fabsf(w[6]), fabsf(w[7])))));
        uint4 bh, bl;
        split_f16x8_scaled(w, s_scale, bh, bl);
        *reinterpret_cast<uint4*>(bo + kb * B_LBO + n * 16) = bh;
        *reinterpret_cast<uint4*>(bo + B_HALF + kb * B_LBO + n * 16) = bl;
      }
    }
    if (false) {
#else
    if (tid < N && !PATFFT_TC16_NOBUILD) {
#endif
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = tq + h * NH;
        float w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = sr[(8 * ko + j) * N + n];
        uint4 bh, bl;
        split_f16x8_scaled(w, s_scale, bh, bl);
        *reinterpret_cast<uint4*>(bo + ko * B_LBO + n * 16) = bh;
        *reinterpret_cast<uint4*>(bo + B_HALF + ko * B_LBO + n * 16) = bl;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (PATFFT_TC16_MBAR) {
      // B of stage g is complete once all threads arrived; only the MMA thread and the
      // load warp wait for it, the other warps go on to stage g + 1
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full_bar[sb])) : "memory");
      if (tid == 0 || warp == 1) mbar_wait_tc(&full_bar[sb], (g >> 1) & 1);
    } else {
      __syncthreads();
    }
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_hi = su32(a_ring + (g % A_SLOTS) * A_SLOT), a_lo = a_hi + A_SLOT / 2;
      const uint32_t b_hi = su32(bo), b_lo = b_hi + B_HALF;
      const uint64_t dah = umma_desc(a_hi, A_LBO, A_SBO), dal = umma_desc(a_lo, A_LBO, A_SBO);
      const uint64_t dbh = umma_desc(b_hi, B_LBO, B_SBO), dbl = umma_desc(b_lo, B_LBO, B_SBO);
      if (!PATFFT_TC16_NOMMA) {
        umma_f16(tmem, dah, dbh, IDESC, cur.c ? 1u : 0u);
        umma_f16(tmem, dah, dbl, IDESC, 1u);
        umma_f16(tmem, dal, dbh, IDESC, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       su32(&mma_bar[sb]))
                   : "memory");
      // offsets of stage g + 4 into slot (g + 4) % 8, last read when stage g - 4's loads were issued
      if (c16_valid(cr)) {
        fetch_offs(g + 4, cr);
        cr_next();
      }
    } else if (warp == 1) {
      // stage g + 2: A slot (g + 2) % 4 was read by stage g - 2 (complete), sample slot sb was
      // read by this stage's B build (all threads arrived above)
      if (c16_valid(cs)) issue_loads(g + 2, cs);
      c16_next(cs, ring);
    }
    if (cur.c == cur.it.nch - 1) epilogue(g);
    c16_next(cur, ring);
  }
  if (p.tc_track) {
    const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(seen_max));  // non-negative floats order as uints
    if (lane == 0 && mb) atomicMax(reinterpret_cast<unsigned*>(p.tc_counter + kCtrSeen), mb);
  }
  if (p.tc_tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

// After the first gridding launch: is the scale hint it used in the 4-binade bucket of the maximum it
// saw?  (Same bucket <=> the launch used exactly the scale the max pass would have given, so the
// result does not depend on the hint's history.)  Otherwise the second launch redoes the gridding.
__global__ void check_scale_kernel(int* __restrict__ ctr, int hint_slot) {
  const unsigned seen = (unsigned)ctr[kCtrSeen], hint = (unsigned)ctr[hint_slot];
  const bool ok = seen == 0 || (hint != 0 && scale_bucket(seen) == scale_bucket(hint));
  ctr[kCtrRedo] = ok ? 0 : 1;
  if (seen) ctr[hint_slot] = (int)seen;
}

template <int N>
cudaError_t go_tc16(const SpreadParams& p, cudaStream_t s) {
  const size_t smem = 4 * 8192 + std::max(2 * (2 * kKC * N * 2), 32768) + 2 * (kKC * N * 4);
  auto k = spread_tc16_kernel<N>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err) return err;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  SpreadParams q = p;
  q.tc_tblocks = (p.t_end - p.t_begin) / N;
  const int blocks = std::min(q.tc_ntiles * q.tc_tblocks, 2 * sms);
  if ((err = cudaMemsetAsync(q.tc_counter, 0, 4 * sizeof(int), s))) return err;  // counters, seen, redo
  if (blocks <= 0 || q.tc_tblocks <= 0) return cudaSuccess;
  // The sample scale 2^es needs max |sample| of the launch.  PATFFT_TC16_SPECULATE=0: a max pass first
  // (one extra read of the samples, 47 us at cfg4).  Default: the launch uses the maximum the
  // previous launch of this plan saw as a hint, records the maximum it sees itself, and a one-thread
  // check compares their 4-binade buckets; only if they differ (first call, data 16x off) a
  // second launch redoes the gridding with the right scale -- otherwise it exits at once.  Same
  // scale either way, so the result is bit-identical to the max-pass form.
  static const bool speculate = [] {
    const char* e = std::getenv("PATFFT_TC16_SPECULATE");
    return e ? std::atoi(e) != 0 : true;
  }();
  if (p.tc_batch_scale) {  // frames of one batch share the scale of the batch's maximum (one max pass per batch)
    q.tc_scale_src = kCtrBatch;
    q.tc_track = 0;
    q.tc_pass = 0;
    k<<<blocks, kThreadsTC, smem, s>>>(q);
    return cudaGetLastError();
  }
  if (!speculate) {
    absmax_kernel<<<4 * sms, 256, 0, s>>>(p.samples, p.tc_m, p.T, p.t_begin, p.t_end,
                                          reinterpret_cast<unsigned*>(q.tc_counter + kCtrSeen));
    if ((err = cudaGetLastError())) return err;
    q.tc_scale_src = kCtrSeen;
    q.tc_track = 0;
    q.tc_pass = 0;
    k<<<blocks, kThreadsTC, smem, s>>>(q);
    return cudaGetLastError();
  }
  q.tc_scale_src = kCtrHint + ((p.t_begin / N) % kHintSlots);
  q.tc_track = 1;
  q.tc_pass = 0;
  k<<<blocks, kThreadsTC, smem, s>>>(q);
  if ((err = cudaGetLastError())) return err;
  check_scale_kernel<<<1, 1, 0, s>>>(q.tc_counter, q.tc_scale_src);
  if ((err = cudaGetLastError())) return err;
  q.tc_track = 0;
  q.tc_pass = 1;
  k<<<blocks, kThreadsTC, smem, s>>>(q);
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

cudaError_t spread_tc16_build(const float* recs, int nstages, void* a16, uint32_t* offs, cudaStream_t s) {
  if (nstages <= 0) return cudaSuccess;
  build_a16_kernel<<<std::min(nstages, 148 * 8), kThreadsTC, 0, s>>>(recs, nstages, static_cast<uint4*>(a16), offs);
  return cudaGetLastError();
}

// max |sample| over `rows` sensor rows (all frames of a batch) into the plan's batch-scale slot
cudaError_t spread_tc16_batch_max(const float* samples, int64_t rows, int T, int* counters, cudaStream_t s) {
  cudaError_t err = cudaMemsetAsync(counters + kCtrBatch, 0, sizeof(int), s);
  if (err) return err;
  absmax_kernel<<<4 * 148, 256, 0, s>>>(samples, (int)std::min<int64_t>(rows, INT32_MAX), T, 0, T,
                                        reinterpret_cast<unsigned*>(counters + kCtrBatch));
  return cudaGetLastError();
}

cudaError_t launch_spread_tc(const SpreadParams& p, cudaStream_t s) {
  const int n = p.tc_n;
  if ((p.t_end - p.t_begin) % n || p.t_begin % n) return cudaErrorInvalidValue;
  if (p.tc_f16) {
    switch (n) {
      case 256: return go_tc16<256>(p, s);
      case 128: return go_tc16<128>(p, s);
      case 64: return go_tc16<64>(p, s);
      case 32: return go_tc16<32>(p, s);
    }
    return cudaErrorInvalidValue;
  }
  switch (n) {
    case 256: return go_tc<256>(p, s);
    case 128: return go_tc<128>(p, s);
    case 64: return go_tc<64>(p, s);
    case 32: return go_tc<32>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace patfft
