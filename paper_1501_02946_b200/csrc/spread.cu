// NED gridding (reference nufft.py:373-404 + the weighting of recon.py:374).
//
// Output-stationary and deterministic (no atomics): a CTA owns a group of R
// consecutive oversampled grid rows, one column segment and 128 consecutive
// time samples (one per thread).  It sweeps the group's sensor records,
// sorted by column window, once: each record carries the sensor's R row
// weights (times h_m/dx^(d-1)) and its 2K column weights.  Every thread
// keeps an R x RING register ring of column accumulators; columns that
// can no longer receive contributions are streamed to HBM in groups of 4
// (coalesced over time).  Records and the sensors' time samples are staged
// into shared memory one chunk ahead with cp.async, so the FFMA stream never
// waits on a dependent global load.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "patfft_internal.h"

namespace patfft {
namespace {

constexpr int kThreads = 128;  // time samples per CTA
constexpr int kChunk = 32;     // records staged per chunk

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Packed FP32 FMA (sm_100a FFMA2): two lanes of work per issue slot; a
// broadcast scalar operand (s, s) is folded into the instruction.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

template <int Q, int R, int RING>
__device__ __forceinline__ void flush_q(float2 (&acc)[R][RING / 2], float* __restrict__ colp, size_t row_stride,
                                        int T, int rows_valid, bool store) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (store && r < rows_valid) {
        colp[(size_t)r * row_stride + (size_t)(2 * c) * T] = acc[r][Q * 2 + c].x;
        colp[(size_t)r * row_stride + (size_t)(2 * c + 1) * T] = acc[r][Q * 2 + c].y;
      }
      acc[r][Q * 2 + c] = make_float2(0.f, 0.f);
    }
  }
}

template <int R, int RING>
__device__ __forceinline__ void flush_group(float2 (&acc)[R][RING / 2], int g, float* __restrict__ base, size_t row_stride,
                                            int T, int c0, int c1, int rows_valid, bool tvalid) {
  const int col = g * 4;
  const bool store = tvalid && col >= c0 && col < c1;
  float* colp = base + (size_t)(store ? col : 0) * T;
  switch (g & (RING / 4 - 1)) {
#define PATFFT_FQ(q) \
  case q:            \
    if (q < RING / 4) flush_q<(q < RING / 4 ? q : 0), R, RING>(acc, colp, row_stride, T, rows_valid, store); \
    break;
    PATFFT_FQ(0) PATFFT_FQ(1) PATFFT_FQ(2) PATFFT_FQ(3) PATFFT_FQ(4) PATFFT_FQ(5) PATFFT_FQ(6) PATFFT_FQ(7)
#undef PATFFT_FQ
  }
}

// Record layout (float words): [0] ws (int bits), [1] sensor m (int bits),
// [2..3] pad, [4..7] row weights (R <= 4), [8..8+RING) column weights
// rotated into ring order: slot (ws + j) mod RING holds tap j, the other
// RING - 2K slots are zero.  Every record then updates the whole ring with
// compile-time register indices (no per-record branch on the rotation).
template <int K2, int R, int RING, bool VEC16>
__global__ void __launch_bounds__(kThreads, 4) spread_kernel(const SpreadParams p) {
  static_assert(K2 + 3 <= RING, "ring too small for the window");
  constexpr int RECW = 8 + RING;
  constexpr int NG = RING / 4;
  constexpr int PIECE = VEC16 ? 4 : 2;                 // floats per cp.async
  constexpr int PIECES = kThreads / PIECE;             // per record
  constexpr int PER_THREAD = kChunk * PIECES / kThreads;
  extern __shared__ float4 smem4[];
  float* rbuf = reinterpret_cast<float*>(smem4);             // [2][kChunk][RECW]
  float* sbuf = rbuf + 2 * kChunk * RECW;                    // [2][kChunk][kThreads]

  const int4 bk = p.blk[blockIdx.x];
  const int grp = p.blk_grp[blockIdx.x];
  const int c0 = bk.z;
  const int c1 = bk.w;
  const int T = p.T;
  const int t0 = p.t_begin + blockIdx.y * kThreads;
  const int tid = threadIdx.x;
  const int t = t0 + tid;
  const bool tvalid = t < p.t_end;
  const int2 rg = make_int2(bk.x, bk.y);
  const int nrec = rg.y - rg.x;
  const int nchunks = (nrec + kChunk - 1) / kChunk;
  const int row0 = grp * R;
  const int rows_valid = min(R, p.nrows - row0);

  // which (record, piece) pairs this thread stages
  const int piece = tid % PIECES;
  const int rec_lane = tid / PIECES;
  constexpr int REC_STEP = kThreads / PIECES;
  const int tp = t0 + piece * PIECE;
  const int src_bytes = max(0, min(PIECE, p.t_end - tp)) * 4;

  int mnext[PER_THREAD];
  auto load_m = [&](int c) {
#pragma unroll
    for (int i = 0; i < PER_THREAD; ++i) {
      const int e = c * kChunk + rec_lane + i * REC_STEP;
      mnext[i] = (e < nrec) ? __ldg(reinterpret_cast<const int*>(p.recs) + (size_t)(rg.x + e) * RECW + 1) : -1;
    }
  };
  auto stage = [&](int c, int b) {
    const int e0 = c * kChunk;
    const int ne = min(kChunk, nrec - e0);
    const float4* srcr = reinterpret_cast<const float4*>(p.recs + (size_t)(rg.x + e0) * RECW);
    float4* dstr = reinterpret_cast<float4*>(rbuf + b * kChunk * RECW);
    for (int i = tid; i < ne * RECW / 4; i += kThreads) cp_async16(dstr + i, srcr + i, 16);
    float* sb = sbuf + b * kChunk * kThreads;
#pragma unroll
    for (int i = 0; i < PER_THREAD; ++i) {
      const int e = rec_lane + i * REC_STEP;
      const int m = mnext[i];
      float* dst = sb + e * kThreads + piece * PIECE;
      if (m >= 0) {
        const float* src = p.samples + (size_t)m * T + (src_bytes > 0 ? tp : 0);
        if (VEC16) cp_async16(dst, src, src_bytes);
        else cp_async8(dst, src, src_bytes);
      }
    }
    cp_commit();
  };

  float2 acc[R][RING / 2];  // column pairs (2c, 2c+1)
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < RING / 2; ++c) acc[r][c] = make_float2(0.f, 0.f);

  const size_t row_stride = (size_t)p.ncols * T;
  float* base = p.grid + (size_t)row0 * row_stride + (tvalid ? t : 0);
  int fg = (c0 >> 2) - NG;  // ring holds column groups [fg, fg + NG)

  if (nchunks > 0) {
    load_m(0);
    stage(0, 0);
    load_m(1);
  }
  for (int c = 0; c < nchunks; ++c) {
    const int b = c & 1;
    if (c + 1 < nchunks) {
      stage(c + 1, b ^ 1);
      load_m(c + 2);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const float* rb = rbuf + b * kChunk * RECW;
    const float* sb = sbuf + b * kChunk * kThreads + tid;
    const int ne = min(kChunk, nrec - c * kChunk);
    for (int e = 0; e < ne; ++e) {
      const float* rec = rb + e * RECW;
      const int ws = __float_as_int(rec[0]);
      const int gs = ws >> 2;
      while (fg < gs) {
        flush_group<R, RING>(acc, fg, base, row_stride, T, c0, c1, rows_valid, tvalid);
        ++fg;
      }
      const float s = sb[e * kThreads];
      const float4 wr4 = *reinterpret_cast<const float4*>(rec + 4);
      const float wrv[4] = {wr4.x, wr4.y, wr4.z, wr4.w};
      float sv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) sv[r] = s * wrv[r];
      const float4* wq = reinterpret_cast<const float4*>(rec + 8);
#pragma unroll
      for (int j = 0; j < RING / 4; ++j) {
        const float4 q = wq[j];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float2 svv = make_float2(sv[r], sv[r]);
          acc[r][2 * j + 0] = ffma2(make_float2(q.x, q.y), svv, acc[r][2 * j + 0]);
          acc[r][2 * j + 1] = ffma2(make_float2(q.z, q.w), svv, acc[r][2 * j + 1]);
        }
      }
    }
    __syncthreads();
  }
  const int gend = c1 >> 2;
  while (fg < gend) {
    flush_group<R, RING>(acc, fg, base, row_stride, T, c0, c1, rows_valid, tvalid);
    ++fg;
  }
}

template <int K2, int R, int RING>
cudaError_t go(const SpreadParams& p, int nblk, cudaStream_t s) {
  constexpr int RECW = 8 + RING;
  const size_t smem = sizeof(float) * 2 * kChunk * (RECW + kThreads);
  dim3 grid((unsigned)nblk, (unsigned)((p.t_end - p.t_begin + kThreads - 1) / kThreads));
  cudaError_t err;
  if (p.T % 4 == 0) {
    auto k = spread_kernel<K2, R, RING, true>;
    if ((err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return err;
    k<<<grid, kThreads, smem, s>>>(p);
  } else {
    auto k = spread_kernel<K2, R, RING, false>;
    if ((err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return err;
    k<<<grid, kThreads, smem, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace

int spread_rows_per_group(int n_lat, int K2) {
  static const int forced = [] {
    const char* e = std::getenv("PATFFT_SPREAD_ROWS");
    return e ? std::atoi(e) : 0;
  }();
  if (n_lat == 1) return 1;
  if ((forced == 2 || forced == 4) && (K2 <= 12 || forced == 2)) return forced;
  return K2 <= 12 ? 4 : 2;
}
int spread_ring(int K2) { return K2 <= 12 ? 16 : 32; }
int spread_record_words(int K2) { return 8 + spread_ring(K2); }
int spread_time_chunks(int T) { return (T + kThreads - 1) / kThreads; }

cudaError_t launch_spread(const SpreadParams& p, int K2, int R, int nblk, cudaStream_t s) {
  if (R == 4) {
    switch (K2) {
      case 2: return go<2, 4, 16>(p, nblk, s);
      case 4: return go<4, 4, 16>(p, nblk, s);
      case 6: return go<6, 4, 16>(p, nblk, s);
      case 8: return go<8, 4, 16>(p, nblk, s);
      case 10: return go<10, 4, 16>(p, nblk, s);
      case 12: return go<12, 4, 16>(p, nblk, s);
    }
  } else if (R == 2) {
    switch (K2) {
      case 2: return go<2, 2, 16>(p, nblk, s);
      case 4: return go<4, 2, 16>(p, nblk, s);
      case 6: return go<6, 2, 16>(p, nblk, s);
      case 8: return go<8, 2, 16>(p, nblk, s);
      case 10: return go<10, 2, 16>(p, nblk, s);
      case 12: return go<12, 2, 16>(p, nblk, s);
      case 14: return go<14, 2, 32>(p, nblk, s);
      case 16: return go<16, 2, 32>(p, nblk, s);
    }
  } else if (R == 1) {
    switch (K2) {
      case 2: return go<2, 1, 16>(p, nblk, s);
      case 4: return go<4, 1, 16>(p, nblk, s);
      case 6: return go<6, 1, 16>(p, nblk, s);
      case 8: return go<8, 1, 16>(p, nblk, s);
      case 10: return go<10, 1, 16>(p, nblk, s);
      case 12: return go<12, 1, 16>(p, nblk, s);
      case 14: return go<14, 1, 32>(p, nblk, s);
      case 16: return go<16, 1, 32>(p, nblk, s);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace patfft
