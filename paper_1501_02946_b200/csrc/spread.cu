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
#ifndef PATFFT_SPREAD_CHUNK
#define PATFFT_SPREAD_CHUNK 32
#endif
constexpr int kChunk = PATFFT_SPREAD_CHUNK;  // records staged per chunk
#ifndef PATFFT_SPREAD_MINB
#define PATFFT_SPREAD_MINB 5
#endif

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
// --- bulk (TMA) copies completing on an mbarrier -------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra WAIT;\n"
      "DONE:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
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

// Accumulators: acc[slot][p] holds rows (2p, 2p+1) of ring column `slot`
// (R = 1: only .x is used).  Flushing a column stores its R rows (coalesced
// over time) and clears the slot.
template <int Q, int R, int NS>
__device__ __forceinline__ void flush_slot(float2 (&acc)[NS][(R + 1) / 2], float* __restrict__ colp,
                                           size_t row_stride, int rows_valid, bool store) {
#pragma unroll
  for (int p = 0; p < (R + 1) / 2; ++p) {
    if (store && 2 * p < rows_valid) colp[(size_t)(2 * p) * row_stride] = acc[Q][p].x;
    if (R > 1 && store && 2 * p + 1 < rows_valid) colp[(size_t)(2 * p + 1) * row_stride] = acc[Q][p].y;
    acc[Q][p] = make_float2(0.f, 0.f);
  }
}

// One record: acc[j][p] += (s*wr[2p], s*wr[2p+1]) * w_j for every ring slot j.
template <int NS, int R>
__device__ __forceinline__ void record_fma(float2 (&acc)[NS][(R + 1) / 2], const float* __restrict__ rec, float s) {
  constexpr int RP = (R + 1) / 2;
  const float4 wr4 = *reinterpret_cast<const float4*>(rec + 4);
  float2 sv[RP];
  if (R == 1) {
    sv[0] = make_float2(s * wr4.x, 0.f);
  } else {
    sv[0] = make_float2(s * wr4.x, s * wr4.y);
    if (RP > 1) sv[RP > 1 ? 1 : 0] = make_float2(s * wr4.z, s * wr4.w);
  }
  const float4* wq = reinterpret_cast<const float4*>(rec + 8);
#pragma unroll
  for (int j4 = 0; j4 < (NS + 3) / 4; ++j4) {
    const float4 q = wq[j4];
    const float wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j4 * 4 + u;
      if (j < NS) {
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          if (R == 1) acc[j < NS ? j : 0][r].x = fmaf(sv[r].x, wv[u], acc[j < NS ? j : 0][r].x);
          else acc[j < NS ? j : 0][r] = ffma2(sv[r], make_float2(wv[u], wv[u]), acc[j < NS ? j : 0][r]);
        }
      }
    }
  }
}

// Record layout (float words): [0] ws (int bits), [1] sensor m (int bits),
// [2..3] pad, [4..7] row weights (R <= 4), [8..8+NS) column weights rotated
// into ring order: slot (ws + j) mod NS holds tap j.  The ring is exactly
// NS = 2K columns wide, so every FMA is useful in the column direction, and
// each record updates the whole ring with compile-time register indices.
// Rows are paired into FFMA2 lanes: acc[j][p] += (s*wr[2p], s*wr[2p+1]) *
// w_j, with the column weight folded in as the broadcast operand.
//
// Column sweep as a state machine: state q means "the ring's oldest column
// fg lives in slot q".  In state q the CTA applies every record starting at
// fg, then flushes slot q (a compile-time register set: no indirect branch
// per column) and moves to state q + 1 mod NS.  The state is dispatched
// dynamically only when a staged chunk of records runs out.
template <int K2, int R, bool VEC16>
__global__ void __launch_bounds__(kThreads, PATFFT_SPREAD_MINB) spread_kernel(const SpreadParams p) {
  constexpr int NS = K2;
  constexpr int RP = (R + 1) / 2;
  constexpr int RECW = 8 + (K2 + 3) / 4 * 4;
  constexpr int PIECE = VEC16 ? 4 : 2;                 // floats per cp.async
  constexpr int PIECES = kThreads / PIECE;             // per record
  constexpr int PER_THREAD = kChunk * PIECES / kThreads;
  static_assert(NS <= 16, "ring states are generated for up to 16 slots");
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

  float2 acc[NS][RP];
#pragma unroll
  for (int j = 0; j < NS; ++j)
#pragma unroll
    for (int q = 0; q < RP; ++q) acc[j][q] = make_float2(0.f, 0.f);

  const size_t row_stride = (size_t)p.ncols * T;
  float* base = p.grid + (size_t)row0 * row_stride + (tvalid ? t : 0);
  // the ring holds columns [fg, fg + NS); start on a multiple of NS so the
  // sweep enters in state 0 (the few extra columns before c0 are not stored)
  int fg = (c0 - NS) >= 0 ? (c0 - NS) / NS * NS : -((NS - (c0 - NS) - 1) / NS) * NS;
  int fs = 0;

  if (nchunks > 0) {
    load_m(0);
    stage(0, 0);
    load_m(1);
  }
  const int npass = max(nchunks, 1);
  for (int c = 0; c < npass; ++c) {
    const int b = c & 1;
    int ne = 0;
    if (c < nchunks) {
      if (c + 1 < nchunks) {
        stage(c + 1, b ^ 1);
        load_m(c + 2);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      ne = min(kChunk, nrec - c * kChunk);
    }
    const bool last = c + 1 >= npass;
    const float* rb = rbuf + b * kChunk * RECW;
    const float* sb = sbuf + b * kChunk * kThreads + tid;
    int e = 0;
    switch (fs) {
      case 0: goto st_0;   case 1: goto st_1;   case 2: goto st_2;   case 3: goto st_3;
      case 4: goto st_4;   case 5: goto st_5;   case 6: goto st_6;   case 7: goto st_7;
      case 8: goto st_8;   case 9: goto st_9;   case 10: goto st_10; case 11: goto st_11;
      case 12: goto st_12; case 13: goto st_13; case 14: goto st_14; default: goto st_15;
    }
#define PATFFT_STATE(q, qn)                                                                          \
  st_##q:                                                                                            \
    if (q < NS) {                                                                                    \
      while (e < ne) {                                                                               \
        const float* rec = rb + e * RECW;                                                            \
        if (__float_as_int(rec[0]) != fg) break;                                                     \
        record_fma<NS, R>(acc, rec, sb[e * kThreads]);                                               \
        ++e;                                                                                         \
      }                                                                                              \
      if (e == ne) {                                                                                 \
        if (!last) {                                                                                 \
          fs = q;                                                                                    \
          goto chunk_end;                                                                            \
        }                                                                                            \
        if (fg >= c1) goto all_done;                                                                 \
      }                                                                                              \
      {                                                                                              \
        const bool store = tvalid && fg >= c0 && fg < c1;                                            \
        flush_slot<(q < NS ? q : 0), R, NS>(acc, base + (size_t)(store ? fg : 0) * T, row_stride,    \
                                            rows_valid, store);                                      \
      }                                                                                              \
      ++fg;                                                                                          \
      if (q + 1 >= NS) goto st_0;                                                                    \
      goto st_##qn;                                                                                  \
    }
    PATFFT_STATE(0, 1) PATFFT_STATE(1, 2) PATFFT_STATE(2, 3) PATFFT_STATE(3, 4)
    PATFFT_STATE(4, 5) PATFFT_STATE(5, 6) PATFFT_STATE(6, 7) PATFFT_STATE(7, 8)
    PATFFT_STATE(8, 9) PATFFT_STATE(9, 10) PATFFT_STATE(10, 11) PATFFT_STATE(11, 12)
    PATFFT_STATE(12, 13) PATFFT_STATE(13, 14) PATFFT_STATE(14, 15) PATFFT_STATE(15, 0)
#undef PATFFT_STATE
  chunk_end:
    __syncthreads();
  }
all_done:;
}

// ---------------------------------------------------------------------------
// Time-pair variant (default for 2-D sensor planes): R = 2 grid rows per
// group and TWO consecutive time samples per thread.  FFMA2 lanes are the
// time pair, the broadcast operand is the precomputed weight product
// wr[r] * wc[j], so one record costs 2K*R FFMA2 with no per-record FMUL and a
// single LDS.64 for the samples; the thinner row groups waste fewer FMAs on
// rows outside a sensor's window ((2K+1)/2K vs (2K+3)/2K for R = 4).
// Record layout (float words): [0] ws, [1] m, [2..3] pad, [4 + j*R + r]
// weight of ring slot j (column (ws + tap) mod NS = j) and group row r.
// ---------------------------------------------------------------------------
#ifndef PATFFT_SPREAD_TP_MINB
#define PATFFT_SPREAD_TP_MINB 5
#endif
#ifndef PATFFT_SPREAD_BULK
#define PATFFT_SPREAD_BULK 1
#endif
#ifndef PATFFT_SPREAD_TP_CHUNK
#define PATFFT_SPREAD_TP_CHUNK 16
#endif
constexpr int kChunkTP = PATFFT_SPREAD_TP_CHUNK;
constexpr int kTimeTP = 2 * kThreads;  // time samples per CTA

template <int NS, int R>
__device__ __forceinline__ void record_fma_tp(float2 (&acc)[NS][R], const float* __restrict__ rec, float2 s2) {
  const float4* wq = reinterpret_cast<const float4*>(rec + 4);
#pragma unroll
  for (int j4 = 0; j4 < (NS * R + 3) / 4; ++j4) {
    const float4 q = wq[j4];
    const float wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = j4 * 4 + u;
      if (idx < NS * R) {
        const int j = idx < NS * R ? idx / R : 0, r = idx < NS * R ? idx % R : 0;
        acc[j][r] = ffma2(s2, make_float2(wv[u], wv[u]), acc[j][r]);
      }
    }
  }
}

template <int Q, int R, int NS, bool TEVEN>
__device__ __forceinline__ void flush_slot_tp(float2 (&acc)[NS][R], float* __restrict__ colp, size_t row_stride,
                                              int rows_valid, bool store, bool t1valid) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (store && r < rows_valid) {
      float* d = colp + (size_t)r * row_stride;
      if (TEVEN) {
        *reinterpret_cast<float2*>(d) = acc[Q][r];
      } else {
        d[0] = acc[Q][r].x;
        if (t1valid) d[1] = acc[Q][r].y;
      }
    }
    acc[Q][r] = make_float2(0.f, 0.f);
  }
}

template <int K2, int R, int PIECE>
__global__ void __launch_bounds__(kThreads, PATFFT_SPREAD_TP_MINB) spread_tp_kernel(const SpreadParams p) {
  constexpr int NS = K2;
  constexpr int RECW = 4 + (NS * R + 3) / 4 * 4;
  constexpr int CH = kChunkTP;
  constexpr int PIECES = kTimeTP / PIECE;  // cp.async pieces per record
  constexpr int PER_THREAD = CH * PIECES / kThreads;
  constexpr bool TEVEN = PIECE >= 2;       // T even: aligned float2 samples and stores
  // T % 4 == 0: records and each record's sample row arrive as bulk (TMA)
  // copies issued by one warp and completing on mbarriers -- no per-thread
  // cp.async address work
  constexpr bool BULK = PIECE == 4 && PATFFT_SPREAD_BULK;
  constexpr int NRB = BULK ? 3 : 2;        // record buffers (bulk: two chunks ahead)
  static_assert(NS <= 16, "ring states are generated for up to 16 slots");
  static_assert((CH * PIECES) % kThreads == 0, "staging split");
  static_assert(CH <= 32, "one lane per record in the bulk issue");
  extern __shared__ float4 smem4[];
  float* rbuf = reinterpret_cast<float*>(smem4);  // [NRB][CH][RECW]
  float* sbuf = rbuf + NRB * CH * RECW;           // [2][CH][kTimeTP]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sbuf + 2 * CH * kTimeTP);  // [NRB] records, [2] samples

  const int4 bk = p.blk[blockIdx.x];
  const int grp = p.blk_grp[blockIdx.x];
  const int c0 = bk.z;
  const int c1 = bk.w;
  const int T = p.T;
  const int t0 = p.t_begin + blockIdx.y * kTimeTP;
  const int tid = threadIdx.x;
  const int t = t0 + 2 * tid;
  const bool tvalid = t < p.t_end;
  const bool t1valid = t + 1 < p.t_end;
  const int nrec = bk.y - bk.x;
  const int nchunks = (nrec + CH - 1) / CH;
  const int row0 = grp * R;
  const int rows_valid = min(R, p.nrows - row0);

  int mnext[PER_THREAD];  // sensor of each (record, piece) this thread stages
  auto load_m = [&](int c) {
#pragma unroll
    for (int i = 0; i < PER_THREAD; ++i) {
      const int flat = tid + i * kThreads;  // (record, piece) pair index within the chunk
      const int e = c * CH + flat / PIECES;
      mnext[i] = (e < nrec) ? __ldg(reinterpret_cast<const int*>(p.recs) + (size_t)(bk.x + e) * RECW + 1) : -1;
    }
  };
  auto stage = [&](int c, int b) {
    const int e0 = c * CH;
    const int ne = min(CH, nrec - e0);
    const float4* srcr = reinterpret_cast<const float4*>(p.recs + (size_t)(bk.x + e0) * RECW);
    float4* dstr = reinterpret_cast<float4*>(rbuf + b * CH * RECW);
    for (int i = tid; i < ne * RECW / 4; i += kThreads) cp_async16(dstr + i, srcr + i, 16);
    float* sb = sbuf + b * CH * kTimeTP;
#pragma unroll
    for (int i = 0; i < PER_THREAD; ++i) {
      const int flat = tid + i * kThreads;
      const int e = flat / PIECES, pc = flat % PIECES;
      const int m = mnext[i];
      if (m >= 0) {
        const int tp = t0 + pc * PIECE;
        const int nb = max(0, min(PIECE, p.t_end - tp)) * 4;
        float* dst = sb + e * kTimeTP + pc * PIECE;
        const float* src = p.samples + (size_t)m * T + (nb > 0 ? tp : 0);
        if (PIECE == 4) cp_async16(dst, src, nb);
        else if (PIECE == 2) cp_async8(dst, src, nb);
        else cp_async4(dst, src, nb);
      }
    }
    cp_commit();
  };

  float2 acc[NS][R];
#pragma unroll
  for (int j = 0; j < NS; ++j)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[j][r] = make_float2(0.f, 0.f);

  const size_t row_stride = (size_t)p.ncols * T;
  float* base = p.grid + (size_t)row0 * row_stride + (tvalid ? t : 0);
  int fg = (c0 - NS) >= 0 ? (c0 - NS) / NS * NS : -((NS - (c0 - NS) - 1) / NS) * NS;
  int fs = 0;

  const int nvalid = min(kTimeTP, p.t_end - t0);  // time samples of this block
  // bulk issue (warp 0): records of chunk cc into record buffer cc % NRB
  auto issue_recs = [&](int cc) {
    const int ne = min(CH, nrec - cc * CH);
    uint64_t* bar = mbar + (cc % NRB);
    mbar_expect_tx(bar, (unsigned)(ne * RECW * 4));
    bulk_g2s(rbuf + (cc % NRB) * CH * RECW, p.recs + (size_t)(bk.x + cc * CH) * RECW, (unsigned)(ne * RECW * 4), bar);
  };
  // samples of chunk cc (its records must have landed): lane e copies record e's row
  auto issue_smp = [&](int cc, int lane) {
    const int ne = min(CH, nrec - cc * CH);
    uint64_t* bar = mbar + NRB + (cc & 1);
    if (lane == 0) mbar_expect_tx(bar, (unsigned)(ne * nvalid * 4));
    __syncwarp();
    if (lane < ne) {
      const int m = __float_as_int(rbuf[((cc % NRB) * CH + lane) * RECW + 1]);
      bulk_g2s(sbuf + ((cc & 1) * CH + lane) * kTimeTP, p.samples + (size_t)m * T + t0, (unsigned)(nvalid * 4), bar);
    }
  };
  if constexpr (BULK) {
    if (tid == 0) {
      for (int i = 0; i < NRB + 2; ++i) mbar_init(mbar + i, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (tid < 32 && nchunks > 0) {
      if (tid == 0) {
        issue_recs(0);
        if (nchunks > 1) issue_recs(1);
      }
      mbar_wait(mbar + 0, 0);
      issue_smp(0, tid);
    }
  } else if (nchunks > 0) {
    load_m(0);
    stage(0, 0);
    load_m(1);
  }
  const int npass = max(nchunks, 1);
  for (int c = 0; c < npass; ++c) {
    const int b = c & 1;
    int ne = 0;
    if (c < nchunks) {
      if constexpr (BULK) {
        if (tid < 32) {
          if (tid == 0 && c + 2 < nchunks) issue_recs(c + 2);
          if (c + 1 < nchunks) {
            mbar_wait(mbar + (c + 1) % NRB, (unsigned)(((c + 1) / NRB) & 1));
            issue_smp(c + 1, tid);
          }
        }
        mbar_wait(mbar + c % NRB, (unsigned)((c / NRB) & 1));
        mbar_wait(mbar + NRB + b, (unsigned)((c >> 1) & 1));
      } else {
        if (c + 1 < nchunks) {
          stage(c + 1, b ^ 1);
          load_m(c + 2);
          cp_wait<1>();
        } else {
          cp_wait<0>();
        }
        __syncthreads();
      }
      ne = min(CH, nrec - c * CH);
    }
    const bool last = c + 1 >= npass;
    const float* rb = rbuf + (BULK ? c % NRB : b) * CH * RECW;
    const float* sb = sbuf + b * CH * kTimeTP + 2 * tid;
    int e = 0;
    switch (fs) {
      case 0: goto st_0;   case 1: goto st_1;   case 2: goto st_2;   case 3: goto st_3;
      case 4: goto st_4;   case 5: goto st_5;   case 6: goto st_6;   case 7: goto st_7;
      case 8: goto st_8;   case 9: goto st_9;   case 10: goto st_10; case 11: goto st_11;
      case 12: goto st_12; case 13: goto st_13; case 14: goto st_14; default: goto st_15;
    }
#define PATFFT_STATE_TP(q, qn)                                                                       \
  st_##q:                                                                                            \
    if (q < NS) {                                                                                    \
      while (e < ne) {                                                                               \
        const float* rec = rb + e * RECW;                                                            \
        if (__float_as_int(rec[0]) != fg) break;                                                     \
        float2 s2;                                                                                   \
        if (TEVEN) s2 = *reinterpret_cast<const float2*>(sb + e * kTimeTP);                          \
        else s2 = make_float2(sb[e * kTimeTP], sb[e * kTimeTP + 1]);                                 \
        record_fma_tp<NS, R>(acc, rec, s2);                                                          \
        ++e;                                                                                         \
      }                                                                                              \
      if (e == ne) {                                                                                 \
        if (!last) {                                                                                 \
          fs = q;                                                                                    \
          goto chunk_end;                                                                            \
        }                                                                                            \
        if (fg >= c1) goto all_done;                                                                 \
      }                                                                                              \
      {                                                                                              \
        const bool store = tvalid && fg >= c0 && fg < c1;                                            \
        flush_slot_tp<(q < NS ? q : 0), R, NS, TEVEN>(acc, base + (size_t)(store ? fg : 0) * T,      \
                                                      row_stride, rows_valid, store, t1valid);       \
      }                                                                                              \
      ++fg;                                                                                          \
      if (q + 1 >= NS) goto st_0;                                                                    \
      goto st_##qn;                                                                                  \
    }
    PATFFT_STATE_TP(0, 1) PATFFT_STATE_TP(1, 2) PATFFT_STATE_TP(2, 3) PATFFT_STATE_TP(3, 4)
    PATFFT_STATE_TP(4, 5) PATFFT_STATE_TP(5, 6) PATFFT_STATE_TP(6, 7) PATFFT_STATE_TP(7, 8)
    PATFFT_STATE_TP(8, 9) PATFFT_STATE_TP(9, 10) PATFFT_STATE_TP(10, 11) PATFFT_STATE_TP(11, 12)
    PATFFT_STATE_TP(12, 13) PATFFT_STATE_TP(13, 14) PATFFT_STATE_TP(14, 15) PATFFT_STATE_TP(15, 0)
#undef PATFFT_STATE_TP
  chunk_end:
    __syncthreads();
  }
all_done:;
}

template <int K2, int R>
cudaError_t go_tp(const SpreadParams& p, int nblk, cudaStream_t s) {
  constexpr int RECW = 4 + (K2 * R + 3) / 4 * 4;
  const size_t smem = sizeof(float) * (3 * kChunkTP * RECW + 2 * kChunkTP * kTimeTP) + 8 * sizeof(uint64_t);
  dim3 grid((unsigned)nblk, (unsigned)((p.t_end - p.t_begin + kTimeTP - 1) / kTimeTP));
  cudaError_t err;
  auto run = [&](auto k) {
    if ((err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return;
    k<<<grid, kThreads, smem, s>>>(p);
    err = cudaGetLastError();
  };
  if (p.T % 4 == 0) run(spread_tp_kernel<K2, R, 4>);
  else if (p.T % 2 == 0) run(spread_tp_kernel<K2, R, 2>);
  else run(spread_tp_kernel<K2, R, 1>);
  return err;
}

template <int K2, int R>
cudaError_t go(const SpreadParams& p, int nblk, cudaStream_t s) {
  constexpr int RECW = 8 + (K2 + 3) / 4 * 4;
  const size_t smem = sizeof(float) * 2 * kChunk * (RECW + kThreads);
  dim3 grid((unsigned)nblk, (unsigned)((p.t_end - p.t_begin + kThreads - 1) / kThreads));
  cudaError_t err;
  if (p.T % 4 == 0) {
    auto k = spread_kernel<K2, R, true>;
    if ((err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return err;
    k<<<grid, kThreads, smem, s>>>(p);
  } else {
    auto k = spread_kernel<K2, R, false>;
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
  (void)K2;
  if (n_lat == 1) return 1;
  if (forced == 1 || forced == 2 || forced == 4) return forced;
  return 2;
}
// R == 2: the time-pair kernel (set PATFFT_SPREAD_TP=0 for the one-sample
// kernel).  2-D sensor lines (R = 1) keep the one-sample kernel: their grids
// are small and need the finer time blocks for parallelism.
bool spread_time_pairs(int R) {
  static const bool on = [] {
    const char* e = std::getenv("PATFFT_SPREAD_TP");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on && R == 2;
}
int spread_ring(int K2) { return K2; }
int spread_ctas_per_sm(int R) { return spread_time_pairs(R) ? PATFFT_SPREAD_TP_MINB : PATFFT_SPREAD_MINB; }
int spread_record_words(int K2, int R) {
  return spread_time_pairs(R) ? 4 + (K2 * R + 3) / 4 * 4 : 8 + (K2 + 3) / 4 * 4;
}
int spread_time_chunks(int T, int R) {
  const int tb = spread_time_pairs(R) ? kTimeTP : kThreads;
  return (T + tb - 1) / tb;
}

cudaError_t launch_spread(const SpreadParams& p, int K2, int R, int nblk, cudaStream_t s) {
  if (p.tc_tiles) return launch_spread_tc(p, s);
  if (spread_time_pairs(R)) {
#define PATFFT_SPREAD_TPK(RR)                       \
    switch (K2) {                                   \
      case 2: return go_tp<2, RR>(p, nblk, s);      \
      case 4: return go_tp<4, RR>(p, nblk, s);      \
      case 6: return go_tp<6, RR>(p, nblk, s);      \
      case 8: return go_tp<8, RR>(p, nblk, s);      \
      case 10: return go_tp<10, RR>(p, nblk, s);    \
      case 12: return go_tp<12, RR>(p, nblk, s);    \
      case 14: return go_tp<14, RR>(p, nblk, s);    \
      case 16: return go_tp<16, RR>(p, nblk, s);    \
    }
    if (R == 2) {
      PATFFT_SPREAD_TPK(2)
    } else {
      PATFFT_SPREAD_TPK(1)
    }
#undef PATFFT_SPREAD_TPK
    return cudaErrorInvalidValue;
  }
#define PATFFT_SPREAD_K(RR)                         \
  switch (K2) {                                     \
    case 2: return go<2, RR>(p, nblk, s);           \
    case 4: return go<4, RR>(p, nblk, s);           \
    case 6: return go<6, RR>(p, nblk, s);           \
    case 8: return go<8, RR>(p, nblk, s);           \
    case 10: return go<10, RR>(p, nblk, s);         \
    case 12: return go<12, RR>(p, nblk, s);         \
    case 14: return go<14, RR>(p, nblk, s);         \
    case 16: return go<16, RR>(p, nblk, s);         \
  }
  if (R == 4) {
    PATFFT_SPREAD_K(4)
  } else if (R == 2) {
    PATFFT_SPREAD_K(2)
  } else if (R == 1) {
    PATFFT_SPREAD_K(1)
  }
#undef PATFFT_SPREAD_K
  return cudaErrorInvalidValue;
}

}  // namespace patfft
