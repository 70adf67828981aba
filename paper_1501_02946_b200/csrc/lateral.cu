// Lateral (sensor-plane) FFTs of the NEDNER pipeline, as tiled shared-memory
// transforms over chunks of consecutive time samples.  The time axis is the
// fastest in every array, so each tile row is one coalesced 128-256 B
// segment and the P transforms of a tile are interleaved (conflict-free).
//
// Forward (replaces nufft.py:406-415 -- oversampled FFT, centred crop,
// deapodisation -- plus the Nyquist-plane Hermitian part of recon.py:218-222):
//   colfft : real FFT along grid columns, two time samples packed per complex
//            transform, only the j1 in [0, N1/2] half that is needed is kept;
//   rowfft : complex FFT along grid rows, crop j0 in [-N0/2, N0/2], deapodise,
//            symmetrise the Nyquist planes -> gh (half spectrum in j1).
// Inverse (replaces the lateral part of recon.py:255 ifftn + fftshift + real):
//   inv_col: complex inverse FFT along j0 (in place);
//   inv_c2r: Hermitian-completed inverse FFT along j1, two time samples packed
//            per transform -> real image rows.
#include <cuda_runtime.h>

#include <cstdlib>

#include "fft_smem.cuh"
#include "patfft_internal.h"

namespace patfft {
namespace {

using fft::TileAddr;

#ifndef PATFFT_C2R_LOADED
#define PATFFT_C2R_LOADED 1
#endif
#ifndef PATFFT_LAT_FUSED
#define PATFFT_LAT_FUSED 1  // colfft/rowfft: last FFT pass evaluated inside the crop/unpack epilogue
#endif
#ifndef PATFFT_LAT_FUSED_MAXR
#define PATFFT_LAT_FUSED_MAXR 1  // largest log2 radix of a last pass that is folded into the colfft unpack
#endif
#ifndef PATFFT_LAT_ROWPTR
#define PATFFT_LAT_ROWPTR 1  // colfft/rowfft first pass: one base pointer + running row offset per item
#endif
#ifndef PATFFT_ROW_FUSED
#define PATFFT_ROW_FUSED 0  // measured slower for rowfft (half the outputs are cropped away anyway)
#endif
#ifndef PATFFT_INVCOL_STORED
#define PATFFT_INVCOL_STORED 1
#endif

// launch bounds (max threads, min CTAs per SM) per kernel; 512 threads is the
// largest tile (P = 16 transforms of 512 points)
#ifndef PATFFT_LB_COL_T
#define PATFFT_LB_COL_T 512
#endif
#ifndef PATFFT_LB_COL_B
#define PATFFT_LB_COL_B 2
#endif
#ifndef PATFFT_LB_ROW_T
#define PATFFT_LB_ROW_T 512
#endif
#ifndef PATFFT_LB_ROW_B
#define PATFFT_LB_ROW_B 2
#endif
#ifndef PATFFT_LB_INV_MINB256
#define PATFFT_LB_INV_MINB256 5  // inverse kernels with <= 256 threads: 5 CTAs/SM (48 regs); measured 4 / 6 slower
#endif

// Grid order of the tiled lateral kernels: 1 = time tiles fastest (CTAs
// launched together read neighbouring time segments of the same rows, i.e.
// the same DRAM pages), 0 = rows / columns fastest.
#ifndef PATFFT_LAT_TFAST
#define PATFFT_LAT_TFAST 1
#endif
__device__ __forceinline__ int lat_line() { return PATFFT_LAT_TFAST ? blockIdx.y : blockIdx.x; }
__device__ __forceinline__ int lat_ttile() { return PATFFT_LAT_TFAST ? blockIdx.x : blockIdx.y; }

int plog_for(int len);

constexpr int nth_for(int L, int PLOG) {
  return ((L >= 4 ? (1 << (L - 4)) : 1) << PLOG) < 64 ? 64
         : (((L >= 4 ? (1 << (L - 4)) : 1) << PLOG) > 512 ? 512 : ((L >= 4 ? (1 << (L - 4)) : 1) << PLOG));
}
constexpr int inv_lb_threads(int PLOG, int LC) { return LC > 0 ? nth_for(LC, PLOG) : 512; }
constexpr int inv_lb_minb(int PLOG, int LC) { return inv_lb_threads(PLOG, LC) <= 256 ? PATFFT_LB_INV_MINB256 : 2; }

struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// One column-FFT tile: grid row u0, packed time pairs [t0, t0 + 2P) -> Y (time
// stride ys, time yt0 at offset 0).  `before_store` runs (all threads) between
// the transform and the first write to Y.
// LC > 0: compile-time transform length 2^LC (launched with nth_for(LC, PLOG) threads)
#ifndef PATFFT_FUSED_NOGRID
#define PATFFT_FUSED_NOGRID 0  // diagnosis: the fused kernel's column tiles transform zeros instead of reading the grid
#endif
#ifndef PATFFT_FUSED_GRIDLD
#define PATFFT_FUSED_GRIDLD 3  // fused kernel: grid row loads (fft::RowsLd mode)
#endif
#ifndef PATFFT_FUSED_FENCEALL
#define PATFFT_FUSED_FENCEALL 0
#endif
#ifndef PATFFT_FUSED_GHCS
#define PATFFT_FUSED_GHCS 1    // fused kernel: gh stored with the streaming (evict-first) hint
#endif
template <int PLOG, int LC, int GMODE = 1, class Hook>
__device__ __forceinline__ void colfft_body(const LateralParams& p, float2* __restrict__ sm, int u0, int t0,
                                            float2* __restrict__ Y, int ys, int yt0, Hook before_store) {
  constexpr int P = 1 << PLOG;
  const int tid = threadIdx.x;
  const int nth = LC > 0 ? nth_for(LC, PLOG) : (int)blockDim.x;
  const int T = p.T, n = p.ncols;
  const TileAddr ad{PLOG};
  const float* __restrict__ src = p.grid + (size_t)u0 * n * T;
  auto ld = [&](int row, int q) {
    const int t = t0 + 2 * q;
    return (t < p.t_end) ? __ldcs(reinterpret_cast<const float2*>(src + (size_t)row * T + t)) : make_float2(0.f, 0.f);
  };
  constexpr int LLAST = LC > 0 ? fft::LastPassLogh<(LC > 0 ? LC : 1), 4, false>::value : 0;
  // the last pass is folded into the unpack only when it is short: a radix-2^r fold costs 2^r
  // complex MACs for each of the 2 ny outputs kept, a radix-16 one three times the pass it replaces
  // (cfg3's 256-point columns: colfft 0.089 -> see DESIGN.md 4)
  constexpr bool FUSED = PATFFT_LAT_FUSED && LC > 0 && LLAST > 0 && (LC - LLAST) <= PATFFT_LAT_FUSED_MAXR;
  if constexpr (LC > 0 && PATFFT_LAT_ROWPTR) {
    fft::fft_ct_loaded<false, LC, 4, false, PLOG, nth_for(LC, PLOG), FUSED>(
        sm, p.tw, tid, fft::TileC<PLOG>(), fft::rows_ld<GMODE>([&](int row, int q) -> const float2* {
          const int t = t0 + 2 * q;
          if (PATFFT_FUSED_NOGRID && GMODE != 1) return nullptr;
          return t < p.t_end ? reinterpret_cast<const float2*>(src + (size_t)row * T + t) : nullptr;
        }, (size_t)(T / 2)));
  } else if constexpr (LC > 0) {
    fft::fft_ct_loaded<false, LC, 4, false, PLOG, nth_for(LC, PLOG), FUSED>(sm, p.tw, tid, fft::TileC<PLOG>(), ld);
  } else {
    fft::staged_copy<8, float2>(
        n * P, tid, nth, [&](int i) { return ld(i >> PLOG, i & (P - 1)); },
        [&](int i, float2 v) { sm[ad(fft::brev(i >> PLOG, p.lcols), i & (P - 1))] = v; });
    __syncthreads();
    fft::fft_inplace<false, 4, false>(sm, p.lcols, PLOG, p.tw, tid, nth, ad);
  }
  // spectrum value at column frequency k (the last pass folded in when FUSED)
  auto zat = [&](int k, int q) {
    if constexpr (FUSED) return fft::last_pass_output<false, (LC > 0 ? LC : 1), (LC > 0 ? LC : 1) - LLAST>(
        sm, p.tw, fft::TileC<PLOG>(), k, q);
    else return sm[ad(k, q)];
  };
  before_store();
  if (p.cplx) {
    // complex values (NedPlan): the packed pair IS one complex sample; keep
    // the full cropped spectrum j1 in [-N1/2, N1/2) in wrapped order
    const int Tc = T / 2;
    float2* __restrict__ dst = Y + (size_t)u0 * p.ny * Tc;
    for (int i = tid; i < p.ny * P; i += nth) {
      const int k = i >> PLOG, q = i & (P - 1);
      const int t = t0 + 2 * q;
      if (t >= p.t_end) continue;
      const int j1 = k < p.N1 / 2 ? k : k - p.N1;
      dst[(size_t)k * Tc + t / 2] = zat(j1 & (n - 1), q);
    }
    return;
  }
  // Y: [nrows][ny][ys] holding times [yt0, yt0 + ys) (the whole record, or a
  // time chunk that stays L2-resident until rowfft consumes it)
  float2* __restrict__ dst = Y + (size_t)u0 * p.ny * ys;
  // each thread keeps one packed time pair q (nth is a multiple of P) and walks the bins k
  const int q = tid & (P - 1);
  const int t = t0 + 2 * q;
  if (t >= p.t_end) return;
  const int kstep = nth >> PLOG;
  const size_t ostep = (size_t)kstep * ys;
  float2* __restrict__ o = dst + (size_t)(tid >> PLOG) * ys + (t - yt0);
  for (int k = tid >> PLOG; k < p.ny; k += kstep, o += ostep) {
    const float2 zk = zat(k, q);
    const float2 zm = fft::conjf2(zat((n - k) & (n - 1), q));
    const float2 d = fft::csub(zk, zm);
    *reinterpret_cast<float4*>(o) =
        make_float4(0.5f * (zk.x + zm.x), 0.5f * (zk.y + zm.y), 0.5f * d.y, -0.5f * d.x);
  }
}

template <int PLOG, int LC>
__global__ void __launch_bounds__(PATFFT_LB_COL_T, PATFFT_LB_COL_B) colfft_kernel(const LateralParams p) {
  extern __shared__ float2 sm[];
  colfft_body<PLOG, LC>(p, sm, lat_line(), p.t_begin + lat_ttile() * (2 << PLOG), p.Y, p.ys, p.yt0, NoHook());
}

// One row-FFT tile: half-spectrum column j1, time samples [t0, t0 + P) of Y
// (time stride ys, time yt0 at offset 0) -> gh.  YMODE: how Y is loaded
// (fft::RowsLd; 2 when other CTAs of the same launch wrote it).
template <int PLOG, int LC, int YMODE>
__device__ __forceinline__ void rowfft_body(const LateralParams& p, float2* __restrict__ sm, int j1, int t0,
                                            const float2* __restrict__ Y, int ys, int yt0) {
  constexpr int P = 1 << PLOG;
  const int tid = threadIdx.x;
  const int nth = LC > 0 ? nth_for(LC, PLOG) : (int)blockDim.x;
  const int T = p.T, nr = p.nrows;
  const TileAddr ad{PLOG};
  const float2* __restrict__ yb = Y - yt0;
  auto ld = [&](int row, int q) {
    const int t = t0 + q;
    return (t < p.t_end) ? __ldcs(yb + ((size_t)row * p.ny + j1) * ys + t) : make_float2(0.f, 0.f);
  };
  constexpr int LLAST = LC > 0 ? fft::LastPassLogh<(LC > 0 ? LC : 1), 4, false>::value : 0;
  constexpr bool FUSED = PATFFT_ROW_FUSED && LC > 0 && LLAST > 0;
  if constexpr (LC > 0 && PATFFT_LAT_ROWPTR) {
    fft::fft_ct_loaded<false, LC, 4, false, PLOG, nth_for(LC, PLOG), FUSED>(
        sm, p.tw, tid, fft::TileC<PLOG>(), fft::rows_ld<YMODE>([&](int row, int q) -> const float2* {
          const int t = t0 + q;
          return t < p.t_end ? yb + ((size_t)row * p.ny + j1) * ys + t : nullptr;
        }, (size_t)p.ny * ys));
  } else if constexpr (LC > 0) {
    fft::fft_ct_loaded<false, LC, 4, false, PLOG, nth_for(LC, PLOG), FUSED>(sm, p.tw, tid, fft::TileC<PLOG>(), ld);
  } else {
    fft::staged_copy<8, float2>(
        nr * P, tid, nth, [&](int i) { return ld(i >> PLOG, i & (P - 1)); },
        [&](int i, float2 v) { sm[ad(fft::brev(i >> PLOG, p.lrows), i & (P - 1))] = v; });
    __syncthreads();
    fft::fft_inplace<false, 4, false>(sm, p.lrows, PLOG, p.tw, tid, nth, ad);
  }
  auto zat = [&](int k, int q) {
    if constexpr (FUSED) return fft::last_pass_output<false, (LC > 0 ? LC : 1), (LC > 0 ? LC : 1) - LLAST>(
        sm, p.tw, fft::TileC<PLOG>(), k, q);
    else return sm[ad(k, q)];
  };
  const int N0 = p.N0, mask = nr - 1;
  const float dp1 = p.dp1[j1];
  if (p.cplx) {
    // NedPlan: full spectrum, centred-grid sign (-1)^(j0+j1), deapodise,
    // centred or wrapped output order (nufft.py:406-417)
    const int j1s = j1 < p.N1 / 2 ? j1 : j1 - p.N1;
    for (int i = tid; i < N0 * P; i += nth) {
      const int j0w = i >> PLOG, q = i & (P - 1);
      const int t = t0 + q;
      if (t >= p.t_end) continue;
      const int a = (N0 > 1) ? (j0w < N0 / 2 ? j0w : j0w - N0) : 0;
      const float sg = ((a + j1s) & 1) ? -1.f : 1.f;
      const float2 v = fft::cscale(zat(a & mask, q), sg * p.dp0[j0w] * dp1);
      const size_t o = p.centered ? (size_t)(a + N0 / 2) * p.ny + (j1s + p.N1 / 2) : (size_t)j0w * p.ny + j1;
      p.gh[o * T + t] = v;
    }
    return;
  }
  const bool nyq1 = (j1 == p.N1 / 2);
  // each thread keeps one time sample q (nth is a multiple of P) and walks the rows j0w
  const int q = tid & (P - 1);
  const int t = t0 + q;
  if (t >= p.t_end) return;
  // gh: [N0][ny][gs] holding times [gt0, gt0 + gs) (the whole slice, or the
  // time chunk one pipelined exchange of the sharded path sends)
  const int kstep = nth >> PLOG;
  const size_t gstep = (size_t)kstep * p.ny * p.gs;
  float2* __restrict__ gp = p.gh + ((size_t)(tid >> PLOG) * p.ny + j1) * p.gs + (t - p.gt0);
  for (int j0w = tid >> PLOG; j0w < N0; j0w += kstep, gp += gstep) {
    const int a = (N0 > 1) ? (j0w < N0 / 2 ? j0w : j0w - N0) : 0;
    const bool nyq0 = (N0 > 1) && (a == -(N0 / 2));
    float2 v;
    if (nyq1) {  // stored j1 = N1/2 is signed -N1/2: X(a,-N1/2) = conj X(-a,+N1/2)
      const float2 v1 = fft::conjf2(zat((-a) & mask, q));
      const float2 v2 = zat((nyq0 ? -a : a) & mask, q);
      v = fft::cscale(fft::cadd(v1, v2), 0.5f);
    } else if (nyq0) {
      v = fft::cscale(fft::cadd(zat(a & mask, q), zat((-a) & mask, q)), 0.5f);
    } else {
      v = zat(a & mask, q);
    }
    const float2 g = fft::cscale(v, __ldg(&p.dp0[j0w]) * dp1);
    if (YMODE == 2 && PATFFT_FUSED_GHCS) __stcs(gp, g);
    else *gp = g;
  }
}

template <int PLOG, int LC>
__global__ void __launch_bounds__(PATFFT_LB_ROW_T, PATFFT_LB_ROW_B) rowfft_kernel(const LateralParams p) {
  extern __shared__ float2 sm[];
  rowfft_body<PLOG, LC, 1>(p, sm, lat_line(), p.t_begin + lat_ttile() * (1 << PLOG), p.Y, p.ys, p.yt0);
}

// ---------------------------------------------------------------------------
// Column and row FFTs in ONE launch, so the column-transformed half spectrum Y
// never travels to HBM: the time axis is cut into chunks of 2P samples (one
// column-FFT tile); CTAs are laid out in rounds
//   round r = [column tiles of chunk r (nrows CTAs)] [row tiles of chunk r - 1 (2 ny CTAs)]
// and Y is a ring of kYSlots chunk buffers (nrows x ny x 2P each, 17 MB at
// cfg4) that stays L2-resident.  A row tile waits until all column tiles of
// its chunk have signalled; a column tile waits, just before it stores, until
// the row tiles that read its ring slot kYSlots chunks earlier have finished.
// Both dependencies point to CTAs with lower block indices -- dispatched
// earlier, hence resident or complete -- so the waits cannot deadlock.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void lat_wait(const int* flag, int need) {
  if (threadIdx.x == 0) {
    int v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if (v >= need) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
}
// (release by one thread after the CTA barrier: cumulative over the other threads' stores)
__device__ __forceinline__ void lat_signal(int* flag) {
#if PATFFT_FUSED_FENCEALL
  __threadfence();
#endif
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(flag) : "memory");
}

template <int PLOG, int L>
__global__ void __launch_bounds__(PATFFT_LB_COL_T, PATFFT_LB_COL_B) latfused_kernel(const LateralParams p) {
  extern __shared__ float2 sm[];
  constexpr int P = 1 << PLOG;
  const int nc = p.nrows, nr = 2 * p.ny, per = nc + nr;
  const int round = blockIdx.x / per, idx = blockIdx.x - round * per;
  const size_t slot = (size_t)p.nrows * p.ny * (2 * P);
  if (idx < nc) {
    const int c = round;
    if (c >= p.f_chunks) return;
    const int t0 = p.t_begin + c * 2 * P;
    colfft_body<PLOG, L, PATFFT_FUSED_GRIDLD>(p, sm, idx, t0, p.Y + (size_t)(c % p.f_slots) * slot, 2 * P, t0, [&]() {
      if (c >= p.f_slots) lat_wait(p.f_flags + p.f_chunks + (c - p.f_slots), nr);
    });
    lat_signal(p.f_flags + c);
  } else {
    const int c = round - 1;
    if (c < 0) return;
    const int tc = p.t_begin + c * 2 * P, i = idx - nc;
    lat_wait(p.f_flags + c, nc);
    rowfft_body<PLOG, L, 2>(p, sm, i >> 1, tc + (i & 1) * P, p.Y + (size_t)(c % p.f_slots) * slot, 2 * P, tc);
    lat_signal(p.f_flags + p.f_chunks + c);
  }
}

template <int PLOG, int LC>
__global__ void __launch_bounds__(inv_lb_threads(PLOG, LC), inv_lb_minb(PLOG, LC)) inv_col_kernel(const LateralParams p) {
  extern __shared__ float2 sm[];
  constexpr int P = 1 << PLOG;
  const int j1 = lat_line();
  const int t0 = lat_ttile() * P;
  const int tid = threadIdx.x;
  const int nth = LC > 0 ? nth_for(LC, PLOG) : (int)blockDim.x;
  const int T = p.Tu, n = p.N0u;
  const TileAddr ad{PLOG};
  float2* __restrict__ z = p.z;
  auto ld = [&](int row, int q) {
    const int t = t0 + q;
    return (t < T) ? z[((size_t)row * p.N1uh + j1) * T + t] : make_float2(0.f, 0.f);
  };
  auto st = [&](int row, int q, float2 v) {
    const int t = t0 + q;
    if (t < T) z[((size_t)row * p.N1uh + j1) * T + t] = v;
  };
  if constexpr (LC > 4 && PATFFT_INVCOL_STORED && PATFFT_LAT_ROWPTR) {
    const size_t rs = (size_t)p.N1uh * T;
    auto rp = [&](int row, int q) -> float2* { return t0 + q < T ? z + (size_t)row * rs + j1 * (size_t)T + t0 + q : nullptr; };
    fft::fft_ct_loaded_stored<true, LC, 4, false, PLOG, nth_for(LC, PLOG)>(
        sm, p.tw, tid, fft::TileC<PLOG>(),
        fft::rows_ld<false>([&](int row, int q) -> const float2* { return rp(row, q); }, rs), fft::rows_st(rp, rs));
  } else if constexpr (LC > 4 && PATFFT_INVCOL_STORED) {
    fft::fft_ct_loaded_stored<true, LC, 4, false, PLOG, nth_for(LC, PLOG)>(sm, p.tw, tid, fft::TileC<PLOG>(), ld, st);
  } else if constexpr (LC > 0) {
    fft::fft_ct_loaded<true, LC, 4, false, PLOG, nth_for(LC, PLOG)>(sm, p.tw, tid, fft::TileC<PLOG>(), ld);
    for (int i = tid; i < n * P; i += nth) st(i >> PLOG, i & (P - 1), sm[ad(i >> PLOG, i & (P - 1))]);
  } else {
    fft::staged_copy<8, float2>(
        n * P, tid, nth, [&](int i) { return ld(i >> PLOG, i & (P - 1)); },
        [&](int i, float2 v) { sm[ad(fft::brev(i >> PLOG, p.l0u), i & (P - 1))] = v; });
    __syncthreads();
    if constexpr (LC > 0) fft::fft_ct<true, LC, 4, false, PLOG, nth_for(LC, PLOG)>(sm, p.tw, tid, fft::TileC<PLOG>());
    else fft::fft_inplace<true, 4, false>(sm, p.l0u, PLOG, p.tw, tid, nth, ad);
    for (int i = tid; i < n * P; i += nth) st(i >> PLOG, i & (P - 1), sm[ad(i >> PLOG, i & (P - 1))]);
  }
}

template <int PLOG, int LC>
__global__ void __launch_bounds__(inv_lb_threads(PLOG, LC), inv_lb_minb(PLOG, LC)) inv_c2r_kernel(const LateralParams p) {
  extern __shared__ float2 sm[];
  constexpr int P = 1 << PLOG;
  const int n0 = lat_line();
  const int t0 = lat_ttile() * 2 * P;
  const int tid = threadIdx.x;
  const int nth = LC > 0 ? nth_for(LC, PLOG) : (int)blockDim.x;
  const int T = p.Tu, n = p.N1u, half = n / 2;
  const TileAddr ad{PLOG};
  const float2* __restrict__ z = p.z + (size_t)n0 * p.N1uh * T;
  float* __restrict__ out = p.out + (size_t)n0 * n * T;
  auto st = [&](int row, int q, float2 v) {
    const int t = t0 + 2 * q;
    if (t < T) *reinterpret_cast<float2*>(out + (size_t)row * T + t) = v;
  };
  if constexpr (LC > 4 && PATFFT_C2R_LOADED) {
    // element r of the packed transform Z = Xa + i Xb (Xa, Xb: the half
    // spectra of time samples t, t+1): r <= n/2 from bin r, else from the
    // conjugate of bin n - r (Z[n-k] = conj(Xa) + i conj(Xb)); each bin is
    // read twice, the second time from L1
    auto ld = [&](int r, int q) {
      const int t = t0 + 2 * q;
      const bool lo = r <= half;
      const int k = lo ? r : n - r;
      // unconditional (clamped) load so the compiler issues all of an item's loads back to back
#if PATFFT_INV_L2PF
      float4 v;
      asm volatile("ld.global.nc.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "l"(reinterpret_cast<const float4*>(z + (size_t)k * T + min(t, T - 2))));
#else
      float4 v = __ldg(reinterpret_cast<const float4*>(z + (size_t)k * T + min(t, T - 2)));
#endif
      if (k == 0 || k == half) {  // C2R semantics: self-conjugate bins are real
        v.y = 0.f;
        v.w = 0.f;
      }
      const float2 o = lo ? make_float2(v.x - v.w, v.y + v.z) : make_float2(v.x + v.w, v.z - v.y);
      return t < T ? o : make_float2(0.f, 0.f);
    };
    if constexpr (PATFFT_LAT_ROWPTR) {
      fft::fft_ct_loaded_stored<true, LC, 4, false, PLOG, nth_for(LC, PLOG)>(
          sm, p.tw, tid, fft::TileC<PLOG>(), ld, fft::rows_st([&](int row, int q) -> float2* {
            const int t = t0 + 2 * q;
            return t < T ? reinterpret_cast<float2*>(out + (size_t)row * T + t) : nullptr;
          }, (size_t)(T / 2)));
    } else {
      fft::fft_ct_loaded_stored<true, LC, 4, false, PLOG, nth_for(LC, PLOG)>(sm, p.tw, tid, fft::TileC<PLOG>(), ld, st);
    }
    return;
  }
  fft::staged_copy<8, float4>(
      (half + 1) * P, tid, nth,
      [&](int i) {
        const int k = i >> PLOG, t = t0 + 2 * (i & (P - 1));
        return (t < T) ? __ldcs(reinterpret_cast<const float4*>(z + (size_t)k * T + t))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      },
      [&](int i, float4 v) {
        const int k = i >> PLOG, q = i & (P - 1);
        if (k == 0 || k == half) {  // C2R semantics: self-conjugate bins are real
          v.y = 0.f;
          v.w = 0.f;
        }
        // Z = Xa + i Xb ; Z[n-k] = conj(Xa) + i conj(Xb)
        sm[ad(fft::brev(k, p.l1u), q)] = make_float2(v.x - v.w, v.y + v.z);
        if (k != 0 && k != half) sm[ad(fft::brev(n - k, p.l1u), q)] = make_float2(v.x + v.w, v.z - v.y);
      });
  __syncthreads();
  if constexpr (LC > 0) fft::fft_ct<true, LC, 4, false, PLOG, nth_for(LC, PLOG)>(sm, p.tw, tid, fft::TileC<PLOG>());
  else fft::fft_inplace<true, 4, false>(sm, p.l1u, PLOG, p.tw, tid, nth, ad);
  for (int i = tid; i < n * P; i += nth) st(i >> PLOG, i & (P - 1), sm[ad(i >> PLOG, i & (P - 1))]);
}

// ---------------------------------------------------------------------------
// Lateral inverse in ONE launch.  inv_col and inv_c2r are bound by HBM (80-85% of the peak), and
// between them the half spectrum z makes a full round trip (0.27 GB written in place, 0.27 GB read
// again at cfg4).  Here the column-inverse tiles write their output into a ring of kSlots chunk
// buffers of 32 depth samples ([N0u][N1uh][32] each, 8.5 MB at cfg4) that stays in L2, and the C2R
// tiles of the same launch read it from there: z is read once, the image written once.  Tiles are
// laid out in rounds [column tiles of chunk r][C2R tiles of chunk r - 1] with the release / acquire
// progress counters of latfused_kernel (dependencies only on lower block indices).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 ld_l2_v4(const float4* a) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a));
  return v;
}

template <int PLOG, int LC>
__global__ void __launch_bounds__(inv_lb_threads(PLOG, LC), inv_lb_minb(PLOG, LC)) invfused_kernel(const LateralParams p) {
  extern __shared__ float2 sm[];
  constexpr int P = 1 << PLOG, CH = 2 * P, NTH = nth_for(LC, PLOG);
  const int tid = threadIdx.x;
  const int T = p.Tu, n = 1 << LC, half = n / 2;
  const int nc = 2 * p.N1uh, nr = p.N0u, per = nc + nr;
  const int round = blockIdx.x / per, idx = blockIdx.x - round * per;
  const size_t slot = (size_t)p.N0u * p.N1uh * CH, rr = (size_t)p.N1uh * CH;
  if (idx < nc) {  // column inverse (along j0) of half-spectrum column j1, 16 depth samples
    const int c = round;
    if (c >= p.f_chunks) return;
    const int j1 = idx >> 1, tl = (idx & 1) * P, t0 = c * CH + tl;
    if (c >= p.f_slots) lat_wait(p.f_flags + p.f_chunks + (c - p.f_slots), nr);
    float2* __restrict__ ring = p.inv_ring + (size_t)(c % p.f_slots) * slot;
    const size_t rs = (size_t)p.N1uh * T;
    fft::fft_ct_loaded_stored<true, LC, 4, false, PLOG, NTH>(
        sm, p.tw, tid, fft::TileC<PLOG>(),
        fft::rows_ld<1>([&](int row, int q) -> const float2* { return p.z + (size_t)row * rs + (size_t)j1 * T + t0 + q; },
                        rs),
        fft::rows_st([&](int row, int q) -> float2* { return ring + (size_t)row * rr + (size_t)j1 * CH + tl + q; }, rr));
    lat_signal(p.f_flags + c);
  } else {  // C2R (along j1) of image row n0, 32 depth samples as 16 packed pairs
    const int c = round - p.f_lead;  // f_lead rounds behind the column tiles it consumes
    if (c < 0) return;
    const int n0 = idx - nc, t0 = c * CH;
    lat_wait(p.f_flags + c, nc);
    const float2* __restrict__ zr = p.inv_ring + (size_t)(c % p.f_slots) * slot + (size_t)n0 * rr;
    float* __restrict__ out = p.out + (size_t)n0 * n * T;
    auto ld = [&](int r, int q) {
      const bool lo = r <= half;
      const int k = lo ? r : n - r;
      float4 v = ld_l2_v4(reinterpret_cast<const float4*>(zr + (size_t)k * CH + 2 * q));
      if (k == 0 || k == half) {  // C2R semantics: self-conjugate bins are real
        v.y = 0.f;
        v.w = 0.f;
      }
      return lo ? make_float2(v.x - v.w, v.y + v.z) : make_float2(v.x + v.w, v.z - v.y);
    };
    fft::fft_ct_loaded_stored<true, LC, 4, false, PLOG, NTH>(
        sm, p.tw, tid, fft::TileC<PLOG>(), ld, fft::rows_st([&](int row, int q) -> float2* {
          return reinterpret_cast<float2*>(out + (size_t)row * T + t0 + 2 * q);
        }, (size_t)(T / 2)));
    lat_signal(p.f_flags + p.f_chunks + c);
  }
}

// Ring slots; 0 (default) = the two-kernel form.  Measured at cfg4: 0.170 ms (6 slots, lead 3)
// against 0.192 ms -- the launch is held back by its tile dependencies rather than sped up by the
// halved HBM traffic -- and slower at cfg3 (0.029-0.056 vs 0.028 ms), so it stays an opt-in.
int inv_fused_slots() {
  const char* e = std::getenv("PATFFT_INV_FUSED_SLOTS");
  return e ? std::max(0, std::min(16, std::atoi(e))) : 0;
}

int inv_fused_lead() {  // rounds between a chunk's column tiles and its C2R tiles
  const char* e = std::getenv("PATFFT_INV_FUSED_LEAD");
  return e ? std::max(1, std::atoi(e)) : 3;
}

bool inverse_fused_supported(const LateralParams& p) {
  return inv_fused_slots() > 0 && p.inv_ring && p.inv_flags && p.N0u == p.N1u &&
         (p.N0u == 64 || p.N0u == 128 || p.N0u == 256 || p.N0u == 512) && plog_for(p.N0u) == 4 && p.Tu % 32 == 0 &&
         p.Tu / 32 >= 2 && p.Tu <= p.inv_capacity;
}

int tile_bytes() {
  static int b = [] {
    const char* e = std::getenv("PATFFT_TILE_KB");
    const int kb = e ? std::atoi(e) : 64;
    return (kb >= 8 && kb <= 128 ? kb : 64) * 1024;
  }();
  return b;
}

int plog_for(int len) {
  // P transforms per tile, tile <= tile_bytes() of float2
  int plog = 4;
  while (plog > 0 && ((size_t)len << plog) * sizeof(float2) > (size_t)tile_bytes()) --plog;
  return plog;
}

int threads_for(int len, int plog) {
  int items = (len >> 4 ? len >> 4 : 1) << plog;  // radix-16 passes
  if (items < 64) items = 64;
  if (items > 512) items = 512;
  return items;
}

#define PATFFT_DEF_LAUNCH(NAME)                                                                        \
  cudaError_t launch_##NAME(const LateralParams& p, int len, dim3 grid_xy, int tpack, cudaStream_t s) { \
    const int plog = plog_for(len);                                                                    \
    const size_t smem = ((size_t)len << plog) * sizeof(float2);                                        \
    const int thr = threads_for(len, plog);                                                            \
    const unsigned ntt = (unsigned)((grid_xy.y + (tpack << plog) - 1) / (tpack << plog));               \
    const dim3 grid = PATFFT_LAT_TFAST ? dim3(ntt, grid_xy.x) : dim3(grid_xy.x, ntt);                  \
    cudaError_t err = cudaSuccess;                                                                     \
    auto run = [&](auto k) {                                                                           \
      err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);           \
      if (err == cudaSuccess) {                                                                        \
        k<<<grid, thr, smem, s>>>(p);                                                                  \
        err = cudaGetLastError();                                                                      \
      }                                                                                                \
    };                                                                                                 \
    if (plog == 4) {                                                                                   \
      switch (len) {                                                                                   \
        case 64: run(NAME##_kernel<4, 6>); return err;                                                 \
        case 128: run(NAME##_kernel<4, 7>); return err;                                                \
        case 256: run(NAME##_kernel<4, 8>); return err;                                                \
        case 512: run(NAME##_kernel<4, 9>); return err;                                                \
      }                                                                                                \
    }                                                                                                  \
    if (plog == 3) {                                                                                   \
      switch (len) {                                                                                   \
        case 256: run(NAME##_kernel<3, 8>); return err;                                                \
        case 512: run(NAME##_kernel<3, 9>); return err;                                                \
        case 1024: run(NAME##_kernel<3, 10>); return err;                                              \
      }                                                                                                \
    }                                                                                                  \
    if (plog == 2 && len == 2048) { run(NAME##_kernel<2, 11>); return err; }                           \
    switch (plog) {                                                                                    \
      case 4: run(NAME##_kernel<4, 0>); break;                                                         \
      case 3: run(NAME##_kernel<3, 0>); break;                                                         \
      case 2: run(NAME##_kernel<2, 0>); break;                                                         \
      case 1: run(NAME##_kernel<1, 0>); break;                                                         \
      default: run(NAME##_kernel<0, 0>); break;                                                        \
    }                                                                                                  \
    return err;                                                                                        \
  }

}  // namespace

namespace {
PATFFT_DEF_LAUNCH(colfft)
PATFFT_DEF_LAUNCH(rowfft)
PATFFT_DEF_LAUNCH(inv_col)
PATFFT_DEF_LAUNCH(inv_c2r)
}  // namespace

cudaError_t launch_lateral_col(const LateralParams& p, cudaStream_t s) {
  return launch_colfft(p, p.ncols, dim3((unsigned)p.nrows, (unsigned)(p.t_end - p.t_begin)), 2, s);
}

cudaError_t launch_lateral_row(const LateralParams& p, cudaStream_t s) {
  return launch_rowfft(p, p.nrows, dim3((unsigned)p.ny, (unsigned)(p.t_end - p.t_begin)), 1, s);
}

// Column + row FFTs of [t_begin, t_end): the two kernels with the whole Y in
// between, or (opt-in, PATFFT_LAT_FUSED_SLOTS) the single-launch form
// (latfused_kernel) for square oversampled planes of 128 / 256 / 512 points a side.
namespace {
// Ring slots of the single-launch form; 0 (default) = the two-kernel form.  Measured at cfg4
// (DESIGN.md 4): the single launch keeps Y in L2 (DRAM traffic of the lateral stage 2.37 ->
// 1.39 GB) but takes 0.606 ms against 0.532 ms -- both forms are bound by the latency of
// their shared-memory passes at 2 CTAs per SM, not by HBM.  Read per launch (tests toggle it).
int fused_slots() {
  const char* e = std::getenv("PATFFT_LAT_FUSED_SLOTS");
  return e ? std::max(0, std::min(16, std::atoi(e))) : 0;
}
}  // namespace

// transforms per tile of the single-launch form: 16 (64 KB tiles at 512 points, 2 CTAs/SM) or 8
// (PATFFT_LAT_FUSED_PLOG=3: 32 KB tiles, 4 CTAs/SM)
int fused_plog() {
  const char* e = std::getenv("PATFFT_LAT_FUSED_PLOG");
  return e && std::atoi(e) == 3 ? 3 : 4;
}

bool lateral_fused_supported(const LateralParams& p) {
  const int len = p.t_end - p.t_begin, ch = 2 << fused_plog();
  return fused_slots() > 0 && !p.ref && p.f_flags && !p.cplx && p.nrows == p.ncols &&
         (p.nrows == 128 || p.nrows == 256 || p.nrows == 512) && len >= 64 &&
         (int64_t)std::min(fused_slots(), (len + ch - 1) / ch) * ch <= (int64_t)p.y_capacity;
}

cudaError_t launch_lateral_forward(const LateralParams& p0, cudaStream_t s) {
  if (p0.ref) return launch_lateral_ref(p0, s);
  if (!lateral_fused_supported(p0)) {
    cudaError_t e = launch_lateral_col(p0, s);
    return e != cudaSuccess ? e : launch_lateral_row(p0, s);
  }
  LateralParams p = p0;
  const int plog = fused_plog(), ch = 2 << plog;
  p.f_chunks = (p.t_end - p.t_begin + ch - 1) / ch;
  p.f_slots = std::min(fused_slots(), p.f_chunks);
  cudaError_t err = cudaMemsetAsync(p.f_flags, 0, sizeof(int) * 2 * (size_t)p.f_chunks, s);
  if (err != cudaSuccess) return err;
  const unsigned grid = (unsigned)((p.f_chunks + 1) * (p.nrows + 2 * p.ny));
  const size_t smem = ((size_t)p.nrows << plog) * sizeof(float2);
  auto run = [&](auto k, int thr) {
    err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err == cudaSuccess) {
      k<<<grid, thr, smem, s>>>(p);
      err = cudaGetLastError();
    }
  };
  if (plog == 3) {
    switch (p.nrows) {
      case 128: run(latfused_kernel<3, 7>, nth_for(7, 3)); break;
      case 256: run(latfused_kernel<3, 8>, nth_for(8, 3)); break;
      default: run(latfused_kernel<3, 9>, nth_for(9, 3)); break;
    }
    return err;
  }
  switch (p.nrows) {
    case 128: run(latfused_kernel<4, 7>, nth_for(7, 4)); break;
    case 256: run(latfused_kernel<4, 8>, nth_for(8, 4)); break;
    default: run(latfused_kernel<4, 9>, nth_for(9, 4)); break;
  }
  return err;
}

cudaError_t launch_lateral_inverse(const LateralParams& p0, cudaStream_t s) {
  if (inverse_fused_supported(p0)) {
    LateralParams p = p0;
    p.f_chunks = p.Tu / 32;
    p.f_slots = std::min(inv_fused_slots(), p.f_chunks);
    p.f_lead = std::max(1, std::min(inv_fused_lead(), p.f_slots - 1));
    p.f_flags = p.inv_flags;
    cudaError_t err = cudaMemsetAsync(p.f_flags, 0, sizeof(int) * 2 * (size_t)p.f_chunks, s);
    if (err != cudaSuccess) return err;
    const unsigned grid = (unsigned)((p.f_chunks + p.f_lead) * (2 * p.N1uh + p.N0u));
    const size_t smem = ((size_t)p.N0u << 4) * sizeof(float2);
    auto run = [&](auto k, int thr) {
      err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (err == cudaSuccess) {
        k<<<grid, thr, smem, s>>>(p);
        err = cudaGetLastError();
      }
    };
    switch (p.N0u) {
      case 64: run(invfused_kernel<4, 6>, nth_for(6, 4)); break;
      case 128: run(invfused_kernel<4, 7>, nth_for(7, 4)); break;
      case 256: run(invfused_kernel<4, 8>, nth_for(8, 4)); break;
      default: run(invfused_kernel<4, 9>, nth_for(9, 4)); break;
    }
    return err;
  }
  const LateralParams& p = p0;
  if (p.N0u > 1) {
    cudaError_t e = launch_inv_col(p, p.N0u, dim3((unsigned)p.N1uh, (unsigned)p.Tu), 1, s);
    if (e != cudaSuccess) return e;
  }
  return launch_inv_c2r(p, p.N1u, dim3((unsigned)p.N0u, (unsigned)p.Tu), 2, s);
}

}  // namespace patfft
