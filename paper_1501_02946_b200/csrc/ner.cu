// NER stage: one CTA per lateral frequency row j = (j0, j1) of the half
// spectrum.  Everything between reading gh[j, :] and writing the depth-
// inverted row z[j, :] stays in shared memory:
//
//  1. even time extension [g0..g_{T-1}, 0, g_{T-1}..g1] (recon.py:263-271)
//     times the pre-window 1/psi(2 pi n/2T - pi) (nufft.py:281-282, 325),
//     zero padded to n_over and stored rotated by -T (so the FFT output is
//     already multiplied by exp(i pi k / c), which removes the per-tap phase
//     of nufft.py:292) and bit-reversed;
//  2. radix-16 FFT of length n_over;
//  3. for every depth frequency l: kappa_e = 2 sign(l) sqrt(j2 + l^2) on the
//     band (recon.py:282-293), 2K-tap Kaiser-Bessel interpolation
//     (nufft.py:287-293, 329-331) with the tap weights evaluated as even/odd
//     split polynomials (no transcendental per tap), one phase
//     exp(-i pi kappa_e) per target, amplitude 2l/kappa, 0.5 and the
//     inverse-FFT normalisation (recon.py:308, 255);
//  4. zero padding / Nyquist split for upsampling (recon.py:225-246) and the
//     inverse FFT along depth (recon.py:255), written out as one z row (or
//     two rows for the lateral Nyquist split).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "fft_smem.cuh"
#include "patfft_internal.h"

namespace patfft {
namespace {

using fft::SwzAddr;

constexpr int kMaxTargetsPerThread = 8;
#ifndef PATFFT_NER_STORED
#define PATFFT_NER_STORED 1
#endif
#ifndef PATFFT_NER_INV_MAXR
#define PATFFT_NER_INV_MAXR 4  // radix-16 depth IFFT passes: fewer shared-memory round trips beat idle threads
#endif

// (cos(pi r), sin(pi r)) for |r| <= 1, ~1e-8 absolute
__device__ __forceinline__ float2 cospi_sinpi(float r) {
  const float q = rintf(2.f * r);
  const float x = 3.14159265358979f * fmaf(-0.5f, q, r);  // |x| <= pi/4
  const float x2 = x * x;
  const float s = x * fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, 2.7557319e-6f, -1.98412698e-4f), 8.33333333e-3f),
                                    -0.166666667f), 1.f);
  const float c = fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, -2.7557319e-7f, 2.48015873e-5f), -1.38888889e-3f),
                                          4.16666667e-2f), -0.5f), 1.f);
  const int qi = ((int)q) & 3;
  switch (qi) {
    case 0: return make_float2(c, s);
    case 1: return make_float2(-s, c);
    case 2: return make_float2(-c, -s);
    default: return make_float2(s, -c);
  }
}

// LOGT > 0: compile-time variant for T = 2^LOGT, n_over = 4T, upsample 1,
// fused depth IFFT, NTH = T/4 threads (clamped to [64, 512]); LOGT = 0: all
// sizes at run time.
constexpr int ner_ct_threads(int logt) {
  return logt <= 0 ? 512 : ((1 << logt) / 4 < 64 ? 64 : ((1 << logt) / 4 > 512 ? 512 : (1 << logt) / 4));
}
// keep <= 80 registers per thread (3 CTAs of 256 threads per SM at T = 1024)
constexpr int ner_ct_minb(int logt) { return logt <= 0 ? 1 : (65536 / 80) / ner_ct_threads(logt); }

template <int K2, int D, int LOGT>
__global__ void __launch_bounds__(ner_ct_threads(LOGT), ner_ct_minb(LOGT)) ner_kernel(const NerParams p) {
  constexpr bool CT = LOGT > 0;
  constexpr int CT_T = CT ? (1 << LOGT) : 1;
  constexpr int CT_NTH = CT ? ner_ct_threads(LOGT) : 1;
  extern __shared__ float2 sbuf[];
  constexpr int K = K2 / 2;
  const int rl = blockIdx.x + p.in_row_off;  // local row of the input array
  const int r = p.row0 + rl;         // global gh row: j0w * N1h + j1
  const int tid = threadIdx.x;
  const int nth = CT ? CT_NTH : (int)blockDim.x;
  const int T = CT ? CT_T : p.T;
  const int n = CT ? 4 * CT_T : p.n_over;
  const int L = CT ? LOGT + 2 : p.log_n_over;
  const SwzAddr ad = SwzAddr::for_log(L);
  // input row rl, time t lives at gh[((t / tci) * rows_local + rl) * tci + t % tci]
  // (tci = T for a single GPU; the power-of-two time slice per source rank
  // when sharded; the division is a shift/mask, shift = 31 for one chunk)
  const int tci = p.in_tchunk;
  const float2* __restrict__ g = p.gh + (size_t)rl * tci;
  const size_t gstride = (size_t)p.rows_local * tci;

  // 1. rotated, windowed even extension -> bit-reversed smem
  // interp mode (reconstruct_interp_fft, recon.py:297-303): plain length-2T
  // FFT of the unwindowed, unrotated extension; NUFFT mode: rotated by -T
  // and pre-windowed (see the header comment).
  const bool interp = !CT && p.interp;
  auto load_ext = [&](int m) {
        const int i = interp ? m : ((m + T) & (n - 1));  // sequence index stored at slot m
        float2 v = make_float2(0.f, 0.f);
        // CT: ext[0] = g0 is left out, so the windowed sequence is exactly even
        // around slot 0 and its transform D(kappa) is even; g0 is added exactly below
        if (i < 2 * T && i != T && !(CT && i == 0)) {
          const int t = i < T ? i : 2 * T - i;
          const float2 gv = __ldcs(&g[(t >> p.in_tshift) * gstride + (t & p.in_tmask)]);
          v = interp ? gv : fft::cscale(gv, __ldg(&p.iw[i]));
        }
        return v;
  };
  auto store_brev = [&](int m, float2 v) { sbuf[ad(fft::brev(m, L), 0)] = v; };
  if constexpr (CT) {
    fft::fft_ct_loaded<false, LOGT + 2, 4, true, 0, CT_NTH>(sbuf, p.tw, tid, fft::SwzC<LOGT + 2>(),
                                                          [&](int m, int) { return load_ext(m); });
  } else {
    fft::staged_copy<8, float2>(n, tid, nth, load_ext, store_brev);
    __syncthreads();
    fft::fft_inplace<false, 4, true>(sbuf, L, 0, p.tw, tid, nth, ad);
  }
  const SwzAddr gad = ad;

  // 2. targets
  const int j0w = r / p.N1h;
  const int j1 = r - j0w * p.N1h;
  const double j2 = p.jt0[j0w] + p.jt1[j1];  // recon.py:210-214 summation order
  const double halfT = (double)T / 2.0;
  const double band_r2 = halfT * halfT;
  // interpolated D(kappa_e) (2K taps, polynomial weights) for kappa_e >= 0
  auto interp_D = [&](double ke) {
    const double xi = __dmul_rn(p.c_eff, ke);
    const double k0d = floor(xi);
    const int k0 = (int)k0d;
    const float z = (float)(xi - k0d) - 0.5f;
    const float z2 = z * z;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      // tap j (dk = j-K+1) and its mirror K2-1-j share one polynomial:
      // w_j = E(z^2) + z O(z^2), w_mirror = E(z^2) - z O(z^2); the E and O
      // Horner chains run side by side in packed FP32 lanes
      constexpr int DE = D % 2 ? D - 1 : D;  // top even / odd degrees
      constexpr int DO = D % 2 ? D : D - 1;
      float2 eo = make_float2(p.poly[j][DE], p.poly[j][DO]);
#pragma unroll
      for (int s2 = 1; s2 <= DO / 2; ++s2)
        eo = fft::f2fma(eo, make_float2(z2, z2), make_float2(p.poly[j][DE - 2 * s2], p.poly[j][DO - 2 * s2]));
#pragma unroll
      for (int d = DE - 2 * (DO / 2) - 2; d >= 0; d -= 2) eo.x = fmaf(eo.x, z2, p.poly[j][d]);
      const float wa = fmaf(z, eo.y, eo.x);
      const float wb = fmaf(-z, eo.y, eo.x);
      const float2 Fa = sbuf[gad((k0 + j - K + 1) & (n - 1), 0)];
      const float2 Fb = sbuf[gad((k0 + K - j) & (n - 1), 0)];
      acc = fft::f2fma(Fa, make_float2(wa, wa), fft::f2fma(Fb, make_float2(wb, wb), acc));
    }
    return acc;
  };

  constexpr int kPairs = 4;  // CT: |l| in [0, T/2], at most 4 per thread
  float2 vals[kMaxTargetsPerThread];
  float2 valsP[kPairs], valsM[kPairs];
  if constexpr (CT) {
    // NER(+-l) = exp(-+ i pi kappa_e) D(kappa_e) + g0 with kappa_e = 2 kappa(j, |l|) >= 0:
    // one interpolation serves both signs of l (recon.py:282-308 targets)
    const float2 g0 = __ldg(&g[0]);
#pragma unroll
    for (int it = 0; it < kPairs; ++it) {
      const int lh = tid + it * nth;
      float2 vp = make_float2(0.f, 0.f), vm = make_float2(0.f, 0.f);
      if (lh <= T / 2 && lh > 0) {
        const double lv = __dmul_rn(__dmul_rn((double)lh, 1.0 / (double)T), (double)T);  // fftfreq(T)*T
        const double r2 = __dadd_rn(j2, __dmul_rn(lv, lv));
        if (r2 <= band_r2) {
          const double kap = sqrt(r2);
          const double ke = 2.0 * kap;
          const float2 Dv = interp_D(ke);
          const double red = ke - 2.0 * floor(0.5 * ke + 0.5);
          const float2 cs = cospi_sinpi((float)red);  // (cos, sin)(pi kappa_e)
          const float amp = __fdividef(2.f * (float)lv, (float)kap);
          const float a = 0.5f * amp * p.scale;
          const float rx = Dv.x * cs.x, ry = Dv.y * cs.x, sx = Dv.x * cs.y, sy = Dv.y * cs.y;
          vp = make_float2(a * (rx + sy + g0.x), a * (ry - sx + g0.y));  // e^{-i pi ke} D + g0
          vm = make_float2(a * (rx - sy + g0.x), a * (ry + sx + g0.y));  // e^{+i pi ke} D + g0
        }
      }
      valsP[it] = vp;
      valsM[it] = vm;
    }
  } else {
#pragma unroll
  for (int it = 0; it < kMaxTargetsPerThread; ++it) {
    const int l = tid + it * nth;
    float2 out = make_float2(0.f, 0.f);
    if (l < T) {
      const int ls = (l < T / 2) ? l : l - T;
      const double lv = __dmul_rn(__dmul_rn((double)ls, 1.0 / (double)T), (double)T);  // fftfreq(T)*T
      const double r2 = __dadd_rn(j2, __dmul_rn(lv, lv));
      if (ls != 0 && r2 <= band_r2) {
        double kap = sqrt(r2);
        if (ls < 0) kap = -kap;
        const double ke = 2.0 * kap;
        if (interp) {  // linear interpolation between the two nearest bins
          const double i0d = floor(ke);
          const int i0 = (int)i0d;
          const float fr = (float)(ke - i0d);
          const float2 Fa = sbuf[gad(i0 & (n - 1), 0)];
          const float2 Fb = sbuf[gad((i0 + 1) & (n - 1), 0)];
          const float amp = __fdividef(2.f * (float)lv, (float)kap);
          const float a = 0.5f * amp * p.scale;
          vals[it] = make_float2(a * fmaf(fr, Fb.x - Fa.x, Fa.x), a * fmaf(fr, Fb.y - Fa.y, Fa.y));
          continue;
        }
        const float2 acc = interp_D(ke);
        // exp(-i pi kappa_e), kappa_e reduced mod 2 in float64
        const double red = ke - 2.0 * floor(0.5 * ke + 0.5);
        const float2 cs = cospi_sinpi((float)red);
        const float amp = __fdividef(2.f * (float)lv, (float)kap);
        const float a = 0.5f * amp * p.scale;
        out = make_float2(a * (acc.x * cs.x + acc.y * cs.y), a * (acc.y * cs.x - acc.x * cs.y));
      }
    }
    vals[it] = out;
  }
  }

  // destination rows in the (possibly upsampled) half spectrum z
  int drow0 = 0, drow1 = -1;
  float dfac = 1.f;
  {
    int j0u = 0, j0u2 = -1;
    float f0 = 1.f;
    if (p.n_lat == 2) {
      const int a = j0w < p.N0 / 2 ? j0w : j0w - p.N0;
      if (p.up == 1) {
        j0u = j0w;
      } else if (a == -(p.N0 / 2)) {  // Nyquist split (recon.py:239-245)
        j0u = p.N0 / 2;
        j0u2 = p.N0u - p.N0 / 2;
        f0 = 0.5f;
      } else {
        j0u = a >= 0 ? a : p.N0u + a;
      }
    }
    const float f1 = (p.up > 1 && j1 == p.N1 / 2) ? 0.5f : 1.f;
    drow0 = j0u * p.N1uh + j1;
    if (j0u2 >= 0) drow1 = j0u2 * p.N1uh + j1;
    dfac = f0 * f1;
  }

  const int Tu = CT ? CT_T : p.Tu;
  __syncthreads();  // forward spectrum fully consumed
  if (CT || p.fused_ifft) {
    const int Lu = CT ? LOGT : p.log_tu;
    const SwzAddr iad = SwzAddr::for_log(Lu);
    if (!CT && p.up > 1) {
      for (int i = tid; i < Tu; i += nth) sbuf[iad(i, 0)] = make_float2(0.f, 0.f);
      __syncthreads();
    }
    if constexpr (CT) {  // up == 1: +l at index l, -l at index T - l
#pragma unroll
      for (int it = 0; it < kPairs; ++it) {
        const int lh = tid + it * nth;
        if (lh > T / 2) break;
        if (lh < T / 2) sbuf[iad(fft::brev(lh, Lu), 0)] = fft::cscale(valsP[it], dfac);
        if (lh > 0) sbuf[iad(fft::brev(T - lh, Lu), 0)] = fft::cscale(valsM[it], dfac);
      }
    } else {
#pragma unroll
    for (int it = 0; it < kMaxTargetsPerThread; ++it) {
      const int l = tid + it * nth;
      if (l >= T) break;
      const int ls = (l < T / 2) ? l : l - T;
      const float2 v = fft::cscale(vals[it], dfac);
      if (ls == -(T / 2) && p.up > 1) {
        const float2 hv = fft::cscale(v, 0.5f);
        sbuf[iad(fft::brev(T / 2, Lu), 0)] = hv;
        sbuf[iad(fft::brev(Tu - T / 2, Lu), 0)] = hv;
      } else {
        sbuf[iad(fft::brev(ls >= 0 ? ls : Tu + ls, Lu), 0)] = v;
      }
    }
    }
    __syncthreads();
    // output row d, depth i lives at z[((i / tco) * rows_out + d) * tco + i % tco]
    const int tco = p.out_tchunk;
    const size_t zstride = (size_t)p.rows_out * tco;
    float2* __restrict__ z0 = p.z + (size_t)(drow0 - p.out_row0) * tco;
    float2* __restrict__ z1 = p.z + (size_t)((drow1 >= 0 ? drow1 : drow0) - p.out_row0) * tco;
    auto st = [&](int i, int, float2 v) {
      const size_t o = (i >> p.out_tshift) * zstride + (i & p.out_tmask);
      z0[o] = v;
      if (drow1 >= 0) z1[o] = v;
    };
    if constexpr (CT && PATFFT_NER_STORED) {
      // the last IFFT pass writes the z row straight to global memory
      fft::fft_ct_stored<true, LOGT, PATFFT_NER_INV_MAXR, true, 0, CT_NTH>(sbuf, p.tw, tid, fft::SwzC<LOGT>(), st);
    } else {
      if constexpr (CT) fft::fft_ct<true, LOGT, PATFFT_NER_INV_MAXR, true, 0, CT_NTH>(sbuf, p.tw, tid, fft::SwzC<LOGT>());
      else fft::fft_inplace<true, 4, true>(sbuf, Lu, 0, p.tw, tid, nth, iad);
#pragma unroll 4
      for (int i = tid; i < Tu; i += nth) st(i, 0, sbuf[iad(i, 0)]);
    }
  } else {
    // spectrum only; z was zero-filled and a batched cuFFT does the depth IFFT
#pragma unroll
    for (int it = 0; it < kMaxTargetsPerThread; ++it) {
      const int l = tid + it * nth;
      if (l >= T) break;
      const int ls = (l < T / 2) ? l : l - T;
      const float2 v = fft::cscale(vals[it], dfac);
      for (int d = 0; d < (drow1 >= 0 ? 2 : 1); ++d) {
        float2* __restrict__ zr = p.z + (size_t)(d ? drow1 : drow0) * Tu;
        if (ls == -(T / 2) && p.up > 1) {
          zr[T / 2] = fft::cscale(v, 0.5f);
          zr[Tu - T / 2] = fft::cscale(v, 0.5f);
        } else {
          zr[ls >= 0 ? ls : Tu + ls] = v;
        }
      }
    }
  }
}

// DCT form of the compile-time NER kernel (T = 2^LOGT, n_over = 4T, default
// window, upsample 1).  The rotated, windowed even extension x (x[-m] =
// x[m], support |m| < T) makes its 4T-point spectrum D[k] = 2 sum_m x_m
// cos(pi m k / 2T) even, so half the FFT is redundant.  The interpolation
// grid is shifted by half a bin, bins at (k + 1/2) / c: the Kaiser-Bessel
// identity holds for any grid offset (nufft.py:287-293 with kappa -> kappa -
// 1/(2c)), the tap weights keep their form in z = frac(c kappa - 1/2) - 1/2,
// and the rotation still absorbs the per-tap phase.  On that grid
//   D'[q] = 2 sum_{m<T} x_m cos(pi m (2q + 1) / 4T),   q = 0 .. 2T-1,
// is a DCT-III of length 2T, computed with ONE 2T-point complex inverse FFT
// (Makhoul): input W_n = exp(i pi n / 4T) (x_n - i x_{2T-n}) (table pre[]
// times the gh sample), output D'[2j] = Z[j], D'[2j+1] = Z[2T-1-j]; bins
// outside [0, 2T) fold by D'[-1-q] = D'[q] = D'[4T-1-q].  Half the points and
// one radix stage fewer than the 4T-point FFT of the plain form.
// Last radix-2^R pass of a compile-time transform, in place: every thread
// first reads and transforms all of its items, then (after a barrier) hands
// each output, natural index n, to store(n, v) -- which may write anywhere in
// the same buffer.  No trailing barrier.
template <int R, bool INV, int L, int LOGH, int NTH, class Addr, class Store>
__device__ __forceinline__ void last_pass_inplace(float2* __restrict__ buf, const float2* __restrict__ tw, int tid,
                                                  Addr addr, Store store) {
  constexpr int PR = 1 << R;
  constexpr int H = 1 << LOGH;
  constexpr int ITEMS = 1 << (L - R);
  constexpr int ITER = (ITEMS + NTH - 1) / NTH;
  float2 e[ITER][PR];
  int base[ITER];
#pragma unroll
  for (int j = 0; j < ITER; ++j) {
    const int q = tid + j * NTH;
    base[j] = -1;
    if ((ITEMS % NTH) != 0 && q >= ITEMS) continue;
    const int k = q & (H - 1);
    base[j] = ((q >> LOGH) << (LOGH + R)) + k;
    const int ab = addr(base[j], 0);
#pragma unroll
    for (int m = 0; m < PR; ++m) e[j][m] = buf[ab ^ addr(m * H, 0)];
    fft::pass_butterflies<R, INV, LOGH>(e[j], k, tw);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < ITER; ++j) {
    if (base[j] < 0) continue;
#pragma unroll
    for (int m = 0; m < PR; ++m) store(base[j] + m * H, e[j][m]);
  }
}

#ifndef PATFFT_NER_DCT_DIV
#define PATFFT_NER_DCT_DIV 8  // threads per CTA = T / 8 (measured: 4 and 16 slower)
#endif
#ifndef PATFFT_NER_POLY_SCALAR
#define PATFFT_NER_POLY_SCALAR 1  // DCT kernel: tap polynomials as scalar FFMAs on constant-bank coefficients
#endif
#ifndef PATFFT_NER_EXTLOAD
#define PATFFT_NER_EXTLOAD 1  // first pass: running pointers into gh and pre[] (NerExtLoad)
#endif
#ifndef PATFFT_NER_DIRECT
#define PATFFT_NER_DIRECT 0  // 1: targets stored straight to a second buffer, loop not unrolled (kernel code
                             // 3672 -> 2152 instructions) -- measured 0.567 vs 0.560 ms, so not the bound
#endif
#ifndef PATFFT_NER_DCT_MAXR
#define PATFFT_NER_DCT_MAXR 4
#endif
constexpr int ner_dct_threads(int logt) {
  return (1 << logt) / PATFFT_NER_DCT_DIV < 64 ? 64
         : ((1 << logt) / PATFFT_NER_DCT_DIV > 512 ? 512 : (1 << logt) / PATFFT_NER_DCT_DIV);
}
#ifndef PATFFT_NER_DCT_REGS
#define PATFFT_NER_DCT_REGS 64  // 8 CTAs of 128 threads per SM (measured best; 48, 56, 72, 80, 96 slower)
#endif
constexpr int ner_dct_minb(int logt) { return (65536 / PATFFT_NER_DCT_REGS) / ner_dct_threads(logt); }

// First-pass operand of the DCT-form NER: element n of the 2T-point input is
// gh[|n - T|] (the even extension folded about T) times pre[n], zero at n = 0
// and n = T.  For an item's elements n = nat0 + k S (S = 2^(L-R)), k < 2^(R-1)
// read gh[T - nat0 - k S] and the rest gh[nat0 + (k - 2^(R-1)) S]: two base
// pointers with running offsets (single-GPU rows are contiguous in time; the
// sharded layout keeps the general addressing).
struct NerExtLoad {
  const float2* g;
  const float2* pre;
  int T;
  bool flat;
  size_t gstride;
  int tshift, tmask;
  __device__ __forceinline__ float2 at(int t) const {
    return __ldcs(flat ? &g[t] : &g[(t >> tshift) * gstride + (t & tmask)]);
  }
};
template <int R, int L>
__device__ __forceinline__ void load_items(float2 (&e)[1 << R], int nat0, int, const NerExtLoad& ld) {
  constexpr int KH = 1 << (R - 1);
  constexpr int S = 1 << (L - R);
  const float2* pr = ld.pre + nat0;
  if (ld.flat) {
    const float2* ga = ld.g + (ld.T - nat0);
    const float2* gb = ld.g + nat0;
#pragma unroll
    for (int k = 0; k < (1 << R); ++k) {
      const float2 v = k < KH ? ((k == 0 && nat0 == 0) ? make_float2(0.f, 0.f) : fft::ld_stream(ga - k * S))
                              : fft::ld_stream(gb + (k - KH) * S);
      e[fft::brev_c(k, R)] = fft::cmul(v, __ldg(pr + k * S));
    }
  } else {
#pragma unroll
    for (int k = 0; k < (1 << R); ++k) {
      const int n = nat0 + k * S;
      const float2 v = (k == 0 && nat0 == 0) ? make_float2(0.f, 0.f) : ld.at(k < KH ? ld.T - n : n - ld.T);
      e[fft::brev_c(k, R)] = fft::cmul(v, __ldg(pr + k * S));
    }
  }
  if (nat0 == 0) e[fft::brev_c(KH, R)] = make_float2(0.f, 0.f);  // n = T
}

// Last-pass store of the depth IFFT into the z row: contiguous on one GPU,
// [time chunk][row][t] in the sharded layout.
struct NerZStore {
  float2* z0;
  bool flat;
  size_t zstride;
  int tshift, tmask;
};
template <int R, int H>
__device__ __forceinline__ void store_items(const float2 (&e)[1 << R], int base, int, const NerZStore& st) {
  if (st.flat) {
    float2* b = st.z0 + base;
#pragma unroll
    for (int m = 0; m < (1 << R); ++m) b[m * H] = e[m];
  } else {
#pragma unroll
    for (int m = 0; m < (1 << R); ++m) {
      const int i = base + m * H;
      st.z0[(i >> st.tshift) * st.zstride + (i & st.tmask)] = e[m];
    }
  }
}

// float2 slots of the DCT kernel's D' array: bins [-16, 2T + 16) with one pad per 16
__host__ __device__ constexpr int ner_dct_dwords(int T) { return (2 * T + 32) + (2 * T + 32) / 16; }

template <int K2, int D, int LOGT>
__global__ void __launch_bounds__(ner_dct_threads(LOGT), ner_dct_minb(LOGT)) ner_dct_kernel(const NerParams p) {
  constexpr int T = 1 << LOGT;
  constexpr int NTH = ner_dct_threads(LOGT);
  constexpr int L = LOGT + 1;  // DCT length 2T
  constexpr int N2 = 2 * T;
  constexpr int K = K2 / 2;
  extern __shared__ float2 sbuf[];
  const int rl = blockIdx.x + p.in_row_off;
  const int r = p.row0 + rl;
  const int tid = threadIdx.x;
  const int tci = p.in_tchunk;
  const float2* __restrict__ g = p.gh + (size_t)rl * tci;
  const size_t gstride = (size_t)p.rows_local * tci;
  const bool flat_in = p.in_tshift >= 31;  // single GPU: one time chunk per row
  auto gload = [&](int t) {
    return __ldcs(flat_in ? &g[t] : &g[(t >> p.in_tshift) * gstride + (t & p.in_tmask)]);
  };
  // natural-order D' array (after the transform): one pad slot per 16, which
  // keeps the stride-~4 tap gathers of neighbouring threads conflict-free.
  // Bins q in [-16, 2T + 16): the folded bins D'[-1-q] = D'[q] and
  // D'[4T-1-q] = D'[q] that taps at the band ends reach are stored too, so
  // the gathers never fold (no per-tap branch).
  auto dpad = [](int q) { return (q + 16) + ((q + 16) >> 4); };

  // 1. DCT-III of the windowed half extension via a 2T-point inverse FFT;
  // the last pass stores D'[q] in natural order (Makhoul output permutation
  // Z[n] -> D'[n < 2T/2 ? 2n : 4T-1-2n]) into the same swizzled buffer
  const fft::SwzC<L> ad;
#if PATFFT_NER_EXTLOAD
  fft::fft_ct_loaded<true, L, PATFFT_NER_DCT_MAXR, true, 0, NTH, true>(
      sbuf, p.tw, tid, ad, NerExtLoad{g, p.pre, T, flat_in, gstride, p.in_tshift, p.in_tmask});
#else
  fft::fft_ct_loaded<true, L, PATFFT_NER_DCT_MAXR, true, 0, NTH, true>(sbuf, p.tw, tid, ad, [&](int n, int) {
    if (n == 0 || n == T) return make_float2(0.f, 0.f);
    const float2 gv = gload(n < T ? T - n : n - T);
    return fft::cmul(gv, __ldg(&p.pre[n]));
  });
#endif
  {
    constexpr int LH = fft::LastPassLogh<L, PATFFT_NER_DCT_MAXR, true>::value;
    last_pass_inplace<L - LH, true, L, LH, NTH>(sbuf, p.tw, tid, ad, [&](int n, float2 v) {
      const int q = n < T ? 2 * n : 4 * T - 1 - 2 * n;
      sbuf[dpad(q)] = v;
      if (q < K) sbuf[dpad(-1 - q)] = v;
      if (q >= N2 - K) sbuf[dpad(4 * T - 1 - q)] = v;
    });
  }
  __syncthreads();

  // 2. targets.  kappa(j, l) = sqrt(j2 + l^2) in float32 pairs: j2 (float64,
  // recon.py:210-214 summation order) splits into hi + lo floats once per
  // row, l^2 is exact, and one Newton step on rsqrt gives kappa = y + yl to
  // ~1e-12 absolute -- the bin k0 and the offset z of c kappa_e - 1/2 =
  // 4 kappa - 1/2 (c_eff = 2) then follow without float64 arithmetic (the
  // fp64 DSQRT / FRND / F2F chain was a quarter of the target phase).  The
  // band test of recon.py:289 (j2 + l^2 <= (T/2)^2 in float64) is a prefix
  // l <= lmax, decided once per row in float64 exactly as the reference does.
  const int j0w = r / p.N1h;
  const int j1 = r - j0w * p.N1h;
  const double j2 = p.jt0[j0w] + p.jt1[j1];  // recon.py:210-214 summation order
  constexpr double halfT = (double)T / 2.0;
  constexpr double band_r2 = halfT * halfT;
  int lmax;
  {
    const double rem = band_r2 - j2;
    int c0 = rem > 0.0 ? (int)sqrt(rem) : 0;
    if (c0 > T / 2) c0 = T / 2;
    while (c0 < T / 2 && j2 + (double)(c0 + 1) * (c0 + 1) <= band_r2) ++c0;
    while (c0 > 0 && !(j2 + (double)c0 * c0 <= band_r2)) --c0;
    lmax = c0;  // targets lh = 1 .. lmax are on the band
  }
  const float j2h = (float)j2;
  const float j2l = (float)(j2 - (double)j2h);
  auto interp_D = [&](int k0, float z) {
    const float z2 = z * z;
    // taps k0-K+1 .. k0+K of D' (natural order, padded).  Inside the band the
    // taps span at most two 16-blocks: tap t sits at base0 + t or base1 + t.
    // Targets at the ends of the band fold by D'[-1-q] = D'[q] = D'[4T-1-q].
    const int kb = k0 - K + 1;
    const int base0 = dpad(kb), tb = 16 - (kb & 15);  // kb >= -K, kb + K2 <= 2T + K
    auto at = [&](int t) { return sbuf[(t < tb ? base0 : base0 + 1) + t]; };
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      constexpr int DE = D % 2 ? D - 1 : D;
      constexpr int DO = D % 2 ? D : D - 1;
      // scalar Horner chains: each FFMA takes its coefficient straight from the
      // constant bank (the packed form needs the pair in registers: LDC + MOV)
      float ev = p.poly[j][DE], ov = p.poly[j][DO];
#pragma unroll
      for (int s2 = 1; s2 <= DO / 2; ++s2) {
        ev = fmaf(ev, z2, p.poly[j][DE - 2 * s2]);
        ov = fmaf(ov, z2, p.poly[j][DO - 2 * s2]);
      }
#pragma unroll
      for (int d = DE - 2 * (DO / 2) - 2; d >= 0; d -= 2) ev = fmaf(ev, z2, p.poly[j][d]);
      const float wa = fmaf(z, ov, ev);
      const float wb = fmaf(-z, ov, ev);
      const float2 Fa = at(j);
      const float2 Fb = at(K2 - 1 - j);
      acc = fft::f2fma(Fa, make_float2(wa, wa), fft::f2fma(Fb, make_float2(wb, wb), acc));
    }
    return acc;
  };
  constexpr int kPairs = (T / 2 + NTH) / NTH;  // |l| in [0, T/2]
#if PATFFT_NER_DIRECT
  // targets go straight into a separate depth-spectrum buffer (bit-reversed,
  // swizzled) behind the D' array: no per-target registers, and the target
  // loop is not unrolled (five inlined copies of the interpolation made the
  // kernel's code larger than the instruction cache)
  float2* __restrict__ obuf = sbuf + ner_dct_dwords(T);
  const fft::SwzC<LOGT> iad;
#else
  float2 valsP[kPairs], valsM[kPairs];
#endif
  const float2 g0 = gload(0);
#if PATFFT_NER_DIRECT
#pragma unroll 1
#else
#pragma unroll
#endif
  for (int it = 0; it < kPairs; ++it) {
    const int lh = tid + it * NTH;
    float2 vp = make_float2(0.f, 0.f), vm = make_float2(0.f, 0.f);
    if (lh <= lmax && lh > 0) {
      // r2 = lh^2 + j2 as an unevaluated float pair (s, rl): TwoSum
      const float l2 = (float)(lh * lh);  // exact (lh <= 2^10)
      const float s = l2 + j2h;
      const float bb = s - l2;
      const float rl = ((l2 - (s - bb)) + (j2h - bb)) + j2l;
      // kappa = sqrt(s + rl) = y + yl (one Newton step from the rsqrt estimate)
      const float rs = rsqrtf(s);
      const float y = s * rs;
      const float yl = (fmaf(-y, y, s) + rl) * (0.5f * rs);
      // c kappa_e - 1/2 = 4 y - 1/2 + 4 yl; 4 y - 1/2 is exact in float32
      const float xh = fmaf(4.f, y, -0.5f);
      float kf = floorf(xh);
      float z = ((xh - kf) - 0.5f) + 4.f * yl;  // in [-1/2, 1/2) up to the yl correction
      if (z < -0.5f) {
        z += 1.f;
        kf -= 1.f;
      } else if (z >= 0.5f) {
        z -= 1.f;
        kf += 1.f;
      }
      const float2 Dv = interp_D((int)kf, z);
      // exp(-+ i pi kappa_e), kappa_e = 2 kappa reduced mod 2: 2 (y - rint(y)) is exact
      const float red = fmaf(2.f, y - rintf(y), 2.f * yl);
      const float2 cs = cospi_sinpi(red);  // (cos, sin)(pi kappa_e)
      const float amp = __fdividef(2.f * (float)lh, y);  // 2 l / kappa (recon.py:290)
      const float a = 0.5f * amp * p.scale;
      const float rx = Dv.x * cs.x, ry = Dv.y * cs.x, sx = Dv.x * cs.y, sy = Dv.y * cs.y;
      vp = make_float2(a * (rx + sy + g0.x), a * (ry - sx + g0.y));  // e^{-i pi ke} D + g0
      vm = make_float2(a * (rx - sy + g0.x), a * (ry + sx + g0.y));  // e^{+i pi ke} D + g0
    }
#if PATFFT_NER_DIRECT
    if (lh <= T / 2) {
      if (lh < T / 2) obuf[iad(fft::brev(lh, LOGT), 0)] = vp;
      if (lh > 0) obuf[iad(fft::brev(T - lh, LOGT), 0)] = vm;
    }
#else
    valsP[it] = vp;
    valsM[it] = vm;
#endif
  }

  // 3. depth inverse FFT (recon.py:255) straight to z (up == 1: row j0w * N1h + j1)
#if PATFFT_NER_DIRECT
  float2* __restrict__ ibuf = obuf;
#else
  float2* __restrict__ ibuf = sbuf;
  __syncthreads();  // spectrum fully consumed
  {
    const fft::SwzC<LOGT> iad;
#pragma unroll
    for (int it = 0; it < kPairs; ++it) {
      const int lh = tid + it * NTH;
      if (lh > T / 2) break;
      if (lh < T / 2) sbuf[iad(fft::brev(lh, LOGT), 0)] = valsP[it];
      if (lh > 0) sbuf[iad(fft::brev(T - lh, LOGT), 0)] = valsM[it];
    }
  }
#endif
  __syncthreads();
  const int tco = p.out_tchunk;
  const size_t zstride = (size_t)p.rows_out * tco;
  float2* __restrict__ z0 = p.z + (size_t)(r - p.out_row0) * tco;
  const bool flat_out = p.out_tshift >= 31;
#if PATFFT_NER_EXTLOAD
  fft::fft_ct_stored<true, LOGT, PATFFT_NER_INV_MAXR, true, 0, NTH>(
      ibuf, p.tw, tid, fft::SwzC<LOGT>(), NerZStore{z0, flat_out, zstride, p.out_tshift, p.out_tmask});
#else
  fft::fft_ct_stored<true, LOGT, PATFFT_NER_INV_MAXR, true, 0, NTH>(
      ibuf, p.tw, tid, fft::SwzC<LOGT>(), [&](int i, int, float2 v) {
        z0[flat_out ? (size_t)i : (i >> p.out_tshift) * zstride + (i & p.out_tmask)] = v;
      });
#endif
}

}  // namespace

size_t ner_smem_bytes(int n_over, int Tu) {
  const int m = n_over > Tu ? n_over : Tu;
  return (size_t)m * sizeof(float2);  // SwzAddr layout: no padding
}

int ner_threads(int n_over) {
  int t = n_over / 16;
  if (t < 64) t = 64;
  if (t > 512) t = 512;
  return t;
}

cudaError_t launch_ner(const NerParams& p, int K2, int degree, cudaStream_t s) {
  if (p.ref) return launch_ner_ref(p, s);
  int threads = ner_threads(p.n_over);
  const size_t smem = ner_smem_bytes(p.n_over, p.fused_ifft ? p.Tu : 0);
  const unsigned rows = (unsigned)(p.rows_launch > 0 ? p.rows_launch : p.rows_local);
  cudaError_t err = cudaSuccess;
  auto go = [&](auto kern) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return;
    kern<<<rows, threads, smem, s>>>(p);
    err = cudaGetLastError();
  };
  // compile-time variant for the default window (2K = 12, degree 8), c_eff = 2,
  // upsample 1 and T = 2^7 .. 2^11
  const bool ct_ok = (K2 == 12 || K2 == 8) && degree == 8 && p.fused_ifft && p.up == 1 && p.n_over == 4 * p.T &&
                     p.Tu == p.T && p.log_n_over >= 9 && p.log_n_over <= 13;
  static const bool dct = [] {
    const char* e = std::getenv("PATFFT_NER_DCT");
    return e ? std::atoi(e) != 0 : true;
  }();
  if (ct_ok && dct && p.pre) {
    // DCT form: 2T-point transform, half the shared memory
    threads = std::max(64, std::min(512, p.T / PATFFT_NER_DCT_DIV));
    const size_t smem2 = (size_t)(ner_dct_dwords(p.T) + (PATFFT_NER_DIRECT ? p.T : 0)) * sizeof(float2);
    auto go2 = [&](auto kern) {
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
      if (err != cudaSuccess) return;
      kern<<<rows, threads, smem2, s>>>(p);
      err = cudaGetLastError();
    };
#define PATFFT_NER_DCT_SWITCH(k2, d)                         \
  switch (p.log_n_over - 2) {                                 \
    case 7: go2(ner_dct_kernel<k2, d, 7>); return err;        \
    case 8: go2(ner_dct_kernel<k2, d, 8>); return err;        \
    case 9: go2(ner_dct_kernel<k2, d, 9>); return err;        \
    case 10: go2(ner_dct_kernel<k2, d, 10>); return err;      \
    case 11: go2(ner_dct_kernel<k2, d, 11>); return err;      \
  }
    if (K2 == 8) {
      if (p.poly7) PATFFT_NER_DCT_SWITCH(8, 7)
      PATFFT_NER_DCT_SWITCH(8, 8)
    } else {
      if (p.poly7) PATFFT_NER_DCT_SWITCH(12, 7)
      PATFFT_NER_DCT_SWITCH(12, 8)
    }
#undef PATFFT_NER_DCT_SWITCH
  }
  if (ct_ok && K2 == 12) {
    threads = ner_threads(p.n_over);
    switch (p.log_n_over - 2) {
      case 7: go(ner_kernel<12, 8, 7>); return err;
      case 8: go(ner_kernel<12, 8, 8>); return err;
      case 9: go(ner_kernel<12, 8, 9>); return err;
      case 10: go(ner_kernel<12, 8, 10>); return err;
      case 11: go(ner_kernel<12, 8, 11>); return err;
    }
  }
#define PATFFT_NER_CASE(k2)                          \
  case k2:                                           \
    if (degree == 8) go(ner_kernel<k2, 8, 0>);       \
    else go(ner_kernel<k2, 12, 0>);                  \
    break;
  switch (K2) {
    PATFFT_NER_CASE(2)
    PATFFT_NER_CASE(4)
    PATFFT_NER_CASE(6)
    PATFFT_NER_CASE(8)
    PATFFT_NER_CASE(10)
    PATFFT_NER_CASE(12)
    PATFFT_NER_CASE(14)
    PATFFT_NER_CASE(16)
    default: return cudaErrorInvalidValue;
  }
#undef PATFFT_NER_CASE
  return err;
}

}  // namespace patfft
