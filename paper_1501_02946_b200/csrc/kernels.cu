// sm_100a kernels of the NEDNER-NUFFT reconstruction.
//
//  spread_kernel : NED gridding (reference nufft.py:373-404, recon.py:374).
//                  Output-stationary, deterministic, no atomics: one thread
//                  owns (grid row, TPT time samples) and sweeps that row's
//                  column-sorted sensor list with a register ring of RING
//                  columns; finished column groups are streamed to HBM.
//  crop_kernel   : centred crop + deapodisation of the oversampled lateral
//                  spectrum (nufft.py:406-415), fused with the lateral
//                  Hermitian symmetrisation of recon.py:218-222 restricted to
//                  the Nyquist planes (the only place it is not a no-op).
//  ner_kernel    : one CTA per lateral frequency row: even time extension +
//                  pre-window (recon.py:263-271, nufft.py:281-282), shared-
//                  memory FFT of length n_over (nufft.py:325), 2K-tap KB
//                  interpolation at kappa_e = 2 kappa(j,l) (nufft.py:287-293,
//                  329-331), amplitude/band epilogue (recon.py:282-308),
//                  spectral zero padding (recon.py:225-246) and the inverse
//                  FFT along depth (recon.py:255) -- all without leaving SMEM.
#include <cuda_runtime.h>

#include <cstdint>

#include "patfft_internal.h"

namespace patfft {

// ===========================================================================
// spread
// ===========================================================================
namespace {

template <int ROT, int K2, int RING, int TPT>
__device__ __forceinline__ void ring_apply(float (&acc)[RING][TPT], const float (&w)[K2], const float (&sv)[TPT]) {
#pragma unroll
  for (int j = 0; j < K2; ++j) {
#pragma unroll
    for (int i = 0; i < TPT; ++i) acc[(ROT + j) % RING][i] = fmaf(w[j], sv[i], acc[(ROT + j) % RING][i]);
  }
}

template <int Q, int RING, int TPT>
__device__ __forceinline__ void ring_flush_q(float (&acc)[RING][TPT], float* __restrict__ colp, int T, int bdim,
                                             bool store, const bool (&tv)[TPT]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
#pragma unroll
    for (int i = 0; i < TPT; ++i) {
      if (store && tv[i]) colp[(size_t)c * T + i * bdim] = acc[Q * 4 + c][i];
      acc[Q * 4 + c][i] = 0.f;
    }
  }
}

template <int RING, int TPT>
__device__ __forceinline__ void ring_flush(float (&acc)[RING][TPT], int g, float* __restrict__ rowp, int T, int bdim,
                                           int c0, int c1, const bool (&tv)[TPT]) {
  const int col = g * 4;
  const bool store = col >= c0 && col < c1;
  float* colp = rowp + (size_t)(store ? col : 0) * T;
  switch (g & (RING / 4 - 1)) {
#define PATFFT_FLUSH_CASE(q) \
  case q:                    \
    if (q < RING / 4) ring_flush_q<(q < RING / 4 ? q : 0), RING, TPT>(acc, colp, T, bdim, store, tv); \
    break;
    PATFFT_FLUSH_CASE(0) PATFFT_FLUSH_CASE(1) PATFFT_FLUSH_CASE(2) PATFFT_FLUSH_CASE(3)
    PATFFT_FLUSH_CASE(4) PATFFT_FLUSH_CASE(5) PATFFT_FLUSH_CASE(6) PATFFT_FLUSH_CASE(7)
#undef PATFFT_FLUSH_CASE
  }
}

template <int K2, int RING, int TPT>
__device__ __forceinline__ void ring_dispatch(int rot, float (&acc)[RING][TPT], const float (&w)[K2],
                                              const float (&sv)[TPT]) {
  switch (rot) {
#define PATFFT_ROT_CASE(r) \
  case r:                  \
    ring_apply<(r % RING), K2, RING, TPT>(acc, w, sv); \
    break;
    PATFFT_ROT_CASE(0) PATFFT_ROT_CASE(1) PATFFT_ROT_CASE(2) PATFFT_ROT_CASE(3)
    PATFFT_ROT_CASE(4) PATFFT_ROT_CASE(5) PATFFT_ROT_CASE(6) PATFFT_ROT_CASE(7)
    PATFFT_ROT_CASE(8) PATFFT_ROT_CASE(9) PATFFT_ROT_CASE(10) PATFFT_ROT_CASE(11)
    PATFFT_ROT_CASE(12) PATFFT_ROT_CASE(13) PATFFT_ROT_CASE(14) PATFFT_ROT_CASE(15)
#undef PATFFT_ROT_CASE
    default:
      if constexpr (RING > 16) {
        switch (rot) {
#define PATFFT_ROT_CASE(r) \
  case r:                  \
    ring_apply<(r % RING), K2, RING, TPT>(acc, w, sv); \
    break;
          PATFFT_ROT_CASE(16) PATFFT_ROT_CASE(17) PATFFT_ROT_CASE(18) PATFFT_ROT_CASE(19)
          PATFFT_ROT_CASE(20) PATFFT_ROT_CASE(21) PATFFT_ROT_CASE(22) PATFFT_ROT_CASE(23)
          PATFFT_ROT_CASE(24) PATFFT_ROT_CASE(25) PATFFT_ROT_CASE(26) PATFFT_ROT_CASE(27)
          PATFFT_ROT_CASE(28) PATFFT_ROT_CASE(29) PATFFT_ROT_CASE(30) PATFFT_ROT_CASE(31)
#undef PATFFT_ROT_CASE
          default:
            break;
        }
      }
      break;
  }
}

// grid: blockIdx.x = row * nseg + seg (rows fastest -> one time chunk of all
// rows is resident in L2 at a time), blockIdx.y = time chunk.
template <int K2, int RING, int TPT>
__global__ void __launch_bounds__(128) spread_kernel(const SpreadParams p) {
  static_assert(K2 + 3 <= RING, "ring too small for the window");
  constexpr int NG = RING / 4;
  const int rs = blockIdx.x;
  const int row = rs / p.nseg;
  const int seg = rs - row * p.nseg;
  const int c0 = seg * p.segw;
  const int c1 = min(p.ncols, c0 + p.segw);
  const int bdim = blockDim.x;
  const int tbase = blockIdx.y * bdim * TPT + threadIdx.x;
  const int T = p.T;

  bool tv[TPT];
#pragma unroll
  for (int i = 0; i < TPT; ++i) tv[i] = tbase + i * bdim < T;

  float acc[RING][TPT];
#pragma unroll
  for (int c = 0; c < RING; ++c)
#pragma unroll
    for (int i = 0; i < TPT; ++i) acc[c][i] = 0.f;

  float* rowp = p.grid + (size_t)row * p.ncols * T + tbase;
  int fg = (c0 >> 2) - NG;  // ring holds column groups [fg, fg + NG)
  const int2 rg = p.seg_range[rs];
  for (int e = rg.x; e < rg.y; ++e) {
    const int4 en = __ldg(&p.entries[e]);
    const int ws = en.y;
    const int gs = ws >> 2;  // arithmetic shift = floor division
    while (fg < gs) {
      ring_flush<RING, TPT>(acc, fg, rowp, T, bdim, c0, c1, tv);
      ++fg;
    }
    const float wr = __int_as_float(en.z);
    const float* src = p.samples + (size_t)en.x * T + tbase;
    float sv[TPT];
#pragma unroll
    for (int i = 0; i < TPT; ++i) sv[i] = tv[i] ? __ldg(src + i * bdim) * wr : 0.f;
    float w[K2];
    const float* cw = p.colw + (size_t)en.x * K2;
#pragma unroll
    for (int j = 0; j < K2; ++j) w[j] = __ldg(cw + j);
    ring_dispatch<K2, RING, TPT>(ws & (RING - 1), acc, w, sv);
  }
  const int gend = c1 >> 2;
  while (fg < gend) {
    ring_flush<RING, TPT>(acc, fg, rowp, T, bdim, c0, c1, tv);
    ++fg;
  }
}

}  // namespace

void spread_config(int K2, int T, int* bdim, int* tpt, int* tchunks) {
  const int t = (K2 <= 12) ? 4 : 2;
  int threads = (T + t - 1) / t;
  threads = ((threads + 31) / 32) * 32;
  if (threads > 128) threads = 128;
  *tpt = t;
  *bdim = threads;
  *tchunks = (T + threads * t - 1) / (threads * t);
}

cudaError_t launch_spread(const SpreadParams& p, int K2, int nrows, cudaStream_t s) {
  int bdim, tpt, tch;
  spread_config(K2, p.T, &bdim, &tpt, &tch);
  dim3 grid((unsigned)(nrows * p.nseg), (unsigned)tch);
  switch (K2) {
    case 2: spread_kernel<2, 16, 4><<<grid, bdim, 0, s>>>(p); break;
    case 4: spread_kernel<4, 16, 4><<<grid, bdim, 0, s>>>(p); break;
    case 6: spread_kernel<6, 16, 4><<<grid, bdim, 0, s>>>(p); break;
    case 8: spread_kernel<8, 16, 4><<<grid, bdim, 0, s>>>(p); break;
    case 10: spread_kernel<10, 16, 4><<<grid, bdim, 0, s>>>(p); break;
    case 12: spread_kernel<12, 16, 4><<<grid, bdim, 0, s>>>(p); break;
    case 14: spread_kernel<14, 32, 2><<<grid, bdim, 0, s>>>(p); break;
    case 16: spread_kernel<16, 32, 2><<<grid, bdim, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ===========================================================================
// crop + deapodise + Nyquist symmetrisation
// ===========================================================================
namespace {

__device__ __forceinline__ float2 x_at(const CropParams& p, int a, int b, int t) {
  // signed lateral frequency (a, b) of the R2C output; b < 0 via Hermitian symmetry
  if (b >= 0) {
    const int ra = ((a % p.nrows) + p.nrows) % p.nrows;
    return p.X[((size_t)ra * p.ncols_h + b) * p.T + t];
  }
  const int ra = (((-a) % p.nrows) + p.nrows) % p.nrows;
  const float2 v = p.X[((size_t)ra * p.ncols_h + (-b)) * p.T + t];
  return make_float2(v.x, -v.y);
}

__global__ void __launch_bounds__(256) crop_kernel(const CropParams p) {
  const int r = blockIdx.x;  // row of gh: j0w * N1h + j1
  const int t = blockIdx.y * blockDim.x + threadIdx.x;
  if (t >= p.T) return;
  const int j0w = r / p.N1h;
  const int j1 = r - j0w * p.N1h;
  const int a = (p.N0 > 1) ? (j0w < p.N0 / 2 ? j0w : j0w - p.N0) : 0;
  const int b = (j1 == p.N1 / 2) ? -(p.N1 / 2) : j1;
  const bool nyq0 = (p.N0 > 1) && (a == -(p.N0 / 2));
  const bool nyq1 = (b == -(p.N1 / 2));
  float2 v = x_at(p, a, b, t);
  if (nyq0 || nyq1) {
    // Hermitian part of the cropped spectrum on the Nyquist planes
    // (recon.py:218-222): 0.5 * (X(j) + X(j')) with Nyquist components flipped.
    const float2 v2 = x_at(p, nyq0 ? -a : a, nyq1 ? -b : b, t);
    v = make_float2(0.5f * (v.x + v2.x), 0.5f * (v.y + v2.y));
  }
  const float sc = p.dp0[j0w] * p.dp1[j1];
  p.gh[(size_t)r * p.T + t] = make_float2(v.x * sc, v.y * sc);
}

}  // namespace

cudaError_t launch_crop(const CropParams& p, cudaStream_t s) {
  dim3 grid((unsigned)(p.N0 * p.N1h), (unsigned)((p.T + 255) / 256));
  crop_kernel<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ===========================================================================
// NER: shared-memory FFT + KB interpolation + epilogue + inverse depth FFT
// ===========================================================================
namespace {

__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }  // bank-conflict padding

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

// exp(-2 pi i j / 16) (conjugated when INV)
template <bool INV>
__device__ __forceinline__ float2 w16(int j) {
  const float c[16] = {1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                       0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                       -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f,
                       0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
  const float s = c[(j + 12) & 15];  // sin(2 pi j/16) = cos(2 pi (j-4)/16)
  return make_float2(c[j & 15], INV ? s : -s);
}

// One in-place radix-2^R decimation-in-time pass over stages logh+1..logh+R
// of a length-2^L FFT whose input sits in bit-reversed order.
template <int R, bool INV>
__device__ __forceinline__ void dit_pass(float2* __restrict__ buf, int L, int logh, const float2* __restrict__ tw,
                                         int tid, int nth) {
  constexpr int P = 1 << R;
  const int h = 1 << logh;
  const int ngroups = 1 << (L - R);
  for (int q = tid; q < ngroups; q += nth) {
    const int k = q & (h - 1);
    const int base = ((q >> logh) << (logh + R)) + k;
    float2 e[P];
#pragma unroll
    for (int m = 0; m < P; ++m) e[m] = buf[spad(base + m * h)];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const float2 wi = __ldg(&tw[k << (L - logh - i - 1)]);  // W_{h 2^{i+1}}^k
#pragma unroll
      for (int r = 0; r < (1 << i); ++r) {
        const float2 t = (r == 0) ? wi : cmul(wi, w16<INV>(r << (3 - i)));
#pragma unroll
        for (int m0 = 0; m0 < P; m0 += (2 << i)) {
          const int m = m0 + r;
          const float2 x = cmul(e[m + (1 << i)], t);
          e[m + (1 << i)] = make_float2(e[m].x - x.x, e[m].y - x.y);
          e[m] = make_float2(e[m].x + x.x, e[m].y + x.y);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < P; ++m) buf[spad(base + m * h)] = e[m];
  }
}

template <bool INV>
__device__ void smem_fft(float2* __restrict__ buf, int L, const float2* __restrict__ tw, int tid, int nth) {
  int logh = 0;
  while (logh < L) {
    const int R = min(4, L - logh);
    switch (R) {
      case 4: dit_pass<4, INV>(buf, L, logh, tw, tid, nth); break;
      case 3: dit_pass<3, INV>(buf, L, logh, tw, tid, nth); break;
      case 2: dit_pass<2, INV>(buf, L, logh, tw, tid, nth); break;
      default: dit_pass<1, INV>(buf, L, logh, tw, tid, nth); break;
    }
    logh += R;
    __syncthreads();
  }
}

// psi_hat(x) / psi_hat(0) in float32 (nufft.py:168-187 normalised)
__device__ __forceinline__ float kb_hat_norm(float x, const NerParams& p) {
  const float b2x2 = (p.beta - x) * (p.beta + x);
  if (b2x2 > 0.f) {
    const float q = sqrtf(b2x2);
    const float s = p.alpha * q;
    if (s > 0.35f) {
      const float d = -p.alpha * x * x / (q + p.beta);  // s - s0 without cancellation
      return (p.s0 / s) * __expf(d) * (1.f - __expf(-2.f * s)) * p.inv_one_minus_e2s0;
    }
    return p.s0_over_sinh_s0 * (1.f + s * s * (1.f / 6.f));
  }
  const float s = p.alpha * sqrtf(-b2x2);
  return p.s0_over_sinh_s0 * (s > 1e-3f ? __sinf(s) / s : 1.f - s * s * (1.f / 6.f));
}

constexpr int kMaxTargetsPerThread = 8;

template <int K2>
__global__ void __launch_bounds__(512) ner_kernel(const NerParams p) {
  extern __shared__ float2 sbuf[];
  const int r = blockIdx.x;  // gh row: j0w * N1h + j1
  const int tid = threadIdx.x, nth = blockDim.x;
  const int T = p.T, n = p.n_over;
  const float2* __restrict__ g = p.gh + (size_t)r * T;

  // 1. even extension [g0..g_{T-1}, 0, g_{T-1}..g1] * pre-window, zero padded
  //    to n_over, stored bit-reversed for the in-place DIT FFT.
  const int shf = 32 - p.log_n_over;
  for (int i = tid; i < n; i += nth) {
    float2 v = make_float2(0.f, 0.f);
    if (i < 2 * T && i != T) {
      const float2 gv = g[i < T ? i : 2 * T - i];
      const float w = __ldg(&p.iw[i]);
      v = make_float2(gv.x * w, gv.y * w);
    }
    sbuf[spad(__brev(i) >> shf)] = v;
  }
  __syncthreads();
  smem_fft<false>(sbuf, p.log_n_over, p.twf, tid, nth);

  // 2. interpolate at kappa_e = 2*sign(l)*sqrt(j2 + l^2) on the band
  const int j0w = r / p.N1h;
  const int j1 = r - j0w * p.N1h;
  const double j2 = p.jt0[j0w] + p.jt1[j1];  // recon.py:210-214 summation order
  const double halfT = (double)T / 2.0;
  const double band_r2 = halfT * halfT;
  float2 vals[kMaxTargetsPerThread];
  int cnt = 0;
  for (int l = tid; l < T; l += nth, ++cnt) {
    const int ls = (l < T / 2) ? l : l - T;
    const double lv = __dmul_rn(__dmul_rn((double)ls, 1.0 / (double)T), (double)T);  // fftfreq(T)*T
    const double r2 = __dadd_rn(j2, __dmul_rn(lv, lv));
    float2 out = make_float2(0.f, 0.f);
    if (ls != 0 && r2 <= band_r2) {
      double kap = sqrt(r2);
      if (ls < 0) kap = -kap;
      const double amp = __ddiv_rn(2.0 * lv, kap);
      const double xi = __dmul_rn(p.c_eff, 2.0 * kap);
      const double k0d = floor(xi);
      const float f = (float)(xi - k0d);
      const int k0 = (int)k0d;
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < K2; ++j) {
        const int dk = j - K2 / 2 + 1;
        const float wv = kb_hat_norm((f - (float)dk) * p.inv_c, p);
        const float2 ph = p.tap_phase[j];
        const float2 F = sbuf[spad((k0 + dk) & (n - 1))];
        const float2 FP = cmul(F, ph);
        acc.x = fmaf(wv, FP.x, acc.x);
        acc.y = fmaf(wv, FP.y, acc.y);
      }
      float sn, cs;
      sincospif(-f * p.inv_c, &sn, &cs);
      const float2 v = cmul(acc, make_float2(cs, sn));
      const float a = (float)(0.5 * amp) * p.scale;
      out = make_float2(v.x * a, v.y * a);
    }
    vals[cnt] = out;
  }

  // destination rows in the (possibly upsampled) half spectrum z
  int drow[2];
  float dfac[2];
  int nd = 1;
  {
    int j0u = 0;
    float f0 = 1.f;
    int j0u2 = -1;
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
    drow[0] = j0u * p.N1uh + j1;
    dfac[0] = f0 * f1;
    if (j0u2 >= 0) {
      drow[1] = j0u2 * p.N1uh + j1;
      dfac[1] = f0 * f1;
      nd = 2;
    }
  }

  const int Tu = p.Tu;
  __syncthreads();  // all reads of the forward spectrum are done
  if (p.fused_ifft) {
    // 3. place l at its (upsampled) frequency slot, bit-reversed
    const int shi = 32 - p.log_tu;
    if (p.up > 1) {
      for (int i = tid; i < Tu; i += nth) sbuf[spad(i)] = make_float2(0.f, 0.f);
      __syncthreads();
    }
    cnt = 0;
    for (int l = tid; l < T; l += nth, ++cnt) {
      const int ls = (l < T / 2) ? l : l - T;
      const float2 v = vals[cnt];
      if (ls == -(T / 2) && p.up > 1) {
        const float2 hv = make_float2(0.5f * v.x, 0.5f * v.y);
        sbuf[spad(__brev(T / 2) >> shi)] = hv;
        sbuf[spad(__brev(Tu - T / 2) >> shi)] = hv;
      } else {
        const int u = ls >= 0 ? ls : Tu + ls;
        sbuf[spad(__brev(u) >> shi)] = v;
      }
    }
    __syncthreads();
    // 4. inverse FFT along depth (unnormalised; scale folded above)
    smem_fft<true>(sbuf, p.log_tu, p.twi, tid, nth);
    for (int d = 0; d < nd; ++d) {
      float2* __restrict__ zr = p.z + (size_t)drow[d] * Tu;
      const float fc = dfac[d];
      for (int i = tid; i < Tu; i += nth) {
        const float2 v = sbuf[spad(i)];
        zr[i] = make_float2(v.x * fc, v.y * fc);
      }
    }
  } else {
    // spectrum only; z was zero-filled and a batched cuFFT does the depth IFFT
    cnt = 0;
    for (int l = tid; l < T; l += nth, ++cnt) {
      const int ls = (l < T / 2) ? l : l - T;
      const float2 v = vals[cnt];
      for (int d = 0; d < nd; ++d) {
        float2* __restrict__ zr = p.z + (size_t)drow[d] * Tu;
        const float fc = dfac[d];
        if (ls == -(T / 2) && p.up > 1) {
          const float2 hv = make_float2(0.5f * fc * v.x, 0.5f * fc * v.y);
          zr[T / 2] = hv;
          zr[Tu - T / 2] = hv;
        } else {
          zr[ls >= 0 ? ls : Tu + ls] = make_float2(fc * v.x, fc * v.y);
        }
      }
    }
  }
}

}  // namespace

size_t ner_smem_bytes(int n_over, int Tu) {
  const int m = n_over > Tu ? n_over : Tu;
  return (size_t)(m + m / 16) * sizeof(float2);
}

int ner_threads(int n_over) {
  int t = n_over / 16;
  if (t < 64) t = 64;
  if (t > 512) t = 512;
  return t;
}

cudaError_t launch_ner(const NerParams& p, int K2, cudaStream_t s) {
  const int threads = ner_threads(p.n_over);
  const size_t smem = ner_smem_bytes(p.n_over, p.fused_ifft ? p.Tu : 0);
  const unsigned rows = (unsigned)(p.N0 * p.N1h);
  cudaError_t err = cudaSuccess;
  auto go = [&](auto kern) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return;
    kern<<<rows, threads, smem, s>>>(p);
    err = cudaGetLastError();
  };
  switch (K2) {
    case 2: go(ner_kernel<2>); break;
    case 4: go(ner_kernel<4>); break;
    case 6: go(ner_kernel<6>); break;
    case 8: go(ner_kernel<8>); break;
    case 10: go(ner_kernel<10>); break;
    case 12: go(ner_kernel<12>); break;
    case 14: go(ner_kernel<14>); break;
    case 16: go(ner_kernel<16>); break;
    default: return cudaErrorInvalidValue;
  }
  return err;
}

// ===========================================================================
// conversions / fills
// ===========================================================================
namespace {
__global__ void f64_to_f32_kernel(const double* __restrict__ s, float* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = (float)s[i];
}
__global__ void f32_to_f64_kernel(const float* __restrict__ s, double* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = (double)s[i];
}
__global__ void fill_kernel(float* __restrict__ d, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = v;
}
unsigned grid_for(size_t n) {
  size_t b = (n + 255) / 256;
  const size_t cap = 148 * 32;
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}
}  // namespace

cudaError_t launch_f64_to_f32(const double* src, float* dst, size_t n, cudaStream_t s) {
  f64_to_f32_kernel<<<grid_for(n), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}
cudaError_t launch_f32_to_f64(const float* src, double* dst, size_t n, cudaStream_t s) {
  f32_to_f64_kernel<<<grid_for(n), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}
cudaError_t launch_fill(float* dst, size_t n, float v, cudaStream_t s) {
  fill_kernel<<<grid_for(n), 256, 0, s>>>(dst, n, v);
  return cudaGetLastError();
}

}  // namespace patfft
