// Reference-length path: the NEDNER stages on the reference's OWN oversampled
// lengths (even 11-smooth, nufft.py:83-89) instead of the power-of-two grids of
// the shared-memory kernels.
//
// An explicit (alpha, beta) window that is inaccurate at the reference's length
// makes the reference return the exact transform PLUS its own truncation /
// aliasing error (up to 1e-3 for admissible but poorly chosen shapes,
// nufft.py:119-149).  A drop-in has to return that same answer, and the error
// depends on the grid length, so such plans run here: same gridding kernels on
// an n_over_ref grid, the uniform FFT stages through cuFFT (any length), and
// two small kernels around them.  This is a compatibility path (taken only
// when the plan's accuracy probe fails, capi.cu), not a tuned one.
//
//   lateral : cuFFT R2C over (rows, cols) for every time sample, then
//             crop_ref_kernel = the rowfft epilogue (crop to the centred box,
//             deapodise, Nyquist-plane Hermitian part; nufft.py:406-415,
//             recon.py:218-222)
//   NER     : ner_ref_prep_kernel (pre-windowed even extension, zero padded;
//             recon.py:263-271, nufft.py:325) -> cuFFT C2C of length n_over ->
//             ner_ref_gather_kernel (2K taps per target with the window
//             transform evaluated directly in float64, nufft.py:287-293; kappa,
//             band, amplitude, recon.py:282-308; zero padding / Nyquist split
//             for upsampling, recon.py:225-246) writing the depth spectrum that
//             the plan's cuFFT inverse consumes.
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>

#include "patfft_internal.h"

namespace patfft {
namespace {

__device__ __forceinline__ int pmodi(int a, int n) {
  const int r = a % n;
  return r < 0 ? r + n : r;
}

// gh[j0w][j1][t] from the oversampled half spectrum X[row][col bin][t]
// and ghd = (own value - conj(Hermitian partner)) / 2, non-zero on the lateral Nyquist planes only
// (see ner_ref_gather_kernel, dpass)
__global__ void crop_ref_kernel(const LateralParams p, const float2* __restrict__ X, int nyo,
                                float2* __restrict__ ghd) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int j1 = blockIdx.y, j0w = blockIdx.z;
  if (t >= p.T) return;
  const int N0 = p.N0, nr = p.nrows;
  const int a = (N0 > 1) ? (j0w < N0 / 2 ? j0w : j0w - N0) : 0;
  const bool nyq0 = (N0 > 1) && (a == -(N0 / 2));
  const bool nyq1 = (j1 == p.N1 / 2);
  auto at = [&](int row) { return X[((size_t)pmodi(row, nr) * nyo + j1) * p.T + t]; };
  float2 v, dv = make_float2(0.f, 0.f);
  if (nyq1) {  // stored j1 = N1/2 is signed -N1/2: X(a, -N1/2) = conj X(-a, +N1/2)
    const float2 v1 = at(-a), v2 = at(nyq0 ? -a : a);
    v = make_float2(0.5f * (v1.x + v2.x), 0.5f * (v2.y - v1.y));
    dv = make_float2(0.5f * (v1.x - v2.x), 0.5f * (-v1.y - v2.y));
  } else if (nyq0) {
    const float2 v1 = at(a), v2 = at(-a);
    v = make_float2(0.5f * (v1.x + v2.x), 0.5f * (v1.y + v2.y));
    dv = make_float2(0.5f * (v1.x - v2.x), 0.5f * (v1.y - v2.y));
  } else {
    v = at(a);
  }
  const float s = p.dp0[j0w] * p.dp1[j1];
  const size_t o = ((size_t)j0w * p.ny + j1) * p.T + t;
  p.gh[o] = make_float2(v.x * s, v.y * s);
  ghd[o] = make_float2(dv.x * s, dv.y * s);
}

// NedPlan (complex values, full spectrum): crop of the in-place C2C spectrum X[row][col][b], the
// centred-grid sign (-1)^(j0+j1), deapodisation, centred or wrapped output order (nufft.py:406-417;
// the rowfft epilogue of lateral.cu for p.cplx)
__global__ void crop_ref_cplx_kernel(const LateralParams p, const float2* __restrict__ X, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int j1 = blockIdx.y, j0w = blockIdx.z;
  if (b >= B) return;
  const int N0 = p.N0, N1 = p.N1;
  const int j1s = j1 < N1 / 2 ? j1 : j1 - N1;
  const int a = (N0 > 1) ? (j0w < N0 / 2 ? j0w : j0w - N0) : 0;
  const float sg = ((a + j1s) & 1) ? -1.f : 1.f;
  const float2 v = X[((size_t)pmodi(a, p.nrows) * p.ncols + pmodi(j1s, p.ncols)) * B + b];
  const float s = sg * p.dp0[j0w] * p.dp1[j1];
  const size_t o = p.centered ? (size_t)(a + N0 / 2) * N1 + (j1s + N1 / 2) : (size_t)j0w * N1 + j1;
  p.gh[o * B + b] = make_float2(v.x * s, v.y * s);
}

// rows [r0, r0 + nrows) of gh -> pre-windowed even extension, zero padded to n_over
__global__ void ner_ref_prep_kernel(const NerParams p, const float2* __restrict__ gh, int r0, int nrows,
                                    float2* __restrict__ fb) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (n >= p.n_over || r >= nrows) return;
  const int T = p.T;
  float2 v = make_float2(0.f, 0.f);
  if (n < 2 * T && n != T) {
    const int t = n < T ? n : 2 * T - n;
    const float2 g = gh[(size_t)(r0 + r) * T + t];
    const float w = p.iw[n];
    v = make_float2(g.x * w, g.y * w);
  }
  fb[(size_t)r * p.n_over + n] = v;
}

__device__ __forceinline__ double psihat_ref(double alpha, double beta, double x) {  // nufft.py:168-187
  const double t = alpha * alpha * (beta * beta - x * x);
  double v;
  if (fabs(t) < 1e-9) v = 1.0 + t / 6.0 + t * t / 120.0;
  else if (t > 0) {
    const double s = sqrt(t);
    v = sinh(s) / s;
  } else {
    const double s = sqrt(-t);
    v = sin(s) / s;
  }
  return 2.0 * alpha * v;
}

// one thread per (row, depth frequency l): the reference's tap sum on the cuFFT spectrum.
//
// Targets with an integer c * kappa_e ("ties").  The reference's tap window for +kappa starts at
// floor(xi) = xi and the one for the Hermitian partner -kappa at floor(-xi) = -xi: the two are not
// mirror images (they are for every other target), and its Hermitian symmetrisation
// (recon.py:218-222) averages what they give: with S0 / S1 the tap sums of the windows at k0 and
// k0 - 1, own = this row's spectrum and part = conj(partner row's),
//   fhat_s = (S0[own] + S1[part]) / 2 = (S0 + S1)[s] / 2 + (S0 - S1)[d] / 2,
// s = (own + part) / 2 (what crop_ref_kernel stores in gh), d = (own - part) / 2 (ghd; zero except on
// the lateral Nyquist planes, whose partner rows are not their conjugates).  dpass = 0 evaluates the
// first term (S0[s] at ordinary targets), dpass = 1 adds the second at the ties of Nyquist-plane rows.
__global__ void ner_ref_gather_kernel(const NerParams p, NerRefWindow w, int r0, int nrows,
                                      const float2* __restrict__ fb, int dpass) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const int rb = blockIdx.y;
  const int T = p.T, n = p.n_over, Tu = p.Tu;
  if (l >= T || rb >= nrows) return;
  const int r = r0 + rb;
  const int j0w = r / p.N1h, j1 = r - j0w * p.N1h;
  if (dpass && !(j1 == p.N1 / 2 || (p.n_lat == 2 && j0w == p.N0 / 2))) return;
  const double j2 = p.jt0[j0w] + p.jt1[j1];
  const double halfT = (double)T / 2.0;
  const int ls = (l < T / 2) ? l : l - T;
  const double lv = __dmul_rn(__dmul_rn((double)ls, 1.0 / (double)T), (double)T);  // fftfreq(T)*T
  const double r2 = __dadd_rn(j2, __dmul_rn(lv, lv));
  float2 out = make_float2(0.f, 0.f);
  if (ls != 0 && r2 <= halfT * halfT) {
    double kap = sqrt(r2);
    if (ls < 0) kap = -kap;
    const double ke = 2.0 * kap;
    const double xi = __dmul_rn(p.c_eff, ke);
    const double k0 = floor(xi);
    // At an integer c * kappa_e the reference's tap windows for +kappa (floor(xi) = xi) and for the
    // Hermitian partner -kappa (floor(-xi) = -xi) are not mirror images, and its Hermitian
    // symmetrisation (recon.py:218-222) averages the two: the window at k0 and the one at k0 - 1.
    const bool tie = xi == k0;
    if (dpass && !tie) return;
    const float2* __restrict__ row = fb + (size_t)rb * n;
    double ar = 0.0, ai = 0.0;
    for (int sh = 0; sh <= (tie ? 1 : 0); ++sh) {
      const double sg = (dpass && sh) ? -1.0 : 1.0;  // S0 + S1, or S0 - S1 in the difference pass
      for (int a = -w.K + 1; a <= w.K; ++a) {
        const double bin = k0 + (double)(a - sh);
        const double off = ke - bin / p.c_eff;
        const double wt = sg * psihat_ref(w.alpha, w.beta, off) * w.inv_psihat0;  // iw[] carries psihat(0) * norm
        double sn, cs;
        sincospi(-off, &sn, &cs);
        const float2 F = row[pmodi((int)bin, n)];
        ar += wt * (cs * F.x - sn * F.y);
        ai += wt * (cs * F.y + sn * F.x);
      }
    }
    if (tie) {
      ar *= 0.5;
      ai *= 0.5;
    }
    const double amp = 0.5 * (2.0 * lv / kap) * (double)p.scale;
    out = make_float2((float)(amp * ar), (float)(amp * ai));
  }
  // destination rows of the (possibly upsampled) half spectrum z (recon.py:225-246)
  int j0u = 0, j0u2 = -1;
  float f0 = 1.f;
  if (p.n_lat == 2) {
    const int a = j0w < p.N0 / 2 ? j0w : j0w - p.N0;
    if (p.up == 1) j0u = j0w;
    else if (a == -(p.N0 / 2)) {
      j0u = p.N0 / 2;
      j0u2 = p.N0u - p.N0 / 2;
      f0 = 0.5f;
    } else j0u = a >= 0 ? a : p.N0u + a;
  }
  const float f1 = (p.up > 1 && j1 == p.N1 / 2) ? 0.5f : 1.f;
  const float2 v = make_float2(out.x * f0 * f1, out.y * f0 * f1);
  for (int d = 0; d < (j0u2 >= 0 ? 2 : 1); ++d) {
    float2* __restrict__ zr = p.z + ((size_t)(d ? j0u2 : j0u) * p.N1uh + j1) * Tu;
    auto put = [&](int i, float2 x) {
      if (dpass) x = make_float2(zr[i].x + x.x, zr[i].y + x.y);
      zr[i] = x;
    };
    if (ls == -(T / 2) && p.up > 1) {
      put(T / 2, make_float2(0.5f * v.x, 0.5f * v.y));
      put(Tu - T / 2, make_float2(0.5f * v.x, 0.5f * v.y));
    } else {
      put(ls >= 0 ? ls : Tu + ls, v);
    }
  }
}

}  // namespace

cudaError_t launch_lateral_ref(const LateralParams& p, cudaStream_t s) {
  const LatRef* R = p.ref;
  if (p.t_begin != 0 || p.t_end != p.T) return cudaErrorInvalidValue;  // whole record only
  if (cufftSetStream(R->r2c, s) != CUFFT_SUCCESS) return cudaErrorUnknown;
  if (cufftExecR2C(R->r2c, const_cast<float*>(p.grid), reinterpret_cast<cufftComplex*>(R->spec)) != CUFFT_SUCCESS)
    return cudaErrorUnknown;
  const dim3 grid((unsigned)((p.T + 127) / 128), (unsigned)p.ny, (unsigned)p.N0);
  crop_ref_kernel<<<grid, 128, 0, s>>>(p, R->spec, R->nyo, R->ghd);
  return cudaGetLastError();
}

// NedPlan on the reference's lengths: in-place C2C over (rows, cols) of the complex grid, then the crop
cudaError_t launch_lateral_ref_cplx(const LateralParams& p, int B, cudaStream_t s) {
  const LatRef* R = p.ref;
  float2* X = reinterpret_cast<float2*>(const_cast<float*>(p.grid));
  if (cufftSetStream(R->c2c, s) != CUFFT_SUCCESS) return cudaErrorUnknown;
  if (cufftExecC2C(R->c2c, reinterpret_cast<cufftComplex*>(X), reinterpret_cast<cufftComplex*>(X), CUFFT_FORWARD) !=
      CUFFT_SUCCESS)
    return cudaErrorUnknown;
  const dim3 grid((unsigned)((B + 127) / 128), (unsigned)p.N1, (unsigned)p.N0);
  crop_ref_cplx_kernel<<<grid, 128, 0, s>>>(p, X, B);
  return cudaGetLastError();
}

cudaError_t launch_ner_ref(const NerParams& p, cudaStream_t s) {
  const NerRef* R = p.ref;
  const int rows = p.N0 * p.N1h;
  if (cufftSetStream(R->c2c, s) != CUFFT_SUCCESS) return cudaErrorUnknown;
  for (int dpass = 0; dpass < 2; ++dpass)  // 0: symmetrised rows (gh); 1: difference rows (ghd) at the ties
    for (int r0 = 0; r0 < rows; r0 += R->rows_blk) {
      const int nb = std::min(R->rows_blk, rows - r0);
      ner_ref_prep_kernel<<<dim3((unsigned)((p.n_over + 255) / 256), (unsigned)nb), 256, 0, s>>>(
          p, dpass ? R->ghd : p.gh, r0, nb, R->fb);
      // the plan transforms rows_blk rows; the rows past nb of the last block are stale but unused
      if (cufftExecC2C(R->c2c, reinterpret_cast<cufftComplex*>(R->fb), reinterpret_cast<cufftComplex*>(R->fb),
                       CUFFT_FORWARD) != CUFFT_SUCCESS)
        return cudaErrorUnknown;
      ner_ref_gather_kernel<<<dim3((unsigned)((p.T + 127) / 128), (unsigned)nb), 128, 0, s>>>(p, R->win, r0, nb,
                                                                                               R->fb, dpass);
    }
  return cudaGetLastError();
}

}  // namespace patfft
