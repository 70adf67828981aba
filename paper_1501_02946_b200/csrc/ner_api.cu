// Standalone non-equispaced-range NUFFT (the reference's NerPlan,
// nufft.py:270-338): out[r, i] ~= sum_k u[r, k] exp(-2 pi i kappa[r, i] k / n).
// One CTA per row: pre-window + rotation by -n/2 into shared memory (so the
// FFT output already carries exp(i pi bin / c) and only one phase
// exp(-i pi kappa) per target remains), radix-16 FFT of length n_over, and a
// 2K-tap Kaiser-Bessel interpolation per target with polynomial tap weights.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fft_smem.cuh"
#include "patfft_internal.h"

namespace patfft {
namespace {

struct NerApiParams {
  const float2* u;       // [rows][n]
  const double* kap;     // [rows][m] or [m] (shared)
  float2* out;           // [rows][m]
  const float* iw;       // [n] psihat(0) * norm / psi(2 pi k/n - pi)
  const float2* tw;      // exp(-2 pi i k / 2^14)
  int n, n_over, L, rows, m, shared;
  double c_eff;
  float poly[kMaxTaps / 2][kMaxPolyDegree + 1];
};

__device__ __forceinline__ float2 cospi_sinpi_api(float r) {
  const float q = rintf(2.f * r);
  const float x = 3.14159265358979f * fmaf(-0.5f, q, r);
  const float x2 = x * x;
  const float s = x * fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, 2.7557319e-6f, -1.98412698e-4f), 8.33333333e-3f),
                                    -0.166666667f), 1.f);
  const float c = fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, -2.7557319e-7f, 2.48015873e-5f), -1.38888889e-3f),
                                          4.16666667e-2f), -0.5f), 1.f);
  switch (((int)q) & 3) {
    case 0: return make_float2(c, s);
    case 1: return make_float2(-s, c);
    case 2: return make_float2(-c, -s);
    default: return make_float2(s, -c);
  }
}

// ---- reference-length form (windows whose approximation error the reference's answer carries, see
// capi.cu / reflen.cu): pre-window + zero padding to the reference's n_over, cuFFT, and the
// reference's own tap sum per target (nufft.py:287-293, floor() bins, window transform in float64)
__global__ void nerplan_ref_prep_kernel(const NerApiParams p, int r0, int nrows, float2* __restrict__ fb) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
  if (k >= p.n_over || r >= nrows) return;
  float2 v = make_float2(0.f, 0.f);
  if (k < p.n) {
    const float2 g = p.u[(size_t)(r0 + r) * p.n + k];
    const float w = p.iw[k];
    v = make_float2(g.x * w, g.y * w);
  }
  fb[(size_t)r * p.n_over + k] = v;
}

__global__ void nerplan_ref_gather_kernel(const NerApiParams p, int r0, int nrows, const float2* __restrict__ fb,
                                          double alpha, double beta, double inv_psihat0, int K) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, rb = blockIdx.y;
  if (i >= p.m || rb >= nrows) return;
  const int r = r0 + rb;
  const double ke = p.shared ? p.kap[i] : p.kap[(size_t)r * p.m + i];
  const double k0 = floor(__dmul_rn(p.c_eff, ke));
  const float2* __restrict__ row = fb + (size_t)rb * p.n_over;
  double ar = 0.0, ai = 0.0;
  for (int a = -K + 1; a <= K; ++a) {
    const double bin = k0 + (double)a;
    const double off = ke - bin / p.c_eff;
    const double t = alpha * alpha * (beta * beta - off * off);  // nufft.py:168-187
    double v;
    if (fabs(t) < 1e-9) v = 1.0 + t / 6.0 + t * t / 120.0;
    else if (t > 0) v = sinh(sqrt(t)) / sqrt(t);
    else v = sin(sqrt(-t)) / sqrt(-t);
    const double wt = 2.0 * alpha * v * inv_psihat0;  // iw[] carries psihat(0) * norm
    double sn, cs;
    sincospi(-off, &sn, &cs);
    int b = (int)fmod(bin, (double)p.n_over);
    if (b < 0) b += p.n_over;
    const float2 F = row[b];
    ar += wt * (cs * F.x - sn * F.y);
    ai += wt * (cs * F.y + sn * F.x);
  }
  p.out[(size_t)r * p.m + i] = make_float2((float)ar, (float)ai);
}

template <int K2, int D>
__global__ void __launch_bounds__(512) nerplan_kernel(const NerApiParams p) {
  extern __shared__ float2 sbuf[];
  constexpr int K = K2 / 2;
  const int row = blockIdx.x;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int n = p.n, no = p.n_over, L = p.L;
  const fft::SwzAddr ad = fft::SwzAddr::for_log(L);
  const float2* __restrict__ u = p.u + (size_t)row * n;
  fft::staged_copy<8, float2>(
      no, tid, nth,
      [&](int s) {
        const int i = (s + n / 2) & (no - 1);  // sequence index stored at slot s
        return i < n ? fft::cscale(__ldcs(&u[i]), __ldg(&p.iw[i])) : make_float2(0.f, 0.f);
      },
      [&](int s, float2 v) { sbuf[ad(fft::brev(s, L), 0)] = v; });
  __syncthreads();
  fft::fft_inplace<false, 4, true>(sbuf, L, 0, p.tw, tid, nth, ad);
  const double* __restrict__ kap = p.shared ? p.kap : p.kap + (size_t)row * p.m;
  float2* __restrict__ out = p.out + (size_t)row * p.m;
  for (int i = tid; i < p.m; i += nth) {
    const double kv = __ldg(&kap[i]);
    const double xi = __dmul_rn(p.c_eff, kv);
    const double k0d = floor(xi);
    const int k0 = (int)k0d;
    const float z = (float)(xi - k0d) - 0.5f;
    const float z2 = z * z;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      float e = p.poly[j][D], o = p.poly[j][D - 1];
#pragma unroll
      for (int d = D - 2; d >= 0; d -= 2) e = fmaf(e, z2, p.poly[j][d]);
#pragma unroll
      for (int d = D - 3; d >= 1; d -= 2) o = fmaf(o, z2, p.poly[j][d]);
      const float wa = fmaf(z, o, e);
      const float wb = fmaf(-z, o, e);
      const float2 Fa = sbuf[ad((k0 + j - K + 1) & (no - 1), 0)];
      const float2 Fb = sbuf[ad((k0 + K - j) & (no - 1), 0)];
      acc.x = fmaf(wa, Fa.x, fmaf(wb, Fb.x, acc.x));
      acc.y = fmaf(wa, Fa.y, fmaf(wb, Fb.y, acc.y));
    }
    const double red = kv - 2.0 * floor(0.5 * kv + 0.5);  // exp(-i pi kappa)
    const float2 cs = cospi_sinpi_api((float)red);
    out[i] = make_float2(acc.x * cs.x + acc.y * cs.y, acc.y * cs.x - acc.x * cs.y);
  }
}

__global__ void c128_to_c64(const double2* __restrict__ s, float2* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = make_float2((float)s[i].x, (float)s[i].y);
}
__global__ void c64_to_c128(const float2* __restrict__ s, double2* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = make_double2(s[i].x, s[i].y);
}


// ---------------------------------------------------------------------------
// Forward model (the reference's forward_fourier, forward.py:105-166): per
// lateral half-spectrum row j, the detected depth spectrum
//   ghat(j, w) = w / (2 ky) * [fh(j, +ky) + fh(j, -ky)],  ky = sqrt(w^2 - |j|^2)
// on the doubled window (2 N_t frequencies w = k/2), zero where |w| <= |j|
// (forward.py:138-153), followed by the depth inverse FFT truncated to the
// first N_t samples (forward.py:155).  fh(j, kappa) is the NER transform of
// the laterally transformed field row; ghat is even in w, so only the
// N_t + 1 values |w| = k/2, k = 0..N_t are evaluated and mirrored.  One CTA
// per row: forward FFT (length n_over) and inverse FFT (length 2 N_t <=
// n_over) both in shared memory, the row overwritten in place.
// ---------------------------------------------------------------------------
struct FwdParams {
  NerApiParams q;       // u/out = the [rows][T] spectrum (in place)
  const double* j2;     // [N0][N1] squared lateral frequency, wrapped (recon.py:200-215)
  int N1, N1h, T, LT;   // LT = log2(2 T)
  float scale;          // 1 / (2 T N0 N1): scipy ifft / ifftn normalisation
};

template <int K2, int D>
__device__ __forceinline__ float2 ner_tap_sum(const NerApiParams& p, const float2* sbuf, fft::SwzAddr ad, double kv) {
  constexpr int K = K2 / 2;
  const int no = p.n_over;
  const double xi = __dmul_rn(p.c_eff, kv);
  const double k0d = floor(xi);
  const int k0 = (int)k0d;
  const float z = (float)(xi - k0d) - 0.5f;
  const float z2 = z * z;
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    float e = p.poly[j][D], o = p.poly[j][D - 1];
#pragma unroll
    for (int d = D - 2; d >= 0; d -= 2) e = fmaf(e, z2, p.poly[j][d]);
#pragma unroll
    for (int d = D - 3; d >= 1; d -= 2) o = fmaf(o, z2, p.poly[j][d]);
    const float wa = fmaf(z, o, e);
    const float wb = fmaf(-z, o, e);
    const float2 Fa = sbuf[ad((k0 + j - K + 1) & (no - 1), 0)];
    const float2 Fb = sbuf[ad((k0 + K - j) & (no - 1), 0)];
    acc.x = fmaf(wa, Fa.x, fmaf(wb, Fb.x, acc.x));
    acc.y = fmaf(wa, Fa.y, fmaf(wb, Fb.y, acc.y));
  }
  const double red = kv - 2.0 * floor(0.5 * kv + 0.5);  // exp(-i pi kappa)
  const float2 cs = cospi_sinpi_api((float)red);
  return make_float2(acc.x * cs.x + acc.y * cs.y, acc.y * cs.x - acc.x * cs.y);
}

template <int K2, int D>
__global__ void __launch_bounds__(512) forward_kernel(const FwdParams f) {
  extern __shared__ float2 sbuf[];
  const NerApiParams& p = f.q;
  const int row = blockIdx.x;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int n = p.n, no = p.n_over, L = p.L, T = f.T, LT = f.LT;
  const fft::SwzAddr ad = fft::SwzAddr::for_log(L);
  const fft::SwzAddr adg = fft::SwzAddr::for_log(LT);
  float2* gbuf = sbuf + no;
  float2* __restrict__ u = p.out + (size_t)row * n;
  fft::staged_copy<8, float2>(
      no, tid, nth,
      [&](int s) {
        const int i = (s + n / 2) & (no - 1);
        return i < n ? fft::cscale(u[i], __ldg(&p.iw[i])) : make_float2(0.f, 0.f);
      },
      [&](int s, float2 v) { sbuf[ad(fft::brev(s, L), 0)] = v; });
  __syncthreads();
  fft::fft_inplace<false, 4, true>(sbuf, L, 0, p.tw, tid, nth, ad);
  const int j0 = row / f.N1h, j1 = row - j0 * f.N1h;
  const double j2 = __ldg(&f.j2[(size_t)j0 * f.N1 + j1]);
  for (int k = tid; k <= T; k += nth) {
    const double w = 0.5 * k, w2 = w * w;
    float2 g = make_float2(0.f, 0.f);
    if (j2 < w2) {  // propagating (strict, forward.py:145)
      const double ky = sqrt(w2 - j2);
      const float2 a = ner_tap_sum<K2, D>(p, sbuf, ad, ky);
      const float2 b = ner_tap_sum<K2, D>(p, sbuf, ad, -ky);
      const float s = (float)(w / (2.0 * ky)) * f.scale;  // forward.py:148
      g = make_float2((a.x + b.x) * s, (a.y + b.y) * s);
    }
    gbuf[adg(fft::brev(k, LT), 0)] = g;
    if (k > 0 && k < T) gbuf[adg(fft::brev(2 * T - k, LT), 0)] = g;
  }
  __syncthreads();
  fft::fft_inplace<true, 4, true>(gbuf, LT, 0, p.tw, tid, nth, adg);
  for (int t = tid; t < T; t += nth) u[t] = gbuf[adg(t, 0)];
}

}  // namespace
int set_last_error(int code, const std::string& msg);  // capi.cu
}  // namespace patfft

using namespace patfft;

struct patfft_ner_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  int n = 0, n_over = 0, K2 = 12, degree = 8;
  Window win;
  // reference-length form: n_over is the reference's even 11-smooth length, cuFFT transforms ref_blk rows at a time
  bool ref_len = false;
  cufftHandle ref_c2c = 0;
  float2* d_ref_fb = nullptr;
  int ref_blk = 0;
  NerApiParams prm{};
  float* d_iw = nullptr;
  float2* d_tw = nullptr;
  // host-path staging
  size_t cap_u64 = 0, cap_u = 0, cap_k = 0, cap_o = 0, cap_o64 = 0;
  double2* d_u64 = nullptr;
  float2* d_u = nullptr;
  double* d_k = nullptr;
  float2* d_o = nullptr;
  double2* d_o64 = nullptr;
};

namespace {
int api_fail(int code, const std::string& m) { return set_last_error(code, m); }
#define API_CUDA(expr)                                                                              \
  do {                                                                                              \
    cudaError_t _e = (expr);                                                                        \
    if (_e != cudaSuccess) return api_fail(PATFFT_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

unsigned gridn(size_t n) {
  const size_t b = (n + 255) / 256;
  return (unsigned)std::max<size_t>(1, std::min<size_t>(b, 148 * 32));
}

int launch_nerplan(patfft_ner_plan* P, const float2* u, const double* kap, int rows, int m, int shared, float2* out,
                   cudaStream_t s) {
  NerApiParams q = P->prm;
  q.u = u;
  q.kap = kap;
  q.out = out;
  q.rows = rows;
  q.m = m;
  q.shared = shared;
  if (P->ref_len) {
    if (cufftSetStream(P->ref_c2c, s) != CUFFT_SUCCESS) return api_fail(PATFFT_ERR_CUDA, "cufftSetStream");
    const double psh0 = kb_psihat(P->win, 0.0);
    for (int r0 = 0; r0 < rows; r0 += P->ref_blk) {
      const int nb = std::min(P->ref_blk, rows - r0);
      nerplan_ref_prep_kernel<<<dim3((unsigned)((P->n_over + 255) / 256), (unsigned)nb), 256, 0, s>>>(q, r0, nb,
                                                                                                   P->d_ref_fb);
      if (cufftExecC2C(P->ref_c2c, reinterpret_cast<cufftComplex*>(P->d_ref_fb),
                       reinterpret_cast<cufftComplex*>(P->d_ref_fb), CUFFT_FORWARD) != CUFFT_SUCCESS)
        return api_fail(PATFFT_ERR_CUDA, "cufftExecC2C");
      if (m > 0)
        nerplan_ref_gather_kernel<<<dim3((unsigned)((m + 127) / 128), (unsigned)nb), 128, 0, s>>>(
            q, r0, nb, P->d_ref_fb, P->win.alpha, P->win.beta, 1.0 / psh0, P->win.K);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return api_fail(PATFFT_ERR_CUDA, cudaGetErrorString(e));
    return PATFFT_OK;
  }
  int threads = P->n_over / 16;
  threads = std::max(64, std::min(512, threads));
  const size_t smem = (size_t)P->n_over * sizeof(float2);
  cudaError_t err = cudaSuccess;
  auto go = [&](auto k) {
    err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err == cudaSuccess && rows > 0) {
      k<<<rows, threads, smem, s>>>(q);
      err = cudaGetLastError();
    }
  };
#define PATFFT_NERAPI_CASE(k2)                     \
  case k2:                                         \
    if (P->degree == 8) go(nerplan_kernel<k2, 8>); \
    else go(nerplan_kernel<k2, 12>);               \
    break;
  switch (P->K2) {
    PATFFT_NERAPI_CASE(2) PATFFT_NERAPI_CASE(4) PATFFT_NERAPI_CASE(6) PATFFT_NERAPI_CASE(8)
    PATFFT_NERAPI_CASE(10) PATFFT_NERAPI_CASE(12) PATFFT_NERAPI_CASE(14) PATFFT_NERAPI_CASE(16)
    default: return api_fail(PATFFT_ERR_PARAMETER, "unsupported K");
  }
#undef PATFFT_NERAPI_CASE
  if (err != cudaSuccess) return api_fail(PATFFT_ERR_CUDA, cudaGetErrorString(err));
  return PATFFT_OK;
}

template <typename T>
int ensure(T** p, size_t* cap, size_t need) {
  if (*cap >= need && *p) return PATFFT_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  API_CUDA(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(1, need) * sizeof(T)));
  *cap = need;
  return PATFFT_OK;
}
}  // namespace

struct patfft_forward_plan {
  int device = 0;
  std::mutex mu;
  patfft_ner_plan* ner = nullptr;  // NerPlan(N_t, spec) tables (forward.py:151)
  int n_lat = 1, N0 = 1, N1 = 0, N1h = 0, T = 0;
  size_t L = 0, Lh = 0;
  double* d_j2 = nullptr;          // [N0][N1]
  float* d_field = nullptr;        // host path staging [N0][N1][T] f32
  double* d_f64 = nullptr;         // host path staging f64 (field in, traces out)
  float2* d_spec = nullptr;        // [N0][N1h][T]
  cufftHandle r2c = 0, c2r = 0;
  bool have_r2c = false, have_c2r = false;
  // power-of-two lateral grids: the reconstruction's own shared-memory lateral FFT kernels
  // (lateral.cu) instead of cuFFT's stride-N_t transforms
  bool custom_lateral = false;
  float2* d_Y = nullptr;           // [N0][N1h][T] column-transformed half spectrum
  float* d_ones = nullptr;         // max(N0, N1) ones: no deapodisation
  LateralParams lat{};
};

namespace {
#define API_CUFFT(expr)                                                                    \
  do {                                                                                     \
    cufftResult _r = (expr);                                                               \
    if (_r != CUFFT_SUCCESS)                                                               \
      return api_fail(PATFFT_ERR_CUDA, std::string(#expr) + " failed (" + std::to_string((int)_r) + ")"); \
  } while (0)

int launch_forward(patfft_forward_plan* F, const float* field, float* traces, cudaStream_t s) {
  patfft_ner_plan* P = F->ner;
  if (F->custom_lateral) {
    // plain lateral FFT of the full grid: the column / row kernels with no oversampling, no crop
    // and unit deapodisation (their Nyquist-plane Hermitian part is the identity on such a grid)
    LateralParams L = F->lat;
    L.grid = field;
    cudaError_t e = launch_lateral_col(L, s);
    if (e == cudaSuccess) e = launch_lateral_row(L, s);
    if (e != cudaSuccess) return api_fail(PATFFT_ERR_CUDA, cudaGetErrorString(e));
  } else {
    API_CUFFT(cufftSetStream(F->r2c, s));
    API_CUFFT(cufftSetStream(F->c2r, s));
    API_CUFFT(cufftExecR2C(F->r2c, const_cast<float*>(field), reinterpret_cast<cufftComplex*>(F->d_spec)));
  }
  FwdParams f{};
  f.q = P->prm;
  f.q.u = F->d_spec;
  f.q.out = F->d_spec;
  f.q.rows = (int)F->Lh;
  f.j2 = F->d_j2;
  f.N1 = F->N1;
  f.N1h = F->N1h;
  f.T = F->T;
  int LT = 0;
  while ((1 << LT) < 2 * F->T) ++LT;
  f.LT = LT;
  f.scale = (float)(1.0 / (2.0 * F->T * (double)F->L));
  const int threads = std::max(64, std::min(512, P->n_over / 16));
  const size_t smem = (size_t)(P->n_over + 2 * F->T) * sizeof(float2);
  cudaError_t err = cudaSuccess;
  auto go = [&](auto k) {
    err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err == cudaSuccess) {
      k<<<(unsigned)F->Lh, threads, smem, s>>>(f);
      err = cudaGetLastError();
    }
  };
#define PATFFT_FWD_CASE(k2)                        \
  case k2:                                         \
    if (P->degree == 8) go(forward_kernel<k2, 8>); \
    else go(forward_kernel<k2, 12>);               \
    break;
  switch (P->K2) {
    PATFFT_FWD_CASE(2) PATFFT_FWD_CASE(4) PATFFT_FWD_CASE(6) PATFFT_FWD_CASE(8)
    PATFFT_FWD_CASE(10) PATFFT_FWD_CASE(12) PATFFT_FWD_CASE(14) PATFFT_FWD_CASE(16)
    default: return api_fail(PATFFT_ERR_PARAMETER, "unsupported K");
  }
#undef PATFFT_FWD_CASE
  if (err != cudaSuccess) return api_fail(PATFFT_ERR_CUDA, cudaGetErrorString(err));
  if (F->custom_lateral) {
    LateralParams L = F->lat;
    L.out = traces;
    const cudaError_t e = launch_lateral_inverse(L, s);
    if (e != cudaSuccess) return api_fail(PATFFT_ERR_CUDA, cudaGetErrorString(e));
    return PATFFT_OK;
  }
  API_CUFFT(cufftExecC2R(F->c2r, reinterpret_cast<cufftComplex*>(F->d_spec), traces));
  return PATFFT_OK;
}
}  // namespace

// host-side helpers defined in capi.cu
namespace patfft {
double fit_ner_poly_public(const Window& w, int D, float (*poly)[kMaxPolyDegree + 1]);
}

extern "C" {

int patfft_ner_plan_create(int n, double c, int K, double alpha, double beta, int device, patfft_ner_plan** out) {
  if (!out) return api_fail(PATFFT_ERR_PARAMETER, "null argument");
  *out = nullptr;
  if (n < 2) return api_fail(PATFFT_ERR_PARAMETER, "input length must be >= 2");  // nufft.py:274-275
  if (n % 2) return api_fail(PATFFT_ERR_UNSUPPORTED, "GPU NerPlan supports even lengths");
  if (!(std::isfinite(c) && c > 1.0)) return api_fail(PATFFT_ERR_PARAMETER, "oversampling factor must exceed 1");
  if (K < 1) return api_fail(PATFFT_ERR_PARAMETER, "interpolation half-width K must be an integer >= 1");
  if (K > kMaxTaps / 2) return api_fail(PATFFT_ERR_UNSUPPORTED, "GPU path supports interpolation half-width K <= 8");
  int64_t no = 1;
  while (no < (int64_t)std::ceil(c * n)) no <<= 1;
  if (no > 16384) return api_fail(PATFFT_ERR_UNSUPPORTED, "GPU NerPlan supports oversampled lengths up to 16384");
  std::unique_ptr<patfft_ner_plan, void (*)(patfft_ner_plan*)> P(new patfft_ner_plan(), &patfft_ner_plan_destroy);
  P->device = device;
  API_CUDA(cudaSetDevice(device));
  P->n = n;
  P->n_over = (int)no;
  P->K2 = 2 * K;
  std::string err;
  if (!resolve_window(c, K, alpha, beta, double(no) / n, &P->win, &err)) return api_fail(PATFFT_ERR_PARAMETER, err);
  // The fast kernel (power-of-two length, rotated input) returns the exact transform when the window
  // is accurate; the reference's answer with an inaccurate window (small K, poor alpha / beta) depends
  // on its own even 11-smooth length and tap sums, so such plans run the reference-length form.
  const int nref = even_fast_len(c * n);
  const bool explicit_window = !std::isnan(alpha) || !std::isnan(beta);
  if (explicit_window || K < 6 || c < 2.0) {
    auto accuracy = [](Window w, int len, int len_over) {
      if (len > 256) {
        len_over = (int)std::lround(double(len_over) / len * 256.0);
        len = 256;
        w.c_eff = double(len_over) / len;
      }
      return window_relative_error(w, len, len_over);
    };
    Window wref;
    if (!resolve_window(c, K, alpha, beta, double(nref) / n, &wref, &err)) return api_fail(PATFFT_ERR_PARAMETER, err);
    if (!(accuracy(wref, n, nref) <= 1e-6) || (nref != no && !(accuracy(P->win, n, (int)no) <= 1e-6))) {
      P->ref_len = true;
      P->win = wref;
      P->n_over = nref;
    }
  }
  const double s0 = kb_psihat(P->win, 0.0), norm = 1.0 / (2.0 * M_PI * P->win.c_eff);
  std::vector<float> iw(n);
  for (int k = 0; k < n; ++k) iw[k] = (float)(s0 * norm / kb_psi(P->win, 2.0 * M_PI * k / n - M_PI));
  const std::vector<float2> tw = make_twiddles();
  P->degree = 8;
  if (P->ref_len) {
    P->ref_blk = (int)std::max<int64_t>(1, std::min<int64_t>(4096, ((int64_t)1 << 24) / P->n_over));
    API_CUDA(cudaMalloc(&P->d_ref_fb, (size_t)P->ref_blk * P->n_over * sizeof(float2)));
    int nl[1] = {P->n_over};
    if (cufftPlanMany(&P->ref_c2c, 1, nl, nl, 1, P->n_over, nl, 1, P->n_over, CUFFT_C2C, P->ref_blk) != CUFFT_SUCCESS)
      return api_fail(PATFFT_ERR_CUDA, "cufftPlanMany (reference-length NerPlan)");
  } else if (fit_ner_poly_public(P->win, 8, P->prm.poly) > 2e-8) {
    P->degree = 12;
    if (fit_ner_poly_public(P->win, 12, P->prm.poly) > 1e-6)
      return api_fail(PATFFT_ERR_UNSUPPORTED, "window transform not representable by the tap polynomials");
  }
  API_CUDA(cudaMalloc(&P->d_iw, n * sizeof(float)));
  API_CUDA(cudaMemcpy(P->d_iw, iw.data(), n * sizeof(float), cudaMemcpyHostToDevice));
  API_CUDA(cudaMalloc(&P->d_tw, tw.size() * sizeof(float2)));
  API_CUDA(cudaMemcpy(P->d_tw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice));
  API_CUDA(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
  NerApiParams& q = P->prm;
  q.iw = P->d_iw;
  q.tw = P->d_tw;
  q.n = n;
  q.n_over = P->n_over;  // (the reference's length in the reference-length form)
  int L = 0;
  while ((1 << L) < no) ++L;
  q.L = L;
  q.c_eff = P->win.c_eff;
  *out = P.release();
  return PATFFT_OK;
}

int patfft_ner_plan_info(const patfft_ner_plan* P, int64_t info[4]) {
  if (!P || !info) return api_fail(PATFFT_ERR_PARAMETER, "null argument");
  info[0] = P->n;
  info[1] = P->n_over;
  info[2] = P->K2;
  info[3] = P->degree;
  return PATFFT_OK;
}

int patfft_ner_execute_device(patfft_ner_plan* P, const void* u, const double* kappas, int rows, int m, int shared,
                              void* out, void* stream) {
  if (!P || (!u && rows) || (!kappas && m) || (!out && rows && m)) return api_fail(PATFFT_ERR_PARAMETER, "null argument");
  std::lock_guard<std::mutex> lk(P->mu);
  API_CUDA(cudaSetDevice(P->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P->stream;
  if (rows == 0 || m == 0) return PATFFT_OK;
  return launch_nerplan(P, static_cast<const float2*>(u), kappas, rows, m, shared, static_cast<float2*>(out), st);
}

int patfft_ner_execute(patfft_ner_plan* P, const double* u, const double* kappas, int rows, int m, int shared,
                       double* out) {
  if (!P) return api_fail(PATFFT_ERR_PARAMETER, "null plan");
  if (rows == 0 || m == 0) return PATFFT_OK;
  if (!u || !kappas || !out) return api_fail(PATFFT_ERR_PARAMETER, "null argument");
  std::lock_guard<std::mutex> lk(P->mu);
  API_CUDA(cudaSetDevice(P->device));
  cudaStream_t st = P->stream;
  const size_t nu = (size_t)rows * P->n, nk = shared ? (size_t)m : (size_t)rows * m, no = (size_t)rows * m;
  int rc;
  if ((rc = ensure(&P->d_u64, &P->cap_u64, nu))) return rc;
  if ((rc = ensure(&P->d_u, &P->cap_u, nu))) return rc;
  if ((rc = ensure(&P->d_k, &P->cap_k, nk))) return rc;
  if ((rc = ensure(&P->d_o, &P->cap_o, no))) return rc;
  if ((rc = ensure(&P->d_o64, &P->cap_o64, no))) return rc;
  API_CUDA(cudaMemcpyAsync(P->d_u64, u, nu * sizeof(double2), cudaMemcpyHostToDevice, st));
  API_CUDA(cudaMemcpyAsync(P->d_k, kappas, nk * sizeof(double), cudaMemcpyHostToDevice, st));
  c128_to_c64<<<gridn(nu), 256, 0, st>>>(P->d_u64, P->d_u, nu);
  if ((rc = launch_nerplan(P, P->d_u, P->d_k, rows, m, shared, P->d_o, st))) return rc;
  c64_to_c128<<<gridn(no), 256, 0, st>>>(P->d_o, P->d_o64, no);
  API_CUDA(cudaMemcpyAsync(out, P->d_o64, no * sizeof(double2), cudaMemcpyDeviceToHost, st));
  API_CUDA(cudaStreamSynchronize(st));
  return PATFFT_OK;
}

void patfft_ner_plan_destroy(patfft_ner_plan* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  if (P->stream) cudaStreamSynchronize(P->stream);
  for (void* p : {(void*)P->d_iw, (void*)P->d_tw, (void*)P->d_u64, (void*)P->d_u, (void*)P->d_k, (void*)P->d_o,
                  (void*)P->d_o64})
    if (p) cudaFree(p);
  if (P->d_ref_fb) cudaFree(P->d_ref_fb);
  if (P->ref_c2c) cufftDestroy(P->ref_c2c);
  if (P->stream) cudaStreamDestroy(P->stream);
  delete P;
}

int patfft_forward_plan_create(int n_lat, const int32_t* n_lateral, int n_time, const double* j2, double c, int K,
                               double alpha, double beta, int device, patfft_forward_plan** out) {
  if (!out || !n_lateral || !j2) return api_fail(PATFFT_ERR_PARAMETER, "null argument");
  *out = nullptr;
  if (n_lat != 1 && n_lat != 2) return api_fail(PATFFT_ERR_PARAMETER, "forward operator supports 2D and 3D fields");
  const int N0 = n_lat == 2 ? n_lateral[0] : 1, N1 = n_lateral[n_lat - 1];
  if (n_time < 2 || n_time % 2 || N1 < 2 || N1 % 2 || (n_lat == 2 && (N0 < 2 || N0 % 2)))
    return api_fail(PATFFT_ERR_PARAMETER, "grid sizes must be even");  // forward.py:118-119
  if (n_time & (n_time - 1)) return api_fail(PATFFT_ERR_UNSUPPORTED, "GPU forward model needs a power-of-two N_t");
  if (2 * (int64_t)n_time > 8192) return api_fail(PATFFT_ERR_UNSUPPORTED, "GPU forward model supports N_t <= 4096");
  std::unique_ptr<patfft_forward_plan, void (*)(patfft_forward_plan*)> F(new patfft_forward_plan(),
                                                                          &patfft_forward_plan_destroy);
  F->device = device;
  int rc = patfft_ner_plan_create(n_time, c, K, alpha, beta, device, &F->ner);
  if (rc) return rc;
  if (F->ner->ref_len)
    return api_fail(PATFFT_ERR_UNSUPPORTED,
                    "the GPU forward model needs a window that makes the transform exact to 1e-6 (K >= 4 at c >= 2 "
                    "with the default alpha/beta): with this one the reference's answer carries the window's own "
                    "approximation error");
  if (F->ner->n_over < 2 * n_time)
    return api_fail(PATFFT_ERR_UNSUPPORTED, "GPU forward model needs an oversampling factor >= 2");
  F->n_lat = n_lat;
  F->N0 = N0;
  F->N1 = N1;
  F->N1h = N1 / 2 + 1;
  F->T = n_time;
  F->L = (size_t)N0 * N1;
  F->Lh = (size_t)N0 * F->N1h;
  API_CUDA(cudaSetDevice(device));
  API_CUDA(cudaMalloc(&F->d_j2, F->L * sizeof(double)));
  API_CUDA(cudaMemcpy(F->d_j2, j2, F->L * sizeof(double), cudaMemcpyHostToDevice));
  API_CUDA(cudaMalloc(&F->d_spec, F->Lh * n_time * sizeof(float2)));
  auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
  static const bool custom_on = [] {
    const char* e = std::getenv("PATFFT_FORWARD_CUSTOM_FFT");
    return e ? std::atoi(e) != 0 : true;
  }();
  if (custom_on && pow2(N1) && N1 >= 4 && N1 <= 16384 && (n_lat == 1 || (pow2(N0) && N0 >= 4 && N0 <= 16384))) {
    F->custom_lateral = true;
    const int mx = std::max(N0, N1);
    std::vector<float> ones((size_t)mx, 1.0f);
    API_CUDA(cudaMalloc(&F->d_ones, mx * sizeof(float)));
    API_CUDA(cudaMemcpy(F->d_ones, ones.data(), mx * sizeof(float), cudaMemcpyHostToDevice));
    API_CUDA(cudaMalloc(&F->d_Y, F->Lh * n_time * sizeof(float2)));
    auto lg = [](int v) { int l = 0; while ((1 << l) < v) ++l; return l; };
    LateralParams& L = F->lat;
    L.ref = nullptr;
    L.grid = nullptr;
    L.Y = F->d_Y;
    L.gh = F->d_spec;
    L.tw = F->ner->d_tw;
    L.dp0 = F->d_ones;
    L.dp1 = F->d_ones;
    L.T = n_time;
    L.nrows = N0; L.lrows = lg(N0);
    L.ncols = N1; L.lcols = lg(N1);
    L.ny = F->N1h; L.N0 = N0; L.N1 = N1;
    L.t_begin = 0; L.t_end = n_time;
    L.ys = n_time; L.yt0 = 0; L.gs = n_time; L.gt0 = 0;
    L.f_flags = nullptr; L.f_chunks = L.f_slots = L.f_lead = 0; L.y_capacity = n_time;
    L.cplx = 0; L.centered = 0;
    L.z = F->d_spec; L.out = nullptr;
    L.inv_ring = nullptr; L.inv_flags = nullptr; L.inv_capacity = 0;
    L.Tu = n_time; L.N0u = N0; L.N1u = N1; L.N1uh = F->N1h; L.l0u = lg(N0); L.l1u = lg(N1);
    *out = F.release();
    return PATFFT_OK;
  }
  // lateral transforms of the [N0][N1][T] volume, time fastest: T interleaved batches
  int nr[2] = {N0, N1}, nc[2] = {N0, F->N1h};
  int* dims = n_lat == 2 ? nr : nr + 1;
  int* cdims = n_lat == 2 ? nc : nc + 1;
  API_CUFFT(cufftPlanMany(&F->r2c, n_lat, dims, dims, n_time, 1, cdims, n_time, 1, CUFFT_R2C, n_time));
  F->have_r2c = true;
  API_CUFFT(cufftPlanMany(&F->c2r, n_lat, dims, cdims, n_time, 1, dims, n_time, 1, CUFFT_C2R, n_time));
  F->have_c2r = true;
  *out = F.release();
  return PATFFT_OK;
}

int patfft_forward_execute_device(patfft_forward_plan* F, const float* field, float* traces, void* stream) {
  if (!F || !field || !traces) return api_fail(PATFFT_ERR_PARAMETER, "null argument");
  std::lock_guard<std::mutex> lk(F->mu);
  API_CUDA(cudaSetDevice(F->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : F->ner->stream;
  return launch_forward(F, field, traces, st);
}

int patfft_forward_execute(patfft_forward_plan* F, const double* field, double* traces) {
  if (!F || !field || !traces) return api_fail(PATFFT_ERR_PARAMETER, "null argument");
  std::lock_guard<std::mutex> lk(F->mu);
  API_CUDA(cudaSetDevice(F->device));
  cudaStream_t st = F->ner->stream;
  const size_t vol = F->L * F->T;
  if (!F->d_field) API_CUDA(cudaMalloc(&F->d_field, vol * sizeof(float)));
  if (!F->d_f64) API_CUDA(cudaMalloc(&F->d_f64, vol * sizeof(double)));
  API_CUDA(cudaMemcpyAsync(F->d_f64, field, vol * sizeof(double), cudaMemcpyHostToDevice, st));
  API_CUDA(launch_f64_to_f32(F->d_f64, F->d_field, vol, st));
  int rc = launch_forward(F, F->d_field, F->d_field, st);
  if (rc) return rc;
  API_CUDA(launch_f32_to_f64(F->d_field, F->d_f64, vol, st));
  API_CUDA(cudaMemcpyAsync(traces, F->d_f64, vol * sizeof(double), cudaMemcpyDeviceToHost, st));
  API_CUDA(cudaStreamSynchronize(st));
  return PATFFT_OK;
}

void patfft_forward_plan_destroy(patfft_forward_plan* F) {
  if (!F) return;
  cudaSetDevice(F->device);
  if (F->ner && F->ner->stream) cudaStreamSynchronize(F->ner->stream);
  if (F->have_r2c) cufftDestroy(F->r2c);
  if (F->have_c2r) cufftDestroy(F->c2r);
  for (void* p : {(void*)F->d_j2, (void*)F->d_field, (void*)F->d_f64, (void*)F->d_spec, (void*)F->d_Y, (void*)F->d_ones})
    if (p) cudaFree(p);
  patfft_ner_plan_destroy(F->ner);
  delete F;
}

}  // extern "C"
