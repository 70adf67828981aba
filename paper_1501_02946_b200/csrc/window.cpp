// Host-side float64 window math: the Kaiser-Bessel pair and FFT sizing.
// Restates the reference's nufft.py:83-187 semantics for plan construction
// (deapodisation / pre-window tables and spreading weights).
#include <cmath>
#include <cstdio>
#include <limits>

#include "patfft_internal.h"

namespace patfft {

namespace {
constexpr double kAlphaFraction = 0.999;  // nufft.py:61

bool smooth11(long n) {
  for (long p : {2L, 3L, 5L, 7L, 11L})
    while (n % p == 0) n /= p;
  return n == 1;
}
}  // namespace

// next_even_fast_len (nufft.py:83-89): smallest even 11-smooth n >= target.
int even_fast_len(double target) {
  long n = static_cast<long>(std::ceil(target));
  if (n < 2) n = 2;
  while (!(smooth11(n) && n % 2 == 0)) ++n;
  return static_cast<int>(n);
}

// WindowSpec.resolved (nufft.py:133-149) + _check_alpha (nufft.py:124-131).
bool resolve_window(double c, int K, double alpha, double beta, double c_eff, Window* out, std::string* err) {
  if (!(c_eff >= c)) {
    if (err) *err = "effective oversampling below requested factor";
    return false;
  }
  double a = std::isnan(alpha) ? kAlphaFraction * M_PI * (2.0 * c_eff - 1.0) : alpha;
  const double hi = M_PI * (2.0 * c_eff - 1.0);
  if (!(a > c_eff && a < hi)) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "window support alpha=%.17g outside admissible range (%.17g, %.17g)", a, c_eff, hi);
    if (err) *err = buf;
    return false;
  }
  if (a <= M_PI) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "window support alpha=%.17g must exceed pi", a);
    if (err) *err = buf;
    return false;
  }
  double b = beta;
  if (std::isnan(beta)) {
    const double rad = (K / c_eff) * (K / c_eff) - (M_PI / a) * (M_PI / a);
    b = rad > 0 ? std::sqrt(rad) : M_PI * K * (2.0 - 1.0 / c_eff) / a;
  }
  out->c_eff = c_eff;
  out->K = K;
  out->alpha = a;
  out->beta = b;
  return true;
}

// Modified Bessel I0 by its power series; all terms are positive, so the
// relative error stays at a few ulp over the range used here (|x| <= ~60).
double bessel_i0(double x) {
  const double q = 0.25 * x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 500; ++k) {
    term *= q / (double(k) * double(k));
    sum += term;
    if (term < sum * 1e-18) break;
  }
  return sum;
}

// psi(theta) = I0(beta*sqrt(alpha^2 - theta^2)), 0 outside (nufft.py:159-165).
double kb_psi(const Window& w, double th) {
  if (std::fabs(th) > w.alpha) return 0.0;
  return bessel_i0(w.beta * std::sqrt(std::fmax(w.alpha * w.alpha - th * th, 0.0)));
}

// psi_hat(x) = 2 alpha sinh(s)/s, s = alpha sqrt(beta^2 - x^2), with the sin
// continuation and the small-|s^2| series (nufft.py:168-187).
double kb_psihat(const Window& w, double x) {
  const double t = w.alpha * w.alpha * (w.beta * w.beta - x * x);
  double v;
  if (std::fabs(t) < 1e-9) {
    v = 1.0 + t / 6.0 + t * t / 120.0;
  } else if (t > 0) {
    const double s = std::sqrt(t);
    v = std::sinh(s) / s;
  } else {
    const double s = std::sqrt(-t);
    v = std::sin(s) / s;
  }
  return 2.0 * w.alpha * v;
}

}  // namespace patfft

namespace patfft {

// Accuracy probe of the windowed-gridding approximation for one transform:
// a length-n NER (nufft.py:270-332) evaluated through an oversampled DFT of
// length n_over with window w, against the exact sum, on a deterministic
// random input and 48 targets in [-n/2, n/2].  Returns the relative L2 error.
// The NED (type-1) transform uses the same window pair on the same grid, so
// this bounds both directions.  O(n * n_over) host work (~10 ms at n_over 8192).
double window_relative_error(const Window& w, int n, int n_over) {
  uint64_t s = 0x9E3779B97F4A7C15ull;
  auto rnd = [&]() {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return (double)(s >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  };
  std::vector<double> ur(n), ui(n), pr(n), pi(n);
  for (int k = 0; k < n; ++k) {
    ur[k] = rnd();
    ui[k] = rnd();
    const double iw = 1.0 / kb_psi(w, 2.0 * M_PI * k / n - M_PI);
    pr[k] = ur[k] * iw;
    pi[k] = ui[k] * iw;
  }
  std::vector<double> Fr(n_over), Fi(n_over);
  for (int q = 0; q < n_over; ++q) {
    double ar = 0.0, ai = 0.0;
    for (int k = 0; k < n; ++k) {
      const double a = -2.0 * M_PI * (double)((int64_t)q * k % n_over) / n_over;
      const double c = std::cos(a), sn = std::sin(a);
      ar += pr[k] * c - pi[k] * sn;
      ai += pr[k] * sn + pi[k] * c;
    }
    Fr[q] = ar;
    Fi[q] = ai;
  }
  const double norm = 1.0 / (2.0 * M_PI * w.c_eff);
  double num = 0.0, den = 0.0;
  for (int t = 0; t < 48; ++t) {
    const double kap = (rnd() * 0.999) * n;  // in [-n/2, n/2)
    double er = 0.0, ei = 0.0;
    for (int k = 0; k < n; ++k) {
      const double a = -2.0 * M_PI * kap * k / n;
      er += ur[k] * std::cos(a) - ui[k] * std::sin(a);
      ei += ur[k] * std::sin(a) + ui[k] * std::cos(a);
    }
    const double k0 = std::floor(w.c_eff * kap);
    double fr = 0.0, fi = 0.0;
    for (int dk = -w.K + 1; dk <= w.K; ++dk) {
      const double bin = k0 + dk;
      const double off = kap - bin / w.c_eff;
      const double wt = norm * kb_psihat(w, off);
      const double c = std::cos(-M_PI * off) * wt, sn = std::sin(-M_PI * off) * wt;
      int64_t b = (int64_t)bin % n_over;
      if (b < 0) b += n_over;
      fr += c * Fr[b] - sn * Fi[b];
      fi += c * Fi[b] + sn * Fr[b];
    }
    num += (fr - er) * (fr - er) + (fi - ei) * (fi - ei);
    den += er * er + ei * ei;
  }
  return std::sqrt(num / den);
}

}  // namespace patfft
