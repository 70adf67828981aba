// Host side of the float64 host-buffer path (patfft_nedner_execute).
//
// The reference API hands the reconstruction float64 samples and wants a
// float64 volume back (recon.py:358-379: SensorRecord widens to float64,
// ScalarField holds float64).  The device computes in float32/complex64, so
// moving float64 over PCIe wastes half the bus: a cfg4 call moves 537 MB in
// and 537 MB out at ~55 GB/s (~19.6 ms) for ~2 ms of device work.  Here the
// host cores narrow the samples to float32 into a pinned staging buffer
// (bit-identical to the device's cvt.rn.f32.f64: IEEE round to nearest even)
// while the copy engine uploads the previous block, and widen the float32
// volume into the caller's float64 buffer while the next block downloads.
// Caller buffers may be pageable (numpy arrays): only the staging is pinned.
//
// The pool is process-wide; one conversion runs at a time (a second caller
// converts on its own thread instead of waiting).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <sched.h>

#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include "patfft_internal.h"

namespace patfft {
namespace {

class HostPool {
 public:
  explicit HostPool(int n) {
    for (int i = 0; i + 1 < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int threads() const { return (int)workers_.size() + 1; }

  // Runs fn(0..ntasks-1) on the workers and the calling thread; returns when all are done.
  void run(int ntasks, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> busy(run_mu_, std::try_to_lock);
    if (!busy.owns_lock() || workers_.empty() || ntasks <= 1) {
      for (int i = 0; i < ntasks; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      ntasks_ = ntasks;
      next_.store(0);
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    const int mine = work();
    std::unique_lock<std::mutex> lk(mu_);
    done_ += mine;
    done_cv_.wait(lk, [&] { return done_ == ntasks_; });
    fn_ = nullptr;
  }

 private:
  int work() {
    int n = 0;
    for (int i; (i = next_.fetch_add(1)) < ntasks_; ++n) (*fn_)(i);
    return n;
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      if (!fn_) continue;
      lk.unlock();
      const int n = work();
      lk.lock();
      done_ += n;
      if (done_ == ntasks_) done_cv_.notify_one();
    }
  }

  std::vector<std::thread> workers_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int ntasks_ = 0, done_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

int pool_threads() {
  if (const char* e = std::getenv("PATFFT_HOST_THREADS")) return std::max(1, std::atoi(e));
  cpu_set_t set;
  int n = 0;
  if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
  if (n <= 0) n = (int)std::thread::hardware_concurrency();
  return std::max(1, std::min(n, 32));
}

HostPool& pool() {
  static HostPool p(pool_threads());
  return p;
}

void narrow_row(const double* s, float* d, int64_t n) {
  int64_t i = 0;
#if defined(__SSE2__)
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) d[i] = (float)s[i];
  for (; i + 4 <= n; i += 4) {
    const __m128 lo = _mm_cvtpd_ps(_mm_loadu_pd(s + i));
    const __m128 hi = _mm_cvtpd_ps(_mm_loadu_pd(s + i + 2));
    _mm_stream_ps(d + i, _mm_movelh_ps(lo, hi));
  }
#endif
  for (; i < n; ++i) d[i] = (float)s[i];
}

inline int64_t nonfinite(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return (u & 0x7f800000u) == 0x7f800000u;
}

// returns the number of non-finite values (the ScalarField check, recon.py:62-63 there)
int64_t widen_run(const float* s, double* d, int64_t n) {
  int64_t i = 0, bad = 0;
#if defined(__SSE2__)
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) {
    d[i] = (double)s[i];
    bad += nonfinite(s[i]);
  }
  const __m128i expo = _mm_set1_epi32(0x7f800000);
  __m128i acc = _mm_setzero_si128();
  for (; i + 4 <= n; i += 4) {
    const __m128 f = _mm_loadu_ps(s + i);
    _mm_stream_pd(d + i, _mm_cvtps_pd(f));
    _mm_stream_pd(d + i + 2, _mm_cvtps_pd(_mm_movehl_ps(f, f)));
    const __m128i e = _mm_and_si128(_mm_castps_si128(f), expo);
    acc = _mm_sub_epi32(acc, _mm_cmpeq_epi32(e, expo));  // +1 per non-finite lane
  }
  alignas(16) int32_t lanes[4];
  _mm_store_si128(reinterpret_cast<__m128i*>(lanes), acc);
  bad += (int64_t)lanes[0] + lanes[1] + lanes[2] + lanes[3];
#endif
  for (; i < n; ++i) {
    d[i] = (double)s[i];
    bad += nonfinite(s[i]);
  }
  return bad;
}

void fence() {
#if defined(__SSE2__)
  _mm_sfence();
#endif
}

constexpr int64_t kTaskBytes = 256 << 10;  // source bytes per task

}  // namespace

int host_threads() { return pool().threads(); }

void host_narrow_rows(const double* src, int64_t src_stride, float* dst, int64_t dst_stride, int64_t rows,
                      int64_t cols) {
  if (rows <= 0 || cols <= 0) return;
  const int64_t rows_per = std::max<int64_t>(1, kTaskBytes / (8 * cols));
  const int ntasks = (int)((rows + rows_per - 1) / rows_per);
  pool().run(ntasks, [&](int t) {
    const int64_t r0 = t * rows_per, r1 = std::min(rows, r0 + rows_per);
    for (int64_t r = r0; r < r1; ++r) narrow_row(src + r * src_stride, dst + r * dst_stride, cols);
    fence();
  });
}

int64_t host_widen(const float* src, double* dst, int64_t n) {
  if (n <= 0) return 0;
  const int64_t per = kTaskBytes / 4;
  const int ntasks = (int)((n + per - 1) / per);
  std::atomic<int64_t> bad{0};
  pool().run(ntasks, [&](int t) {
    const int64_t a = t * per, b = std::min(n, a + per);
    const int64_t k = widen_run(src + a, dst + a, b - a);
    fence();
    if (k) bad.fetch_add(k);
  });
  return bad.load();
}

int64_t host_count_nonfinite(const double* x, int64_t n) {
  if (n <= 0) return 0;
  const int64_t per = kTaskBytes / 8;
  const int ntasks = (int)((n + per - 1) / per);
  std::atomic<int64_t> bad{0};
  pool().run(ntasks, [&](int t) {
    const int64_t a = t * per, b = std::min(n, a + per);
    int64_t k = 0;
    for (int64_t i = a; i < b; ++i) k += !std::isfinite(x[i]);
    if (k) bad.fetch_add(k);
  });
  return bad.load();
}

}  // namespace patfft
