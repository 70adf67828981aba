// Host-side probe for the end-to-end path: pinned H2D/D2H bandwidth for the
// cfg4 float64 record (537 MB) vs a float32 copy (268 MB), and the throughput
// of multi-threaded float64 -> float32 narrowing / float32 -> float64 widening
// on the host, alone and overlapped with the copies.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -O3,-march=native,-pthread h2d_probe.cu -o h2d_probe
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void narrow(const double* s, float* d, size_t n, int threads) {
  std::vector<std::thread> ts;
  size_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    size_t a = t * per, b = std::min(n, a + per);
    ts.emplace_back([=] { for (size_t i = a; i < b; ++i) d[i] = (float)s[i]; });
  }
  for (auto& t : ts) t.join();
}
static void widen(const float* s, double* d, size_t n, int threads) {
  std::vector<std::thread> ts;
  size_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    size_t a = t * per, b = std::min(n, a + per);
    ts.emplace_back([=] { for (size_t i = a; i < b; ++i) d[i] = (double)s[i]; });
  }
  for (auto& t : ts) t.join();
}

int main() {
  const size_t n = 65536ull * 1024;
  double *h64p, *h64b; float *h32p;
  cudaMallocHost(&h64p, n * 8);
  cudaMallocHost(&h32p, n * 4);
  h64b = (double*)malloc(n * 8);  // pageable (numpy-like)
  void* d; cudaMalloc(&d, n * 8);
  for (size_t i = 0; i < n; ++i) { h64p[i] = i * 1e-9; h64b[i] = i * 1e-9; }
  memset(h32p, 0, n * 4);
  cudaStream_t st; cudaStreamCreate(&st);
  auto bw = [&](const char* what, void* dst, const void* src, size_t bytes, cudaMemcpyKind k) {
    cudaMemcpyAsync(dst, src, bytes, k, st); cudaStreamSynchronize(st);
    double t0 = now();
    for (int r = 0; r < 3; ++r) cudaMemcpyAsync(dst, src, bytes, k, st);
    cudaStreamSynchronize(st);
    double dt = (now() - t0) / 3;
    printf("%-28s %8.2f ms  %6.1f GB/s\n", what, dt * 1e3, bytes / dt / 1e9);
  };
  bw("H2D f64 pinned", d, h64p, n * 8, cudaMemcpyHostToDevice);
  bw("H2D f32 pinned", d, h32p, n * 4, cudaMemcpyHostToDevice);
  bw("D2H f64 pinned", h64p, d, n * 8, cudaMemcpyDeviceToHost);
  bw("D2H f32 pinned", h32p, d, n * 4, cudaMemcpyDeviceToHost);
  bw("H2D f64 pageable", d, h64b, n * 8, cudaMemcpyHostToDevice);
  for (int th : {1, 2, 4, 8, 16, 32}) {
    narrow(h64p, h32p, n, th);
    double t0 = now();
    narrow(h64p, h32p, n, th);
    double t1 = now();
    widen(h32p, h64p, n, th);
    double t2 = now();
    narrow(h64b, h32p, n, th);
    double t3 = now();
    printf("threads %2d: narrow pinned %7.2f ms  widen %7.2f ms  narrow pageable %7.2f ms\n", th,
           (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3);
  }
  // pipelined: narrow chunk k (threads) while chunk k-1 copies
  for (int th : {4, 8, 16}) {
    for (int chunks : {8, 16, 32}) {
      size_t cn = n / chunks;
      cudaEvent_t ev[64];
      for (int c = 0; c < chunks; ++c) cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming);
      double t0 = now();
      for (int c = 0; c < chunks; ++c) {
        narrow(h64p + c * cn, h32p + c * cn, cn, th);
        cudaMemcpyAsync((char*)d + c * cn * 4, h32p + c * cn, cn * 4, cudaMemcpyHostToDevice, st);
      }
      cudaStreamSynchronize(st);
      double t1 = now();
      // download + widen pipelined
      for (int c = 0; c < chunks; ++c) {
        cudaMemcpyAsync(h32p + c * cn, (char*)d + c * cn * 4, cn * 4, cudaMemcpyDeviceToHost, st);
        cudaEventRecord(ev[c], st);
      }
      for (int c = 0; c < chunks; ++c) {
        cudaEventSynchronize(ev[c]);
        widen(h32p + c * cn, h64b + c * cn, cn, th);
      }
      double t2 = now();
      printf("pipelined th %2d chunks %2d: up %7.2f ms  down %7.2f ms  total %7.2f\n", th, chunks,
             (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t2 - t0) * 1e3);
      for (int c = 0; c < chunks; ++c) cudaEventDestroy(ev[c]);
    }
  }
  return 0;
}
