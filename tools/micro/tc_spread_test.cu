// Standalone check of the tensor-core gridding kernel (spread_tc.cu) on one
// or a few tiles with hand-made records, against a double-precision CPU sum.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include \
//        tools/micro/tc_spread_test.cu -o /tmp/tc_test
#include "../../paper_1501_02946_b200/csrc/spread_tc.cu"

#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

using namespace patfft;

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 256;
  const int nsens = argc > 2 ? atoi(argv[2]) : 16;   // records in the tile (multiple of 16)
  const int mode = argc > 3 ? atoi(argv[3]) : 0;     // 0 random, 1 A=1, 2 one-hot
  const int nrows = 8, ncols = 16, M = 64;
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> samples((size_t)M * T), recs((size_t)nsens * 32, 0.f);
  for (auto& v : samples) v = mode == 2 ? 0.f : U(rng);
  if (mode == 2) for (int m = 0; m < M; ++m) samples[(size_t)m * T + (m % T)] = 1.f + m;
  for (int k = 0; k < nsens; ++k) {
    int m = (k * 7) % M;
    unsigned off = (unsigned)m * T;
    std::memcpy(&recs[k * 32], &off, 4);
    for (int r = 0; r < 8; ++r) recs[k * 32 + 8 + r] = mode ? (mode == 2 ? (r == (k % 8)) : 1.f) : U(rng);
    for (int c = 0; c < 16; ++c) recs[k * 32 + 16 + c] = mode ? (mode == 2 ? (c == (k % 16)) : 1.f) : U(rng);
  }
  std::vector<double> want((size_t)nrows * ncols * T, 0.0);
  for (int k = 0; k < nsens; ++k) {
    unsigned off;
    std::memcpy(&off, &recs[k * 32], 4);
    int m = off / T;
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 16; ++c)
        for (int t = 0; t < T; ++t)
          want[((size_t)r * ncols + c) * T + t] +=
              (double)recs[k * 32 + 8 + r] * recs[k * 32 + 16 + c] * samples[(size_t)m * T + t];
  }
  float *ds, *dr, *dg;
  int4* dt;
  cudaMalloc(&ds, samples.size() * 4);
  cudaMalloc(&dr, recs.size() * 4);
  cudaMalloc(&dg, want.size() * 4);
  cudaMalloc(&dt, sizeof(int4));
  cudaMemcpy(ds, samples.data(), samples.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, recs.data(), recs.size() * 4, cudaMemcpyHostToDevice);
  int4 tile = make_int4(0, nsens, 0, 0);
  cudaMemcpy(dt, &tile, sizeof tile, cudaMemcpyHostToDevice);
  cudaMemset(dg, 0xFF, want.size() * 4);
  SpreadParams p{};
  p.samples = ds;
  p.grid = dg;
  p.T = T;
  p.ncols = ncols;
  p.nrows = nrows;
  p.t_begin = 0;
  p.t_end = T;
  p.tc_recs = dr;
  p.tc_tiles = dt;
  p.tc_ntiles = 1;
  p.tc_nonempty = 1;
  cudaMalloc(&p.tc_counter, sizeof(int));
  p.tc_n = spread_tc_block(T);
  cudaError_t e = launch_spread_tc(p, 0);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("launch %s sync %s N=%d\n", cudaGetErrorString(e), cudaGetErrorString(e2), p.tc_n);
  std::vector<float> got(want.size());
  cudaMemcpy(got.data(), dg, got.size() * 4, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  int shown = 0;
  for (size_t i = 0; i < want.size(); ++i) {
    const double d = got[i] - want[i];
    num += d * d;
    den += want[i] * want[i];
    if (std::fabs(d) > 1e-4 * (1 + std::fabs(want[i])) && shown < 12) {
      const int t = i % T, pc = (i / T) % ncols, pr = i / T / ncols;
      printf("  p=(%d,%d) t=%d got %.6f want %.6f\n", pr, pc, t, got[i], want[i]);
      ++shown;
    }
  }
  printf("rel-L2 %.3e\n", std::sqrt(num / (den > 0 ? den : 1)));
  return 0;
}
