// Internal declarations shared by the host plan builder, the kernels and
// the C ABI.  Not part of the public interface (include/patfft_b200.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <array>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/patfft_b200.h"

namespace patfft {

// ---------------------------------------------------------------------------
// Window pair (reference nufft.py:92-187), evaluated in float64 on the host.
// ---------------------------------------------------------------------------
struct Window {
  double c_eff = 2.0;  // effective oversampling the window is resolved for
  int K = 6;           // half-width; 2K taps
  double alpha = 0.0;  // support half-width
  double beta = 0.0;   // shape
};

// WindowSpec.resolved(c_eff) (nufft.py:133-149).  Returns false + message
// when the support is inadmissible (reference raises ParameterError).
bool resolve_window(double c, int K, double alpha_or_nan, double beta_or_nan, double c_eff, Window* out,
                    std::string* err);
double bessel_i0(double x);                   // scipy.special.i0 equivalent
double kb_psi(const Window& w, double th);    // window_eval (nufft.py:159-165)
double kb_psihat(const Window& w, double x);  // window_ft_eval (nufft.py:168-187)
int even_fast_len(double target);             // next_even_fast_len (nufft.py:83-89)
double window_relative_error(const Window& w, int n, int n_over);
// FFT twiddle table of the shared-memory transforms (fft_smem.cuh): the
// 2^14-point table exp(-2 pi i k / 2^14) followed by the per-pass tables
// (kPassTwOffset); float2 pairs, float64-accurate (window.cpp)
std::vector<float2> make_twiddles();  // accuracy probe (window.cpp)

// ---------------------------------------------------------------------------
// Device-side parameter blocks
// ---------------------------------------------------------------------------
constexpr int kMaxTaps = 16;  // 2K <= 16 (K <= 8)
constexpr int kMaxPolyDegree = 12;

struct SpreadParams {
  const float* samples;   // [M][T] float32, device
  const float* recs;      // per (row group) column-sorted records, see spread.cu
  const int4* blk;        // per CTA column: {lo, hi, c0, c1} -- records [lo, hi), columns [c0, c1)
  const int* blk_grp;     // per CTA column: row group
  float* grid;            // [nrows][ncols][T] centred oversampled grid
  int T, ncols, nrows;
  int t_begin, t_end;     // time range processed by this launch (multiples of 128)
  // tensor-core gridding (spread_tc.cu); tc_tiles == nullptr selects the SIMT kernels
  const float* tc_recs = nullptr;   // [records][32]: sample row offset m*T (u32), row weights at [8..15], column weights at [16..31]
  const int4* tc_tiles = nullptr;   // per tile (launch order): {first record, records (multiple of 16), row0, col0}
  int tc_ntiles = 0, tc_nonempty = 0;  // tiles (the non-empty ones first, longest first)
  int tc_n = 0, tc_tblocks = 0;       // time samples per block, time blocks per launch
  int* tc_counter = nullptr;          // 32 ints: work counters, |sample| max bits, redo flag, batch max, scale hints (spread_tc.cu)
  int tc_batch_scale = 0;  // 1: the scale comes from the batch maximum (frames; spread_tc16_batch_max)
  int tc_pass = 0, tc_track = 0, tc_scale_src = 1;  // fp16 gridding: launch 0 / 1, record the max, scale source slot
  // fp16 two-term operands (kind::f16): records pre-scaled by 2^tc_wexp at plan
  // time, samples by a power of two from their max per launch, undone in the epilogue
  int tc_f16 = 0, tc_wexp = 0;
  int tc_m = 0;                        // sensor rows of `samples`
  const uint4* tc_a16 = nullptr;       // per stage: A operands hi/lo (fp16, UMMA layout), 8 KB
  const uint32_t* tc_off = nullptr;    // per stage: 16 sample row offsets
  int tc_tma_store = 0;                // 1: epilogue stores through tc_gmap (TMA tensor stores)
  CUtensorMap tc_gmap;                 // grid [nrows][ncols][T] f32, box 32 t x 16 cols x 2 rows, 128B swizzle
};

// Reference-length path (reflen.cu): host-side state of the cuFFT stages.  The
// pointers ride in the kernel parameter blocks but are only read on the host.
struct LatRef {
  cufftHandle r2c = 0;     // (rows, cols) real-to-complex per time sample, stride T
  cufftHandle c2c = 0;     // NedPlan: (rows, cols) complex in place, stride T / 2
  float2* spec = nullptr;  // [nrows][ncols / 2 + 1][T]
  float2* ghd = nullptr;   // = NerRef::ghd
  int nyo = 0;             // ncols / 2 + 1
};
struct NerRefWindow {
  double alpha, beta, inv_psihat0;
  int K;
};
struct NerRef {
  cufftHandle c2c = 0;     // length n_over, rows_blk rows per call
  float2* fb = nullptr;    // [rows_blk][n_over]
  float2* ghd = nullptr;   // [N0][N1h][T] difference rows of the lateral Nyquist planes (reflen.cu)
  int rows_blk = 0;
  NerRefWindow win;
};

struct LateralParams {
  const LatRef* ref;   // non-null: reference-length plan (cuFFT lateral stage)
  // forward
  const float* grid;   // [nrows][ncols][T]
  float2* Y;           // [nrows][ny][T]  column-transformed half spectrum
  float2* gh;          // [N0][ny][T]     symmetrised, deapodised lateral spectrum
  const float2* tw;    // exp(-2 pi i k / 2^14)
  const float* dp0;    // [N0] deapodisation (wrapped index)
  const float* dp1;    // [N1]
  int T, nrows, lrows, ncols, lcols, ny, N0, N1;
  int t_begin, t_end;  // forward kernels: time range processed by this launch
  int ys, yt0;         // Y time stride and the time stored at Y offset 0 (whole record: T, 0)
  int gs, gt0;         // the same for gh
  // single-launch column + row FFTs (lateral.cu, latfused_kernel): Y is a ring of
  // f_slots chunk buffers of 32 time samples; f_flags[c] counts the finished column
  // tiles of chunk c, f_flags[f_chunks + c] its finished row tiles
  int* f_flags;        // 2 * ceil(T / 32) ints (nullptr: two-kernel form only)
  int f_chunks, f_slots, f_lead;
  int y_capacity;      // time samples per (row, bin) the Y allocation holds
  int cplx;            // 1: NedPlan mode (complex values, full spectrum, no Hermitian fix-up)
  int centered;        // NedPlan output order
  // inverse
  float2* z;           // [N0u][N1uh][Tu]
  float* out;          // [N0u][N1u][Tu]
  // single-launch inverse (lateral.cu, invfused_kernel): ring of chunk buffers [slots][N0u][N1uh][32],
  // progress counters, and the depth length the counters were sized for (nullptr: two kernels)
  float2* inv_ring;
  int* inv_flags;
  int inv_capacity;
  int Tu, N0u, N1u, N1uh, l0u, l1u;
};

struct NerParams {
  const NerRef* ref;   // non-null: reference-length plan (cuFFT NER stage)
  const float2* gh;    // [N0][N1h][T]
  float2* z;           // [N0u][N1uh][Tu]
  const float* iw;     // [2T] psihat(0)*norm/psi(theta_n) (nufft.py:281-284)
  const float2* pre;   // [2T] DCT-III input twiddle x pre-window (ner_dct_kernel)
  const float2* tw;    // exp(-2 pi i k / 2^14)
  const double* jt0;   // [N0] (j0*ratio0)^2 on the wrapped grid (recon.py:211)
  const double* jt1;   // [N1h]
  int T, n_over, log_n_over, Tu, log_tu;
  int N0, N1, N1h, N0u, N1uh, up, n_lat;
  int fused_ifft;      // 1: inverse depth FFT in shared memory, 0: write spectrum
  int interp;          // 1: linear interpolation of the plain 2T FFT (reconstruct_interp_fft)
  // row / time layout (single GPU: row0 = out_row0 = 0, rows_local = N0*N1h,
  // rows_out = N0u*N1uh, in_tchunk = T, out_tchunk = Tu)
  int row0, rows_local, in_tchunk, in_tshift, in_tmask;
  int in_row_off, rows_launch;  // rows [in_row_off, in_row_off + rows_launch) of the input (0, 0: all)
  int out_row0, rows_out, out_tchunk, out_tshift, out_tmask;
  double c_eff;        // n_over / (2T)
  float scale;         // 1/(N0*N1*T): scipy ifftn normalisation * up^d
  float poly[kMaxTaps / 2][kMaxPolyDegree + 1];  // psihat((z + K-1/2-j)/c)/psihat(0), z in [-1/2,1/2]
  int poly7;           // 1: poly has degree 7 (coefficient 8 zero): ner_dct_kernel<.., 7, ..>
};

// Kernel launchers
cudaError_t launch_spread(const SpreadParams& p, int K2, int R, int nblk, cudaStream_t s);
cudaError_t launch_spread_tc(const SpreadParams& p, cudaStream_t s);
cudaError_t spread_tc16_build(const float* recs, int nstages, void* a16, uint32_t* offs, cudaStream_t s);
cudaError_t spread_tc16_batch_max(const float* samples, int64_t rows, int T, int* counters, cudaStream_t s);
bool spread_tc_supported(int n_lat, int nrows, int ncols, int T);
int spread_tc_block(int T);
int spread_rows_per_group(int n_lat, int K2);
int spread_record_words(int K2, int R);
int spread_ctas_per_sm(int R);
bool spread_time_pairs(int R);
int spread_time_chunks(int T, int R);
cudaError_t launch_lateral_col(const LateralParams& p, cudaStream_t s);
cudaError_t launch_lateral_row(const LateralParams& p, cudaStream_t s);
bool lateral_fused_supported(const LateralParams& p);
cudaError_t launch_lateral_forward(const LateralParams& p, cudaStream_t s);  // fused when supported, else col + row
cudaError_t launch_lateral_inverse(const LateralParams& p, cudaStream_t s);
cudaError_t launch_ner(const NerParams& p, int K2, int degree, cudaStream_t s);
cudaError_t launch_lateral_ref(const LateralParams& p, cudaStream_t s);  // reflen.cu
cudaError_t launch_ner_ref(const NerParams& p, cudaStream_t s);
cudaError_t launch_lateral_ref_cplx(const LateralParams& p, int B, cudaStream_t s);
size_t ner_smem_bytes(int n_over, int Tu);
int ner_threads(int n_over);
cudaError_t launch_f64_to_f32(const double* src, float* dst, size_t n, cudaStream_t s);
cudaError_t launch_f64_to_f32_cols(const double* src, float* dst, int M, int T, int tb, int te, cudaStream_t s);
cudaError_t launch_f32_to_f64(const float* src, double* dst, size_t n, cudaStream_t s);
cudaError_t launch_f32_to_f64_count(const float* src, double* dst, size_t n, unsigned long long* bad,
                                    cudaStream_t s);
cudaError_t launch_fill(float* dst, size_t n, float v, cudaStream_t s);
cudaError_t launch_gather_rows(const float* samples, const int* gidx, float* grid, int M, int T, cudaStream_t s);

// host-side float64 <-> float32 staging (hoststage.cpp), parallel over a process-wide thread pool
int host_threads();
void host_narrow_rows(const double* src, int64_t src_stride, float* dst, int64_t dst_stride, int64_t rows,
                      int64_t cols);
int64_t host_widen(const float* src, double* dst, int64_t n);  // returns #non-finite
int64_t host_count_nonfinite(const double* x, int64_t n);

}  // namespace patfft

// ---------------------------------------------------------------------------
// The plan (opaque to C callers)
// ---------------------------------------------------------------------------
struct patfft_nedner_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // lateral FFTs overlapped with the spread
  cudaEvent_t ev_chunk[4] = {}, ev_fork = nullptr, ev_join = nullptr;
  // host-buffer path: H2D of time chunk k on copy_stream, compute waits ev_h2d[k]
  static constexpr int kMaxH2dChunks = 16;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_h2d[kMaxH2dChunks] = {};
  int h2d_chunks = 8;
  // host conversion (hoststage.cpp): float32 crosses PCIe, the host cores narrow/widen
  bool host_convert = true;
  bool host_trace = false;  // PATFFT_HOST_TRACE=1: per-call phase times on stderr
  int host_blocks = 4;       // row blocks per time chunk (upload) / volume blocks (download, x4)
  float* h_stage = nullptr;  // pinned, max(M*T, out voxels) floats
  // pinned caller buffers: this fraction of the samples / voxels crosses PCIe as
  // float64 by DMA (device converts) instead of through the host cores
  double direct_in = 0.25;  // measured at cfg4: upload 8.2 -> 7.0 ms
  double direct_out = 0.0;  // measured at cfg4: download 7.5 -> 7.9 ms at 0.2 (host memory bound either way)
  unsigned long long* d_bad = nullptr;  // non-finite count of the direct part
  size_t h_stage_n = 0;
  cudaEvent_t ev_d2h[kMaxH2dChunks] = {}, ev_done = nullptr;
  int overlap_chunks = 1;  // time chunks of the overlapped forward stages (1 = off)
  int lat_chunk = 0;       // time samples per colfft -> rowfft chunk (0 = whole record)
  // CUDA graphs of the last executed (samples, image, frames) triples (the
  // batch path alternates two buffer sets)
  bool use_graphs = true;
  struct GraphSlot {
    cudaGraphExec_t exec = nullptr;
    const float* in = nullptr;
    float* out = nullptr;
    int frames = 0;
  };
  static constexpr int kGraphSlots = 4;
  GraphSlot graphs[kGraphSlots];
  int graph_next = 0;
  // pipelined batch of host records (patfft_nedner_execute_batch): two sets of
  // device input/output buffers and pinned staging, one per record in flight
  struct BatchSet {
    float* d_in = nullptr;
    double* d_in64 = nullptr;  // direct (float64 DMA) sensor rows
    float* d_out = nullptr;
    double* d_out64 = nullptr;  // direct voxels, widened on the device
    unsigned long long* d_bad = nullptr;
    float* h_in = nullptr;   // pinned staging of the narrowed rows
    float* h_out = nullptr;  // pinned staging of the downloaded float32 voxels
    unsigned long long* h_bad = nullptr;
    cudaEvent_t ev_in = nullptr, ev_comp = nullptr, ev_out = nullptr;
    cudaEvent_t ev_blk[16] = {};
  };
  BatchSet bset[2];
  bool batch_ready = false;
  cudaStream_t copy_out_stream = nullptr;
  double batch_direct_in = 0.4, batch_direct_out = 0.4;
  std::mutex mu;

  // sizes
  int mode = 0;  // 0 NEDNER, 1 equispaced NUFFT, 2 equispaced interp
  int n_lat = 2, N0 = 1, N1 = 0, T = 0, up = 1, M = 0;
  int nrows = 1, ncols = 0, N1h = 0;
  int N0u = 1, N1u = 0, N1uh = 0, Tu = 0;
  int n_over_t = 0, K2 = 12, K2t = 12, poly_degree = 8;  // K2: lateral taps, K2t: NER taps
  int R = 4, ngroups = 0, nblk = 0;
  int64_t n_records = 0;
  bool fused_ifft = true;
  bool custom_inverse = true;
  // explicit window that is inaccurate at the reference's own oversampled length: the plan
  // runs on those lengths (reflen.cu) so that it reproduces the reference's approximation
  bool ref_len = false;
  // sliced plan (general multi-GPU schedule): NED stages / lateral inverse on Tr (x up) samples,
  // NER on caller-provided row ranges with the full N_t
  bool sliced = false;
  bool batch_scale = false;  // set while the frames of one batch are enqueued (execute_graphed)
  patfft::LatRef lat_ref;
  patfft::NerRef ner_ref;

  patfft::Window win_lat[2], win_t;

  // device buffers
  float* d_samples = nullptr;   // [M][T] f32 (host path staging)
  double* d_samples64 = nullptr;
  float* d_grid = nullptr;      // [nrows][ncols][T]
  float2* d_Y = nullptr;        // [nrows][N1h][T]
  int* d_lat_flags = nullptr;   // progress counters of the single-launch lateral FFTs
  float2* d_inv_ring = nullptr; // single-launch lateral inverse: L2-resident ring between its two FFTs
  int* d_inv_flags = nullptr;
  float2* d_gh = nullptr;       // [N0][N1h][T]
  float2* d_z = nullptr;        // [N0u][N1uh][Tu]
  float* d_out = nullptr;       // [N0u][N1u][Tu] f32 (host path staging)
  double* d_out64 = nullptr;
  float* d_recs = nullptr;
  float* d_tc_recs = nullptr;   // tensor-core gridding records (spread_tc.cu)
  int4* d_tc_tiles = nullptr;
  int* d_tc_counter = nullptr;  // 32 ints (zero-initialised: no scale hints yet)
  uint4* d_tc_a16 = nullptr;
  bool tc_tma_store = false;
  CUtensorMap tc_gmap;
  uint32_t* d_tc_off = nullptr;
  int tc_f16 = 0, tc_wexp = 0;
  int tc_ntiles = 0, tc_nonempty = 0, tc_n = 0;
  int64_t tc_records = 0;
  int* d_gidx = nullptr;      // equispaced modes: grid row of each sensor
  int4* d_blk = nullptr;
  int* d_blkgrp = nullptr;
  float* d_dp0 = nullptr;
  float* d_dp1 = nullptr;
  float* d_iw = nullptr;
  float2* d_pre = nullptr;
  float2* d_tw = nullptr;
  double* d_jt0 = nullptr;
  double* d_jt1 = nullptr;

  cufftHandle fft_c2r = 0, fft_l = 0;
  bool have_c2r = false, have_l = false;

  patfft::NerParams ner{};
  // sharding (time-sliced NED / inverse, row-sliced NER); world = 1 for a single GPU
  int rank = 0, world = 1, Tr = 0;          // Tr: local time slice length
  int rows_total = 0, row_begin = 0, rows_mine = 0;
  std::vector<int> row_starts;              // world + 1 row boundaries
  patfft::LateralParams lat{};

  // profiling
  bool profiling = false;
  cudaEvent_t ev[PATFFT_N_STAGES + 1] = {};
  double stage_ms[PATFFT_N_STAGES] = {};
  int64_t stage_launches[PATFFT_N_STAGES] = {};
};
