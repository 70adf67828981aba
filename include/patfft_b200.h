/*
 * patfft_b200.h -- C ABI of the B200-native NEDNER-NUFFT reconstruction.
 *
 * The reference (`patfft`, pure Python) has no FFI; its public entry point
 * for this path is
 *
 *     patfft.recon.reconstruct_nedner(rec, out_dims=None, upsample=1, spec=None)
 *         /root/reference/pkg/src/patfft/recon.py:358-379
 *
 * which builds a NedPlan (nufft.py:345-418), a NerPlan (nufft.py:270-332)
 * and inverts the spectrum (recon.py:249-260).  This header is what a
 * ctypes binding of that path binds: plain pointers,
 * sizes and status codes, no torch or numpy types.
 *
 * Conventions
 *  - Every function returns PATFFT_OK (0) or a PATFFT_ERR_* code; the
 *    message of the last failure on the calling thread is returned by
 *    patfft_last_error().  The Python shim maps PARAMETER -> ParameterError,
 *    DATA -> DataValidationError, everything else -> RuntimeError, i.e. the
 *    reference's error classes (errors.py:4-13).
 *  - Input validation that the reference performs in SensorRecord
 *    (recon.py:115-164) happens in the shim before the ABI is crossed.
 *  - The caller owns all host buffers.  The plan owns its device buffers,
 *    cuFFT plans and CUDA stream.  A plan is immutable after creation;
 *    execute calls on one plan are serialised internally (they share
 *    scratch), different plans run concurrently.
 *  - Results are bit-deterministic for a given plan and device (fixed
 *    per-element accumulation order, no floating-point atomics).
 */
#ifndef PATFFT_B200_H
#define PATFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PATFFT_OK = 0,
  PATFFT_ERR_PARAMETER = 1,   /* -> ParameterError (spec / upsample / sizes) */
  PATFFT_ERR_DATA = 2,        /* -> DataValidationError (record contents)    */
  PATFFT_ERR_CUDA = 3,        /* CUDA / cuFFT / NCCL runtime failure         */
  PATFFT_ERR_UNSUPPORTED = 4  /* legal for the reference, not yet on the GPU */
};

/* Geometry + window of one reconstruction.  Mirrors the arguments of
 * reconstruct_nedner (recon.py:358-363) after SensorRecord validation. */
typedef struct patfft_nedner_desc {
  int32_t n_lat;          /* d-1: number of lateral axes, 1 or 2                  */
  int32_t out_dims[2];    /* lateral output grid per axis, even (recon.py:372)    */
  int32_t n_time;         /* N_t, even (recon.py:127)                             */
  int32_t upsample;       /* integer >= 1 (recon.py:392-394)                      */
  int32_t n_sensors;      /* M                                                    */
  double lat_ratio[2];    /* N_t*dy/(n_lateral*dx) per axis (recon.py:340-342)    */
  double spec_c;          /* WindowSpec.c (nufft.py:109)                          */
  int32_t spec_K;         /* WindowSpec.K (nufft.py:110)                          */
  double spec_alpha;      /* WindowSpec.alpha, NaN = resolve at plan time         */
  double spec_beta;       /* WindowSpec.beta,  NaN = resolve at plan time         */
} patfft_nedner_desc;

typedef struct patfft_nedner_plan patfft_nedner_plan;

/* Build a plan for fixed sensor positions (replaces NedPlan.__init__ +
 * spread_matrix, nufft.py:352-398, and NerPlan.__init__, nufft.py:273-285).
 *   grid_positions : M x n_lat, row-major, in output-grid units, i.e.
 *                    rec.grid_positions() * out_dims / n_lateral (recon.py:376)
 *   sensor_scale   : M, h_m / dx^(d-1) (recon.py:374)
 *   device         : CUDA device ordinal                                     */
int patfft_nedner_plan_create(const patfft_nedner_desc* desc, const double* grid_positions,
                              const double* sensor_scale, int device, patfft_nedner_plan** out);

/* Complete-grid variants (every lateral grid node has exactly one sensor):
 *   time_eval = 0 : reconstruct_equispaced  (recon.py:345-355) -- plain lateral
 *                   FFT of the cube, NER NUFFT along time;
 *   time_eval = 1 : reconstruct_interp_fft  (recon.py:382-389) -- plain lateral
 *                   FFT, linear interpolation of the length-2N_t FFT.
 *   grid_index : M, flat lateral grid index (row-major over n_lateral) of each
 *                sensor row, as recon.py:311-324 computes it.
 * Weights are not used (the reference ignores them on these paths); execute
 * with the same patfft_nedner_execute* calls.                              */
int patfft_equispaced_plan_create(const patfft_nedner_desc* desc, const int64_t* grid_index, int time_eval,
                                  int device, patfft_nedner_plan** out);

/* Output volume shape (N0*up, N1*up, Nt*up) or (N*up, Nt*up); returns rank. */
int patfft_nedner_output_shape(const patfft_nedner_plan* plan, int64_t shape[3]);

/* Full drop-in execution from host memory (recon.py:370-379):
 *   samples : M x N_t float64 host (pinned or pageable), row-major
 *   image   : output float64 host, C order, lateral axes centred (fftshift)
 *   imag_residual : optional; receives max|Im|/max|Re| of the inverse FFT.
 *                   The GPU inverts the Hermitian half spectrum with a C2R
 *                   transform, so the value is exactly 0.                  */
int patfft_nedner_execute(patfft_nedner_plan* plan, const double* samples, double* image,
                          double* imag_residual);

/* Pipelined patfft_nedner_execute over n records that share the plan's sensor
 * layout (e.g. the frames of a time series; BASELINE config 5): samples[k] /
 * images[k] as in patfft_nedner_execute.  Record k+1 is narrowed and uploaded
 * and record k-1 downloaded and widened while the device reconstructs record
 * k; each record's result is bit-identical to a single call.  nonfinite
 * (optional, n entries) receives each volume's non-finite voxel count. */
int patfft_nedner_execute_batch(patfft_nedner_plan* plan, int n, const double* const* samples,
                                double* const* images, int64_t* nonfinite);

/* patfft_nedner_execute that also counts the non-finite voxels of the image
 * (written to *nonfinite when non-NULL) in the same host pass that widens the
 * float32 volume to float64, so the caller can apply the ScalarField
 * finiteness rule (reference recon.py:62-63, DataValidationError) without a
 * second sweep over the volume.                                           */
int patfft_nedner_execute_checked(patfft_nedner_plan* plan, const double* samples, double* image,
                                  double* imag_residual, int64_t* nonfinite);

/* Device-resident execution on `stream` (NULL = the plan's own stream):
 *   samples_dev : M x N_t float32 on the plan's device
 *   image_dev   : output float32 on the plan's device
 * Enqueues work and returns without synchronising.                       */
int patfft_nedner_execute_device(patfft_nedner_plan* plan, const float* samples_dev,
                                 float* image_dev, void* stream);

/* Frames sharing one sensor layout (config 5): samples F x M x N_t float32,
 * images F x out-volume float32, both device-resident.                    */
int patfft_nedner_execute_frames_device(patfft_nedner_plan* plan, int n_frames,
                                        const float* samples_dev, float* images_dev, void* stream);

void patfft_nedner_plan_destroy(patfft_nedner_plan* plan);

/* ---- standalone NER NUFFT (the reference's NerPlan / nufft_ner, nufft.py:270-338) ----
 * out[r, i] ~= sum_k u[r, k] exp(-2 pi i kappa[r, i] k / n); kappas are per row
 * (rows x m) or shared (m) when `shared` != 0.  u/out complex (interleaved).
 * The host call takes complex128 u/out and float64 kappas; the device call
 * complex64 u/out (float2) and float64 kappas.  Range checks (finite, |kappa| <=
 * kappa_max) are the caller's (nufft.py:305-308, done in the Python shim).   */
typedef struct patfft_ner_plan patfft_ner_plan;
int patfft_ner_plan_create(int n, double c, int K, double alpha_or_nan, double beta_or_nan, int device,
                           patfft_ner_plan** out);
/* info: n, n_over, 2K, tap polynomial degree */
int patfft_ner_plan_info(const patfft_ner_plan* plan, int64_t info[4]);
int patfft_ner_execute(patfft_ner_plan* plan, const double* u, const double* kappas, int rows, int m, int shared,
                       double* out);
int patfft_ner_execute_device(patfft_ner_plan* plan, const void* u, const double* kappas, int rows, int m,
                              int shared, void* out, void* stream);
void patfft_ner_plan_destroy(patfft_ner_plan* plan);

/* ---- standalone NED NUFFT (the reference's NedPlan / nufft_ned, nufft.py:345-423) ----
 * out[j, b] ~= sum_m values[m, b] exp(-2 pi i (j . x_m) / N), j on the centred
 * grid out_dims (1 or 2 axes), x_m = grid_positions (n_points x n_lat, grid
 * units).  values: n_points x n_values complex128 (interleaved) host; out:
 * out_dims x n_values complex128 host, centred (centered != 0) or wrapped
 * order (nufft.py:414-417).  The plan is tied to the positions.              */
int patfft_ned_plan_create(int n_lat, const int32_t* out_dims, int n_values, double spec_c, int spec_K,
                           double spec_alpha, double spec_beta, const double* grid_positions, int n_points,
                           int device, patfft_nedner_plan** out);
int patfft_ned_execute(patfft_nedner_plan* plan, const double* values, double* out, int centered);

/* ---- multi-GPU (one process per GPU; the caller runs the two exchanges) ----
 * A sharded plan splits one reconstruction over `world` ranks:
 *   forward  : NED spread + lateral FFT of the rank's time slice
 *              samples_slice [M][Tr] (Tr = N_t/world)  ->  gh_send [rows_total][Tr]
 *   exchange : all-to-all, rank q receives rows [row_start[q], row_start[q+1])
 *              of every rank's gh_send                 ->  gh_recv [world][rows_mine][Tr]
 *   ner      : NER + depth inverse FFT of the rank's rows
 *              gh_recv                                 ->  z_send [world][rows_mine][Tr]
 *   exchange : all-to-all of the world blocks          ->  z_recv [rows_total][Tr]
 *   inverse  : lateral inverse FFT of the time slice   ->  image_slice [N0][N1][Tr]
 * (complex buffers are float32 pairs).  Requires upsample == 1 and a
 * power-of-two Tr.  All stages enqueue on `stream` and do not synchronise. */
int patfft_nedner_plan_create_sharded(const patfft_nedner_desc* desc, const double* grid_positions,
                                      const double* sensor_scale, int device, int rank, int world,
                                      patfft_nedner_plan** out);
/* info: rank, world, Tr, rows_total, row_begin, rows_mine, N0u, N1u */
int patfft_nedner_shard_info(const patfft_nedner_plan* plan, int64_t info[8]);
int patfft_nedner_shard_rows(const patfft_nedner_plan* plan, int64_t* row_starts, int n);
int patfft_nedner_shard_forward(patfft_nedner_plan* plan, const float* samples_slice, void* gh_send, void* stream);
int patfft_nedner_shard_ner(patfft_nedner_plan* plan, const void* gh_recv, void* z_send, void* stream);
int patfft_nedner_shard_inverse(patfft_nedner_plan* plan, const void* z_recv, float* image_slice, void* stream);
/* Pipelined variants (paper_1501_02946_b200/parallel.py overlaps each exchange
 * with the next piece of compute):
 *  spread: gridding of the whole local time slice into the plan's grid;
 *  lateral: lateral FFTs of local times [t_begin, t_end) (multiples of 32) of
 *    that grid into gh_chunk = [rows_total][t_end - t_begin];
 *  ner_rows: NER + depth IFFT of the rank's local rows [row_begin, row_end)
 *    from gh_recv laid out [t / in_tchunk][rows_mine][in_tchunk] (in_tchunk a
 *    power of two) into z_block = [dst rank][row_end - row_begin][N_t / world]. */
int patfft_nedner_shard_spread(patfft_nedner_plan* plan, const float* samples_slice, void* stream);
int patfft_nedner_shard_lateral(patfft_nedner_plan* plan, int t_begin, int t_end, void* gh_chunk, void* stream);
int patfft_nedner_shard_ner_rows(patfft_nedner_plan* plan, const void* gh_recv, int in_tchunk, int row_begin,
                                 int row_end, void* z_block, void* stream);

/* General multi-GPU schedule (any even N_t, any upsample, any lateral size the plan supports;
 * paper_1501_02946_b200/parallel.py, GeneralShardedNedNer): a SLICED plan runs the NED stages on a
 * time slice of t_slice samples and the lateral inverse on a depth slice of upsample * t_slice
 * samples, with the same kernels as the single-GPU plan:
 *   patfft_nedner_shard_forward : samples_slice [M][t_slice] -> gh [rows_total][t_slice]
 *   patfft_nedner_slice_ner     : rows [row_begin, row_end) with the full N_t, [rows][N_t]
 *                                 -> their rows of z_full = [N0u * N1uh][Tu] (depth-inverted;
 *                                 recon.py:225-246 row placement, Nyquist rows written twice)
 *   patfft_nedner_shard_inverse : z_slice [N0u * N1uh][upsample * t_slice] -> image slice
 * The exchanges between them (rows <-> time slices) belong to the caller. */
int patfft_nedner_plan_create_slice(const patfft_nedner_desc* desc, const double* grid_positions,
                                    const double* sensor_scale, int device, int t_slice, patfft_nedner_plan** out);
int patfft_nedner_slice_ner(patfft_nedner_plan* plan, const void* gh_rows, int row_begin, int row_end, void* z_full,
                            void* stream);

/* ---- forward model: the reference's forward_fourier (forward.py:105-166) --
 * Full-grid sensor traces of an initial pressure field on an
 * (N0, N1, N_t) or (N, N_t) grid (time/depth fastest, dt = dz / c):
 * lateral FFT of the field (cuFFT R2C), per lateral frequency row the NER
 * transform at +-ky = +-sqrt(w^2 - |j|^2) on the doubled window with the
 * w/(2 ky) Jacobian and the propagating mask (sm_100a kernel, depth inverse
 * FFT in shared memory), lateral inverse (cuFFT C2R).  The ifftshift of the
 * field and the fftshift of the traces (forward.py:124,157) cancel for even
 * sizes and are both omitted.
 *   n_lateral : n_lat lateral sizes, even (forward.py:118-119)
 *   n_time    : N_t, a power of two <= 4096 on the GPU
 *   j2        : N0*N1 float64, _lateral_freq_sq(n_lateral, ratios) on the
 *               wrapped grid (recon.py:200-215, forward.py:141-143)
 *   c, K, alpha, beta : WindowSpec of the NerPlan(N_t, spec) (forward.py:151) */
typedef struct patfft_forward_plan patfft_forward_plan;
int patfft_forward_plan_create(int n_lat, const int32_t* n_lateral, int n_time, const double* j2, double c, int K,
                               double alpha, double beta, int device, patfft_forward_plan** out);
/* field: N0*N1*N_t float64 host; traces: N0*N1*N_t float64 host, one row of
 * N_t samples per grid node in C order (forward.py:158-166). */
int patfft_forward_execute(patfft_forward_plan* plan, const double* field, double* traces);
/* Device-resident float32 variant; field and traces may alias.  Enqueues on
 * `stream` (NULL = the plan's stream) without synchronising. */
int patfft_forward_execute_device(patfft_forward_plan* plan, const float* field_dev, float* traces_dev, void* stream);
void patfft_forward_plan_destroy(patfft_forward_plan* plan);

/* Per-stage device timing (CUDA events on the plan's stream).  When enabled
 * every execute records one event per stage boundary; patfft_nedner_stage_times
 * returns the accumulated milliseconds per stage and the launch count per
 * stage since the last reset, and the stage names via patfft_nedner_stage_name. */
enum { PATFFT_STAGE_SPREAD = 0,       /* NED gridding onto the oversampled plane      */
       PATFFT_STAGE_LATERAL_COL = 1,  /* real FFT along grid columns (half kept)      */
       PATFFT_STAGE_LATERAL_ROW = 2,  /* FFT along rows + crop + deapodise + Nyquist  */
       PATFFT_STAGE_NER = 3,          /* fused NER + epilogue + depth inverse FFT     */
       PATFFT_STAGE_INVERSE = 4,      /* lateral inverse FFT (C2R) to the image       */
       PATFFT_N_STAGES = 5 };
int patfft_nedner_set_profiling(patfft_nedner_plan* plan, int enabled);
int patfft_nedner_stage_times(patfft_nedner_plan* plan, double* ms, int64_t* launches, int n);
const char* patfft_nedner_stage_name(int stage);
/* Algorithmic bytes per launch of each stage (roofline table). */
int patfft_nedner_stage_bytes(const patfft_nedner_plan* plan, double* bytes, int n);
/* Number of kernels one execute_device launches: own sm_100a kernels and
 * library (cuFFT) kernels (the latter only on fallback sizes). */
int patfft_nedner_launches_per_execute(const patfft_nedner_plan* plan, int* own, int* library);

/* Gridding (spread) kernel of the plan: info[0] = 2 for the tcgen05 tensor-core
 * kernel with fp16 two-term operands (spread_tc.cu, default), 1 for its 3xTF32
 * form (PATFFT_SPREAD_F16=0), 0 for the SIMT kernel; info[1] = records (tensor
 * core: tile x sensor pairs, padded to 16 per tile -- each is 128 grid points
 * x N_t MACs per product); info[2] = tiles (or SIMT blocks); info[3] = time
 * samples per tensor-core work item. */
int patfft_nedner_spread_info(const patfft_nedner_plan* plan, int64_t info[4]);

/* Windows the plan evaluates (nufft.py:133-149 semantics): taps[0] = 2K of the
 * lateral gridding, taps[1] = 2K of the NER (8 when the float32-grade window
 * replaced an auto-resolved K > 4), taps[2] = degree
 * of the NER tap polynomials; win[0..2] = (c_eff, alpha, beta) of the lateral
 * window along the last axis, win[3..5] = the same for the NER window. */
int patfft_nedner_window_info(const patfft_nedner_plan* plan, int64_t taps[3], double win[6]);

/* ---- small runtime helpers used by the Python shim and bench.py ---------- */
const char* patfft_last_error(void);
const char* patfft_version(void);
int patfft_device_count(int* count);
int patfft_device_alloc(int device, size_t bytes, void** ptr);
int patfft_device_free(void* ptr);
int patfft_host_alloc(size_t bytes, void** ptr);          /* pinned */
int patfft_host_free(void* ptr);
int patfft_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int patfft_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int patfft_stream_sync(void* stream);
int patfft_plan_stream(const patfft_nedner_plan* plan, void** stream);
/* f64 <-> f32 conversion on device (for the host-buffer path). */
int patfft_convert_f64_to_f32(const double* src, float* dst, size_t n, void* stream);
int patfft_convert_f32_to_f64(const float* src, double* dst, size_t n, void* stream);
/* Write `bytes` of a scratch buffer larger than L2 (cache flush between
 * timed iterations). */
int patfft_l2_flush(void* scratch, size_t bytes, void* stream);
/* CUDA-event timing on a stream: record/elapsed.  Events are opaque. */
int patfft_event_create(void** ev);
int patfft_event_record(void* ev, void* stream);
int patfft_event_elapsed_ms(void* start, void* stop, float* ms);
int patfft_event_destroy(void* ev);

#ifdef __cplusplus
}
#endif

#endif /* PATFFT_B200_H */
