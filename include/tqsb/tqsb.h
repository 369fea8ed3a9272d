/* tqsb.h -- C ABI of the B200-native RL-JSDE reconstruction library (libtqsb.so).
 *
 * Drop-in boundary for the reference entry point
 *     ReconstructionReport tqs::reconstruct(const MeasurementFrame&, const QuadrantPattern&,
 *                                           const ReconstructionConfig&, KernelCache* = nullptr,
 *                                           const Image* reference = nullptr);
 * (/root/reference/proj/include/tqs/pipeline.hpp:45-47, src/pipeline.cpp:62-185).
 *
 * A plan (tqsb_plan) plays the role of the reference's external KernelCache
 * (rljsde.hpp:81-100, pipeline.cpp:110-133): it owns the per-offset-class
 * tables resident in device memory and reuses them across calls. Plain
 * pointers and sizes only; no exceptions cross the ABI. Status codes map to the
 * reference's exception types in include/tqsb/reconstruct.hpp:
 *   TQSB_EINVAL -> std::invalid_argument   (pipeline.cpp:27-42, 66-67, 74-75, 180-181)
 *   TQSB_ELOGIC -> std::logic_error         (pipeline.cpp:146-147)
 *   TQSB_ECUDA / TQSB_ENOMEM / TQSB_ENODEV / TQSB_EIO -> std::runtime_error
 * The message of the last failure on the calling thread is tqsb_last_error().
 */
#ifndef TQSB_H
#define TQSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TQSB_OK 0
#define TQSB_EINVAL 1
#define TQSB_ECUDA 2
#define TQSB_ENOMEM 3
#define TQSB_ELOGIC 4
#define TQSB_ENODEV 5
#define TQSB_EIO 6     /* file format / I/O failure -> std::runtime_error ("<path>: <what>") */

/* Reference Precision (rljsde.hpp:22): storage precision of the reference's tables. */
#define TQSB_PRECISION_SINGLE 0
#define TQSB_PRECISION_DOUBLE 1

/* Device arithmetic of the block loop. FP32 is the product path (tables
 * accumulated in fp64, stored fp32; loop in fp32 with FFMA2). FP64 is the parity
 * mode: fp64 tables and loop, reproducing the reference's greedy paths. */
#define TQSB_COMPUTE_FP32 0
#define TQSB_COMPUTE_FP64 1

/* Reference Algorithm (pipeline.hpp:15): L-JSDE is the baseline block solver
 * (ljsde.cpp, re-summed every iteration, always fp64 on the device); RL-JSDE the
 * recurrent solver (the product path). */
#define TQSB_ALGO_LJSDE 0
#define TQSB_ALGO_RLJSDE 1

/* Mirrors ReconstructionConfig field for field (pipeline.hpp:17-26), with
 * SolverOptions (basis.hpp:77-82) and WeightingConfig (basis.hpp:15-18) inlined.
 * `threads` has no device meaning; the device set is given to tqsb_plan_create. */
typedef struct tqsb_config {
    int window;                /* W, default 32 (pipeline.hpp:18); any even W >= 2 like the
                                  reference -- W > 32 runs on the fp64 kernel in either
                                  compute mode */
    int block;                 /* B, default 4 (pipeline.hpp:19) */
    int max_iterations;        /* nu, default 200 (basis.hpp:78) */
    double step_width;         /* gamma_odc in (0,1], default 0.5 (basis.hpp:79) */
    double spatial_decay;      /* default 0.8 (basis.hpp:16) */
    double frequency_exponent; /* default 2.0 (basis.hpp:17) */
    int precision;             /* TQSB_PRECISION_*, default DOUBLE (pipeline.hpp:22) */
    int clip_output;           /* default 1 (pipeline.hpp:23) */
    int threads;               /* accepted and validated (>= 0) like the reference; unused */
    int compute;               /* TQSB_COMPUTE_*, default FP32 (the product kernel, W <= 32) */
    int hot_columns;           /* C' columns held in tensor memory; -1 = auto */
    int algorithm;             /* TQSB_ALGO_*, default RLJSDE (pipeline.hpp:15, 25) */
    int early_stop;            /* L-JSDE energy stop (basis.hpp:80), default 0 */
    double early_stop_scale;   /* stop once sum_m w_m |r_m|^2 < scale * L (basis.hpp:81), 1e-14 */
} tqsb_config;

/* Mirrors ReconstructionReport (pipeline.hpp:28-39) minus the output image,
 * which the caller owns. */
typedef struct tqsb_report {
    double seconds;            /* block-phase device time (CUDA events, max over devices) */
    double warm_seconds;       /* table precompute time of this call */
    double e2e_seconds;        /* host wall time of the whole call (copies included) */
    long long blocks_processed;
    long long classes_total;
    long long classes_interior;
    long long classes_created; /* cache misses of this call */
    long long cache_hits;      /* blocks served from resident tables (reference semantics) */
    long long cache_misses;
    double psnr_db;            /* vs reference when supplied; +inf when identical */
    int has_psnr;
    int gpu_launches;          /* kernels launched by this call */
    int compute;               /* TQSB_COMPUTE_* the call actually ran in: FP32 = the product
                                  kernel; FP64 = the reference's fp64 arithmetic (compute=fp64,
                                  L-JSDE, or W > 32 / B > 16, outside the fp32 kernel) */
} tqsb_report;

typedef struct tqsb_plan tqsb_plan;

const char* tqsb_last_error(void);
const char* tqsb_version(void);

/* Fills the reference defaults. */
void tqsb_config_default(tqsb_config* cfg);

/* validate_config (pipeline.cpp:27-42) without a device: TQSB_OK or TQSB_EINVAL. */
int tqsb_validate_config(const tqsb_config* cfg, int period);

/* Block/class census of pipeline.cpp:84-106 (host only): out[0] = blocks,
 * out[1] = classesTotal, out[2] = classesInterior. */
int tqsb_census(int frame_rows, int frame_cols, const tqsb_config* cfg, int period,
                long long out[3]);

/* Plan: validates like pipeline.cpp:27-42 and binds the pattern
 * (opaque = (period/2)^2 quadrant indices, grid.hpp:19-34) to `n_devices`
 * CUDA devices. The plan is the reference's KernelCache: the fp64 B, C, D tables of
 * each offset class are built on first use and stay resident (per device,
 * replicated), and nothing else is pinned by them. `cfg` is the default per-call
 * configuration; the *_with entry points take the configuration per call instead
 * (max_iterations, step_width, frequency_exponent, block, clip_output, compute,
 * algorithm and early stop may differ from call to call; the fp32 product tables of
 * each (frequency_exponent, step_width) are derived from the cached planes on first
 * use). Like the reference's cache, which is keyed by offset class only, classes
 * already resident are reused as built (spatial_decay and precision of the call that
 * created them); a call with a different window fails with TQSB_ELOGIC
 * ("kernel cache holds a different window size", pipeline.cpp:146-147).
 * devices = NULL uses 0..n_devices-1; a device may be listed more than once (each
 * entry is an independent context with its own streams, e.g. to exercise the
 * multi-device band split on one GPU). */
int tqsb_plan_create(const uint8_t* opaque, int period, const tqsb_config* cfg,
                     const int* devices, int n_devices, tqsb_plan** out);
int tqsb_plan_destroy(tqsb_plan* plan);

/* Host-buffer entry point, the drop-in for tqs::reconstruct: frame is
 * frame_rows x frame_cols float64 row-major (MeasurementFrame, grid.hpp:41-53),
 * out receives (2*frame_rows) x (2*frame_cols) float64 (Image, image.hpp:10-27).
 * reference (same shape as out) may be NULL; rep may be NULL. Work is split
 * across the plan's devices in block-row bands. */
int tqsb_reconstruct(tqsb_plan* plan, const double* frame, int frame_rows, int frame_cols,
                     double* out, const double* reference, tqsb_report* rep);
/* The same with a per-call configuration (NULL = the plan's): the drop-in for
 * tqs::reconstruct(frame, pattern, config, &cache, reference), pipeline.hpp:45-47. */
int tqsb_reconstruct_with(tqsb_plan* plan, const tqsb_config* config, const double* frame,
                          int frame_rows, int frame_cols, double* out, const double* reference,
                          tqsb_report* rep);

/* Band form (one process per GPU): reconstruct only output block rows
 * [block_row_begin, block_row_end) of the padded image on the plan's first
 * device. frame is the FULL host frame (only the rows the band's windows need,
 * halo included, are read); out_band receives rows
 * [block_row_begin*B, min(block_row_end*B, 2*frame_rows)) x (2*frame_cols). */
int tqsb_reconstruct_band(tqsb_plan* plan, const double* frame, int frame_rows, int frame_cols,
                          int block_row_begin, int block_row_end, double* out_band,
                          tqsb_report* rep);
int tqsb_reconstruct_band_with(tqsb_plan* plan, const tqsb_config* config, const double* frame,
                               int frame_rows, int frame_cols, int block_row_begin,
                               int block_row_end, double* out_band, tqsb_report* rep);

/* Multi-frame form (a video stream): n_frames frames of identical shape, frames[i]
 * and outs[i] host pointers (pinned buffers are used in place; pageable ones are
 * staged). Frames are distributed whole across the plan's devices; on each device
 * the H2D of frame i+1 overlaps the solve of frame i and outputs are written by
 * the kernel straight into pinned host memory. rep->blocks_processed counts all
 * frames; rep->seconds is the device span of the batch (max over devices). */
int tqsb_reconstruct_batch(tqsb_plan* plan, const double* const* frames, int n_frames,
                           int frame_rows, int frame_cols, double* const* outs, tqsb_report* rep);
int tqsb_reconstruct_batch_with(tqsb_plan* plan, const tqsb_config* config,
                                const double* const* frames, int n_frames, int frame_rows,
                                int frame_cols, double* const* outs, tqsb_report* rep);

/* Device-resident form on the plan's first device: d_frame / d_out are device
 * pointers (same layouts as tqsb_reconstruct), stream a cudaStream_t (NULL =
 * legacy default). Asynchronous: returns after enqueueing; rep->seconds is 0.
 * Tables for the frame's classes must be resident (tqsb_plan_warm) or are
 * built synchronously first. Every launch takes its own task-queue head from a
 * ring of 64 (zeroed on the launch stream), so up to 64 reconstructions may be in
 * flight on different streams at once. */
int tqsb_reconstruct_device(tqsb_plan* plan, const double* d_frame, int frame_rows,
                            int frame_cols, double* d_out, void* stream, tqsb_report* rep);
int tqsb_reconstruct_device_with(tqsb_plan* plan, const tqsb_config* config, const double* d_frame,
                                 int frame_rows, int frame_cols, double* d_out, void* stream,
                                 tqsb_report* rep);

/* Band form of the device-resident entry point (rows as tqsb_reconstruct_band;
 * d_frame is the full frame in device memory, d_out_band the band). */
int tqsb_reconstruct_band_device(tqsb_plan* plan, const double* d_frame, int frame_rows,
                                 int frame_cols, int block_row_begin, int block_row_end,
                                 double* d_out_band, void* stream, tqsb_report* rep);

/* Build (if missing) the tables of every class a frame of this size touches,
 * on every device of the plan (the reference's serial warm pass,
 * pipeline.cpp:127-133). warm_seconds may be NULL. */
int tqsb_plan_warm(tqsb_plan* plan, int frame_rows, int frame_cols, double* warm_seconds);

/* Resident table classes and their device bytes (all devices' copies of one device). */
int tqsb_plan_stats(const tqsb_plan* plan, long long* classes, long long* device_bytes);

/* Table export for parity tests (KernelSet planes, rljsde.hpp:34-52): the
 * tables of the class of window origin (origin_row, origin_col), built on the
 * plan's first device, copied to host as fp64: b (K*L complex, k-major [k*L+m]),
 * c (K*K complex, column-major [uk*K+sk]), d (K). Pass NULL b to query L. */
int tqsb_plan_export_tables(tqsb_plan* plan, int origin_row, int origin_col, int* local_out,
                            double* b_re, double* b_im, double* c_re, double* c_im, double* d);

/* TQSK table persistence (save_kernel_cache / load_kernel_cache, rljsde.cpp:337-475):
 * the same header (window, period, precision, spatial decay, frequency exponent,
 * pattern digest) and per-class planes in the config's precision, so files move
 * between this library and the reference. save writes every resident class;
 * load rejects a header that does not match the plan (TQSB_EIO, "<path>: kernel
 * cache does not match the current configuration") and makes the file's classes
 * resident on every device of the plan without the fp64 precompute. */
int tqsb_plan_save_tables(tqsb_plan* plan, const char* path, int* classes_out);
int tqsb_plan_load_tables(tqsb_plan* plan, const char* path, int* classes_out);
/* pattern_digest (rljsde.cpp:322-333): FNV-1a over the period's 4 LE bytes, then the
 * (period/2)^2 quadrant indices. */
uint64_t tqsb_pattern_digest(const uint8_t* opaque, int period);
/* kernel_memory_report (rljsde.cpp:322-335): out = {B, C, D, total} bytes of
 * `classes` table sets (local < 0: W*W/4), TQSB_PRECISION_* storage. */
int tqsb_kernel_memory_report(int classes, int window, int precision, int local, uint64_t out[4]);

/* Greedy path of one block on the device (parity diagnostics, the analogue of
 * rljsde_block's IterationHook, rljsde.hpp:75-77): y_local (L values, the
 * gather_local_values order) for a window at (origin_row, origin_col); picks
 * receive chosen flat indices, gd the scaled deltas (re, im interleaved),
 * window_out (optional) the full W*W synthesis. Returns iterations completed
 * through *n_out. Uses the plan's compute mode. */
int tqsb_plan_block_trace(tqsb_plan* plan, int origin_row, int origin_col, const double* y_local,
                          int* picks, double* gd, double* window_out, int* n_out);

/* Host helpers (test support / input side; no device needed). */
/* generate_pattern (grid.cpp:8-26): mt19937_64, low two bits per cell. */
int tqsb_generate_pattern(uint64_t seed, int period, int block, uint8_t* opaque_out);
/* simulate_measurement (grid.cpp:46-66): image rows x cols (even) -> frame. */
int tqsb_simulate(const double* image, int rows, int cols, const uint8_t* opaque, int period,
                  double* frame_out);
/* synthetic test image (tests/support/synthetic.cpp:9-80), values in [0.02, 0.98]. */
int tqsb_synthetic_image(int rows, int cols, uint64_t seed, double* out);
/* Input side on the device (no host round trip): the synthetic scene evaluated on
 * `device` into d_out (rows x cols float64; parameters drawn like the host version,
 * pixels within a few ulp of it), and the plan's sensor readout of a device image
 * (simulate_measurement, grid.cpp:46-66; image rows x cols even -> frame
 * rows/2 x cols/2 in d_frame) on the plan's first device. Asynchronous on `stream`. */
int tqsb_synthetic_image_device(int device, int rows, int cols, uint64_t seed, double* d_out,
                                void* stream);
int tqsb_plan_simulate_device(tqsb_plan* plan, const double* d_image, int rows, int cols,
                              double* d_frame, void* stream);
/* psnr (pipeline.cpp:221-233): +inf when identical. */
double tqsb_psnr(const double* reference, const double* estimate, long long n);

/* File formats (include/tqs/io.hpp:1-35, src/io.cpp of the reference); byte-identical
 * output, the same acceptance rules and "<path>: <what>" messages. No device needed.
 * tqsb_io_read: kind TQSB_IO_PGM (P5, 8/16-bit, samples / maxval), TQSB_IO_TQSM
 * (frame or raw image dump) or TQSB_IO_ANY (sniffs "TQSM", else PGM: read_image_any).
 * Pass out = NULL to query rows/cols; out receives rows*cols float64 row-major. */
#define TQSB_IO_ANY 0
#define TQSB_IO_PGM 1
#define TQSB_IO_TQSM 2
int tqsb_io_read(const char* path, int kind, int* rows, int* cols, double* out);
/* write_pgm (io.cpp:99-131): bits 8 or 16, values clamped to [0,1] and rounded. */
int tqsb_io_write_pgm(const char* path, const double* image, int rows, int cols, int bits);
/* TQSM container: "TQSM", u32 rows, u32 cols (LE), float64 payload (write_frame /
 * write_raw_image). */
int tqsb_io_write_tqsm(const char* path, const double* values, int rows, int cols);
/* TQSP pattern text (read_pattern / write_pattern, io.cpp:133-199). rng receives the
 * generator name (NUL-terminated, truncated to rng_cap-1); opaque (nullable) receives
 * (period/2)^2 quadrant indices. */
int tqsb_io_read_pattern(const char* path, int* period, uint64_t* seed, char* rng, size_t rng_cap,
                         uint8_t* opaque);
int tqsb_io_write_pattern(const char* path, int period, uint64_t seed, const char* rng,
                          const uint8_t* opaque);

/* Pinned host memory for zero-staging transfers (cudaHostAlloc). */
void* tqsb_host_alloc(size_t bytes);
void tqsb_host_free(void* p);
int tqsb_device_count(void);

/* Diagnostics: measured roofline denominators of `device` -- FP32 pipe peak
 * (FFMA2 chains, TFLOP/s) and shared-memory load bandwidth (LDS.128, TB/s). */
int tqsb_probe_peaks(int device, double* fp32_tflops, double* smem_tbps);

#ifdef __cplusplus
}
#endif
#endif /* TQSB_H */
