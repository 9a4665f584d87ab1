/*
 * holospots_b200.h -- C ABI of the B200-native CS-WGS hologram solver.
 *
 * The reference (`holospots`, pure Python + numba) has no FFI; its hot-path
 * boundary is the module-level Python API (holospots/__init__.py:18-29).
 * Each entry point below replaces one of those calls; the Python package
 * `paper_2003_05293_b200` binds them with ctypes and
 * keeps the reference signatures, argument meanings and exceptions.
 *
 *   hs_plan_create   <- geometry upload that the reference repeats on every
 *                       call (Pupil arrays, optics.py:63-214)
 *   hs_set_spots     <- spot_tables (kernels.py:177-183, _build_tables 78-96)
 *   hs_superpose     <- superpose (kernels.py:186-214)
 *   hs_forward       <- forward_project (kernels.py:217-246)
 *   hs_quality       <- quality_report / spot_intensities (metrics.py:33-79)
 *   hs_solve         <- rs / wgs / cswgs / solve (solvers.py:179-282), batched
 *   hs_get_*         <- the (Hologram, SolverTrace) / QualityReport results
 *
 * Conventions
 *   - All host arrays are plain C arrays (float64 unless noted), row-major.
 *   - Complex values are interleaved (re, im) float64 pairs.
 *   - Pixel arrays are in the pupil's storage order (optics.py:184-192).
 *   - Every call is synchronous with respect to host buffers: when it
 *     returns, host outputs are written and host inputs may be reused.
 *     hs_solve_async is the exception (device-resident; see below).
 *   - A plan is bound to one CUDA device and one stream; it is not
 *     thread-safe (like the reference's process-global worker pool,
 *     kernels.py:154-165).
 *   - Results never depend on launch configuration, batch size or batch
 *     position of a pattern (fixed-shape reductions), mirroring the
 *     reference determinism contract (kernels.py:16-21).
 *
 * Status codes (returned by every int function; the Python layer maps them
 * onto the holospots.errors hierarchy, errors.py:4-29):
 */
#ifndef HOLOSPOTS_B200_H
#define HOLOSPOTS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_OK 0
#define HS_EINVAL 1        /* InvalidParameterError */
#define HS_EGEOMETRY 2     /* GeometryMismatchError */
#define HS_EDEGENERATE 3   /* DegenerateFieldError: all spot fields vanished */
#define HS_EDIVERGED 4     /* DegenerateFieldError: weights left float range */
#define HS_ECUDA 5         /* device / launch / allocation failure */
#define HS_EZEROILLUM 6    /* ZeroIlluminationError */
#define HS_EUNDEFINED 7    /* UndefinedUniformityError */

#define HS_ALG_RS 0
#define HS_ALG_WGS 1
#define HS_ALG_CSWGS 2

/* hs_solve flags */
#define HS_WANT_FIELDS 1   /* fuse the full-range e/u projection into the last pass */
#define HS_WANT_RASTER 2   /* also write the SLM gray raster (default linear LUT) */
#define HS_WANT_PHASE32 4  /* fp32 solves: the last pass stores 4-byte phase codes; hs_get_phase
                              widens them on the host to the identical f64 phases (half the
                              device->host bytes; hs_solve_host always does this) */

/* Pixel-pass arithmetic (hs_set_precision).  The reference computes in fp64
 * throughout (holospots/kernels.py:78-144).  FP32: fp32 pixel products with
 * fp64 tables / folds / updates (the fast kernels).  FP64: every pixel
 * product in fp64.  AUTO (default): FP64 when the smallest pixel set a call
 * projects over has fewer than 512 pixels per spot, or n > 1024; else FP32. */
#define HS_PREC_AUTO 0
#define HS_PREC_FP32 1
#define HS_PREC_FP64 2

typedef struct hs_plan hs_plan;

/* Human-readable message for the last failing call on this thread. */
const char *hs_last_error(void);

/* Number of visible CUDA devices (0 on a host without a GPU). */
int hs_device_count(int *count);

/* Largest spot count one pattern may carry (4096; above 1024 spots the
 * passes run in fp64). */
int hs_max_spots(void);

/* Upload pupil geometry once.  rows/cols/amplitude: m storage-order pixels;
 * axis: side grid-line coordinates (Pupil.axis_coords, optics.py:111-115);
 * prism/lens: Pupil.prism_coeff / lens_coeff (optics.py:101-109);
 * sum_amplitude: Pupil.sum_amplitude (optics.py:213). */
int hs_plan_create(int device, int side, int64_t m, const int64_t *rows,
                   const int64_t *cols, const double *amplitude,
                   const double *axis, double prism, double lens,
                   double sum_amplitude, hs_plan **out);
void hs_plan_destroy(hs_plan *plan);

/* Precision mode of the plan's pixel passes (HS_PREC_*); the environment
 * variable HS_PRECISION=auto|fp32|fp64 sets the default of new plans.
 * hs_get_precision: the mode, and the precision the last solve ran in
 * (HS_PREC_FP32 or HS_PREC_FP64). */
int hs_set_precision(hs_plan *plan, int mode);
int hs_get_precision(hs_plan *plan, int *mode, int *last_solve);

/* Spot targets of `batch` independent patterns with n spots each:
 * x, y, z, a0 are [batch][n].  Builds the per-pattern phasor tables on
 * the device (kernels.py:78-96). */
int hs_set_spots(hs_plan *plan, int batch, int n, const double *x,
                 const double *y, const double *z, const double *a0);

/* Test hook: one device weight update (rebalance_weights, solvers.py:104-129)
 * of n spots from weights w_in[n] and fields[2n] (a0 = 1) on the current
 * device.  w_out / mags_out receive the new weights and the magnitudes used
 * (floored); status: HS_OK, HS_EDEGENERATE (all fields zero) or HS_EDIVERGED
 * (a weight left float range; outputs then undefined); degenerate: 1 when
 * a zero magnitude was floored. */
int hs_debug_update(int n, const double *w_in, const double *fields, double *w_out,
                    double *mags_out, int *status, int *degenerate);

/* Phasor tables of pattern 0 (SpotTables, kernels.py:61-76, 177-183):
 * gx_re/gx_im/gy_re/gy_im are [side][n] fp64 row-major.
 * hs_get_tables builds them on the device (the reference's operation order
 * for the arguments, fp64 sincos) and copies them out.
 * hs_set_tables installs caller tables for pattern 0 (batch 1, n spots) --
 * the `tables=` argument of superpose / forward_project: the following API
 * passes use them (rounded once to fp32 on the fp32 passes) until the spot
 * set changes or a solve rebuilds the tables from the spots. */
int hs_get_tables(hs_plan *plan, double *gx_re, double *gx_im, double *gy_re, double *gy_im);
int hs_set_tables(hs_plan *plan, int n, const double *gx_re, const double *gx_im,
                  const double *gy_re, const double *gy_im);

/* Backward pass of pattern 0 over storage pixels [start, stop):
 * out[stop-start] receives wrapped phases (kernels.py:186-214).
 * amplitude/theta: [n] superposition coefficients (SpotCoefficients). */
int hs_superpose(hs_plan *plan, const double *amplitude, const double *theta,
                 int64_t start, int64_t stop, double *out);

/* Forward pass of pattern 0: phase[m] storage order; fields[2n] receives
 * the per-spot complex sums over [start, stop) (kernels.py:217-246). */
int hs_forward(hs_plan *plan, const double *phase, int64_t start, int64_t stop,
               double *fields);

/* Full-range projection + metrics of pattern 0 (metrics.py:71-79):
 * e, u scalars; intensities[n], relative[n]; fields[2n] (may be NULL). */
int hs_quality(hs_plan *plan, const double *phase, double *e, double *u,
               double *intensities, double *relative, double *fields);

/* Far-field probe intensities (simulate.py:48-63): |E|^2 / (sum A)^2 of the
 * hologram phase[m] at npts probe positions xyz[npts][3], evaluated in
 * chunks of `batch` probes with the same kernels and normalisation as
 * hs_quality (a probe on a target spot reproduces its intensity bit for
 * bit).  Replaces the plan's current spot set. */
int hs_probe(hs_plan *plan, const double *phase, int64_t npts, const double *xyz,
             int batch, double *out);

/* SLM gray raster [side][side] (uint8, 0 outside the aperture) of a
 * storage-order phase[m] through a 256-entry phase LUT (NULL = the default
 * linear table); equals write_hologram_pgm's raster (fileio.py:233-241,
 * PhaseLut.gray fileio.py:202-213) bit for bit. */
int hs_raster(hs_plan *plan, const double *phase, const double *lut, unsigned char *out);

/* Rasters [count][side][side] built by the last pass of a solve run with
 * HS_WANT_RASTER (linear LUT fused into the phase write). */
int hs_get_raster(hs_plan *plan, int first, int count, unsigned char *out);

/* Run `algorithm` on all patterns of the current spot batch.
 * iterations: I (ignored for RS); subset: ceil(c*M) for CS-WGS (M for WGS);
 * theta0: [batch][n] starting phase offsets (solvers.py:169-170).
 * hs_solve_async only enqueues work on the plan stream (results stay on the
 * device; poll with hs_sync); hs_solve also waits for completion. */
int hs_solve_async(hs_plan *plan, int algorithm, int iterations,
                   int64_t subset, const double *theta0, int flags);
int hs_solve(hs_plan *plan, int algorithm, int iterations, int64_t subset,
             const double *theta0, int flags);
int hs_sync(hs_plan *plan);

/* Results of the last solve.
 * hs_get_status: status[batch] per pattern (HS_OK / HS_EDEGENERATE /
 *   HS_EDIVERGED), degenerate[batch] trace flags (solvers.py:116-122).
 * hs_get_trace: weights, mags [batch][iterations][n] (StepRecord,
 *   solvers.py:61-70).
 * hs_get_phase: phase[count][m] for patterns first..first+count-1.
 * hs_get_quality: e[batch], u[batch], intensities/relative [batch][n],
 *   fields [batch][2n]; any pointer may be NULL.  Needs HS_WANT_FIELDS. */
int hs_get_status(hs_plan *plan, int32_t *status, int32_t *degenerate);
int hs_get_trace(hs_plan *plan, double *weights, double *mags);
int hs_get_phase(hs_plan *plan, int first, int count, double *phase);
int hs_get_quality(hs_plan *plan, double *e, double *u, double *intensities,
                   double *relative, double *fields);

/* End-to-end call used by bench.py's e2e leg: uploads spots + theta0 from
 * host memory, solves, and copies phases [batch][m], e[batch], u[batch]
 * back to host memory.  Equivalent to hs_set_spots + hs_solve +
 * hs_get_phase + hs_get_quality.  fp32 solves split the phase download:
 * the first hs_host_copy_split patterns are widened to f64 on the device and
 * copied as f64, the rest cross the link as 4-byte codes and are widened on
 * the host threads (HS_E2E_F64_FRAC, default 0.375; HS_E2E_CODES=0 ships all
 * as f64) -- identical f64 bits either way. */
int hs_host_copy_split(hs_plan *plan, int batch, int *f64_patterns);
int hs_solve_host(hs_plan *plan, int algorithm, int iterations, int64_t subset,
                  int batch, int n, const double *x, const double *y,
                  const double *z, const double *a0, const double *theta0,
                  double *phase, double *e, double *u);

/* Pipelined form of hs_solve_host: returns once the work is enqueued.  Host
 * buffers must be page-locked (hs_host_alloc) and stay valid until hs_sync.
 * The phase download of call k runs on a copy stream and overlaps the solve
 * of call k+1 (device phase outputs are double-buffered). */
int hs_solve_host_async(hs_plan *plan, int algorithm, int iterations, int64_t subset,
                        int batch, int n, const double *x, const double *y,
                        const double *z, const double *a0, const double *theta0,
                        double *phase, double *e, double *u);

/* Row-sharded solve of one batch across `world` processes (one per GPU,
 * SURVEY.md 8(e)).  Every rank calls, with identical spots and theta0:
 *   hs_shard_begin(...);
 *   for j in 0 .. passes-1   (passes = 1 for RS, iterations + 1 otherwise):
 *       hs_shard_pass(j, local, &g_lo, &g_hi, &ngroups);
 *       all_groups = all-gather(local) in rank order   (caller: NCCL / gloo)
 *       hs_shard_update(j, all_groups, ngroups);
 * `local` / `all_groups` hold complex128 group partials laid out
 * [batch][groups][np] (np = hs_padded_spots).  Ranks own fold-group-aligned
 * chunk ranges (pixel-row slabs), so every rank folds the same group
 * sequence: fields, weights, e/u are bitwise identical on all ranks and to
 * hs_solve.  Phases of pixels another rank owns are NaN in hs_get_phase. */
int hs_shard_begin(hs_plan *plan, int algorithm, int iterations, int64_t subset,
                   const double *theta0, int rank, int world);
int hs_shard_pass(hs_plan *plan, int pass, double *local_groups, int *g_lo, int *g_hi,
                  int *ngroups);
int hs_shard_update(hs_plan *plan, int pass, const double *all_groups, int ngroups);
/* Group range [g_lo, g_hi) of this rank and the total group count of pass j. */
int hs_shard_groups(hs_plan *plan, int pass, int *g_lo, int *g_hi, int *ngroups);

/* The same sharded solve with the exchange over peer memory (NVLink P2P
 * through CUDA IPC) instead of a host round trip per pass
 * (csrc/hs_xchg.cuh).  After hs_shard_begin:
 *   hs_shard_p2p_setup(handle)            this rank's exchange buffer; writes
 *                                         its cudaIpcMemHandle (HS_IPC_HANDLE_BYTES)
 *   handles = all-gather(handle)          rank order, caller (once per solve)
 *   hs_shard_p2p_open(handles)            maps the peers' buffers
 *   for j: hs_shard_p2p_pass(j)           enqueues the rank's chunk range, the
 *                                         publish of its group partials into every
 *                                         rank's buffer and the gather + update;
 *                                         no host synchronisation
 *   hs_sync(); hs_shard_p2p_close()
 * Results are bitwise identical to hs_shard_pass / hs_shard_update and to
 * hs_solve.  A peer that never publishes times out after ~2 s (status 5). */
#define HS_IPC_HANDLE_BYTES 64
int hs_shard_p2p_setup(hs_plan *plan, unsigned char *ipc_handle_out);
int hs_shard_p2p_open(hs_plan *plan, const unsigned char *ipc_handles);
int hs_shard_p2p_pass(hs_plan *plan, int pass);
/* All passes of the begun sharded solve in one call: captured into a CUDA
 * graph on first use (per algorithm, iterations, subset, batch, n, rank and
 * world) and replayed; equal to calling hs_shard_p2p_pass for every pass. */
int hs_shard_p2p_solve(hs_plan *plan);
int hs_shard_p2p_close(hs_plan *plan);
int hs_padded_spots(hs_plan *plan);

/* Instrumentation for bench.py: the plan's cudaStream_t, the number of
 * kernels the last solve launched, and the mean device time (CUDA events,
 * `reps` back-to-back launches on the plan stream) of the kernel `which`
 * (0 = full-range fused pass, 1 = compressed-window fused pass,
 * 2 = full-range fused pass of the final iteration, with the f64 phase
 * written in storage order, 3 = the same storing 4-byte phase codes, as
 * solves do) with the current spot batch. */
void *hs_plan_stream(hs_plan *plan);
int hs_last_launch_count(hs_plan *plan, int64_t *launches);
int hs_time_kernel(hs_plan *plan, int which, int64_t subset, int reps,
                   double *ms_per_launch, double *pairs_per_launch);

/* Measured FP32 FFMA throughput of `device` in TFLOP/s (2 FLOP per FFMA),
 * the roofline denominator for the FMA-bound pass kernel. */
int hs_fma_peak(int device, double *tflops);

/* Page-locked host buffers for the e2e path (cudaHostAlloc / cudaFreeHost). */
void *hs_host_alloc(int64_t bytes);
void hs_host_free(void *ptr);

#ifdef __cplusplus
}
#endif
#endif /* HOLOSPOTS_B200_H */
