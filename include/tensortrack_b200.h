/*
 * tensortrack_b200 — C ABI of the B200-native online tensor-subspace tracker.
 *
 * Drop-in boundary for the hot path of the reference package `tensortrack`
 * (arXiv 1609.04104 reference, /root/reference/pkg/src/tensortrack). The
 * reference has no FFI of its own: its boundary is the Python function API
 * (`__init__.py:3-62`). These entry points are what that API binds to; the
 * Python mirror lives in `paper_1609_04104_b200/` and the ctypes binding a
 * maintainer would add is shown in INTEGRATION.md.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers unless stated otherwise.
 *  - complex64 arrays are interleaved (re, im) float pairs; complex128 are
 *    interleaved doubles.
 *  - Factor matrices are row-major (N, R) per slice: [nslices][N][R].
 *  - "k-space factors" Ah = F_x A, Bh = F_y B (ortho, unshifted DFT down the
 *    columns, observation.py:225-226). The row-mask step runs on them; the
 *    image-domain factors are A = F_x^-1 Ah (tt_fft_cols, inverse=1).
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*),
 *    takes no locks, never aborts, and returns a status code:
 *      TT_OK          0  success
 *      TT_EINVAL      1  invalid argument  -> ValueError   (observation.py:41-55)
 *      TT_EUNSUPPORTED 2 unsupported shape/descriptor -> TypeError (tracker.py:238)
 *      TT_ENONFINITE  3  non-finite result -> NumericalError (experiment.py:66)
 *      TT_ECUDA       4  CUDA error        -> RuntimeError
 *    Device-side problems (bad row ids in a table, non-finite gamma) are
 *    OR-ed into the caller's `status` array (TT_ST_* bits) for a later read.
 *  - tt_last_error() returns a thread-local message for the last failure.
 */
#ifndef TENSORTRACK_B200_H
#define TENSORTRACK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { TT_OK = 0, TT_EINVAL = 1, TT_EUNSUPPORTED = 2, TT_ENONFINITE = 3, TT_ECUDA = 4 };

/* device status bits */
enum { TT_ST_BADROW = 1, TT_ST_DUPROW = 2, TT_ST_NONFINITE = 4, TT_ST_ZEROCOL = 8, TT_ST_OVERFLOW = 16 };

enum { TT_POLICY_STATIC = 0, TT_POLICY_INFORMATIVE = 1 };
enum { TT_Y_GATHER = 0, TT_Y_PACKED = 1 };
enum { TT_STEP_FIXED = 0, TT_STEP_HESSIAN = 1 };

const char* tt_version(void);
const char* tt_last_error(void);

/* ------------------------------------------------------------------ FFT
 * Batched ortho 1-D DFT down the columns of `batch` row-major (n x ncols)
 * complex64 matrices, in place. inverse=0: F (np.fft.fft(.., axis=0,
 * norm="ortho")); inverse=1: F^-1. Replaces observation.py:225-226 (build_phi
 * Fourier branch) and the x/y inverse transforms inside _scatter_theta
 * (tracker.py:186-188) by the separable identity F(a b^T) = (F a)(F b)^T.
 * n = 16 ... 1024 (powers of two) use a two-level register transform (one
 * shared-memory exchange), other powers of two <= 4096 shared-memory Stockham
 * passes; other n use a direct DFT (exact same convention). */
int tt_fft_cols(void* stream, float* data, int n, int ncols, int batch, int inverse);
/* The same ortho DFT along the LAST axis: `nrows` contiguous rows of n complex64, in place (n a power of two
 * from 16 to 1024; other n: TT_EUNSUPPORTED). tt_fft_cols then tt_fft_rows over a batch of (nx x ny) frames is the
 * unshifted ortho 2-D DFT of observation.py:171-183 (np.fft.fft2(.., norm="ortho")) without transposes. */
int tt_fft_rows(void* stream, float* data, long long nrows, int n, int inverse);

/* ------------------------------------------------------------------ row-mask step
 * Persistent fused online step for Cartesian row masks (the path of
 * tracker.track_step with a FourierMask whose indices are full phase-encode
 * lines, tracker.py:367-411, and of experiment.run_adaptive's per-frame body,
 * experiment.py:482-530). One thread-block cluster of `cluster` CTAs per
 * slice runs `frames` consecutive frames: [informative draw] -> gather y ->
 * separable Gram/rhs -> fp64 LDL^H ridge solve -> Lipschitz/fixed step ->
 * k-space factor update. State stays resident in shared memory across frames.
 */
typedef struct tt_rows_args {
  int32_t nslices, nx, ny, rank, frames, max_rows, cluster;
  int64_t t0;                 /* tracker time of frame 0 (same for every slice) */
  const float* ah_in;         /* [nslices][nx][rank] complex64 k-space factors */
  const float* bh_in;         /* [nslices][ny][rank] */
  float* ah_out;              /* may alias ah_in */
  float* bh_out;              /* may alias bh_in */
  double* alpha_bar;          /* [nslices] in/out (HessianBound running sum) */
  int32_t policy;             /* TT_POLICY_* */
  const int32_t* rows_tab;    /* static: [frames][nslices][max_rows] */
  const int32_t* rows_cnt;    /* static: [frames][nslices] */
  int32_t k_draws;            /* informative: trials K (forced lines count) */
  const int32_t* forced;      /* informative: sorted unique forced rows */
  int32_t nforced;
  double beta;                /* uniform blend weight (sampler.py:32) */
  uint64_t key0, key1;        /* Philox key; slice s draws with (key0, key1 + s) */
  uint64_t* philox_pos;       /* [nslices] stream positions, in/out */
  int32_t y_mode;             /* TT_Y_* */
  const float* ysrc;          /* GATHER: truth k-space, frame f slice s row i at
                                 ysrc + (f*y_frame_stride + s*y_slice_stride + i*ny)*2
                                 PACKED: [frames][nslices][max_rows][ny] */
  int64_t y_frame_stride, y_slice_stride; /* complex elements (GATHER) */
  double lam;
  int32_t step_mode;          /* TT_STEP_* */
  double mu, c_floor, c_cap;
  float* gamma_out;           /* [frames][nslices][rank] complex64 or NULL */
  double* cost_out;           /* [frames][nslices] or NULL */
  double* mu_out;             /* [frames][nslices] or NULL */
  double* alpha_out;          /* [frames][nslices] or NULL */
  int32_t* rows_out;          /* [frames][nslices][max_rows] or NULL */
  int32_t* cnt_out;           /* [frames][nslices] or NULL */
  float* resid_out;           /* [frames][nslices][max_rows][ny] complex64 or NULL */
  float* ah_hist;             /* [frames][nslices][nx][rank] post-update or NULL */
  float* bh_hist;             /* [frames][nslices][ny][rank] or NULL */
  int32_t* status;            /* [nslices] OR-ed TT_ST_* bits */
  void* scratch;              /* tt_rows_scratch_bytes() bytes */
  int64_t* phase_clock;       /* optional profiling: [frames][32] SM clock64 stamps of CTA 0, or NULL */
  /* Row sharding across GPUs (BASELINE config 4; 0 = off). Rank `shard_rank` of
   * `shard_world` owns k-space rows [nx*rank/world, nx*(rank+1)/world) of Ah; ah_in/ah_out
   * then hold only those rows, Bh is replicated. Each frame is two launches:
   * phase 1 writes this rank's partial payload (xw: W = Y^T conj(Ah_S) [ny][rank]
   * complex128 (fp64 sums of exact products); xg: packed GA (R(R+1)/2 complex128), ||Y||^2,
   * ||Ah||^2 as doubles), all doubles, so a caller that places xg right after xw
   * (xg = xw + 2*ny*rank) all-reduces the frame's payload in ONE sum over the ranks
   * (2*ny*rank + tt_rows_shard_xg_len(rank) doubles); phase 2 solves
   * redundantly and updates the owned rows and the replicated Bh. Static row
   * policy, nslices = 1, frames = 1 per launch. */
  int32_t shard_rank, shard_world, shard_phase;
  double* xw;
  double* xg;
  /* Local multi-rank launch (appended; 0 = off): all shard_world ranks are clusters of one launch
   * on this GPU (shard_rank ignored). ah_in/ah_out/ah_hist hold all nx rows; xw/xg hold one
   * payload slot per rank; tt_rows_shard_reduce sums the slots into slot 0, which phase 2 reads. */
  int32_t shard_local;
  /* Fused local multi-rank launch (appended; 0 = off; needs shard_local, static rows): one
   * cooperative cluster launch runs all `frames` frames, both phases per frame, with two
   * inter-cluster barriers per frame on `grid_sync` (one zeroed uint32 per launch) around an
   * in-kernel payload reduction in tt_rows_shard_reduce's order. xw/xg then hold two sets of
   * shard_world slots (frame parity). */
  int32_t shard_fused;
  uint32_t* grid_sync;
  /* Informative draws without replacement (appended; 0 = with replacement): draw_samples(replacement=False)
   * (sampler.py:163-169): the forced rows' weights zeroed, k - nforced sequential renormalised draws
   * (observation.py:279-297, one uniform each), union with the forced rows, sorted. */
  int32_t draw_wor;
  /* TrackerConfig.norm_cap (tracker.py:406-408; appended): when norm_out is non-NULL,
   * norm_out[f][s] = 1 if frame f's post-update ||A||_F or ||B||_F exceeds norm_cap, else 0 (the DFT is
   * unitary, so ||Ah||_F = ||A||_F; 0 for a frame without samples, which does not update). Not with
   * row sharding. */
  double norm_cap;
  int32_t* norm_out;
  /* Informative draws under row sharding (appended; NULL = off): the raw row scores of all nx rows
   * (tt_rows_shard_scores over the all-gathered row energies), identical on every rank, so every rank
   * draws the same rows from the shared Philox stream. Phase 1 only, one GPU per rank: the full drawn
   * row set goes to rows_out / cnt_out (frame 0 slots), which the caller passes to phase 2 as its
   * static table. */
  const double* sraw_in;
  /* Truth in host memory (appended; 0 = device memory): ysrc is a page-locked host buffer addressed through
   * unified virtual addressing, and the kernel reads only the frame's sampled rows over the host link
   * (zero-copy: the truth is consulted only at the sampled rows, as run_adaptive's StreamingProvider
   * consults it, experiment.py:70-111) instead of the caller uploading every frame. */
  int32_t y_host;
} tt_rows_args;
/* Row energies of a rank's owned k-space rows: energy [nx][rank] (fp64) gets E[i][r] = |Ah_ir|^2 for the owned
 * rows [r0, r0 + nrows) (ah_rows [nrows][rank] complex64) and 0 elsewhere, so a sum all-reduce over the ranks
 * assembles the full matrix exactly (x + 0 = x). */
int tt_rows_shard_energy(void* stream, int nx, int rank, int r0, int nrows, const float* ah_rows, double* energy);
/* Raw row scores from the full energy matrix (row_scores before normalisation, sampler.py:115-126):
 * nrm_r = sum_i E[i][r] (fixed order), s_i = (ny sum_r E[i][r] / nrm_r + R) / (R (nx + ny)) -> sraw [nx];
 * a zero column ORs TT_ST_ZEROCOL into status[0]. Identical bits on every rank for identical inputs. */
int tt_rows_shard_scores(void* stream, int nx, int ny, int rank, const double* energy, double* sraw, int32_t* status);
/* plan of a row-mask launch at `cluster` (0: smallest that fits): out[6] = cluster, rows per k tile,
 * shared-memory bytes, tight plan (0/1), padded Y row stride, K-split buffer entries (diagnostics) */
int tt_rows_plan_info(int nx, int ny, int rank, int max_rows, int cluster, int* out);
/* how many clusters of `cluster` CTAs of the row-mask kernel (this shape's shared-memory plan) the current
 * device holds at once (cudaOccupancyMaxActiveClusters): a launch with more slices than this runs in waves, so
 * the host picks the widest cluster whose count covers the slices (the reference has no counterpart: its
 * slices are a Python loop, experiment.py:332-441) */
int tt_rows_max_clusters(int nx, int ny, int rank, int max_rows, int cluster, int* nclusters);
/* doubles in the fp64 payload xg of a sharded launch */
size_t tt_rows_shard_xg_len(int rank);
/* 1 when tt_track_rows runs the mirrored kernel for this shape at `cluster` (every CTA holds the whole Ah;
 * two cluster barriers per frame, exchanges through distributed shared memory; opt-in with the environment
 * variable TT_ROWS_MIRROR=1), else 0 (the L2-exchange kernel runs); diagnostics / tests. */
int tt_rows_mirror_fits(int nx, int ny, int rank, int max_rows, int cluster);
/* sum the `world` payload slots of a local multi-rank phase-1 launch into slot 0 (fixed order) */
int tt_rows_shard_reduce(void* stream, int world, int ny, int rank, double* xw, double* xg);

/* Choose the cluster size (if *cluster <= 0) and report the dynamic shared
 * memory per CTA; TT_EUNSUPPORTED if no cluster size fits. */
int tt_rows_plan(int nx, int ny, int rank, int max_rows, int policy, int* cluster, size_t* smem_bytes);
size_t tt_rows_scratch_bytes(int nslices, int nx, int ny, int rank, int max_rows, int cluster);
int tt_track_rows(void* stream, const tt_rows_args* a);

/* ------------------------------------------------------------------ generic index step
 * One frame of tracker.track_step for an arbitrary (i, j) index list
 * (FourierMask / EntryMask, observation.py:58-90) on measurement-domain
 * factors: Gram over |Omega| samples (fp64), ridge solve, residual, dense
 * back-projection P = Xi conj(Bh), Q = Xi^T conj(Ah) (the collapsed form of
 * tracker.py:176-228), closed-form Lipschitz bound, update. */
typedef struct tt_entries_args {
  int32_t nx, ny, rank, nmeas;
  int64_t t;
  const float* ah_in;
  const float* bh_in;
  float* ah_out;
  float* bh_out;
  double* alpha_bar;          /* [1] */
  const int32_t* idx;         /* [nmeas][2] (i, j) */
  const float* y;             /* [nmeas] complex64 */
  double lam;
  int32_t step_mode;
  double mu, c_floor, c_cap;
  float* gamma_out;           /* [rank] */
  double* cost_out;           /* [1] */
  double* mu_out;             /* [1] */
  double* alpha_out;          /* [1] */
  float* resid_out;           /* [nmeas] or NULL */
  int32_t* status;            /* [1] */
  void* scratch;
  /* Optional device-side count (appended): when non-NULL the step uses
   * *nmeas_dev measurements and `nmeas` is only the capacity of idx / y.
   * An empty batch then runs as a zero step (mu = 0) on the device, so the
   * whole per-frame chain can be captured in a CUDA graph. */
  const int32_t* nmeas_dev;
  /* Optional flat-index form (appended): when `omega` is non-NULL the step reads entry l as
   * w = omega[l], (i, j) = (w / ny, w % ny), y = frame[w] (frame [nx][ny] complex64, the resident
   * truth) and ignores idx / y, so a device-side draw feeds the step without a gather pass. */
  const int32_t* omega;
  const float* frame;
} tt_entries_args;
/* Scratch for tt_track_entries: zero-fill it before its first use and reuse it for later steps
 * of the same shape (it carries a per-step stamp that replaces clearing the residual image). */
size_t tt_entries_scratch_bytes(int nx, int ny, int rank, int nmeas);
int tt_track_entries(void* stream, const tt_entries_args* a);

/* Acquisition at drawn entries (adaptive_step's truth lookup, sampler.py:204-206)
 * on the device: omega [cap] flat indices i*ny + j (sorted unique, the first
 * *count valid), frame [nx][ny] complex64 -> idx_out [cap][2] (i, j) and
 * y_out [cap] complex64 for the first *count entries. */
int tt_gather_entries(void* stream, int nx, int ny, const float* frame, const int32_t* omega,
                      const int32_t* count, int cap, int32_t* idx_out, float* y_out);

/* ------------------------------------------------------------------ standalone step pieces
 * For the reference API functions called on their own, on measurement-domain
 * factors (Fourier masks: Ah = F_x A, Bh = F_y B) and an (i, j) index list:
 *  tt_residual:   e = y - Phi gamma (tracker.py:388; instantaneous_cost :163-173)
 *  tt_data_terms: D_A = conj(gamma) . Xi conj(Bh) (nx x R), D_B = conj(gamma) . Xi^T conj(Ah)
 *                 (ny x R), Xi = scatter(e) (_gradient_data_terms, tracker.py:208-228), and
 *                 cmax[r] = max(max_i sum_{j:(i,j)} |Bh_jr|^2, max_j sum_i |Ah_ir|^2), the exact
 *                 curvature of hessian_bound (tracker.py:337-364).
 * gamma is complex64 [R]; scratch: tt_terms_scratch_bytes(). */
size_t tt_terms_scratch_bytes(int nx, int ny, int rank);
int tt_residual(void* stream, int nx, int ny, int rank, int nmeas, const float* ah, const float* bh,
                const int32_t* idx, const float* y, const float* gamma, float* e_out);
int tt_data_terms(void* stream, int nx, int ny, int rank, int nmeas, const float* ah, const float* bh,
                  const int32_t* idx, const float* e, const float* gamma, float* dA, float* dB, double* cmax,
                  void* scratch);

/* ------------------------------------------------------------------ sampling
 * row_scores (sampler.py:115-128) on the factor `a` ([nslices][nx][rank]):
 * s(i) = (ny e_i + R)/(R (nx + ny)), e_i = sum_r |a_ir|^2/||a_r||^2,
 * normalised, blended with beta/nx, renormalised; fp64 out [nslices][nx]. */
int tt_row_scores(void* stream, int nslices, int nx, int ny, int rank, const float* a, double beta,
                  double* probs_out, int32_t* status);
/* entry_scores (sampler.py:95-112): [nx][ny] fp64 */
int tt_entry_scores(void* stream, int nx, int ny, int rank, const float* a, const float* b, double beta,
                    double* probs_out, int32_t* status);
/* the same with a caller-owned workspace of tt_entry_scores_ws_bytes(nx, ny) bytes (no per-call
 * allocation; the form the device engines and captured graphs use) */
size_t tt_entry_scores_ws_bytes(int nx, int ny);
int tt_entry_scores_ws(void* stream, int nx, int ny, int rank, const float* a, const float* b, double beta,
                       double* probs_out, int32_t* status, void* ws);
/* draw_samples(replacement=True) (sampler.py:146-162): k - nforced draws of
 * Generator(Philox(key)).choice(n, p=probs) at stream positions pos[s]..,
 * union with forced -> sorted unique rows. Bit-exact with numpy for the
 * same probabilities (sequential fp64 cumsum semantics). */
int tt_draw_with_replacement(void* stream, int nslices, int n, const double* probs, int k,
                             const int32_t* forced, int nforced, uint64_t key0, uint64_t key1,
                             uint64_t* pos, int32_t* omega_out, int32_t* count_out);
/* The same draw over a domain too large for one CTA (entry sampling over
 * nx*ny): two-level parallel scan in global memory, one binary search per
 * draw, exact sequential fallback near bucket edges, compaction. One slice;
 * omega_out [k] sorted unique, *count_out valid; *pos advances by k - nforced.
 * The flags in scratch must start zeroed (cudaMemset once) and are left
 * zeroed. scratch: tt_draw_scratch_bytes(n). Graph-capturable. */
size_t tt_draw_scratch_bytes(int n);
int tt_draw_with_replacement_large(void* stream, int n, const double* probs, int k, const int32_t* forced,
                                   int nforced, uint64_t key0, uint64_t key1, uint64_t* pos,
                                   int32_t* omega_out, int32_t* count_out, void* scratch);
/* weighted_draw_without_replacement (observation.py:279-297): k sequential
 * renormalised draws, draw order; consumes k uniforms from pos[0]. */
int tt_draw_without_replacement(void* stream, int n, const double* weights, int k, uint64_t key0,
                                uint64_t key1, uint64_t* pos, int32_t* out, int32_t* status);
/* variable_density_rows (observation.py:300-323) for `frames` frames of `nslices` slices in one launch:
 * frame f of slice s is the DC row then n_rows - 1 sequential draws without replacement with `weights`
 * (the reference's d**alpha / 2 per row, DC 0; computed by the caller) from the Philox stream
 * (key0, key1 + s) at position pos0[s] + f (n_rows - 1) (pos0 NULL: 0), in draw order ->
 * out [frames][nslices][n_rows]. The VD phase of run_adaptive (experiment.py:484-497) for a block of
 * frames. */
int tt_vd_rows_batch(void* stream, int frames, int nslices, int n, const double* weights, int n_rows,
                     uint64_t key0, uint64_t key1, const uint64_t* pos0, int32_t* out);
/* The three draws with caller-supplied uniforms instead of the Philox stream: uniforms[m] is the
 * Generator.random() value draw m consumes (one per draw, as numpy's choice and the sequential draws
 * consume them), so a caller holding any other bit generator (np.random.default_rng(seed), PCG64,
 * as the reference builds them: experiment.py:257,338,453) draws them on the host with rng.random(k)
 * and gets numpy's result for the same probabilities. _u: uniforms [nslices][k - nforced];
 * large_u: [k - nforced], pos is an 8-byte device scratch word; without_u: [k]. */
int tt_draw_with_replacement_u(void* stream, int nslices, int n, const double* probs, int k,
                               const int32_t* forced, int nforced, const double* uniforms,
                               int32_t* omega_out, int32_t* count_out);
int tt_draw_with_replacement_large_u(void* stream, int n, const double* probs, int k, const int32_t* forced,
                                     int nforced, const double* uniforms, uint64_t* pos, int32_t* omega_out,
                                     int32_t* count_out, void* scratch);
int tt_draw_without_replacement_u(void* stream, int n, const double* weights, int k, const double* uniforms,
                                  int32_t* out, int32_t* status);

/* ------------------------------------------------------------------ CTEN container (cten.py:1-74)
 * "CTEN" | u8 version 1 | u8 dtype (0 f32 pairs, 1 f64 pairs) | u8 ndim | ndim x u32 dims | payload.
 * Malformed files -> TT_EINVAL (CtenFormatError). Host memory only.
 *  tt_cten_info:     dtype code, ndim and dims (max_dims entries) of a file.
 *  tt_cten_read:     payload into `out` (count complex elements) as complex64 (out_is_f64 = 0)
 *                    or complex128 (1); bit-exact when the file holds the same precision.
 *  tt_cten_write:    data complex64 (src_is_f64 = 0) or complex128 (1), stored as dtype_code. */
int tt_cten_info(const char* path, int* dtype_code, int* ndim, uint32_t* dims, int max_dims);
int tt_cten_read(const char* path, void* out, size_t count, int out_is_f64);
int tt_cten_write(const char* path, const void* data, int src_is_f64, int dtype_code, int ndim, const uint32_t* dims);

/* ------------------------------------------------------------------ values
 * Reconstruction X_f = A_f diag(gamma_f) B_f^T (core.py:91-104,
 * mri.py:107-121), batched over frames: a [frames][nx][rank],
 * b [frames][ny][rank], gamma [frames][rank] -> x [frames][nx][ny]. */
int tt_reconstruct(void* stream, int frames, int nx, int ny, int rank, const float* a, const float* b,
                   const float* gamma, float* x_out);
/* NMSE per frame (metrics.nmse, metrics.py:53-62): out[f] = ||truth_f - est_f||^2 / ||truth_f||^2 over
 * `frames` complex64 frames of n elements (NaN for an all-zero truth frame; the Python mirror raises
 * ValueError there as the reference does). `work` holds tt_nmse_work_doubles(frames) doubles. Fixed
 * summation order: repeat calls are bit-identical. */
int tt_nmse(void* stream, int frames, size_t n, const float* truth, const float* est, double* work, double* out);
size_t tt_nmse_work_doubles(int frames);
/* Squared Frobenius norms (fp64, fixed order) of `batch` complex64 matrices of n elements each -> out[batch]:
 * the post-update factor norms a factor history needs for StepConfig.norm_cap (tracker.py:406-408). */
int tt_factor_norms2(void* stream, int batch, size_t n, const float* x, double* out);
/* rebalance (core.py:138-166) in place on [nslices][n][rank] factor pairs. */
int tt_rebalance(void* stream, int nslices, int nx, int ny, int rank, float* a, float* b, int32_t* status);

/* Per-patch independent trackers (experiment._run_tracking_patched, experiment.py:332-441;
 * mri.PatchGrid / patch_partition / patch_assemble, mri.py:48-177). The nx x ny frame is tiled
 * row-major into (nx/pn1) x (ny/pn2) patches of pn1 x pn2; each is a rank-`rank` EntryMask tracker
 * (track_step, tracker.py:367-411) on its entries in local coordinates.
 *
 * tt_patch_bin: patch_batches' stable filter (experiment.py:352-370) for `frames` frames at once:
 *   entries [total][2] global (i, j), frame f's list at [offsets[f], offsets[f+1]) in measurement
 *   order (offsets [frames + 1], int64), frame_data
 *   [frames][nx][ny] complex64 (pre-noised truth) -> per (frame, patch) lists in measurement order:
 *   pidx [frames][npatch][pn1*pn2] local flat index i*pn2 + j, py [...] complex64 values,
 *   pcnt [frames][npatch]. Out-of-range entries -> TT_ST_BADROW, overflow -> TT_ST_OVERFLOW in
 *   status[0].
 * tt_track_patches: one CTA per patch runs the schedule's steps (frame indices into the binned
 *   table) in order on patches [patch0, patch0 + npatch_local); factors a [npatch_local][pn1][rank],
 *   b [npatch_local][pn2][rank] complex64 (the EntryMask factors), t / alpha_bar [npatch_local]
 *   in/out. Per step outputs [nsteps][npatch_local](...) when non-NULL. With `project` != 0 the
 *   factors are not updated: each scheduled frame's gamma is the ridge solve on the current
 *   subspace (experiment.py:419-431) and, with recon_out [frames][nx][ny], the patch tile
 *   A diag(gamma) B^T is written into the assembled frame (patch_assemble). Ranks up to 16; the
 *   patch must fit one CTA's shared memory (tt_patches_smem_bytes) -> else TT_EUNSUPPORTED. */
typedef struct tt_patches_args {
  int32_t nx, ny, pn1, pn2, rank;
  int32_t patch0, npatch_local;
  int32_t frames;
  const int32_t* pidx;
  const float* py;
  const int32_t* pcnt;
  int32_t nsteps;
  const int32_t* sched;       /* [nsteps] device frame indices */
  float* a;
  float* b;
  int64_t* t;
  double* alpha_bar;
  double lam;
  int32_t step_mode;          /* 0 Fixed(mu), 1 HessianBound(c_floor, c_cap) */
  double mu, c_floor, c_cap;
  int32_t project;
  float* gamma_out;           /* [nsteps][npatch_local][rank] */
  double* cost_out;           /* [nsteps][npatch_local] */
  double* mu_out;             /* [nsteps][npatch_local] */
  float* resid_out;           /* [nsteps][npatch_local][pn1*pn2], measurement order */
  float* recon_out;           /* project: [frames][nx][ny] */
  int32_t* status;            /* [npatch_local] OR-ed TT_ST_* bits */
} tt_patches_args;
size_t tt_patches_smem_bytes(int pn1, int pn2, int rank);
int tt_patch_bin(void* stream, int nx, int ny, int pn1, int pn2, int frames, const float* frame_data,
                 const int32_t* entries, const int64_t* offsets, int32_t* pidx, float* py, int32_t* pcnt,
                 int32_t* status);
int tt_track_patches(void* stream, const tt_patches_args* a);
/* solve_gamma (tracker.py:139-156) for a dense complex128 Phi [L][R]:
 * (Phi^H Phi + lam I)^-1 Phi^H y in fp64 (LDL^H); gamma_out complex128 [R].
 * scratch: tt_solve_scratch_bytes(R). */
size_t tt_solve_scratch_bytes(int L, int R);
int tt_solve_gamma(void* stream, int L, int R, const double* phi, const double* y, double lam, double* gamma_out,
                   void* scratch);

#ifdef __cplusplus
}
#endif
#endif /* TENSORTRACK_B200_H */
