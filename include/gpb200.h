/*
 * gpb200 -- C ABI of the B200-native tiled Gaussian-process hot path.
 *
 * This is the drop-in boundary for the reference's model API
 * (taskgp 0.1.0, /root/reference/pkg/src/taskgp/model.py) and its tile-kernel
 * plugin registry (tiles.py:98-117).  Plain pointers and sizes only: every
 * array is float64, C-contiguous (row-major), in HOST memory unless the
 * function name ends in _device.  Every entry point returns a gpb_status;
 * gpb_last_error() gives the message of the last failure on this thread.
 *
 * Threading: calls on one model must be serialised by the caller
 * (model.py:104-108); distinct models may be used from different threads.
 * Every call blocks until its device work is complete (run_as_root,
 * runtime.py:250-262).
 */
#ifndef GPB200_H
#define GPB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python layer maps each onto the reference exception
 * class of the same meaning (errors.py:4-52). */
typedef enum gpb_status {
  GPB_OK = 0,
  GPB_INVALID_CONFIG = 1,  /* InvalidConfig        (errors.py:8)  */
  GPB_ALREADY_RUNNING = 2, /* AlreadyRunning       (errors.py:12) */
  GPB_NOT_RUNNING = 3,     /* NotRunning           (errors.py:16) */
  GPB_TILING = 4,          /* TilingError          (errors.py:20) */
  GPB_DIM = 5,             /* DimensionMismatch    (errors.py:24) */
  GPB_NOT_PD = 6,          /* NotPositiveDefinite  (errors.py:28) */
  GPB_SINGULAR = 7,        /* SingularTriangular   (errors.py:32) */
  GPB_NUMERIC = 8,         /* NumericalConsistencyError (errors.py:36) */
  GPB_CUDA = 9,            /* device error (no reference equivalent) */
  GPB_NCCL = 10,
  GPB_NO_MEMORY = 11
} gpb_status;

typedef struct gpb_ctx gpb_ctx;     /* a started runtime */
typedef struct gpb_model gpb_model; /* a GP model bound to a runtime */

/* ---- runtime lifecycle: start_runtime / stop_runtime (runtime.py:369-403) */
int gpb_init(int device, gpb_ctx** out);      /* GPB_ALREADY_RUNNING if live */
int gpb_finalize(gpb_ctx* ctx);               /* GPB_NOT_RUNNING if not live */
gpb_ctx* gpb_current(void);                   /* current_runtime(), or NULL */
const char* gpb_last_error(void);
int gpb_abi_version(void);

/* ---- model: GPModel(train, params, tiles_per_dim) (model.py:111-131) ------
 * z: n x d, y: n.  GPB_TILING unless 1 <= tiles_per_dim and it divides n. */
int gpb_model_create(gpb_ctx* ctx, const double* z, const double* y, int64_t n, int64_t d,
                     int64_t tiles_per_dim, gpb_model** out);
/* same, z and y already in device memory of ctx's GPU */
int gpb_model_create_device(gpb_ctx* ctx, const double* z_dev, const double* y_dev, int64_t n,
                            int64_t d, int64_t tiles_per_dim, gpb_model** out);
int gpb_model_destroy(gpb_model* m);
/* train setter (model.py:139-147): re-uploads, invalidates the factor */
int gpb_model_set_train(gpb_model* m, const double* z, const double* y, int64_t n, int64_t d);
/* params setter (model.py:153-156): (lengthscale, vertical_scale,
 * noise_variance) + trainable flags; invalidates factor, beta, alpha.
 * GPB_INVALID_CONFIG if l <= 0, nu <= 0 or s2 < 0 (covariance.py:50-62). */
int gpb_model_set_params(gpb_model* m, double lengthscale, double vertical_scale,
                         double noise_variance, const uint8_t trainable[3]);
int gpb_model_get_params(gpb_model* m, double out[3]);

/* ---- hot path ------------------------------------------------------------
 * gpb_cholesky: assemble K + tiled Cholesky (model.py:169-177), cached.
 *   L_out (n x n, lower, upper = 0) may be NULL; it is written in strips of
 *   rows through a bounded (<= 256 MB) device staging buffer.  GPB_NOT_PD on failure,
 *   with gpb_last_pivot giving the first failing index; the cache is
 *   invalidated (model.py:210-217). */
int gpb_cholesky(gpb_model* m, double* L_out);
int gpb_last_pivot(gpb_model* m, int64_t* pivot);
/* log marginal likelihood (model.py:316-339); compute_loss = -this */
int gpb_log_likelihood(gpb_model* m, double* out);
/* dNLL/d(l, nu, s2) (model.py:341-435); zeros for non-trainable */
int gpb_loss_gradients(gpb_model* m, double out[3]);
/* Gradient terms of a set of internal K^-1 tile columns (tiles of gpb_layout's
 * out[0] size), for splitting loss_gradients across ranks that each hold the
 * factor (model.py:362-432 restated per tile column):
 *   out[0] = sum w (K^-1 - a a^T) o E o D2,  out[1] = sum w (K^-1 - a a^T) o E,
 *   out[2] = sum of the real diagonal entries of K^-1   (w = 2 off the diagonal),
 * each over the lower tiles (i >= J) of the columns J in cols (strictly increasing).
 * Summed over a partition of [0, T): dNLL/dl = nu / (2 l^3) out[0],
 * dNLL/dnu = out[1] / 2, dNLL/ds2 = (out[2] - |alpha|^2) / 2.
 * GPB_NO_MEMORY if the (n - cols[0] b) x ncols b panel does not fit. */
int gpb_loss_gradient_terms(gpb_model* m, const int* cols, int64_t ncols, double out[3]);
/* Adam on log-parameters (model.py:437-485). history: iterations NLLs.
 * On GPB_NOT_PD the message is prefixed "iteration k: ". */
int gpb_optimize(gpb_model* m, double learning_rate, double beta1, double beta2,
                 double epsilon, int64_t iterations, double* history);
/* predict / predict_variance / predict_with_full_cov (model.py:221-314).
 * zt: m x d.  mean (m) required; var (m) and cov (m x m) optional.
 * Variances are clamped like _clamp_variances (model.py:488-496):
 * GPB_NUMERIC if any < -1e-9.  GPB_DIM on a feature-count mismatch. */
int gpb_predict(gpb_model* m, const double* zt, int64_t mt, int64_t d, double* mean,
                double* var, double* cov);
/* same with zt, mean, var in device memory (no clamp check; raw values) */
int gpb_predict_device(gpb_model* m, const double* zt_dev, int64_t mt, int64_t d,
                       double* mean_dev, double* var_dev);
/* Building blocks of the test-point-sharded full covariance (multi-GPU):
 * gpb_predict_solve_device writes V = L^-1 K*^T of mt test points into V_dev
 * (n_p x ldv row-major, n_p = gpb_layout out[2]; rows at padded positions are
 * 0) and optionally the mean.  GPB_NO_MEMORY if all mt columns do not fit at once.
 * gpb_cov_block_device writes out (ma x mb, ld ldo) = K**(za, zb) - Va^T Vb
 * (model.py:254-269 for one block of Sigma); Va / Vb are n_p x ldv blocks
 * from gpb_predict_solve_device with ldv >= m rounded up to 128. */
int gpb_predict_solve_device(gpb_model* m, const double* zt_dev, int64_t mt, int64_t d,
                             double* mean_dev, double* V_dev, int64_t ldv);
int gpb_cov_block_device(gpb_model* m, const double* za, int64_t ma, const double* Va, int64_t ldva,
                         const double* zb, int64_t mb, const double* Vb, int64_t ldvb, double* out,
                         int64_t ldo);

/* _clamp_variances (model.py:488-496) on a host vector, in place: entries in
 * [-1e-9, 0) become 0; GPB_NUMERIC (nothing changed) if any is below -1e-9.
 * gpb_predict applies it to var and to the diagonal of cov. */
int gpb_clamp_variances(double* v, int64_t n);
/* Adam state of optimize (model.py:446-448: moments and step count persist
 * across calls); get/set let a caller carry it across a model re-creation */
int gpb_model_get_adam(gpb_model* m, double moment1[3], double moment2[3], int64_t* step);
int gpb_model_set_adam(gpb_model* m, const double moment1[3], const double moment2[3], int64_t step);

/* per-phase device times (ms, CUDA events on the model stream) of the last
 * calls: [0] assembly, [1] factorisation, [2] alpha solves, [3] predict
 * cross+mean, [4] predict TRSM+variance, [5] gradient, [6] full-cov SYRK */
int gpb_model_timings(gpb_model* m, double* ms_out, int n);
/* launches of this library's kernels since the model was created */
int gpb_model_launch_count(gpb_model* m, int64_t* out);

/* tcgen05 digit-plane products (csrc/ozaki.cuh): the long-k products of the
 * path -- the factorisation's trailing updates (tiled.py:187-204), the
 * prediction sweep (tiled.py:263-298) and the full-covariance V^T V
 * (model.py:254-269) -- on the int8 tensor pipe from `slices` signed 7-bit
 * digit planes per operand (8, the default: every kept term of the FP64
 * product; 0: off, every product on the FP64 DMMA kernels).  GPB_OZAKI sets
 * the default of new models.  Changing the count drops the cached factor
 * when it changes the panel grouping.  `fallbacks` counts phases repeated on
 * the DMMA kernels because an operand exceeded its fixed-point scale. */
int gpb_model_set_ozaki(gpb_model* m, int slices);
int gpb_model_get_ozaki(gpb_model* m, int* slices, int64_t* fallbacks);
/* the CUDA stream (cudaStream_t) the model's kernels run on */
int gpb_model_stream(gpb_model* m, void** stream);
/* per-kernel-class profiling with CUDA events around every launch:
 * class 0 grouped DMMA GEMM, 1 POTRF/TRTRI tile, 2 SEK assembly, 3 solves,
 * 4 plane slicing and other small kernels, 5 tcgen05 digit-plane products.
 * set_profiling resets the counters; kernel_stats returns the totals
 * (device ms, executed flops, launches) since then. */
int gpb_model_set_profiling(gpb_model* m, int on);
int gpb_model_kernel_stats(gpb_model* m, double ms[8], double flops[8], int64_t count[8]);
/* per class: length of the union of its launch intervals since set_profiling
 * (the launches of the critical and main streams overlap, so the summed
 * durations of kernel_stats can exceed wall time; this cannot) */
int gpb_model_kernel_busy(gpb_model* m, double busy_ms[8]);
/* sustained FP64 tensor-pipe (DMMA.8x8x4) throughput of this GPU, TFLOP/s */
int gpb_fp64_peak_probe(gpb_ctx* ctx, double seconds, double* tflops);
/* the same for the int8 tcgen05 pipe: tcgen05.mma kind::i8 128 x 128 x 32 issued back to back from
 * shared memory on every SM for about `seconds`; int8 operations per second, in units of 1e12 */
int gpb_int8_peak_probe(gpb_ctx* ctx, double seconds, double* tops);

/* ---- device-level tile operations (external schedulers) -------------------
 * Used by the multi-GPU driver (2D block-cyclic tiled Cholesky, tiled.py:168-204,
 * and blocked solves, tiled.py:215-260, scheduled across ranks).  All pointers are
 * device pointers on the runtime's GPU; `stream` is a cudaStream_t (NULL: legacy
 * default stream).  Tiles are b x b row-major with b a multiple of 128.
 *
 * gpb_layout: the padded internal layout the library uses for (n, tiles_per_dim):
 *   out = {tile size b, tiles per dim T, padded order n_p, pad.bp, pad.b, user tile}.
 *   A padded position P is real iff P % pad.bp < pad.b. */
int gpb_layout(int64_t n, int64_t tiles_per_dim, int64_t out[6]);
typedef struct gpb_tile_desc { int32_t i, j; double* ptr; } gpb_tile_desc;
typedef struct gpb_gemm_job {
  const double* a; const double* b; const double* cin; double* cout;
  int32_t k; int32_t lower;  /* lower: skip 128-blocks above the block diagonal */
} gpb_gemm_job;
typedef struct gpb_gemv_job { const double* a; const double* x; double* y; } gpb_gemv_job;
/* pad rows of src (n x d, or a vector when d == 0) into the padded layout (n_p rows) */
int gpb_dev_pad(gpb_ctx* ctx, void* stream, const double* src, int64_t n_p, int64_t d,
                int64_t pad_bp, int64_t pad_b, double* dst);
/* SEK tiles (covariance.py:118-164): tile (i,j) of K(zp) (+ s2 on the global diagonal) */
int gpb_dev_assemble(gpb_ctx* ctx, void* stream, const double* zp, int64_t d, int64_t b,
                     int64_t pad_bp, int64_t pad_b, double lengthscale, double vertical_scale,
                     double noise_variance, int add_noise, const gpb_tile_desc* tiles,
                     int64_t ntiles);
/* POTRF + TRTRI of one diagonal tile in place (tiles.py:132-137); writes dinv = L^-1,
 * *logdiag_out = sum log l_jj over real pivots, *info_dev = first failing index
 * (must be -1 on entry; the kernel is skipped when it is already >= 0) */
int gpb_dev_potrf(gpb_ctx* ctx, void* stream, double* tile, double* dinv, int64_t b,
                  int64_t tile_off, int64_t pad_bp, int64_t pad_b, double* logdiag_out,
                  int* info_dev);
/* grouped DMMA GEMM, b x b outputs: cout = alpha * a b^T + beta * cin (operand
 * layouts per a_kmajor / b_kmajor as in the single-GPU path) */
int gpb_dev_gemm(gpb_ctx* ctx, void* stream, const gpb_gemm_job* jobs, int64_t njobs, int64_t b,
                 int64_t lda, int64_t ldb, int64_t ldc, int a_kmajor, int b_kmajor, double alpha,
                 double beta);
/* same with a tiled-k walk on both (K-major) operands: k runs through
 * consecutive ktile-deep tiles kstride doubles apart -- the update of a tile
 * by several panels held in one buffer, K = (number of panels) * ktile */
int gpb_dev_gemm_tiled(gpb_ctx* ctx, void* stream, const gpb_gemm_job* jobs, int64_t njobs,
                       int64_t b, int64_t lda, int64_t ldb, int64_t ldc, int a_kmajor, int b_kmajor,
                       int64_t ktile, int64_t kstride, double alpha, double beta);
/* gpb_dev_gemm_tiled whose jobs also store their output tiles at mirror
 * addresses: job j's element at offset o from its cout is written to
 * mirrors[j * nmirror + r] + o for every non-null entry -- the TRSM of the
 * multi-GPU schedule pushing its panel tiles into peer ranks' panel buffers
 * (CUDA IPC mappings, NVLink stores) from the GEMM epilogue */
int gpb_dev_gemm_mirror(gpb_ctx* ctx, void* stream, const gpb_gemm_job* jobs, int64_t njobs,
                        int64_t b, int64_t lda, int64_t ldb, int64_t ldc, int a_kmajor, int b_kmajor,
                        int64_t ktile, int64_t kstride, double alpha, double beta,
                        double* const* mirrors, int64_t nmirror);
/* peer memory and stream-ordered flags for the fused panel exchange:
 * zeroed device memory with its CUDA IPC handle (GPB_IPC_HANDLE_BYTES bytes),
 * a peer's mapping of it, and 64-bit flags written / awaited in stream order
 * (cuStreamWriteValue64 after a fence; cuStreamWaitValue64 >=, no SM spins) */
#define GPB_IPC_HANDLE_BYTES 64
int gpb_dev_ipc_alloc(gpb_ctx* ctx, int64_t bytes, void** ptr, void* handle);
int gpb_dev_ipc_open(gpb_ctx* ctx, const void* handle, void** ptr);
int gpb_dev_ipc_close(gpb_ctx* ctx, void* ptr);
int gpb_dev_free(gpb_ctx* ctx, void* ptr);
int gpb_dev_signal(gpb_ctx* ctx, void* stream, uint64_t* flag, uint64_t value);
int gpb_dev_wait(gpb_ctx* ctx, void* stream, const uint64_t* flag, uint64_t value);
/* batched tile GEMV: y (+)= alpha * op(a) x; outputs must be distinct per call */
int gpb_dev_gemv(gpb_ctx* ctx, void* stream, const gpb_gemv_job* jobs, int64_t njobs, int64_t b,
                 int trans, double alpha, int accumulate);
/* batched device copies of `bytes` each: dst_i <- src_i (jobs: {src, dst} pairs) */
typedef struct gpb_copy_job { const double* src; double* dst; } gpb_copy_job;
int gpb_dev_copy(gpb_ctx* ctx, void* stream, const gpb_copy_job* jobs, int64_t njobs, int64_t bytes);
/* out = base - sum_p parts[p] (fixed order), vectors of length len */
int gpb_dev_combine(gpb_ctx* ctx, void* stream, const double* base, const double* parts,
                    int64_t nparts, int64_t len, double* out);
/* hand a factor computed elsewhere (packed row-major lower tiles in the model's layout,
 * inverse diagonal tiles, per-tile log-diagonal sums, beta, alpha; all device) to a
 * model: its caches become valid and prediction / likelihood use it */
int gpb_model_adopt_factor(gpb_model* m, const double* tiles, const double* dinv,
                           const double* logdiag, const double* beta, const double* alpha);
/* the model's own device buffers (written in place by an external scheduler,
 * then published with gpb_model_mark_factored) */
int gpb_model_factor_buffers(gpb_model* m, double** tiles, double** dinv, double** logdiag,
                             double** beta, double** alpha);
int gpb_model_mark_factored(gpb_model* m);

/* ---- multi-GPU runtime: one process per GPU, 2D block-cyclic tile grid ------
 * Replaces the reference's runtime lifecycle (runtime.py:369-403) and its
 * task DAG (tiled.py:168-324, model.py:169-485) across the GPUs of one box.
 * SURVEY.md 8(b) lists gpb_init(ndev, devs); here every rank runs its own
 * process with its own gpb_init(device), and gpb_dist_init joins them: ranks
 * form a P x Q process grid (rank = p * Q + q), lower tile (i, j) lives on
 * rank (i mod P) * Q + (j mod Q), and the library creates its NCCL
 * communicators itself -- the world communicator from a unique id that rank 0
 * makes with gpb_nccl_unique_id and the caller passes to every rank out of
 * band, then ncclCommSplit into the process-row and process-column
 * communicators the panel exchanges run on.  NCCL is loaded at run time
 * (GPB_NCCL_LIB, else libnccl.so.2); GPB_NCCL if it cannot be.
 * gpb_dist_init_host runs the same schedule with host-staged collectives
 * supplied by the caller (tests, or ranks without NCCL): buffers passed to the
 * callbacks are host memory; group 0 = world, 1 = this rank's process row
 * (ranks ordered by q), 2 = its process column (ordered by p); root and the
 * callback's rank numbering are within the group.  A callback returns 0 on
 * success.  Every gpb_dist_* call below is COLLECTIVE: all ranks make it with
 * the same arguments, and results are returned on every rank. */
typedef struct gpb_dist gpb_dist;
typedef struct gpb_dmodel gpb_dmodel;
#define GPB_NCCL_ID_BYTES 128
typedef struct gpb_host_coll {
  int (*bcast)(void* user, int group, void* buf, int64_t bytes, int root);
  int (*reduce_sum)(void* user, int group, double* buf, int64_t count, int root);  /* in place, at root */
  int (*allreduce_sum)(void* user, int group, double* buf, int64_t count);        /* in place */
  void* user;
} gpb_host_coll;
int gpb_nccl_unique_id(void* id_out);  /* GPB_NCCL_ID_BYTES bytes */
int gpb_dist_init(gpb_ctx* ctx, int rank, int world, int P, int Q, const void* nccl_id, gpb_dist** out);
int gpb_dist_init_host(gpb_ctx* ctx, int rank, int world, int P, int Q, const gpb_host_coll* coll,
                       gpb_dist** out);
/* Timing emulation: rank `rank` of the grid alone on this GPU, every collective a
 * no-op (results are meaningless; the schedule's kernels run as they would on
 * that rank).  Measures each rank's compute time when only one GPU is at hand. */
int gpb_dist_init_emulate(gpb_ctx* ctx, int rank, int world, int P, int Q, gpb_dist** out);
int gpb_dist_finalize(gpb_dist* dc);  /* GPB_INVALID_CONFIG while models of dc are alive */
/* Panel exchange of the factorisation for models created afterwards:
 * 0 (default) collectives (row / column broadcasts); 1 peer memory -- the
 * panel TRSM's epilogue stores every solved tile straight into the row- and
 * column-panel buffers of the ranks that read it (CUDA IPC mappings, NVLink
 * stores), readiness and buffer reuse ordered by stream-written 64-bit flags
 * (no SM waits).  Needs every rank's GPU to map every other's memory. */
int gpb_dist_set_exchange(gpb_dist* dc, int mode);
/* GPModel(train, params, tiles_per_dim) sharded: every rank passes the whole
 * (replicated) z, y and keeps only its tiles of K / L */
int gpb_dist_model_create(gpb_dist* dc, const double* z, const double* y, int64_t n, int64_t d,
                          int64_t tiles_per_dim, gpb_dmodel** out);
int gpb_dist_model_destroy(gpb_dmodel* m);
int gpb_dist_set_params(gpb_dmodel* m, double lengthscale, double vertical_scale, double noise_variance,
                        const uint8_t trainable[3]);
int gpb_dist_get_params(gpb_dmodel* m, double out[3]);
/* assemble + block-cyclic tiled Cholesky + beta / alpha solves (cached);
 * GPB_NOT_PD as gpb_cholesky, the pivot is the smallest failing index over ranks */
int gpb_dist_factor(gpb_dmodel* m);
int gpb_dist_last_pivot(gpb_dmodel* m, int64_t* pivot);
int gpb_dist_log_likelihood(gpb_dmodel* m, double* out);
/* replica-free: distributed TRTRI + LAUUM on the block-cyclic tiles, trace
 * pass on each rank's K^-1 tiles, all-reduce of three partial sums */
int gpb_dist_loss_gradients(gpb_dmodel* m, double out[3]);
int gpb_dist_optimize(gpb_dmodel* m, double learning_rate, double beta1, double beta2, double epsilon,
                      int64_t iterations, double* history);
/* test points sharded over ranks (each rank gathers the factor once into a
 * local replica); mean / var / cov (m x m) as gpb_predict, on every rank */
int gpb_dist_predict(gpb_dmodel* m, const double* zt, int64_t mt, int64_t d, double* mean, double* var,
                     double* cov);
/* dense n x n lower factor on every rank (through the replica) */
int gpb_dist_cholesky(gpb_dmodel* m, double* L_out);
/* device ms of the last calls: [0] assembly, [1] factorisation, [2] solves,
 * [3] prediction, [4] gradient, [5] replica gather; [6] host enqueue us per
 * panel step of the last factorisation; [7] collectives issued by this rank */
int gpb_dist_timings(gpb_dmodel* m, double* ms_out, int n);
int gpb_dist_launch_count(gpb_dmodel* m, int64_t* out);

/* The schedule IR.  gpb_dist_plan emits, for one rank, the ordered operation
 * list of a phase (0 factorisation, 1 beta / alpha solves, 2 gradient): what
 * the device executor runs (kernels on two streams, collectives on the row /
 * column / world communicators) and what the CPU interpreter of the tests
 * replays on numpy tiles.  Host-only (no GPU needed).  Buffers are numbered
 * GPB_BUF_*; offsets and counts are in doubles.  With ops == NULL only the
 * counts are returned. meta (16): bi, Ti, n_p, P, Q, G, owned tiles, events,
 * vector offsets {Y, BETA, ALPHA, LOGDIAG, ACC, TMP, RECV, RED}. */
enum {
  GPB_BUF_L = 0, GPB_BUF_DINV, GPB_BUF_ROW, GPB_BUF_COL, GPB_BUF_VEC, GPB_BUF_X, GPB_BUF_KINV,
  GPB_BUF_XCOL, GPB_BUF_XROW, GPB_BUF_LCOL, GPB_NBUF
};
enum {
  GPB_OP_ASSEMBLE = 1, GPB_OP_POTRF, GPB_OP_GEMM, GPB_OP_COPY, GPB_OP_GEMV, GPB_OP_COMBINE, GPB_OP_BCAST,
  GPB_OP_REDUCE, GPB_OP_ALLREDUCE, GPB_OP_RECORD, GPB_OP_WAIT, GPB_OP_ZERO, GPB_OP_SOLVE_FLOW, GPB_OP_TRACE,
  /* peer-memory exchange: MIRROR lists extra stores of the preceding GEMM's outputs
   * (job: k = index of the GEMM job, i = destination rank, buf[3] / off[3] = where
   * in that rank's buffers); SIGNAL sets flag `j` (0 ready, 1 free) of rank i to
   * count; WAITFLAG waits until this rank's flag j of source rank i reaches count */
  GPB_OP_MIRROR, GPB_OP_SIGNAL, GPB_OP_WAITFLAG,
  /* digit planes (csrc/ozaki.cuh): SLICE writes the planes of `count` consecutive
   * bi x bi tiles from buf[0] / off[0] (a row or column panel) into the executor's
   * plane buffer of that panel; a GEMM with flag = 1 is the same product computed
   * from those planes on the int8 tensor pipe */
  GPB_OP_SLICE
};
typedef struct gpb_op {
  int32_t kind, stream, group, root;  /* stream 0 main, 1 critical; group 0 world, 1 row, 2 column */
  int32_t buf[3], flag;               /* flag: ASSEMBLE add_noise, GEMV trans, GEMM digit planes */
  int64_t off[3];
  int64_t count, job0, njobs;         /* count: doubles (collectives, COPY per job, ZERO, COMBINE) */
  int32_t mblk, nblk, ak, bk;         /* GEMM: blocks of 128 per job, K-major operands */
  int64_t lda, ldb, ldc;
  int64_t a_ktile, a_kstride, b_ktile, b_kstride; /* tiled-k walks (0: none) */
  double alpha, beta;                 /* GEMM cout = alpha a b^T + beta cin; GEMV beta 1 = accumulate */
  int32_t i, j;                       /* POTRF tile k; RECORD / WAIT event */
} gpb_op;
typedef struct gpb_op_job {
  int32_t buf[4];                     /* A, B, Cin, Cout (-1: none) */
  int64_t off[4];
  int32_t k, lower, i, j;             /* GEMM depth and diagonal-tile flag; tile coordinates */
} gpb_op_job;
/* exchange: as gpb_dist_set_exchange */
int gpb_dist_plan(int rank, int world, int P, int Q, int64_t n, int64_t tiles_per_dim, int phase, int exchange,
                  gpb_op* ops, int64_t* nops, gpb_op_job* jobs, int64_t* njobs, int64_t bufsz[GPB_NBUF],
                  int64_t meta[16]);

/* ---- BASELINE input generator on the device ---------
 * u, noise: the n draws of the host generator (numpy default_rng, SURVEY.md
 * Appendix A.1), device memory.  Writes y (n) = mass-spring-damper position +
 * noise (semi-implicit Euler, bitwise the host recurrence) and z (n x n_reg)
 * = lag features u_t, u_{t-1}, ... (0 before the start). */
int gpb_msd_series_device(gpb_ctx* ctx, const double* u_dev, const double* noise_dev, int64_t n, int64_t n_reg,
                          double dt, double mass, double damping, double stiffness, double* z_dev, double* y_dev);

/* ---- tile-kernel plugin (tiles.py:23-46, 132-164) -------------------------
 * Host buffers, fresh outputs, inputs never mutated.  Square tiles b x b;
 * trsm solves X l^T = b_in for rows x b b_in. */
int gpb_tile_potrf(gpb_ctx* ctx, const double* a, int64_t b, double* out);
int gpb_tile_trsm(gpb_ctx* ctx, const double* l, const double* b_in, int64_t rows, int64_t b,
                  double* out);
int gpb_tile_syrk(gpb_ctx* ctx, const double* a, const double* c, int64_t b, int64_t k,
                  double* out);
int gpb_tile_gemm(gpb_ctx* ctx, const double* a, const double* bm, const double* c, int64_t m,
                  int64_t n, int64_t k, double* out);

#ifdef __cplusplus
}
#endif
#endif /* GPB200_H */
