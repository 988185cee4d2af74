/*
 * p2g.h — C ABI of the B200-native SPARTan PARAFAC2-ALS engine.
 *
 * This is the drop-in boundary.  The reference exposes a
 * header-only C++ API (/root/reference/proj/include/parafac2); there is no
 * FFI in the reference, so each entry point below names the reference
 * function it replaces (file:line).  The C++ drop-in headers in
 * include/parafac2/ headers re-create the reference's signatures on top of this
 * ABI; INTEGRATION.md shows how a maintainer binds it.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Host buffers are borrowed for the
 *    duration of the call.  Dense matrices are column-major (the layout of
 *    Eigen::MatrixXd, common.hpp:30) unless stated otherwise.
 *  - Every function returns a status: 0 ok; P2G_EINVAL (std::invalid_argument),
 *    P2G_EDATA (DataError, CLI exit 2), P2G_ENUM (NumericalError, CLI exit 3),
 *    P2G_ECUDA (CUDA/NCCL failure).  p2g_last_error() returns the message of
 *    the last failure on the calling thread (solver/common.hpp messages are
 *    preserved where the reference defines them).
 *  - One context drives one GPU.  Multi-GPU: one process (rank) per GPU,
 *    each with its own context; subjects are sharded by
 *    partition_weighted(nnz_k + I_k, world) (parallel.hpp:51-79,
 *    solver.hpp:263-267) and the per-iteration J x R / R x R partials are
 *    combined with ncclAllReduce.  A context is not thread-safe.
 *  - There is no CPU fallback: every compute entry point runs on the GPU and
 *    fails with P2G_ECUDA when no device is usable.
 *
 * Data layout of the sparse tensor (flattened CSR):
 *    subj_row_ptr[K+1]  int64  first global row of subject k
 *    row_ptr[NR+1]      int64  first entry of global row r (NR = sum_k I_k)
 *    col_idx[nnz]       int32  column ids, strictly ascending within a row
 *    val[nnz]           fp64   stored values (non-zero)
 *  Packed per-subject factors Q_k (I_k x R) are stored as one ROW-MAJOR
 *  (sum_k I_k) x R array, subject k occupying rows subj_row_ptr[k]...
 */
#ifndef P2G_H_
#define P2G_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P2G_OK 0
#define P2G_EINVAL 1
#define P2G_EDATA 2
#define P2G_ENUM 3
#define P2G_ECUDA 4

/* Procrustes flags per subject (canonical rule D5). */
#define P2G_FLAG_FULL_RANK 0   /* rank(A_k) = R: unique polar factor            */
#define P2G_FLAG_DEFICIENT 1   /* rank(A_k) < R: canonical completion           */
#define P2G_FLAG_ACCURATE 2    /* ill-conditioned: solved by the Jacobi-SVD path */
#define P2G_FLAG_DEGENERATE 3  /* completion itself degenerate (not parity-safe) */

/* Last error message of the calling thread ("" if none). */
const char* p2g_last_error(void);
/* Library version / build string. */
const char* p2g_version(void);

/* ------------------------------------------------------------------------
 * Host-side utilities (no GPU required)
 * ------------------------------------------------------------------------ */

/* partition_weighted (parallel.hpp:51-79): contiguous [begin,end) ranges of
 * roughly equal cumulative weight.  begin_end receives 2*n_out int64 values;
 * it must hold 2*n_chunks.  Bit-exact with the reference. */
int p2g_partition_weighted(const uint64_t* weights, int64_t n, int32_t n_chunks, int64_t* begin_end,
                           int32_t* n_out);

/* Synthetic BASELINE workloads (decisions D1, D10, D11).
 * Deterministic function of the spec: subject k draws from
 * Rng(substream_seed(seed, k+1)) (common.hpp:65-121).  */
typedef struct {
  int64_t K;           /* subjects                                            */
  int64_t J;           /* variables (columns)                                 */
  int32_t rows_dist;   /* 0: I_k ~ U{rows_lo..rows_hi}; 1: Geometric(1/rows_mean) capped at rows_hi */
  int64_t rows_lo, rows_hi;
  double rows_mean;
  int64_t min_rows;    /* D1: I_k <- max(I_k, min_rows) (= R)                 */
  int32_t nnz_dist;    /* 0: nnz_row ~ U{nnz_lo..nnz_hi}; 1: 1 + Poisson(nnz_lambda) */
  int64_t nnz_lo, nnz_hi;
  double nnz_lambda;
  int32_t col_dist;    /* 0: uniform over [0,J); 1: Zipf(zipf_s), rank = column id */
  double zipf_s;
  int32_t val_dist;    /* 0: 1 - uniform() in (0,1]; 1: 1 + below(5)          */
  uint64_t seed;
  int32_t threads;     /* host threads (0 = hardware concurrency); result independent of it */
} p2g_gen_spec;

typedef struct p2g_gen p2g_gen;

/* Fills *spec with BASELINE.json config `config_id` (1..5) at rank R. */
int p2g_gen_baseline_spec(int32_t config_id, int32_t R, p2g_gen_spec* spec);
int p2g_gen_create(const p2g_gen_spec* spec, p2g_gen** out, int64_t* n_rows, int64_t* nnz);
int p2g_gen_export(const p2g_gen* g, int64_t* subj_row_ptr, int64_t* row_ptr, int32_t* col_idx, double* val);
void p2g_gen_free(p2g_gen* g);

/* Initial factors for the BASELINE configs (D2): H = I_R; V (J x R) from
 * Rng(seed) r-outer / j-inner exactly as solver.hpp:128-132, then W (K x R)
 * continuing the same stream r-outer / k-inner.  Column-major outputs. */
int p2g_init_factors(uint64_t seed, int64_t K, int64_t J, int32_t R, double* H, double* V, double* W);

/* The reference's random initialisation (solver.hpp:124-132): H = I,
 * S = ones, V from Rng(seed).  Validation of rank/tol/max_iters/I_k/J as in
 * initialize() (solver.hpp:104-122). */
int p2g_initialize_random(uint64_t seed, int64_t K, int64_t J, int32_t R, double* H, double* S, double* V);

/* ------------------------------------------------------------------------
 * Device context
 * ------------------------------------------------------------------------ */
typedef struct p2g_ctx p2g_ctx;

/* 128-byte NCCL unique id for multi-GPU contexts (call on rank 0, share). */
int p2g_nccl_unique_id(char out_id[128]);
/* world == 1: nccl_id may be NULL (no NCCL).  device: CUDA ordinal. */
int p2g_create(int32_t device, int32_t rank, int32_t world, const char* nccl_id, p2g_ctx** out);
int p2g_destroy(p2g_ctx* ctx);

/* Uploads this rank's shard of the full tensor (all K subjects given).
 * Validates the CSR (DataError on bad indices / empty tensor). */
int p2g_load_csr(p2g_ctx* ctx, int64_t K, int64_t J, const int64_t* subj_row_ptr, const int64_t* row_ptr,
                 const int32_t* col_idx, const double* val);
/* This rank's subject range [k_begin, k_end) and its row / nnz counts. */
int p2g_shard_info(const p2g_ctx* ctx, int64_t* k_begin, int64_t* k_end, int64_t* n_rows, int64_t* nnz);

/* Shard-local load: a rank passes only its own subjects [k_begin, k_end) of
 * a K-subject tensor, with subj_row_ptr[k_end-k_begin+1] and row_ptr rebased
 * to the shard (both start at 0).  The ranges must tile [0, K) in rank order
 * (bit-exact shards: p2g_partition_weighted over nnz_k + I_k, the weights of
 * solver.hpp:263-267).  Checks, ||X||^2 and the verdict are collective:
 * every rank returns the same status.  Afterwards W0 / W arguments are this
 * rank's rows only ((k_end-k_begin) x R).  Replaces the per-rank slice of
 * IrregularTensor construction (sparse.hpp:176-215). */
int p2g_load_shard(p2g_ctx* ctx, int64_t K, int64_t J, int64_t k_begin, int64_t k_end, const int64_t* subj_row_ptr,
                   const int64_t* row_ptr, const int32_t* col_idx, const double* val);

/* Host-staged collective, used instead of NCCL: fn reduces `count` doubles
 * in place across all ranks (op 0 = sum, 1 = max) and returns 0 on success.
 * A context created with world > 1 and nccl_id == NULL must set one before
 * loading.  (The reference reduces thread partials with merge_tree,
 * parallel.hpp:115-124; this is the cross-process analogue's seam.) */
typedef int (*p2g_host_allreduce_fn)(double* buf, int64_t count, int32_t op, void* user);
int p2g_set_host_collective(p2g_ctx* ctx, p2g_host_allreduce_fn fn, void* user);

/* Fault injection (tests): kind 1 makes this rank's W-NNLS report a failure
 * at the given iteration (1-based); kind 0 clears.  The error is agreed over
 * all ranks in the iteration's last collective, so every rank raises
 * NumericalError("NNLS did not converge") (kernels.hpp:137) together. */
int p2g_inject_fault(p2g_ctx* ctx, int32_t kind, int32_t iteration);

/* ------------------------------------------------------------------------
 * The fused PARAFAC2-ALS loop — replaces fit_parafac2 (solver.hpp:251-321).
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t rank;       /* R >= 1                                 (solver.hpp:51) */
  int32_t max_iters;  /* >= 1                                   (solver.hpp:52) */
  double tol;         /* > 0; relative fit change stop          (solver.hpp:53) */
  int32_t nonneg;     /* NNLS on V and W                        (solver.hpp:54) */
  int32_t init;       /* 0: random V from seed, H=I, W=ones (solver.hpp:124-132);
                         1: eye: V = |top-R eigenvectors of sum_k X_k^T X_k|,
                            H=I, W=ones (solver.hpp:133-164), on the device;
                         2: explicit H0/V0/W0 (D2). */
  uint64_t seed;      /*                                        (solver.hpp:56) */
} p2g_fit_config;

typedef struct {
  int32_t iterations;
  int32_t converged;
  double total_ms;
  double norm_x;      /* ||X||_F^2 */
} p2g_fit_summary;

/* H0 (R x R), V0 (J x R), W0 (K x R, all subjects) used when init == 2.
 * Outputs (any may be NULL): H_out (R x R), V_out (J x R), W_out (this
 * rank's shard rows, (k_end-k_begin) x R), Q_out (this rank's packed Q,
 * row-major), flags_out (per shard subject, last iteration),
 * fit / resid / ms per iteration (length >= max_iters). */
int p2g_fit(p2g_ctx* ctx, const p2g_fit_config* cfg, const double* H0, const double* V0, const double* W0,
            double* H_out, double* V_out, double* W_out, double* Q_out, int32_t* flags_out, double* fit_trace,
            double* resid_trace, double* ms_trace, p2g_fit_summary* summary);

/* initialize(..., Init::eye) (solver.hpp:133-164) on the loaded tensor: V_out
 * (J x R, column-major) = entry-wise |leading R eigenvectors| of the column
 * Gram matrix sum_k X_k^T X_k over non-zero column pairs.  Same validation
 * as initialize() (rank, J >= R, I_k >= R). */
int p2g_initialize_eye(p2g_ctx* ctx, int32_t R, double* V_out);

/* IterationStats of the last p2g_fit (solver.hpp:70-77): per iteration
 * {ms_procrustes, ms_project, ms_cp} from CUDA events on the context's
 * stream.  ms_procrustes includes the fused mode-1 partial; ms_project is 0
 * (the loop is Q-based and never forms Y_k). */
int p2g_fit_phase_ms(const p2g_ctx* ctx, int32_t max_iters, double* out /* 3 * max_iters */, int32_t* n_out);

/* fit_parafac2 with per-iteration dumps of the loop kernels' own outputs
 * (parity tests): for iteration t (0-based) the mode-1/2/3 MTTKRPs
 * m1 (R x R), m2 (J x R), m3 (shard K x R) of cp.hpp:108,116,127 and the
 * updated H, V, W, all column-major at offset t * size.  Any may be NULL.
 * Stops like p2g_fit; *n_iters = iterations run. */
int p2g_fit_dumps(p2g_ctx* ctx, const p2g_fit_config* cfg, const double* H0, const double* V0, const double* W0,
                  double* m1, double* m2, double* m3, double* H, double* V, double* W, double* fit_trace,
                  int32_t* n_iters);

/* Device-resident variant for benchmarking: runs `iters` iterations from the
 * state left by the previous call (or from explicit factors when reset != 0),
 * all inputs already in HBM.  Reports per-iteration device time (ms, CUDA
 * events, max over ranks when world > 1). */
int p2g_bench_iterations(p2g_ctx* ctx, const p2g_fit_config* cfg, const double* H0, const double* V0,
                         const double* W0, int32_t reset, int32_t iters, double* ms_per_iter, double* fit_trace);

/* Process-wide number of CUDA kernels this library has launched so far. */
int64_t p2g_launch_count(void);

/* Per-kernel device time of the last p2g_bench_iterations call, averaged per
 * launch: names "procrustes", "mode2", "mode3", "nnls_v", "nnls_w", ... */
int p2g_kernel_times(const p2g_ctx* ctx, int32_t max_entries, char* names /* max_entries*32 */,
                     double* ms_per_launch, int64_t* launches, int32_t* n_out);

/* ------------------------------------------------------------------------
 * Per-step entry points (teacher-forced parity hooks; all on this shard)
 * ------------------------------------------------------------------------ */

/* procrustes_update over all shard subjects (solver.hpp:173-193 + the
 * run_chunks loop :279-284), fused with the mode-1 MTTKRP partial
 * M1 = sum_k Q_k^T (X_k V) diag(W_k) (mttkrp.hpp:81-106 in Q form).
 * H (R x R), V (J x R), W (K x R full).  Q_out packed row-major; flags per
 * shard subject; m1_out (R x R, allreduced).  Any output may be NULL. */
int p2g_procrustes(p2g_ctx* ctx, int32_t R, const double* H, const double* V, const double* W, double* Q_out,
                   int32_t* flags_out, double* m1_out);

/* Q-based slice-wise MTTKRP (north_star forms) from packed Q of this shard:
 *  mode 1: sum_k Q_k^T (X_k V) diag(W_k)            -> R x R (allreduced)
 *  mode 2: sum_k X_k^T (Q_k H diag(W_k))            -> J x R (allreduced)
 *  mode 3: row k = colwise-dot(Q_k H, X_k V)        -> shard K x R
 * Equal to mttkrp(project_slices(X, Q), H, V, W, mode) (mttkrp.hpp:187-196). */
int p2g_mttkrp_q(p2g_ctx* ctx, int32_t mode, int32_t R, const double* Q, const double* H, const double* V,
                 const double* W, double* out);

/* project_slices (solver.hpp:212-235): packed Y_k = Q_k^T X_k (R x c_k,
 * column-major per subject, subjects concatenated) and the column ids.
 * ycol_ptr[K_shard+1] offsets (in columns) are written first; call with
 * Y_out == NULL to obtain sizes only. */
int p2g_project(p2g_ctx* ctx, int32_t R, const double* Q, int64_t* ycol_ptr, int32_t* ycols, double* Y_out);

/* mttkrp on packed projected slices — replaces mttkrp(ProjectedSlices,...)
 * (mttkrp.hpp:187-196) with its shape checks (:170-181).  Standalone: does
 * not need load_csr.  ycol_ptr[K+1], ycols (ascending per slice), Y packed
 * (R x c_k column-major blocks).  H R x R, V J x R, W K x R. */
int p2g_mttkrp_packed(p2g_ctx* ctx, int32_t mode, int64_t K, int64_t J, int32_t R, const int64_t* ycol_ptr,
                      const int32_t* ycols, const double* Y, const double* H, const double* V, const double* W,
                      double* out);

/* cp_als_iteration on packed projected slices (cp.hpp:99-145): H, V, W in/out
 * (column-major), lambda_out (R), m3_out (K x R) optional. */
int p2g_cp_als_iteration(p2g_ctx* ctx, int64_t K, int64_t J, int32_t R, const int64_t* ycol_ptr,
                         const int32_t* ycols, const double* Y, double* H, double* V, double* W, int32_t nonneg,
                         int32_t normalize_w, double* lambda_out, double* m3_out);

/* nnls_rowwise (kernels.hpp:194-211): X (n x R) = argmin_{X>=0} rowwise
 * x G x^T - 2 x b^T; max_iter 0 -> 30 R.  Column-major G (R x R), B, X. */
int p2g_nnls_rowwise(p2g_ctx* ctx, const double* G, const double* B, int64_t n, int32_t R, int32_t max_iter,
                     double* X);

/* naive_mttkrp (mttkrp.hpp:198-235) on the device: the dense mode-n
 * unfolding and the full Khatri-Rao product materialised in HBM, then one
 * DGEMM.  Same arguments and shape checks as p2g_mttkrp_packed.  The
 * baseline the slice-wise kernels beat. */
int p2g_naive_mttkrp(p2g_ctx* ctx, int32_t mode, int64_t K, int64_t J, int32_t R, const int64_t* ycol_ptr,
                     const int32_t* ycols, const double* Y, const double* H, const double* V, const double* W,
                     double* out);
/* naive_mttkrp_bytes (mttkrp.hpp:241-253); 0 for a bad mode. */
uint64_t p2g_naive_mttkrp_bytes(int64_t K, int64_t J, int64_t R, int32_t mode);

/* bench_mttkrp (bench.hpp:90-215) on the device over the loaded tensor:
 * Y_k = Q_k^T X_k with seeded random orthonormal Q_k (generator.hpp:36-47,
 * stream substream_seed(seed, k+1)) and seeded uniform H, V, W; `reps`
 * timed sweeps (CUDA events, medians; one untimed warm-up sweep each) of the
 * specialized kernels, then of the naive kernel per mode unless its
 * materialisation exceeds budget_bytes (0 = free device memory - 2 GiB),
 * which marks the cell out-of-memory as the reference does. */
typedef struct {
  int64_t K, J;
  int32_t R;
  int64_t nnz;
  int32_t reps;
  uint64_t budget_bytes;
  double specialized_ms[3];    /* median per mode */
  double naive_ms[3];          /* median per mode, -1 when out of memory */
  uint64_t naive_bytes[3];     /* materialisation bytes per mode */
  int32_t naive_oom[3];
  double specialized_sweep_ms; /* median of the 3-mode sweeps */
  double naive_sweep_ms;       /* 0 when any naive mode was skipped */
  int32_t naive_sweep_oom;
  double speedup;              /* naive / specialized sweep, 0 if unknown */
  uint64_t specialized_device_bytes; /* device bytes the specialized path holds */
  double checksum_specialized, checksum_naive; /* sums of the outputs (anti-elision) */
} p2g_bench_report;
int p2g_bench_mttkrp(p2g_ctx* ctx, int32_t R, int32_t reps, uint64_t budget_bytes, uint64_t seed,
                     p2g_bench_report* report);

/* pinv_small (kernels.hpp:68-87) and gram (kernels.hpp:57-63) on device. */
int p2g_pinv_small(p2g_ctx* ctx, const double* G, int32_t n, double* out);
int p2g_gram(p2g_ctx* ctx, const double* A, int64_t rows, int32_t cols, double* out);

/* economy_svd (kernels.hpp:92-107): thin SVD M = P diag(sigma) Z^T of the
 * column-major rows x cols matrix M, rho = min(rows, cols); P is rows x rho,
 * Z is cols x rho (both column-major), sigma non-increasing.  A zero matrix
 * yields zero singular values and identity-block factors (kernels.hpp:101-104);
 * non-finite entries: P2G_ENUMERICAL ("svd operand").  min(rows, cols) <= 128. */
int p2g_economy_svd(p2g_ctx* ctx, const double* M, int64_t rows, int64_t cols, double* P, double* sigma, double* Z);

/* ---------------------------------------------------------------------------
 * Ingest and export (host side).  No GPU needed.
 * ------------------------------------------------------------------------- */

/* A parsed/loaded host CSR tensor owned by the library. */
typedef struct p2g_csr p2g_csr;

/* parse_coordinate_stream / parse_coordinate_file (io.hpp:100-177): '#'
 * comments and blank lines skipped, "K J" header, entries "k i j v" (0-based),
 * duplicates summed, zero sums dropped, all-zero rows removed (counted in
 * filtered_rows), empty subjects rejected.  Errors are P2G_EDATA with the
 * reference's messages ("... at line N").  threads 0 = all host threads. */
int p2g_coo_parse(const char* text, int64_t len, int32_t threads, p2g_csr** out);
int p2g_coo_read(const char* path, int32_t threads, p2g_csr** out);
int p2g_csr_info(const p2g_csr* t, int64_t* K, int64_t* J, int64_t* n_rows, int64_t* nnz, int64_t* filtered_rows);
int p2g_csr_copy(const p2g_csr* t, int64_t* subj_row_ptr, int64_t* row_ptr, int32_t* col_idx, double* val);
void p2g_csr_free(p2g_csr* t);

/* write_coordinate_file (io.hpp:179-204): canonical order (subject, column,
 * row), "%.17g" values, optional "# comment" lines first. */
int p2g_coo_write(const char* path, int64_t K, int64_t J, const int64_t* subj_row_ptr, const int64_t* row_ptr,
                  const int32_t* col_idx, const double* val, const char* const* comments, int32_t n_comments);

/* Binary CSR cache ("P2GCSR01" + K, J, NR, nnz + the four arrays): reloads a
 * parsed tensor at storage speed. */
int p2g_csr_cache_write(const char* path, int64_t K, int64_t J, const int64_t* subj_row_ptr, const int64_t* row_ptr,
                        const int32_t* col_idx, const double* val);
int p2g_csr_cache_read(const char* path, p2g_csr** out);

/* write_matrix_file / read_matrix_file (io.hpp:206-268).  Column-major data.
 * read: pass colmajor = NULL to query rows/cols. */
int p2g_matrix_write(const char* path, int64_t rows, int64_t cols, const double* colmajor, const char* title);
int p2g_matrix_read(const char* path, int64_t* rows, int64_t* cols, double* colmajor, int64_t capacity);
int p2g_matrix_parse(const char* text, int64_t len, int64_t* rows, int64_t* cols, double* colmajor, int64_t capacity);

/* write_factors (io.hpp:270-305): V.txt, S.txt, H.txt, U_<k>.txt with
 * U_k = Q_k H (assemble_U, solver.hpp:238-243), manifest.json.  H, V, S
 * column-major; Q packed row-major (sum I_k) x R; metadata_json is embedded
 * as "config" (may be NULL). */
int p2g_write_factors(const char* dir, int64_t K, int64_t J, int32_t R, const int64_t* subj_row_ptr, const double* H,
                      const double* V, const double* S, const double* Q, const char* metadata_json);

/* write_trace_tsv (io.hpp:307-315): "iter\tresidual_sq\tfit". */
int p2g_write_trace(const char* path, int32_t n, const int32_t* iters, const double* residual_sq, const double* fit);

#ifdef __cplusplus
}
#endif

#endif /* P2G_H_ */
