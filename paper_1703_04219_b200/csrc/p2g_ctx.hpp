// Device context of libp2g (one per rank / GPU) and the launcher
// declarations shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "p2g_common.hpp"

struct cublasContext;  // cuBLAS handle (cublasHandle_t), dlopen'ed on first use

namespace p2g {

#define P2G_CUDA(call)                                                                                   \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess)                                                                               \
      throw ::p2g::CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + __FILE__ + \
                             ":" + std::to_string(__LINE__));                                            \
  } while (0)

/// Process-wide count of kernels this library launched (bench gpu_launches).
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> n{0};
  return n;
}

/// Call right after each <<<>>> launch: error check + launch count.
#define P2G_LAUNCHED(nkernels)                  \
  do {                                          \
    ::p2g::launch_counter() += (nkernels);      \
    P2G_CUDA(cudaGetLastError());               \
  } while (0)

/// Owning device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  std::size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void resize(std::size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) return;
    P2G_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  T* get() const { return p; }
};

/// Grows a per-warp scratch buffer to `count` elements, refusing with a clear
/// message when the device cannot hold it (the generic large-R and accurate
/// Procrustes paths size their slabs by the longest subject, max_rows).
template <typename T>
inline void grow_scratch(DBuf<T>& b, std::size_t count, const char* what, std::int64_t max_rows) {
  if (count <= b.n && b.p) return;
  std::size_t free_b = 0, total_b = 0;
  P2G_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const std::size_t need = count * sizeof(T);
  if (need > free_b + b.n * sizeof(T))
    throw CudaError(std::string(what) + ": per-warp scratch for subjects of up to " + std::to_string(max_rows) +
                    " rows needs " + std::to_string(need >> 20) + " MiB, " + std::to_string(free_b >> 20) +
                    " MiB free on the device");
  b.resize(count);
}

/// Per-phase device timing collected by the fused loop (bench / profiling).
struct PhaseTimer {
  std::vector<std::string> names;
  std::vector<cudaEvent_t> start, stop;
  std::map<std::string, std::pair<double, std::int64_t>> acc;  // total ms, launches
};

/// Device arguments of the sparse shard (CSR rebased to the shard).
struct ShardArgs {
  const std::int64_t* srp;  // K_s + 1, rows (rebased)
  const std::int64_t* rp;   // NR_s + 1, nnz offsets (rebased)
  const std::int32_t* ci;
  const double* val;
  std::int64_t K;  // shard subjects
  std::int64_t NR;
  std::int64_t nnz;
  std::int64_t J;
};

struct NcclState;  // opaque, defined in p2g_api.cu

/// Device workspace of the NNLS kernels (per context: two contexts, or two
/// streams, never share one).
struct NnlsWork {
  DBuf<double> slab;        // pinv fallback, 3 RP^2 per warp
  DBuf<double> ginv;        // G^{-1} (+ validity) for the warm fast path, R > 16
  DBuf<double> ginv_small;  // G^{-1} (+ validity) for the cold thread-per-row start, R <= 16
};

}  // namespace p2g

struct p2g_ctx {
  int device = 0;
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  p2g::NcclState* nccl = nullptr;
  // Host-staged collective (p2g_set_host_collective): used instead of NCCL
  // when set, e.g. by a gloo process group in tests.
  int (*host_coll)(double*, int64_t, int32_t, void*) = nullptr;
  void* host_coll_user = nullptr;
  double* coll_pinned = nullptr;
  std::size_t coll_pinned_n = 0;
  // Fault injection (p2g_inject_fault): force a rank-local error at an iteration.
  int fault_kind = 0, fault_iter = 0;
  int num_sms = 148;

  // Shard of the sparse tensor.
  std::int64_t K_total = 0, J = 0;
  std::int64_t k_begin = 0, k_end = 0;
  std::int64_t NR = 0, nnz = 0;  // shard rows / nnz
  std::int64_t max_rows = 0;     // max I_k in the shard
  std::int64_t min_rows_global = 0;
  std::int64_t nnz_total = 0;
  double norm_x = 0.0;  // ||X||_F^2 over ALL subjects (allreduced)
  bool loaded = false;
  bool shard_local = false;  // loaded by p2g_load_shard: W0 / W arguments are this rank's rows only
  p2g::DBuf<std::int64_t> srp, rp;
  p2g::DBuf<std::int32_t> ci;
  p2g::DBuf<double> val;

  // Factor state (row-major on device).
  int R = 0;
  p2g::DBuf<double> H, V, W, Q;       // R*R, J*R, K_s*R, NR*R
  p2g::DBuf<double> gramW, gramV;     // R*R each
  p2g::DBuf<double> nH, nV;           // R each
  p2g::DBuf<double> m1, M2, m3;       // R*R, J*R, K_s*R
  p2g::DBuf<double> G1, G2, G3, gramH; // R*R
  p2g::DBuf<double> gvraw, gwc;       // R*R, R*R+1
  p2g::DBuf<double> stage;            // host<->device staging (col-major)
  std::vector<std::int64_t> srp_host;  // this shard's subj_row_ptr (global row numbers; validation)
  double* pinned = nullptr;           // small pinned host block for per-iteration scalars
  p2g::DBuf<double> pinvbuf;          // R*R
  p2g::DBuf<double> partials;         // scratch for per-block partials
  p2g::DBuf<double> scal;             // small scalars (fit, cross, residual ...)
  p2g::DBuf<std::int32_t> flags;      // K_s
  p2g::DBuf<std::int32_t> fb_list;    // compacted fallback subject ids
  p2g::DBuf<std::int32_t> counters;   // [0]=n_fallback, [1]=nnls error, ...
  p2g::NnlsWork nnls_ws;
  // Diagnostics and experiment switches, read once from the environment at
  // p2g_create (P2G_DEBUG, P2G_TIMING, P2G_WARM, P2G_POLAR_NOSORT); the
  // defaults are the production configuration.
  struct Options {
    bool debug = false;        // sweep / convergence counters to stderr (adds atomics)
    bool timing = false;       // per-phase event timing on every call
    bool polar_warm = false;   // R <= 12: warm-start the polar Jacobi from the last eigenvectors
    bool polar_sort = true;    // R <= 12: order subjects by last sweep count (load balance)
  } opt;
  p2g::DBuf<double> acc_scratch;      // accurate Procrustes path slabs
  p2g::DBuf<std::int32_t> acc_list;   // flagged subjects (ascending) + count
  p2g::DBuf<unsigned char> acc_bytes, acc_temp;
  p2g::DBuf<double> Cbuf, Sbuf, Ebuf; // small-R pipeline: per-subject packed C, S; E / Shat of flagged subjects
  p2g::DBuf<double> Chat;             // completion term of flagged subjects (K_s x R x R)
  p2g::DBuf<double> Ewarm;            // per-subject Jacobi eigenvectors (warm start / preconditioner)
  bool ew_valid = false;              // Ewarm holds eigenvectors from a previous Procrustes step
  p2g::DBuf<double> Hp, Vp, Wp;       // factors the last Procrustes step used (Q-free reconstruction)
  bool c_valid = false;               // Cbuf holds Gram of X V for the current V
  bool xv_valid = false;              // R <= 16: Ubuf holds the X V rows of the current V (last mode-3 pass)
  p2g::DBuf<std::int32_t> redo;       // NNLS rows re-solved by the warp (pinv) kernel
  p2g::DBuf<double> m2part;           // per-range J x R partials of the on-chip mode-2 kernel
  // column-major copy of the shard for the atomics-free mode-2 pass (k_csc.cu)
  p2g::DBuf<std::int64_t> col_ptr, seg_ptr, seg_beg, seg_end;
  p2g::DBuf<std::int32_t> csc_row, seg_ids;
  p2g::DBuf<double> csc_val, seg_part, Ubuf;
  p2g::DBuf<unsigned long long> seg_next;  // R > 16 CSC SpMM: next unclaimed segment chunk
  std::int64_t nseg = 0;
  // The CSC build runs on `side` behind the load's upload (phase A: the big
  // sort, overlapping the first Procrustes step) and is finished at its first
  // use (phase B needs the segment count on the host): build_csc / ensure_csc.
  cudaStream_t side = nullptr;
  cudaEvent_t ev_upload = nullptr, ev_csc = nullptr;
  bool csc_pending = false;
  p2g::DBuf<std::int32_t> csc_rowof, csc_iota, csc_perm, csc_ids;
  p2g::DBuf<std::uint64_t> csc_keys, csc_skeys, csc_ck, csc_sck;
  p2g::DBuf<std::int64_t> csc_mark, csc_runstart, csc_nsel;
  p2g::DBuf<unsigned char> csc_head, csc_temp;
  p2g::DBuf<unsigned> mask_v, mask_w; // NNLS passive sets of the previous iteration (warm start)
  p2g::DBuf<unsigned long long> mask64_v, mask64_w;  // same, R > 16
  p2g::DBuf<std::uint8_t> polar_sweeps, polar_keys;  // per-subject Jacobi sweeps of the last polar step
  p2g::DBuf<std::int32_t> polar_perm;                // subjects sorted by those counts (+ iota scratch)
  p2g::DBuf<unsigned char> polar_temp;
  bool polar_sweeps_valid = false;
  bool masks_valid = false;
  bool state_valid = false;

  // Per-iteration phase times of the last p2g_fit (the reference's
  // IterationStats ms_procrustes / ms_project / ms_cp, solver.hpp:70-77).
  std::vector<double> fit_phase_ms;
  cudaEvent_t ev_it[3] = {nullptr, nullptr, nullptr};

  // Timing.
  bool timing = false;
  p2g::PhaseTimer timer;
  std::vector<cudaEvent_t> ev_pool;
  std::size_t ev_used = 0;
  std::vector<std::pair<std::string, std::pair<std::size_t, std::size_t>>> pending;  // name, (ev0, ev1)
};

namespace p2g {

// ---- launchers (defined in the kernel translation units) ----
// Accurate Jacobi-SVD path over the subjects flagged P2G_FLAG_ACCURATE;
// writes one R x R m1 partial per block (count = procrustes_accurate_blocks).
void build_csc(p2g_ctx* c);
void ensure_csc(p2g_ctx* c);
void sync_csc(p2g_ctx* c);
void launch_csc_mode2(p2g_ctx* c, int R, const double* U, double* M2, cudaStream_t s);
void launch_urows_large(p2g_ctx* c, int R, const double* Q, const double* H, const double* W, const double* nH,
                        double* U, cudaStream_t s);
int launch_procrustes_large(p2g_ctx* c, int R, const double* H, const double* V, const double* W, double* Q,
                            std::int32_t* flags, double* m1_partials, double* Ewarm, int ew_valid, int max_blocks,
                            cudaStream_t s, const double* XV_in = nullptr);
int launch_procrustes_accurate(p2g_ctx* c, int R, const double* H, const double* V, const double* W, double* Q,
                               std::int32_t* flags, double* m1_partials, const double* Ebuf, double* Shat,
                               double* Chat, cudaStream_t s);
int procrustes_accurate_blocks(p2g_ctx* c, int R);

// Small-rank (Q-free, thread-per-subject) pipeline (k_small.cu) up to R = 12;
// larger R takes the warp-per-subject pipeline (k_large.cu).  Its R = 16
// instantiation of k_polar_small spilled 14.6 KB per thread (ptxas), so
// R = 13..16 runs faster on the large-R path.
constexpr int kSmallRankMax = 12;
void launch_gram_c(p2g_ctx* c, int R, const double* V, double* Cbuf, cudaStream_t s);
int launch_polar_small(p2g_ctx* c, int R, const double* H, const double* W, const double* Cbuf, double* Sbuf,
                       double* Ewarm, int warm, std::int32_t* flags, double* m1_partials, int max_blocks,
                       cudaStream_t s);
void launch_qrows(p2g_ctx* c, int R, const double* H, const double* V, const double* W, const double* Sbuf,
                  const double* Shat, const double* Chat, const std::int32_t* flags, double* Q, cudaStream_t s);
void launch_mode2_qf(p2g_ctx* c, int R, const double* Hprev, const double* Vprev, const double* Wprev,
                     const double* Ht, const double* nH, const double* Sbuf, const double* Shat, const double* Chat,
                     const std::int32_t* flags, double* M2, cudaStream_t s, const double* XV = nullptr);
void launch_mode3_qf(p2g_ctx* c, int R, const double* Hprev, const double* Vprev, const double* Wprev,
                     const double* Ht, const double* Vt, const double* Sbuf, const double* Shat, const double* Chat,
                     const std::int32_t* flags, double* M3, double* Cnext, cudaStream_t s, double* XV = nullptr,
                     int xv_in = 0);
void launch_nnls_thread(int R, std::int64_t n, const double* G, const double* B, double* X, int max_iter,
                        std::int32_t* err, std::int32_t* redo, std::int32_t* n_redo, unsigned* masks, int warm,
                        cudaStream_t s, const double* ginv = nullptr);
void launch_mode2(p2g_ctx* c, int R, const double* Q, const double* H, const double* W, const double* nH,
                  double* M2, cudaStream_t s);
/// X V rows (NR x R) of the shard into XV, exact R in {24, 32, 40} (the first
/// R = 40 Procrustes step of a fit, before any mode-3 pass has left them).
void launch_xv_rows(p2g_ctx* c, int R, const double* V, double* XV, cudaStream_t s);
void launch_mode3(p2g_ctx* c, int R, const double* Q, const double* H, const double* V, double* m3,
                  cudaStream_t s, double* XV_out = nullptr);
void launch_mode1_q(p2g_ctx* c, int R, const double* Q, const double* V, const double* W, double* m1_partials,
                    int nblocks, cudaStream_t s);
void launch_project(p2g_ctx* c, int R, const double* Q, const std::int64_t* ycol_ptr, const std::int32_t* ycols,
                    double* Y, cudaStream_t s);
int packed_mode1_blocks(int num_sms);
// Packed-Y MTTKRP (boundary): mode 1 -> nblocks R x R partials in out; mode 3 -> K x R rows.
void launch_packed_mode13(int mode, std::int64_t K, std::int64_t J, int R, const std::int64_t* ycol_ptr,
                          const std::int32_t* ycols, const double* Y, const double* H, const double* V,
                          const double* W, double* out, int nblocks, cudaStream_t s);
// Packed-Y mode 2, deterministic via the per-column occurrence list (c, k) pairs.
void launch_packed_mode2(std::int64_t K, std::int64_t J, int R, const std::int64_t* ycol_ptr,
                         const std::int32_t* ycols, const double* Y, const double* H, const double* W,
                         const std::int64_t* occ_ptr, const std::int64_t* occ, double* out, cudaStream_t s);

// Naive MTTKRP (k_naive.cu, mttkrp.hpp:198-253): materialised unfolding x
// Khatri-Rao product on the device; scratch reused across calls.
struct NaiveScratch {
  DBuf<double> A, KRP;
  DBuf<std::int64_t> subj_of;
  cublasContext* blas = nullptr;
  NaiveScratch() = default;
  NaiveScratch(const NaiveScratch&) = delete;
  NaiveScratch& operator=(const NaiveScratch&) = delete;
  ~NaiveScratch();
  void prepare(p2g_ctx* c, int mode, std::int64_t K, std::int64_t J, int R, const std::int64_t* ptr, std::int64_t nc);
};
std::uint64_t naive_bytes(std::int64_t K, std::int64_t J, std::int64_t R, int mode);
void naive_mttkrp(p2g_ctx* c, NaiveScratch& s, int mode, std::int64_t K, std::int64_t J, int R,
                  const std::int64_t* ptr, const std::int32_t* cols, const double* Y, std::int64_t nc, const double* H,
                  const double* V, const double* W, double* out);

// Eye initialisation (k_init.cu): C = sum_k X_k^T X_k of this shard into C
// (J x J), then V (row-major J x R) = |top-R eigenvectors of C| (C destroyed).
void build_column_gram(p2g_ctx* c, double* C);
void eye_vectors(p2g_ctx* c, double* C, int R, double* V);

// Dense helpers (k_dense.cu).
int gram_partials(int R, std::int64_t n, const double* A, const double* B, double* partials, int max_blocks,
                  cudaStream_t s);  // returns #partials; each partial R*R (+1 cross if B)
void reduce_partials(const double* partials, int nparts, std::int64_t len, double* out, cudaStream_t s);
// work: n+1 ints of scratch (thread-per-row path for R <= 16) or null.
// masks / masks64: n passive-set bit masks (R <= 16 / R <= 64) carried across
// calls for the warm start (warm != 0 uses them), or null.
// ws: the NNLS device workspace (pinv-fallback slab, G^{-1} for the warm fast
// path and the cold thread-per-row start), owned by the caller's context.
void launch_nnls_rows(NnlsWork& ws, int R, std::int64_t n, const double* G, const double* B, double* X, int max_iter,
                      std::int32_t* err, std::int32_t* work, cudaStream_t s, unsigned* masks = nullptr,
                      int warm = 0, unsigned long long* masks64 = nullptr);
void launch_rows_times(int R, std::int64_t n, const double* B, const double* P, double* X,
                       cudaStream_t s);  // X = B * P (row-major rows)
void launch_pinv(int n, const double* G, double* out, cudaStream_t s);
/// economy_svd (kernels.hpp:92-107), k_svd.cu: one-sided Jacobi SVD of W (mm x nn row-major, mm >= nn).
int svd_max_cols();
void launch_economy_svd(int mm, int nn, double* W, double* V, double* Uo, double* Vo, double* sig, int* status,
                        cudaStream_t s);
// Replicated R x R steps of the CP iteration (cp.hpp:99-145):
void launch_solve_h(int R, const double* m1, const double* gramW, const double* gramV, double* H, double* nH,
                    double* gramH, double* G2, cudaStream_t s);  // H update + normalize + G2 for the V step
void launch_normalize_v(int R, std::int64_t J, double* V, const double* gramV_raw, double* gramV, double* nV,
                        const double* gramH, double* G3, cudaStream_t s);
void launch_fit(int R, const double* gramW_cross, const double* gramH, const double* gramV, double norm_x,
                double* gramW, double* scal, cudaStream_t s);
// A[:, c] /= norms[c] for a row-major n x R matrix.
void launch_scale_cols(int R, std::int64_t n, double* A, const double* norms, cudaStream_t s);
void launch_transpose(const double* in, double* out, std::int64_t rows, std::int64_t cols, cudaStream_t s);
void launch_fill_identity(double* A, int n, cudaStream_t s);
void launch_fill(double* A, std::int64_t n, double v, cudaStream_t s);
void launch_hadamard(const double* A, const double* B, double* C, int n, cudaStream_t s);

}  // namespace p2g
