// C-ABI implementation (include/p2g.h): device context, CSR upload and
// sharding, the fused PARAFAC2-ALS loop (fit_parafac2, solver.hpp:251-321)
// and the per-step parity hooks.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <thread>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "p2g_ctx.hpp"

namespace p2g {

void partition_weighted(const std::uint64_t* w, std::int64_t n, std::int32_t n_chunks,
                        std::vector<std::pair<std::int64_t, std::int64_t>>& out);

// ---------------------------------------------------------------------------
// NCCL, loaded lazily (dlopen) so a process that already has torch's NCCL
// reuses it and a single-GPU context never touches NCCL.
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl_api() {
  static NcclApi api;
  if (!api.h) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw CudaError("NCCL unavailable: cannot dlopen libnccl.so.2");
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.CommDestroy)
      throw CudaError("NCCL unavailable: missing symbols");
    api.h = h;
  }
  return api;
}

struct NcclState {
  ncclComm_t comm = nullptr;
};

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw CudaError(std::string("NCCL ") + what + " failed: " +
                    (nccl_api().GetErrorString ? nccl_api().GetErrorString(r) : "?"));
}

/// Allreduce of fp64 values in device memory, in place (no-op on one rank);
/// op 0 = sum, 1 = max.  NCCL on the context's stream, or the host-staged
/// collective when one is set (p2g_set_host_collective).  The collectives of
/// an iteration: M1 (R x R), M2 (J x R), [gram(W), cross, error flags].
static void allreduce_op(p2g_ctx* c, double* buf, std::size_t count, int op) {
  if (c->world <= 1 || count == 0) return;
  if (c->host_coll) {
    if (c->coll_pinned_n < count) {
      if (c->coll_pinned) P2G_CUDA(cudaFreeHost(c->coll_pinned));
      c->coll_pinned = nullptr;
      c->coll_pinned_n = 0;
      P2G_CUDA(cudaMallocHost(&c->coll_pinned, count * sizeof(double)));
      c->coll_pinned_n = count;
    }
    P2G_CUDA(cudaMemcpyAsync(c->coll_pinned, buf, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    if (c->host_coll(c->coll_pinned, static_cast<int64_t>(count), op, c->host_coll_user) != 0)
      throw CudaError("host collective failed");
    P2G_CUDA(cudaMemcpyAsync(buf, c->coll_pinned, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    return;
  }
  if (!c->nccl) throw InvalidArgument("world > 1 without NCCL: set a host collective first");
  nccl_check(nccl_api().AllReduce(buf, buf, count, ncclFloat64, op == 1 ? ncclMax : ncclSum, c->nccl->comm,
                                  c->stream),
             "allreduce");
}

static void allreduce(p2g_ctx* c, double* buf, std::size_t count) { allreduce_op(c, buf, count, 0); }

/// Allreduce of host values through the device path (one-time setup values:
/// ||X||^2, validation verdicts).
static void allreduce_host(p2g_ctx* c, double* host, std::size_t count, int op) {
  if (c->world <= 1 || count == 0) return;
  c->scal.resize(std::max<std::size_t>(8, count));
  P2G_CUDA(cudaMemcpyAsync(c->scal.get(), host, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  allreduce_op(c, c->scal.get(), count, op);
  P2G_CUDA(cudaMemcpyAsync(host, c->scal.get(), count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  P2G_CUDA(cudaStreamSynchronize(c->stream));
}

DBuf<double>& scratch_partials(p2g_ctx* c, std::size_t count) {
  c->partials.resize(count);
  return c->partials;
}

namespace {

// ---- timing helpers --------------------------------------------------------
struct Phase {
  p2g_ctx* c;
  std::string name;
  std::size_t ev0 = 0;
  Phase(p2g_ctx* ctx, const char* n) : c(ctx), name(n) {
    if (!c->timing) return;
    ev0 = next_event();
    P2G_CUDA(cudaEventRecord(c->ev_pool[ev0], c->stream));
  }
  ~Phase() noexcept(false) {
    if (!c->timing) return;
    const std::size_t ev1 = next_event();
    P2G_CUDA(cudaEventRecord(c->ev_pool[ev1], c->stream));
    c->pending.push_back({name, {ev0, ev1}});
  }
  std::size_t next_event() {
    if (c->ev_used == c->ev_pool.size()) {
      cudaEvent_t e;
      P2G_CUDA(cudaEventCreate(&e));
      c->ev_pool.push_back(e);
    }
    return c->ev_used++;
  }
};

void collect_timing(p2g_ctx* c) {
  if (!c->timing) return;
  for (auto& p : c->pending) {
    float ms = 0.f;
    P2G_CUDA(cudaEventElapsedTime(&ms, c->ev_pool[p.second.first], c->ev_pool[p.second.second]));
    auto& slot = c->timer.acc[p.first];
    slot.first += ms;
    slot.second += 1;
  }
  c->pending.clear();
  c->ev_used = 0;
}

void require_loaded(const p2g_ctx* c) {
  if (!c) throw InvalidArgument("null context");
  if (!c->loaded) throw InvalidArgument("no tensor loaded (call p2g_load_csr first)");
}

void set_device(const p2g_ctx* c) { P2G_CUDA(cudaSetDevice(c->device)); }

std::int64_t Ks(const p2g_ctx* c) { return c->k_end - c->k_begin; }

/// Host column-major (rows x cols) -> device row-major.
void upload_colmajor(p2g_ctx* c, const double* host, std::int64_t rows, std::int64_t cols, double* dev) {
  c->stage.resize(static_cast<std::size_t>(rows * cols));
  P2G_CUDA(cudaMemcpyAsync(c->stage.get(), host, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, c->stream));
  launch_transpose(c->stage.get(), dev, rows, cols, c->stream);
}

/// Host column-major (K_total x R) -> device row-major shard rows.
void upload_shard_rows(p2g_ctx* c, const double* host, std::int64_t total_rows, int R, double* dev) {
  const std::int64_t n = Ks(c);
  // after p2g_load_shard the caller passes this rank's rows only
  const std::int64_t rows = c->shard_local ? n : total_rows, off = c->shard_local ? 0 : c->k_begin;
  c->stage.resize(static_cast<std::size_t>(n * R));
  for (int r = 0; r < R; ++r)
    P2G_CUDA(cudaMemcpyAsync(c->stage.get() + static_cast<std::int64_t>(r) * n, host + r * rows + off,
                             sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  launch_transpose(c->stage.get(), dev, n, R, c->stream);
}

/// Device row-major (rows x cols) -> host column-major.
void download_colmajor(p2g_ctx* c, const double* dev, std::int64_t rows, std::int64_t cols, double* host) {
  // transpose on the device (row-major rows x cols viewed as column-major
  // cols x rows), then one copy straight into the caller's buffer
  c->stage.resize(static_cast<std::size_t>(std::max<std::int64_t>(rows * cols, 1)));
  launch_transpose(dev, c->stage.get(), cols, rows, c->stream);
  P2G_CUDA(cudaMemcpyAsync(host, c->stage.get(), sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, c->stream));
  P2G_CUDA(cudaStreamSynchronize(c->stream));
}

void check_finite_host(const double* a, std::int64_t n, const char* what) {
  for (std::int64_t i = 0; i < n; ++i)
    if (!std::isfinite(a[i])) throw NumericalError(std::string(what) + ": non-finite entries");
}

/// First shard subject with I_k < R as (global index, I_k), or (-1, 0).
std::pair<std::int64_t, std::int64_t> first_short_subject(const p2g_ctx* c, int R) {
  for (std::int64_t k = 0; k + 1 < static_cast<std::int64_t>(c->srp_host.size()); ++k) {
    const std::int64_t I = c->srp_host[static_cast<std::size_t>(k + 1)] - c->srp_host[static_cast<std::size_t>(k)];
    if (I < R) return {c->k_begin + k, I};
  }
  return {-1, 0};
}

/// Config validation of initialize() (solver.hpp:106-122).  The I_k >= R
/// check runs on each rank's shard; with several ranks the first failing
/// subject over all ranks is agreed collectively, so every rank throws the
/// same error (none is left waiting in a later collective).
void validate_fit(p2g_ctx* c, const p2g_fit_config* cfg) {
  const int R = cfg->rank;
  if (R < 1) throw InvalidArgument("rank must be at least 1");
  if (!(cfg->tol > 0.0)) throw InvalidArgument("convergence tolerance must be positive");
  if (cfg->max_iters < 1) throw InvalidArgument("iteration limit must be at least 1");
  if (R > 40) throw InvalidArgument("rank above 40 unsupported on device");
  if (c->J < R) throw DataError("rank exceeds variables: J = " + std::to_string(c->J) + " < rank " + std::to_string(R));
  if (cfg->init < 0 || cfg->init > 2) throw InvalidArgument("init must be 0 (random), 1 (eye) or 2 (explicit factors)");
  auto [k, I] = first_short_subject(c, R);
  if (c->world > 1) {  // max of (K - k): the smallest failing global index wins
    double v[2] = {k >= 0 ? static_cast<double>(c->K_total - k) : 0.0, 0.0};
    allreduce_host(c, v, 1, 1);
    const std::int64_t kk = v[0] > 0.0 ? c->K_total - static_cast<std::int64_t>(v[0]) : -1;
    double iv[1] = {kk >= 0 && kk == k ? static_cast<double>(I) : 0.0};
    allreduce_host(c, iv, 1, 0);  // only the owning rank contributes I_k
    k = kk;
    I = static_cast<std::int64_t>(iv[0]);
  }
  if (k >= 0)
    throw DataError("rank exceeds observations for subject " + std::to_string(k) + ": I_k = " + std::to_string(I) +
                    " < rank " + std::to_string(R));
}

void alloc_state(p2g_ctx* c, int R) {
  const std::size_t RR = static_cast<std::size_t>(R) * R;
  c->R = R;
  c->H.resize(RR);
  c->V.resize(static_cast<std::size_t>(c->J) * R);
  c->W.resize(static_cast<std::size_t>(std::max<std::int64_t>(Ks(c), 1)) * R);
  c->Q.resize(static_cast<std::size_t>(std::max<std::int64_t>(c->NR, 1)) * R);
  c->gramW.resize(RR);
  c->gramV.resize(RR);
  c->gramH.resize(RR);
  c->gvraw.resize(RR);
  c->gwc.resize(RR + 3);
  c->nH.resize(R);
  c->nV.resize(R);
  c->m1.resize(RR);
  c->M2.resize(static_cast<std::size_t>(c->J) * R);
  c->m3.resize(static_cast<std::size_t>(std::max<std::int64_t>(Ks(c), 1)) * R);
  c->G1.resize(RR);
  c->G2.resize(RR);
  c->G3.resize(RR);
  c->pinvbuf.resize(RR);
  c->scal.resize(8);
  c->flags.resize(static_cast<std::size_t>(std::max<std::int64_t>(Ks(c), 1)));
  c->counters.resize(32);
  c->redo.resize(static_cast<std::size_t>(std::max<std::int64_t>(c->J, Ks(c)) + 1));
  c->Hp.resize(RR);
  c->Vp.resize(static_cast<std::size_t>(c->J) * R);
  c->Wp.resize(static_cast<std::size_t>(std::max<std::int64_t>(Ks(c), 1)) * R);
  if (R <= kSmallRankMax) {
    const std::size_t ks = static_cast<std::size_t>(std::max<std::int64_t>(Ks(c), 1));
    const std::size_t nt = static_cast<std::size_t>(R) * (R + 1) / 2;
    c->Cbuf.resize(ks * nt);
    c->Sbuf.resize(ks * nt);
    c->Ebuf.resize(ks * RR);
    c->Chat.resize(ks * RR);
    c->Ewarm.resize(ks * RR);
    c->Ubuf.resize(static_cast<std::size_t>(std::max<std::int64_t>(c->NR, 1)) * R);  // X V rows between passes
    c->mask_v.resize(static_cast<std::size_t>(std::max<std::int64_t>(c->J, 1)));
    c->mask_w.resize(ks);
  } else {
    // right singular vectors per subject: warm start / preconditioner (12.8 KB per subject at R = 40)
    c->Ewarm.resize(static_cast<std::size_t>(std::max<std::int64_t>(Ks(c), 1)) * RR);
    c->Ubuf.resize(static_cast<std::size_t>(std::max<std::int64_t>(c->NR, 1)) * R);
    c->mask64_v.resize(static_cast<std::size_t>(std::max<std::int64_t>(c->J, 1)));
    c->mask64_w.resize(static_cast<std::size_t>(std::max<std::int64_t>(Ks(c), 1)));
  }
}

template <typename T>
void swap_buf(DBuf<T>& a, DBuf<T>& b) {
  std::swap(a.p, b.p);
  std::swap(a.n, b.n);
}

constexpr int kMaxPartials = 148 * 8;

/// m1 partials of one Procrustes step: up to kMaxPartials from the polar /
/// large-R kernel plus one per block of the accurate path, whose grid is
/// 4 x (or 2 x) the device's SM count.
std::size_t procrustes_partials(const p2g_ctx* c) {
  return static_cast<std::size_t>(kMaxPartials) + 4 * static_cast<std::size_t>(std::max(c->num_sms, 148));
}

bool small_rank(const p2g_ctx* c) { return c->R <= kSmallRankMax; }

/// Procrustes step over the shard (solver.hpp:279-284) with the factors
/// c->H, c->V, c->W, fused with the mode-1 partials (into `part`; returns
/// their count).  R <= 16 (Q-free): Gram C (unless mode 3 already produced
/// it), thread-per-subject polar factor -> S_k, accurate path -> Shat/Chat;
/// Q is not materialised.  Larger R: the warp-per-subject K1 writes Q.
/// Flagged subjects go through the accurate Jacobi-SVD path either way.
int procrustes_step(p2g_ctx* c, double* part) {
  const int R = c->R;
  const std::size_t RR = static_cast<std::size_t>(R) * R;
  cudaStream_t s = c->stream;
  int n1 = 0, n2 = 0;
  if (small_rank(c)) {
    if (!c->c_valid) {
      Phase ph(c, "gram_c");
      launch_gram_c(c, R, c->V.get(), c->Cbuf.get(), s);
      c->c_valid = true;
    }
    {
      Phase ph(c, "polar");
      n1 = launch_polar_small(c, R, c->H.get(), c->W.get(), c->Cbuf.get(), c->Sbuf.get(), c->Ewarm.get(),
                              (c->ew_valid && c->opt.polar_warm) ? 1 : 0, c->flags.get(), part,
                              kMaxPartials, s);
      c->ew_valid = true;
    }
    Phase ph(c, "procrustes_accurate");
    n2 = launch_procrustes_accurate(c, R, c->H.get(), c->V.get(), c->W.get(), nullptr, c->flags.get(),
                                    part + static_cast<std::size_t>(n1) * RR, c->Ewarm.get(), c->Ebuf.get(),
                                    c->Chat.get(), s);
  } else {
    {
      Phase ph(c, "procrustes");
      // c_valid: the last mode-3 pass left X V (current V) in Ubuf
      n1 = launch_procrustes_large(c, R, c->H.get(), c->V.get(), c->W.get(), c->Q.get(), c->flags.get(), part,
                                   c->Ewarm.get(), c->ew_valid ? 1 : 0, kMaxPartials, s,
                                   c->c_valid ? c->Ubuf.get() : nullptr);
      c->ew_valid = true;
    }
    Phase ph(c, "procrustes_accurate");
    n2 = launch_procrustes_accurate(c, R, c->H.get(), c->V.get(), c->W.get(), c->Q.get(), c->flags.get(),
                                    part + static_cast<std::size_t>(n1) * RR, c->Ewarm.get(), nullptr, nullptr, s);
  }
  return n1 + n2;
}

/// Materialises Q of the last Procrustes step (factors Hp, Vp, Wp after an
/// iteration, or H, V, W for the per-step hook) — export only.
void export_q(p2g_ctx* c, const double* H, const double* V, const double* W) {
  if (!small_rank(c)) return;  // large R: K1 already wrote Q
  launch_qrows(c, c->R, H, V, W, c->Sbuf.get(), c->Ebuf.get(), c->Chat.get(), c->flags.get(), c->Q.get(), c->stream);
}

/// Rank-local error counters <-> the two doubles after [gram(W), cross], so
/// that the iteration's last allreduce also agrees on the errors: a rank
/// whose W-NNLS failed (or whose Procrustes operand was non-finite) makes
/// every rank throw, instead of throwing alone and leaving the others in the
/// next collective.  `inject` adds a fault (p2g_inject_fault).
__global__ void k_err_pack(std::int32_t* counters, double* tail, int inject) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (inject) counters[1] += 1;
    tail[0] = static_cast<double>(counters[1]);
    tail[1] = static_cast<double>(counters[2]);
  }
}
__global__ void k_err_unpack(std::int32_t* counters, const double* tail) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    counters[1] = static_cast<std::int32_t>(tail[0]);
    counters[2] = static_cast<std::int32_t>(tail[1]);
  }
}

/// gram(W) and the cross term over this shard, allreduced -> c->gwc; with
/// `errors`, also the error counters (k_err_pack).
void gram_w_cross(p2g_ctx* c, const double* W, const double* m3_or_null, bool errors = false, int inject = 0) {
  const int R = c->R;
  const std::size_t RR = static_cast<std::size_t>(R) * R;
  DBuf<double>& part = scratch_partials(c, kMaxPartials * (RR + 1));
  const int np = gram_partials(R, Ks(c), W, m3_or_null, part.get(), kMaxPartials, c->stream);
  reduce_partials(part.get(), np, static_cast<std::int64_t>(RR + 1), c->gwc.get(), c->stream);
  if (!errors) {
    allreduce(c, c->gwc.get(), RR + 1);
    return;
  }
  k_err_pack<<<1, 32, 0, c->stream>>>(c->counters.get(), c->gwc.get() + RR + 1, inject);
  P2G_LAUNCHED(1);
  allreduce(c, c->gwc.get(), RR + 3);
  if (c->world > 1) {
    k_err_unpack<<<1, 32, 0, c->stream>>>(c->counters.get(), c->gwc.get() + RR + 1);
    P2G_LAUNCHED(1);
  }
}

/// gram(V) (replicated, no collective) -> out.
void gram_v(p2g_ctx* c, const double* V, double* out) {
  const int R = c->R;
  const std::size_t RR = static_cast<std::size_t>(R) * R;
  DBuf<double>& part = scratch_partials(c, kMaxPartials * (RR + 1));
  const int np = gram_partials(R, c->J, V, nullptr, part.get(), 148, c->stream);
  reduce_partials(part.get(), np, static_cast<std::int64_t>(RR + 1), c->gwc.get(), c->stream);
  P2G_CUDA(cudaMemcpyAsync(out, c->gwc.get(), sizeof(double) * RR, cudaMemcpyDeviceToDevice, c->stream));
}

/// Initial state: H, V (J x R), W (shard) on device plus gram(W), gram(V).
void init_state(p2g_ctx* c, const p2g_fit_config* cfg, const double* H0, const double* V0, const double* W0) {
  const int R = cfg->rank;
  alloc_state(c, R);
  if (cfg->init == 2) {
    if (!H0 || !V0 || !W0) throw InvalidArgument("explicit init needs H0, V0 and W0");
    upload_colmajor(c, H0, R, R, c->H.get());
    upload_colmajor(c, V0, c->J, R, c->V.get());
    upload_shard_rows(c, W0, c->K_total, R, c->W.get());
  } else if (cfg->init == 1) {
    // solver.hpp:133-164: H = I, S = ones, V = |leading eigenvectors of sum_k X_k^T X_k|
    std::vector<double> h(static_cast<std::size_t>(R) * R, 0.0);
    for (int r = 0; r < R; ++r) h[static_cast<std::size_t>(r) * R + r] = 1.0;
    upload_colmajor(c, h.data(), R, R, c->H.get());
    DBuf<double> C;
    C.resize(static_cast<std::size_t>(c->J) * static_cast<std::size_t>(c->J));
    build_column_gram(c, C.get());
    allreduce(c, C.get(), static_cast<std::size_t>(c->J) * static_cast<std::size_t>(c->J));
    eye_vectors(c, C.get(), R, c->V.get());
    launch_fill(c->W.get(), Ks(c) * R, 1.0, c->stream);
    P2G_CUDA(cudaStreamSynchronize(c->stream));
  } else {
    // solver.hpp:124-132: H = I, S = ones, V = Rng(seed).uniform() r-outer j-inner.
    std::vector<double> h(static_cast<std::size_t>(R) * R), v(static_cast<std::size_t>(c->J) * R);
    if (p2g_initialize_random(cfg->seed, c->K_total, c->J, R, h.data(), nullptr, v.data()) != P2G_OK)
      throw InvalidArgument(p2g_last_error());
    upload_colmajor(c, h.data(), R, R, c->H.get());
    upload_colmajor(c, v.data(), c->J, R, c->V.get());
    launch_fill(c->W.get(), Ks(c) * R, 1.0, c->stream);
  }
  gram_v(c, c->V.get(), c->gramV.get());
  gram_w_cross(c, c->W.get(), nullptr);
  P2G_CUDA(cudaMemcpyAsync(c->gramW.get(), c->gwc.get(), sizeof(double) * R * R, cudaMemcpyDeviceToDevice, c->stream));
  c->c_valid = false;
  c->xv_valid = false;
  c->ew_valid = false;
  c->masks_valid = false;
  c->polar_sweeps_valid = false;
  c->state_valid = true;
  c->fit_phase_ms.clear();
}

struct IterOut {
  double fit, resid;
};

/// One PARAFAC2-ALS iteration on device (solver.hpp:274-306).  Reads the
/// t-1 factors from H, V, W and writes the t factors into Hp, Vp, Wp, then
/// swaps, so afterwards Hp, Vp, Wp hold the factors this Procrustes step
/// used (Q export).
IterOut iterate(p2g_ctx* c, bool nonneg, int iter) {
  const int R = c->R;
  const std::size_t RR = static_cast<std::size_t>(R) * R;
  cudaStream_t s = c->stream;
  const bool qf = small_rank(c);
  for (cudaEvent_t& e : c->ev_it)
    if (!e) P2G_CUDA(cudaEventCreate(&e));
  P2G_CUDA(cudaEventRecord(c->ev_it[0], s));
  P2G_CUDA(cudaMemsetAsync(c->counters.get(), 0, sizeof(std::int32_t) * 32, s));
  {
    DBuf<double>& part = scratch_partials(c, procrustes_partials(c) * RR);
    const int np = procrustes_step(c, part.get());
    Phase ph(c, "m1_reduce");
    reduce_partials(part.get(), np, static_cast<std::int64_t>(RR), c->m1.get(), s);
    allreduce(c, c->m1.get(), RR);
  }
  P2G_CUDA(cudaEventRecord(c->ev_it[1], s));
  {
    Phase ph(c, "solve_h");  // H_t -> Hp
    launch_solve_h(R, c->m1.get(), c->gramW.get(), c->gramV.get(), c->Hp.get(), c->nH.get(), c->gramH.get(),
                   c->G2.get(), s);
  }
  {
    Phase ph(c, "mode2");
    // row factors U (small R: into the Q buffer, unused until export), then
    // M2 = X^T U from the CSC copy (atomics-free, deterministic)
    double* U = qf ? c->Q.get() : c->Ubuf.get();
    if (qf)
      launch_mode2_qf(c, R, c->H.get(), c->V.get(), c->W.get(), c->Hp.get(), c->nH.get(), c->Sbuf.get(),
                      c->Ebuf.get(), c->Chat.get(), c->flags.get(), U, s, c->xv_valid ? c->Ubuf.get() : nullptr);
    else
      launch_urows_large(c, R, c->Q.get(), c->Hp.get(), c->W.get(), c->nH.get(), U, s);
    launch_csc_mode2(c, R, U, c->M2.get(), s);
    allreduce(c, c->M2.get(), static_cast<std::size_t>(c->J) * R);
  }
  {
    Phase ph(c, "update_v");  // V_t -> Vp
    if (nonneg) {
      launch_nnls_rows(c->nnls_ws, R, c->J, c->G2.get(), c->M2.get(), c->Vp.get(), 0, c->counters.get() + 1, c->redo.get(), s,
                       c->mask_v.get(), c->masks_valid ? 1 : 0, c->mask64_v.get());
    } else {
      launch_pinv(R, c->G2.get(), c->pinvbuf.get(), s);
      launch_rows_times(R, c->J, c->M2.get(), c->pinvbuf.get(), c->Vp.get(), s);
    }
    gram_v(c, c->Vp.get(), c->gvraw.get());
    launch_normalize_v(R, c->J, c->Vp.get(), c->gvraw.get(), c->gramV.get(), c->nV.get(), c->gramH.get(),
                       c->G3.get(), s);
  }
  {
    Phase ph(c, "mode3");
    if (qf)
      launch_mode3_qf(c, R, c->H.get(), c->V.get(), c->W.get(), c->Hp.get(), c->Vp.get(), c->Sbuf.get(),
                      c->Ebuf.get(), c->Chat.get(), c->flags.get(), c->m3.get(), c->Cbuf.get(), s, c->Ubuf.get(),
                      c->xv_valid ? 1 : 0);
    else
      launch_mode3(c, R, c->Q.get(), c->Hp.get(), c->Vp.get(), c->m3.get(), s, c->Ubuf.get());  // U is dead here
  }
  {
    Phase ph(c, "update_w");  // W_t -> Wp
    if (nonneg) {
      launch_nnls_rows(c->nnls_ws, R, Ks(c), c->G3.get(), c->m3.get(), c->Wp.get(), 0, c->counters.get() + 1, c->redo.get(), s,
                       c->mask_w.get(), c->masks_valid ? 1 : 0, c->mask64_w.get());
      c->masks_valid = true;
    } else {
      launch_pinv(R, c->G3.get(), c->pinvbuf.get(), s);
      launch_rows_times(R, Ks(c), c->m3.get(), c->pinvbuf.get(), c->Wp.get(), s);
    }
  }
  {
    Phase ph(c, "fit");
    gram_w_cross(c, c->Wp.get(), c->m3.get(), true, c->fault_kind == 1 && c->fault_iter == iter);
    launch_fit(R, c->gwc.get(), c->gramH.get(), c->gramV.get(), c->norm_x, c->gramW.get(), c->scal.get(), s);
  }
  swap_buf(c->H, c->Hp);
  swap_buf(c->V, c->Vp);
  swap_buf(c->W, c->Wp);
  c->c_valid = true;  // mode 3 produced the Gram (R <= 16) or X V rows (R > 16) for the new V
  c->xv_valid = qf;   // and, for R <= 16, the X V rows in Ubuf
  P2G_CUDA(cudaEventRecord(c->ev_it[2], s));
  // One host sync per iteration: fit scalars + error counters.
  P2G_CUDA(cudaMemcpyAsync(c->pinned, c->scal.get(), sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
  P2G_CUDA(cudaMemcpyAsync(c->pinned + 4, c->counters.get(), sizeof(std::int32_t) * 8, cudaMemcpyDeviceToHost, s));
  P2G_CUDA(cudaStreamSynchronize(s));
  collect_timing(c);
  {  // IterationStats (solver.hpp:70-77): procrustes (+ fused mode-1 partial), project (none: the loop is
     // Q-based and never forms Y), cp (MTTKRP modes 2-3, the H/V/W updates and the fit scalars)
    float a = 0.f, b = 0.f;
    P2G_CUDA(cudaEventElapsedTime(&a, c->ev_it[0], c->ev_it[1]));
    P2G_CUDA(cudaEventElapsedTime(&b, c->ev_it[1], c->ev_it[2]));
    c->fit_phase_ms.push_back(a);
    c->fit_phase_ms.push_back(0.0);
    c->fit_phase_ms.push_back(b);
  }
  const std::int32_t* cnt = reinterpret_cast<const std::int32_t*>(c->pinned + 4);
  if (c->opt.debug && cnt[7] > 0) {
    if (small_rank(c))
      std::fprintf(stderr, "[p2g] iter %d polar sweeps: mean %.2f max %d mean-warp-max %.2f\n", iter,
                   static_cast<double>(cnt[4]) / static_cast<double>(std::max<std::int64_t>(Ks(c), 1)), cnt[5],
                   static_cast<double>(cnt[6]) / cnt[7]);
    else
    {
      std::fprintf(stderr, "[p2g] iter %d large-R Jacobi sweeps: mean %.2f per pass, max %d, redone %d of %d\n", iter,
                   static_cast<double>(cnt[4]) / (cnt[7] + cnt[6]), cnt[5], cnt[6], cnt[7]);
      std::int32_t h[24];
      P2G_CUDA(cudaMemcpy(h, c->counters.get() + 8, sizeof(h), cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "[p2g]   warm max scaled off-diag, log10 bins <-8..>=0:");
      for (int b = 0; b < 10; ++b) std::fprintf(stderr, " %d", h[b]);
      std::fprintf(stderr, "\n[p2g]   sweeps per pass 0..9+:");
      for (int b = 0; b < 10; ++b) std::fprintf(stderr, " %d", h[12 + b]);
      std::fprintf(stderr, "\n");
    }
  }
  if (cnt[2] > 0) throw NumericalError("svd operand: non-finite entries");
  if (cnt[1] > 0) throw NumericalError("NNLS did not converge");
  IterOut o{c->pinned[0], c->pinned[1]};
  if (!std::isfinite(o.fit) || !std::isfinite(o.resid))
    throw NumericalError("numerical divergence at iteration " + std::to_string(iter));
  return o;
}

}  // namespace
}  // namespace p2g

using namespace p2g;

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------
extern "C" int p2g_nccl_unique_id(char out_id[128]) {
  return guarded([&] {
    ncclUniqueId id;
    nccl_check(nccl_api().GetUniqueId(&id), "get unique id");
    static_assert(sizeof(ncclUniqueId) == 128, "unexpected NCCL id size");
    std::memcpy(out_id, &id, 128);
  });
}

extern "C" int p2g_create(int32_t device, int32_t rank, int32_t world, const char* nccl_id, p2g_ctx** out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("null output");
    if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("bad rank/world");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) throw CudaError("no CUDA device available (the GPU path has no CPU fallback)");
    if (device < 0 || device >= ndev) throw InvalidArgument("device ordinal out of range");
    auto c = std::make_unique<p2g_ctx>();
    c->device = device;
    c->rank = rank;
    c->world = world;
    P2G_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    P2G_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
      throw CudaError("libp2g is built for sm_100a (B200) only; found sm_" + std::to_string(prop.major) +
                      std::to_string(prop.minor));
    c->num_sms = prop.multiProcessorCount;
    c->opt.debug = std::getenv("P2G_DEBUG") != nullptr;
    c->opt.timing = std::getenv("P2G_TIMING") != nullptr;
    c->opt.polar_warm = std::getenv("P2G_WARM") != nullptr;
    c->opt.polar_sort = std::getenv("P2G_POLAR_NOSORT") == nullptr;
    P2G_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    P2G_CUDA(cudaMallocHost(&c->pinned, 64 * sizeof(double)));
    if (world > 1 && nccl_id) {  // (without an id: a host collective must be set before the load)
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, 128);
      c->nccl = new NcclState();
      nccl_check(nccl_api().CommInitRank(&c->nccl->comm, world, id, rank), "comm init");
    }
    *out = c.release();
  });
}

extern "C" int p2g_destroy(p2g_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->nccl) {
      if (c->nccl->comm) nccl_api().CommDestroy(c->nccl->comm);
      delete c->nccl;
    }
    if (c->side) {
      cudaStreamSynchronize(c->side);
      cudaStreamDestroy(c->side);
      cudaEventDestroy(c->ev_upload);
      cudaEventDestroy(c->ev_csc);
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_it)
      if (e) cudaEventDestroy(e);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->coll_pinned) cudaFreeHost(c->coll_pinned);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
  });
}

extern "C" int p2g_set_host_collective(p2g_ctx* c, p2g_host_allreduce_fn fn, void* user) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    c->host_coll = fn;
    c->host_coll_user = user;
  });
}

extern "C" int p2g_inject_fault(p2g_ctx* c, int32_t kind, int32_t iteration) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    if (kind < 0 || kind > 1) throw InvalidArgument("fault kind must be 0 (none) or 1 (W-NNLS failure)");
    c->fault_kind = kind;
    c->fault_iter = iteration;
  });
}

namespace p2g {
namespace {
/// Host threads for an O(n) pass: fixed by n (not by timing), so chunked
/// reductions are reproducible on a given machine.
int host_threads(std::int64_t n) {
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(std::min(hw, 32), n / (1 << 20) + 1)));
}
template <typename Fn>
void run_host_parallel(int n, Fn&& fn) {
  if (n == 1) {
    fn(0);
    return;
  }
  std::vector<std::thread> ts;
  for (int t = 0; t < n; ++t) ts.emplace_back([&fn, t] { fn(t); });
  for (auto& th : ts) th.join();
}
__global__ void k_rebase(std::int64_t* a, std::int64_t n, std::int64_t off) {
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    a[i] -= off;
}
void launch_rebase(std::int64_t* a, std::int64_t n, std::int64_t off, cudaStream_t s) {
  if (off == 0 || n == 0) return;
  k_rebase<<<static_cast<int>(std::min<std::int64_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(a, n, off);
}

// Device-side checks of a single-rank load (the host loops of
// IrregularTensor::from_slices, sparse.hpp:176-193, read 0.7 GB of host
// memory at cfg2): the first failing row in row order wins, as on the host.
__global__ void k_check_rowptr(const std::int64_t* __restrict__ rp, std::int64_t NR,
                               unsigned long long* __restrict__ bad) {
  for (std::int64_t r = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < NR;
       r += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    if (rp[r + 1] < rp[r]) atomicMin(bad, static_cast<unsigned long long>(r));
}
/// bad = 4 * row + {2: column out of range, 3: not strictly ascending}, the
/// first failing entry of the first failing row (host loop order).
__global__ void k_check_cols(const std::int64_t* __restrict__ rp, const std::int32_t* __restrict__ ci,
                             std::int64_t NR, std::int64_t J, unsigned long long* __restrict__ bad) {
  for (std::int64_t r = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < NR;
       r += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t p0 = rp[r], p1 = rp[r + 1];
    for (std::int64_t p = p0; p < p1; ++p) {
      const std::int32_t j = ci[p];
      int t = 0;
      if (j < 0 || j >= J)
        t = 2;
      else if (p > p0 && j <= ci[p - 1])
        t = 3;
      if (t) {
        atomicMin(bad, static_cast<unsigned long long>(r) * 4ull + static_cast<unsigned long long>(t));
        break;
      }
    }
  }
}
/// ||X||_F^2 partials: block b sums the fixed chunk [b n / B, (b + 1) n / B)
/// with a fixed tree (deterministic); the host adds the B partials in order.
constexpr int kNormBlocks = 1024;
__global__ void __launch_bounds__(256) k_sumsq(const double* __restrict__ v, std::int64_t n, double* __restrict__ out) {
  __shared__ double red[256];
  const std::int64_t b0 = n * blockIdx.x / gridDim.x, b1 = n * (blockIdx.x + 1) / gridDim.x;
  double a = 0.0;
  for (std::int64_t p = b0 + threadIdx.x; p < b1; p += blockDim.x) a = fma(v[p], v[p], a);
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}
}  // namespace
}  // namespace p2g

extern "C" int p2g_load_csr(p2g_ctx* c, int64_t K, int64_t J, const int64_t* srp, const int64_t* rp,
                            const int32_t* ci, const double* val) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    set_device(c);
    const bool tim = c->opt.timing;
    const auto tl0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (tim)
        std::fprintf(stderr, "[p2g] load %-12s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl0).count());
    };
    if (c->world > 1 && !c->nccl && !c->host_coll)
      throw InvalidArgument("world > 1 needs an NCCL unique id or a host collective");
    c->shard_local = false;
    // IrregularTensor::from_slices (sparse.hpp:176-193) validation.
    if (J <= 0) throw DataError("tensor must have at least one column");
    if (K <= 0) throw DataError("tensor must have at least one slice");
    if (!srp || !rp) throw InvalidArgument("null CSR arrays");
    if (srp[0] != 0) throw DataError("subj_row_ptr must start at 0");
    for (int64_t k = 0; k < K; ++k)
      if (srp[k + 1] < srp[k]) throw DataError("subj_row_ptr must be non-decreasing");
    const int64_t NRt = srp[K];
    if (rp[0] != 0) throw DataError("row_ptr must start at 0");
    // One rank holds the whole tensor: the row-pointer / column checks and
    // ||X||^2 run on the device after the upload (same errors, same order).
    const bool dev_checks = c->world == 1;
    if (!dev_checks) {
    // Row pointers first (over all rows, as the serial check), then column
    // range / ascending order within rows: both in parallel over fixed row
    // ranges, the first failing range reports.
    const int nthr = host_threads(NRt);
    std::vector<int> bad(static_cast<std::size_t>(nthr), 0);
    run_host_parallel(nthr, [&](int t) {
      for (int64_t r = NRt * t / nthr; r < NRt * (t + 1) / nthr; ++r)
        if (rp[r + 1] < rp[r]) {
          bad[static_cast<std::size_t>(t)] = 1;
          break;
        }
    });
    for (int b : bad)
      if (b) throw DataError("row_ptr must be non-decreasing");
    if (rp[NRt] > 0 && (!ci || !val)) throw InvalidArgument("null CSR arrays");
    run_host_parallel(nthr, [&](int t) {
      for (int64_t r = NRt * t / nthr; r < NRt * (t + 1) / nthr && !bad[static_cast<std::size_t>(t)]; ++r)
        for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
          if (ci[p] < 0 || ci[p] >= J) {
            bad[static_cast<std::size_t>(t)] = 2;
            break;
          }
          if (p > rp[r] && ci[p] <= ci[p - 1]) {
            bad[static_cast<std::size_t>(t)] = 3;
            break;
          }
        }
    });
    for (int b : bad) {
      if (b == 2) throw DataError("column index out of range");
      if (b == 3) throw DataError("column indices must be strictly ascending within a row");
    }
    }
    lap("validated");
    const int64_t nnz_t = rp[NRt];
    if (nnz_t < 0) throw DataError("row_ptr must be non-decreasing");  // rp[0] = 0 > rp[NR]
    if (nnz_t > 0 && (!ci || !val)) throw InvalidArgument("null CSR arrays");
    sync_csc(c);        // a previous load's CSC build may still read the shard buffers
    c->loaded = false;  // the device checks below may still reject the tensor
    // Shard by partition_weighted(nnz_k + I_k, world) (solver.hpp:263-267);
    // one rank takes [0, K) (partition_weighted's single chunk).
    std::vector<std::pair<std::int64_t, std::int64_t>> parts;
    if (c->world == 1) {
      parts.emplace_back(0, K);
    } else {
      std::vector<std::uint64_t> w(static_cast<std::size_t>(K));
      for (int64_t k = 0; k < K; ++k)
        w[static_cast<std::size_t>(k)] =
            static_cast<std::uint64_t>(rp[srp[k + 1]] - rp[srp[k]]) + static_cast<std::uint64_t>(srp[k + 1] - srp[k]);
      partition_weighted(w.data(), K, c->world, parts);
    }
    if (static_cast<int>(parts.size()) != c->world) throw DataError("fewer subjects than ranks");
    c->K_total = K;
    c->J = J;
    c->k_begin = parts[static_cast<std::size_t>(c->rank)].first;
    c->k_end = parts[static_cast<std::size_t>(c->rank)].second;
    c->srp_host.assign(srp + c->k_begin, srp + c->k_end + 1);
    const int64_t row0 = srp[c->k_begin], row1 = srp[c->k_end];
    const int64_t nz0 = rp[row0], nz1 = rp[row1];
    c->NR = row1 - row0;
    c->nnz = nz1 - nz0;
    c->nnz_total = nnz_t;
    c->max_rows = 0;
    for (int64_t k = c->k_begin; k < c->k_end; ++k) c->max_rows = std::max<std::int64_t>(c->max_rows, srp[k + 1] - srp[k]);
    // Upload the shard as is and rebase row pointers on the device (the
    // caller's buffers are read once; pinned ones copy at link speed).
    c->srp.resize(static_cast<std::size_t>(c->k_end - c->k_begin + 1));
    c->rp.resize(static_cast<std::size_t>(c->NR + 1));
    c->ci.resize(static_cast<std::size_t>(std::max<int64_t>(c->nnz, 1)));
    c->val.resize(static_cast<std::size_t>(std::max<int64_t>(c->nnz, 1)));
    P2G_CUDA(cudaMemcpyAsync(c->srp.get(), srp + c->k_begin, sizeof(int64_t) * (c->k_end - c->k_begin + 1),
                             cudaMemcpyHostToDevice, c->stream));
    P2G_CUDA(cudaMemcpyAsync(c->rp.get(), rp + row0, sizeof(int64_t) * (c->NR + 1), cudaMemcpyHostToDevice, c->stream));
    launch_rebase(c->srp.get(), c->k_end - c->k_begin + 1, row0, c->stream);
    launch_rebase(c->rp.get(), c->NR + 1, nz0, c->stream);
    if (c->nnz > 0) {
      P2G_CUDA(cudaMemcpyAsync(c->ci.get(), ci + nz0, sizeof(int32_t) * c->nnz, cudaMemcpyHostToDevice, c->stream));
      P2G_CUDA(cudaMemcpyAsync(c->val.get(), val + nz0, sizeof(double) * c->nnz, cudaMemcpyHostToDevice, c->stream));
    }
    lap("h2d issued");
    if (dev_checks) {
      DBuf<unsigned long long> bad;
      bad.resize(2);
      DBuf<double> part;
      part.resize(kNormBlocks);
      P2G_CUDA(cudaMemsetAsync(bad.get(), 0xff, sizeof(unsigned long long) * 2, c->stream));
      const int g = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((NRt + 255) / 256, 148 * 8)));
      k_check_rowptr<<<g, 256, 0, c->stream>>>(c->rp.get(), NRt, bad.get());
      k_sumsq<<<kNormBlocks, 256, 0, c->stream>>>(c->val.get(), nnz_t, part.get());
      unsigned long long hb[2];
      std::vector<double> hp(kNormBlocks);
      P2G_CUDA(cudaMemcpyAsync(hb, bad.get(), sizeof(hb), cudaMemcpyDeviceToHost, c->stream));
      P2G_CUDA(cudaStreamSynchronize(c->stream));
      if (hb[0] != ~0ull) throw DataError("row_ptr must be non-decreasing");
      k_check_cols<<<g, 256, 0, c->stream>>>(c->rp.get(), c->ci.get(), NRt, J, bad.get() + 1);
      P2G_CUDA(cudaMemcpyAsync(hb + 1, bad.get() + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
      P2G_CUDA(cudaMemcpyAsync(hp.data(), part.get(), sizeof(double) * kNormBlocks, cudaMemcpyDeviceToHost, c->stream));
      P2G_CUDA(cudaStreamSynchronize(c->stream));
      if (hb[1] != ~0ull) {
        if ((hb[1] & 3ull) == 2ull) throw DataError("column index out of range");
        throw DataError("column indices must be strictly ascending within a row");
      }
      double acc = 0.0;
      for (double v : hp) acc += v;
      c->norm_x = acc;
    } else {
    // ||X||_F^2 (sparse.hpp:219-223): slice order then entry order over all
    // subjects; the full host tensor is available on every rank.
    // fixed chunks summed in order: deterministic for a given thread count
    {
      const int nt = host_threads(nnz_t);
      std::vector<double> part(static_cast<std::size_t>(nt), 0.0);
      run_host_parallel(nt, [&](int t) {
        double a = 0.0;
        for (int64_t p = nnz_t * t / nt; p < nnz_t * (t + 1) / nt; ++p) a += val[p] * val[p];
        part[static_cast<std::size_t>(t)] = a;
      });
      double acc = 0.0;
      for (double v : part) acc += v;
      c->norm_x = acc;
    }
    }
    lap("norm");
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    lap("h2d done");
    build_csc(c);
    lap("csc built");
    c->loaded = true;
    c->state_valid = false;
  });
}

/// Shard-local load: this rank's subjects only (arrays rebased to the shard).
/// The CSR is checked on the device with the same rules as p2g_load_csr;
/// the verdict (first failing check in rank order), the subject ranges and
/// ||X||^2 are agreed collectively, so every rank sees the same error.
extern "C" int p2g_load_shard(p2g_ctx* c, int64_t K, int64_t J, int64_t k_begin, int64_t k_end, const int64_t* srp,
                              const int64_t* rp, const int32_t* ci, const double* val) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    set_device(c);
    if (c->world > 1 && !c->nccl && !c->host_coll)
      throw InvalidArgument("world > 1 needs an NCCL unique id or a host collective");
    if (!srp || !rp) throw InvalidArgument("null CSR arrays");
    const int64_t Kl = k_end - k_begin;
    // ranges must tile [0, K) in rank order: gather every rank's (begin, end)
    std::vector<double> rng(static_cast<std::size_t>(2 * c->world), 0.0);
    rng[static_cast<std::size_t>(2 * c->rank)] = static_cast<double>(k_begin);
    rng[static_cast<std::size_t>(2 * c->rank + 1)] = static_cast<double>(k_end);
    allreduce_host(c, rng.data(), rng.size(), 0);
    double expect = 0.0;
    bool tiled = true;
    for (int r = 0; r < c->world; ++r) {
      tiled &= rng[static_cast<std::size_t>(2 * r)] == expect && rng[static_cast<std::size_t>(2 * r + 1)] > expect;
      expect = rng[static_cast<std::size_t>(2 * r + 1)];
    }
    if (J <= 0) throw DataError("tensor must have at least one column");
    if (K <= 0) throw DataError("tensor must have at least one slice");
    if (!tiled || expect != static_cast<double>(K))
      throw InvalidArgument("shard ranges must tile [0, K) in rank order with at least one subject per rank");
    // local structure checks (host, cheap): error code per rank, agreed below
    // 1 subj_row_ptr, 2 row_ptr start, then the device checks 3 row_ptr order,
    // 4 column range, 5 column order
    int code = 0;
    if (srp[0] != 0) code = 1;
    for (int64_t k = 0; k < Kl && !code; ++k)
      if (srp[k + 1] < srp[k]) code = 1;
    const int64_t NR = code ? 0 : srp[Kl];
    if (!code && rp[0] != 0) code = 2;
    sync_csc(c);
    c->loaded = false;
    c->K_total = K;
    c->J = J;
    c->k_begin = k_begin;
    c->k_end = k_end;
    c->NR = NR;
    c->srp_host.assign(srp, srp + (code ? 1 : Kl + 1));
    double norm_local = 0.0;
    if (!code) {
      const int64_t nnz = rp[NR];
      if (nnz < 0) code = 3;
      if (!code && nnz > 0 && (!ci || !val)) throw InvalidArgument("null CSR arrays");
      if (!code) {
        c->nnz = nnz;
        c->max_rows = 0;
        for (int64_t k = 0; k < Kl; ++k) c->max_rows = std::max<std::int64_t>(c->max_rows, srp[k + 1] - srp[k]);
        c->srp.resize(static_cast<std::size_t>(Kl + 1));
        c->rp.resize(static_cast<std::size_t>(NR + 1));
        c->ci.resize(static_cast<std::size_t>(std::max<int64_t>(nnz, 1)));
        c->val.resize(static_cast<std::size_t>(std::max<int64_t>(nnz, 1)));
        P2G_CUDA(cudaMemcpyAsync(c->srp.get(), srp, sizeof(int64_t) * (Kl + 1), cudaMemcpyHostToDevice, c->stream));
        P2G_CUDA(cudaMemcpyAsync(c->rp.get(), rp, sizeof(int64_t) * (NR + 1), cudaMemcpyHostToDevice, c->stream));
        if (nnz > 0) {
          P2G_CUDA(cudaMemcpyAsync(c->ci.get(), ci, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, c->stream));
          P2G_CUDA(cudaMemcpyAsync(c->val.get(), val, sizeof(double) * nnz, cudaMemcpyHostToDevice, c->stream));
        }
        DBuf<unsigned long long> bad;
        bad.resize(2);
        DBuf<double> part;
        part.resize(kNormBlocks);
        P2G_CUDA(cudaMemsetAsync(bad.get(), 0xff, sizeof(unsigned long long) * 2, c->stream));
        const int g = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((NR + 255) / 256, 148 * 8)));
        k_check_rowptr<<<g, 256, 0, c->stream>>>(c->rp.get(), NR, bad.get());
        k_sumsq<<<kNormBlocks, 256, 0, c->stream>>>(c->val.get(), nnz, part.get());
        P2G_LAUNCHED(2);
        unsigned long long hb[2];
        std::vector<double> hp(kNormBlocks);
        P2G_CUDA(cudaMemcpyAsync(hb, bad.get(), sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
        P2G_CUDA(cudaStreamSynchronize(c->stream));
        if (hb[0] != ~0ull) {
          code = 3;
        } else {
          k_check_cols<<<g, 256, 0, c->stream>>>(c->rp.get(), c->ci.get(), NR, J, bad.get() + 1);
          P2G_LAUNCHED(1);
          P2G_CUDA(cudaMemcpyAsync(hb + 1, bad.get() + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                   c->stream));
          P2G_CUDA(cudaMemcpyAsync(hp.data(), part.get(), sizeof(double) * kNormBlocks, cudaMemcpyDeviceToHost,
                                   c->stream));
          P2G_CUDA(cudaStreamSynchronize(c->stream));
          if (hb[1] != ~0ull) code = (hb[1] & 3ull) == 2ull ? 4 : 5;
          for (double v : hp) norm_local += v;
        }
      }
    }
    // agree: the lowest rank with an error decides (max of world - rank), then ||X||^2
    double v[2] = {code ? static_cast<double>(c->world - c->rank) : 0.0, 0.0};
    allreduce_host(c, v, 1, 1);
    const int bad_rank = v[0] > 0.0 ? c->world - static_cast<int>(v[0]) : -1;
    double cv[1] = {bad_rank == c->rank ? static_cast<double>(code) : 0.0};
    allreduce_host(c, cv, 1, 0);
    switch (static_cast<int>(cv[0])) {
      case 1: throw DataError("subj_row_ptr must start at 0 and be non-decreasing");
      case 2: throw DataError("row_ptr must start at 0");
      case 3: throw DataError("row_ptr must be non-decreasing");
      case 4: throw DataError("column index out of range");
      case 5: throw DataError("column indices must be strictly ascending within a row");
      default: break;
    }
    double nx[1] = {norm_local};
    allreduce_host(c, nx, 1, 0);
    c->norm_x = nx[0];
    double tot[1] = {static_cast<double>(c->nnz)};
    allreduce_host(c, tot, 1, 0);
    c->nnz_total = static_cast<std::int64_t>(tot[0]);
    build_csc(c);
    c->loaded = true;
    c->shard_local = true;
    c->state_valid = false;
  });
}

extern "C" int p2g_shard_info(const p2g_ctx* c, int64_t* k_begin, int64_t* k_end, int64_t* n_rows, int64_t* nnz) {
  return guarded([&] {
    require_loaded(c);
    if (k_begin) *k_begin = c->k_begin;
    if (k_end) *k_end = c->k_end;
    if (n_rows) *n_rows = c->NR;
    if (nnz) *nnz = c->nnz;
  });
}

// ---------------------------------------------------------------------------
// Fused loop
// ---------------------------------------------------------------------------
extern "C" int p2g_fit(p2g_ctx* c, const p2g_fit_config* cfg, const double* H0, const double* V0, const double* W0,
                       double* H_out, double* V_out, double* W_out, double* Q_out, int32_t* flags_out,
                       double* fit_trace, double* resid_trace, double* ms_trace, p2g_fit_summary* summary) {
  return guarded([&] {
    require_loaded(c);
    if (!cfg) throw InvalidArgument("null config");
    set_device(c);
    const auto t_start = std::chrono::steady_clock::now();
    validate_fit(c, cfg);
    if (!(c->norm_x > 0.0)) throw DataError("tensor has no non-zero entries");
    init_state(c, cfg, H0, V0, W0);
    if (c->opt.timing) {
      P2G_CUDA(cudaStreamSynchronize(c->stream));
      std::fprintf(stderr, "[p2g] fit init_state %8.2f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    }
    double prev_fit = 0.0;
    int iters = 0;
    bool converged = false;
    for (int it = 1; it <= cfg->max_iters; ++it) {
      const auto t0 = std::chrono::steady_clock::now();
      const IterOut o = iterate(c, cfg->nonneg != 0, it);
      ++iters;
      if (fit_trace) fit_trace[it - 1] = o.fit;
      if (resid_trace) resid_trace[it - 1] = o.resid;
      if (ms_trace)
        ms_trace[it - 1] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      const double change = std::abs(o.fit - prev_fit) / std::max(prev_fit, std::numeric_limits<double>::epsilon());
      prev_fit = o.fit;
      if (change < cfg->tol) {
        converged = true;
        break;
      }
    }
    const int R = cfg->rank;
    if (H_out) download_colmajor(c, c->H.get(), R, R, H_out);
    if (V_out) download_colmajor(c, c->V.get(), c->J, R, V_out);
    if (W_out) download_colmajor(c, c->W.get(), Ks(c), R, W_out);
    if (Q_out) {
      export_q(c, c->Hp.get(), c->Vp.get(), c->Wp.get());  // factors of the last Procrustes step
      P2G_CUDA(cudaMemcpyAsync(Q_out, c->Q.get(), sizeof(double) * c->NR * R, cudaMemcpyDeviceToHost, c->stream));
    }
    if (flags_out)
      P2G_CUDA(cudaMemcpyAsync(flags_out, c->flags.get(), sizeof(int32_t) * Ks(c), cudaMemcpyDeviceToHost, c->stream));
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    if (c->opt.timing)
      std::fprintf(stderr, "[p2g] fit total      %8.2f ms (%d iterations)\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(), iters);
    if (summary) {
      summary->iterations = iters;
      summary->converged = converged ? 1 : 0;
      summary->norm_x = c->norm_x;
      summary->total_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    }
  });
}

extern "C" int p2g_initialize_eye(p2g_ctx* c, int32_t R, double* V_out) {
  return guarded([&] {
    require_loaded(c);
    set_device(c);
    if (!V_out) throw InvalidArgument("null output");
    p2g_fit_config cfg{R, 1, 1.0, 1, 1, 0};
    validate_fit(c, &cfg);
    DBuf<double> C, V;
    C.resize(static_cast<std::size_t>(c->J) * static_cast<std::size_t>(c->J));
    V.resize(static_cast<std::size_t>(c->J) * R);
    build_column_gram(c, C.get());
    allreduce(c, C.get(), static_cast<std::size_t>(c->J) * static_cast<std::size_t>(c->J));
    eye_vectors(c, C.get(), R, V.get());
    download_colmajor(c, V.get(), c->J, R, V_out);
  });
}

extern "C" int p2g_fit_phase_ms(const p2g_ctx* c, int32_t max_iters, double* out, int32_t* n_out) {
  return guarded([&] {
    if (!c || !out || !n_out) throw InvalidArgument("null argument");
    const int n = static_cast<int>(std::min<std::size_t>(static_cast<std::size_t>(std::max(max_iters, 0)),
                                                         c->fit_phase_ms.size() / 3));
    std::memcpy(out, c->fit_phase_ms.data(), sizeof(double) * 3 * static_cast<std::size_t>(n));
    *n_out = n;
  });
}

extern "C" int p2g_fit_dumps(p2g_ctx* c, const p2g_fit_config* cfg, const double* H0, const double* V0,
                             const double* W0, double* m1, double* m2, double* m3, double* H, double* V, double* W,
                             double* fit_trace, int32_t* n_iters) {
  return guarded([&] {
    require_loaded(c);
    if (!cfg) throw InvalidArgument("null config");
    set_device(c);
    validate_fit(c, cfg);
    if (!(c->norm_x > 0.0)) throw DataError("tensor has no non-zero entries");
    init_state(c, cfg, H0, V0, W0);
    const int R = cfg->rank;
    const std::size_t RR = static_cast<std::size_t>(R) * R, JR = static_cast<std::size_t>(c->J) * R,
                      KR = static_cast<std::size_t>(Ks(c)) * R;
    double prev_fit = 0.0;
    int iters = 0;
    for (int it = 1; it <= cfg->max_iters; ++it) {
      const IterOut o = iterate(c, cfg->nonneg != 0, it);
      const std::size_t t = static_cast<std::size_t>(it - 1);
      // the loop kernels' own outputs of iteration `it` (cp.hpp:108,116,127 and the updated factors)
      if (m1) download_colmajor(c, c->m1.get(), R, R, m1 + t * RR);
      if (m2) download_colmajor(c, c->M2.get(), c->J, R, m2 + t * JR);
      if (m3) download_colmajor(c, c->m3.get(), Ks(c), R, m3 + t * KR);
      if (H) download_colmajor(c, c->H.get(), R, R, H + t * RR);
      if (V) download_colmajor(c, c->V.get(), c->J, R, V + t * JR);
      if (W) download_colmajor(c, c->W.get(), Ks(c), R, W + t * KR);
      if (fit_trace) fit_trace[t] = o.fit;
      ++iters;
      const double change = std::abs(o.fit - prev_fit) / std::max(prev_fit, std::numeric_limits<double>::epsilon());
      prev_fit = o.fit;
      if (change < cfg->tol) break;
    }
    if (n_iters) *n_iters = iters;
  });
}

extern "C" int p2g_bench_iterations(p2g_ctx* c, const p2g_fit_config* cfg, const double* H0, const double* V0,
                                    const double* W0, int32_t reset, int32_t iters, double* ms_per_iter,
                                    double* fit_trace) {
  return guarded([&] {
    require_loaded(c);
    if (!cfg) throw InvalidArgument("null config");
    set_device(c);
    if (reset || !c->state_valid || c->R != cfg->rank) {
      validate_fit(c, cfg);
      if (!(c->norm_x > 0.0)) throw DataError("tensor has no non-zero entries");
      init_state(c, cfg, H0, V0, W0);
    }
    c->timer.acc.clear();  // per-call kernel times (the timed steps only)
    c->timing = true;
    cudaEvent_t e0, e1;
    P2G_CUDA(cudaEventCreate(&e0));
    P2G_CUDA(cudaEventCreate(&e1));
    try {
      for (int it = 0; it < iters; ++it) {
        P2G_CUDA(cudaEventRecord(e0, c->stream));
        const IterOut o = iterate(c, cfg->nonneg != 0, it + 1);
        P2G_CUDA(cudaEventRecord(e1, c->stream));
        P2G_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        P2G_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        double msd = ms;
        allreduce_host(c, &msd, 1, 1);  // max over ranks
        if (ms_per_iter) ms_per_iter[it] = msd;
        if (fit_trace) fit_trace[it] = o.fit;
      }
    } catch (...) {
      c->timing = false;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      throw;
    }
    c->timing = false;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

extern "C" int64_t p2g_launch_count(void) { return launch_counter().load(); }

extern "C" int p2g_kernel_times(const p2g_ctx* c, int32_t max_entries, char* names, double* ms_per_launch,
                                int64_t* launches, int32_t* n_out) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    int n = 0;
    for (const auto& kv : c->timer.acc) {
      if (n >= max_entries) break;
      std::memset(names + 32 * n, 0, 32);
      std::strncpy(names + 32 * n, kv.first.c_str(), 31);
      ms_per_launch[n] = kv.second.second ? kv.second.first / kv.second.second : 0.0;
      launches[n] = kv.second.second;
      ++n;
    }
    *n_out = n;
  });
}

// ---------------------------------------------------------------------------
// Per-step hooks
// ---------------------------------------------------------------------------
extern "C" int p2g_procrustes(p2g_ctx* c, int32_t R, const double* H, const double* V, const double* W,
                              double* Q_out, int32_t* flags_out, double* m1_out) {
  return guarded([&] {
    require_loaded(c);
    set_device(c);
    if (R < 1 || R > 40) throw InvalidArgument("rank out of range");
    if (!H || !V || !W) throw InvalidArgument("null factor");
    if (first_short_subject(c, R).first >= 0) throw InvalidArgument("rank exceeds observations in procrustes step");
    alloc_state(c, R);
    upload_colmajor(c, H, R, R, c->H.get());
    upload_colmajor(c, V, c->J, R, c->V.get());
    upload_shard_rows(c, W, c->K_total, R, c->W.get());
    c->c_valid = false;
  c->xv_valid = false;
    c->ew_valid = false;  // cold Jacobi start for a teacher-forced step
    const std::size_t RR = static_cast<std::size_t>(R) * R;
    P2G_CUDA(cudaMemsetAsync(c->counters.get(), 0, sizeof(std::int32_t) * 32, c->stream));
    DBuf<double>& part = scratch_partials(c, procrustes_partials(c) * RR);
    const int np = procrustes_step(c, part.get());
    reduce_partials(part.get(), np, static_cast<std::int64_t>(RR), c->m1.get(), c->stream);
    allreduce(c, c->m1.get(), RR);
    std::int32_t cnt[8];
    P2G_CUDA(cudaMemcpyAsync(cnt, c->counters.get(), sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    if (cnt[2] > 0) throw NumericalError("svd operand: non-finite entries");
    if (Q_out) {
      export_q(c, c->H.get(), c->V.get(), c->W.get());
      P2G_CUDA(cudaMemcpyAsync(Q_out, c->Q.get(), sizeof(double) * c->NR * R, cudaMemcpyDeviceToHost, c->stream));
      P2G_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (flags_out) P2G_CUDA(cudaMemcpy(flags_out, c->flags.get(), sizeof(int32_t) * Ks(c), cudaMemcpyDeviceToHost));
    if (m1_out) download_colmajor(c, c->m1.get(), R, R, m1_out);
    c->state_valid = false;
  });
}

extern "C" int p2g_mttkrp_q(p2g_ctx* c, int32_t mode, int32_t R, const double* Q, const double* H, const double* V,
                            const double* W, double* out) {
  return guarded([&] {
    require_loaded(c);
    set_device(c);
    if (mode < 1 || mode > 3) throw InvalidArgument("mttkrp: mode must be 1, 2 or 3");
    if (R < 1 || R > 40) throw InvalidArgument("rank out of range");
    if (!Q || !H || !V || !W || !out) throw InvalidArgument("null argument");
    alloc_state(c, R);
    P2G_CUDA(cudaMemcpyAsync(c->Q.get(), Q, sizeof(double) * c->NR * R, cudaMemcpyHostToDevice, c->stream));
    upload_colmajor(c, H, R, R, c->H.get());
    upload_colmajor(c, V, c->J, R, c->V.get());
    upload_shard_rows(c, W, c->K_total, R, c->W.get());
    c->c_valid = false;
  c->xv_valid = false;
    const std::size_t RR = static_cast<std::size_t>(R) * R;
    if (mode == 1) {
      const int nb = 2 * c->num_sms;
      DBuf<double>& part = scratch_partials(c, static_cast<std::size_t>(nb) * RR);
      launch_mode1_q(c, R, c->Q.get(), c->V.get(), c->W.get(), part.get(), nb, c->stream);
      reduce_partials(part.get(), nb, static_cast<std::int64_t>(RR), c->m1.get(), c->stream);
      allreduce(c, c->m1.get(), RR);
      download_colmajor(c, c->m1.get(), R, R, out);
    } else if (mode == 2) {
      launch_mode2(c, R, c->Q.get(), c->H.get(), c->W.get(), nullptr, c->M2.get(), c->stream);
      allreduce(c, c->M2.get(), static_cast<std::size_t>(c->J) * R);
      download_colmajor(c, c->M2.get(), c->J, R, out);
    } else {
      launch_mode3(c, R, c->Q.get(), c->H.get(), c->V.get(), c->m3.get(), c->stream);
      download_colmajor(c, c->m3.get(), Ks(c), R, out);
    }
    c->state_valid = false;
  });
}

namespace {
/// Distinct sorted columns per shard subject (nnz_cols of each slice,
/// sparse.hpp:96-98), from the device CSR.
void shard_cols(p2g_ctx* c, std::vector<std::int64_t>& ptr, std::vector<std::int32_t>& cols) {
  std::vector<std::int64_t> srp(static_cast<std::size_t>(Ks(c) + 1)), rp(static_cast<std::size_t>(c->NR + 1));
  std::vector<std::int32_t> ci(static_cast<std::size_t>(c->nnz));
  P2G_CUDA(cudaMemcpy(srp.data(), c->srp.get(), sizeof(std::int64_t) * srp.size(), cudaMemcpyDeviceToHost));
  P2G_CUDA(cudaMemcpy(rp.data(), c->rp.get(), sizeof(std::int64_t) * rp.size(), cudaMemcpyDeviceToHost));
  if (c->nnz) P2G_CUDA(cudaMemcpy(ci.data(), c->ci.get(), sizeof(std::int32_t) * ci.size(), cudaMemcpyDeviceToHost));
  ptr.assign(static_cast<std::size_t>(Ks(c) + 1), 0);
  cols.clear();
  std::vector<std::int32_t> tmp;
  for (std::int64_t k = 0; k < Ks(c); ++k) {
    tmp.assign(ci.begin() + rp[static_cast<std::size_t>(srp[static_cast<std::size_t>(k)])],
               ci.begin() + rp[static_cast<std::size_t>(srp[static_cast<std::size_t>(k + 1)])]);
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    cols.insert(cols.end(), tmp.begin(), tmp.end());
    ptr[static_cast<std::size_t>(k + 1)] = static_cast<std::int64_t>(cols.size());
  }
}
}  // namespace

extern "C" int p2g_project(p2g_ctx* c, int32_t R, const double* Q, int64_t* ycol_ptr, int32_t* ycols, double* Y_out) {
  return guarded([&] {
    require_loaded(c);
    set_device(c);
    if (R < 1 || R > 40) throw InvalidArgument("rank out of range");
    std::vector<std::int64_t> ptr;
    std::vector<std::int32_t> cols;
    shard_cols(c, ptr, cols);
    if (ycol_ptr) std::memcpy(ycol_ptr, ptr.data(), sizeof(int64_t) * ptr.size());
    if (!Y_out) return;
    if (!Q || !ycols) throw InvalidArgument("null argument");
    std::memcpy(ycols, cols.data(), sizeof(int32_t) * cols.size());
    alloc_state(c, R);
    DBuf<std::int64_t> dptr;
    DBuf<std::int32_t> dcols;
    DBuf<double> dY;
    dptr.resize(ptr.size());
    dcols.resize(std::max<std::size_t>(cols.size(), 1));
    dY.resize(std::max<std::size_t>(cols.size() * R, 1));
    P2G_CUDA(cudaMemcpyAsync(c->Q.get(), Q, sizeof(double) * c->NR * R, cudaMemcpyHostToDevice, c->stream));
    P2G_CUDA(cudaMemcpyAsync(dptr.get(), ptr.data(), sizeof(std::int64_t) * ptr.size(), cudaMemcpyHostToDevice, c->stream));
    if (!cols.empty())
      P2G_CUDA(cudaMemcpyAsync(dcols.get(), cols.data(), sizeof(std::int32_t) * cols.size(), cudaMemcpyHostToDevice, c->stream));
    launch_project(c, R, c->Q.get(), dptr.get(), dcols.get(), dY.get(), c->stream);
    if (!cols.empty())
      P2G_CUDA(cudaMemcpyAsync(Y_out, dY.get(), sizeof(double) * cols.size() * R, cudaMemcpyDeviceToHost, c->stream));
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    c->state_valid = false;
  });
}

namespace {

struct PackedDev {
  DBuf<std::int64_t> ptr, occ_ptr, occ;
  DBuf<std::int32_t> cols;
  DBuf<double> Y, H, V, W, out, part;
};

/// Shape checks of check_mttkrp_input / ProjectedSlices::from_packed
/// (mttkrp.hpp:170-181, slices.hpp:43-67) and upload.
void upload_packed(p2g_ctx* c, std::int64_t K, std::int64_t J, int R, const int64_t* ycol_ptr, const int32_t* ycols,
                   const double* Y, PackedDev& d) {
  if (R <= 0) throw InvalidArgument("slice rank must be positive");
  if (R > 40) throw InvalidArgument("rank above 40 unsupported on device");
  if (K < 0 || J < 0 || !ycol_ptr) throw InvalidArgument("bad packed slices");
  if (ycol_ptr[0] != 0) throw InvalidArgument("ycol_ptr must start at 0");
  for (std::int64_t k = 0; k < K; ++k) {
    if (ycol_ptr[k + 1] < ycol_ptr[k]) throw InvalidArgument("packed block width differs from column list");
    for (std::int64_t t = ycol_ptr[k]; t < ycol_ptr[k + 1]; ++t) {
      if (ycols[t] < 0 || ycols[t] >= J) throw InvalidArgument("packed column index out of range");
      if (t > ycol_ptr[k] && ycols[t] <= ycols[t - 1]) throw InvalidArgument("packed column indices must be ascending");
    }
  }
  const std::int64_t nc = ycol_ptr[K];
  d.ptr.resize(static_cast<std::size_t>(K + 1));
  d.cols.resize(static_cast<std::size_t>(std::max<std::int64_t>(nc, 1)));
  d.Y.resize(static_cast<std::size_t>(std::max<std::int64_t>(nc * R, 1)));
  P2G_CUDA(cudaMemcpyAsync(d.ptr.get(), ycol_ptr, sizeof(int64_t) * (K + 1), cudaMemcpyHostToDevice, c->stream));
  if (nc > 0) {
    P2G_CUDA(cudaMemcpyAsync(d.cols.get(), ycols, sizeof(int32_t) * nc, cudaMemcpyHostToDevice, c->stream));
    P2G_CUDA(cudaMemcpyAsync(d.Y.get(), Y, sizeof(double) * nc * R, cudaMemcpyHostToDevice, c->stream));
  }
  // per-column occurrence lists for the deterministic mode-2 kernel
  std::vector<std::int64_t> cnt(static_cast<std::size_t>(J + 1), 0);
  for (std::int64_t t = 0; t < nc; ++t) cnt[static_cast<std::size_t>(ycols[t]) + 1]++;
  for (std::int64_t j = 0; j < J; ++j) cnt[static_cast<std::size_t>(j + 1)] += cnt[static_cast<std::size_t>(j)];
  std::vector<std::int64_t> occ(static_cast<std::size_t>(2 * std::max<std::int64_t>(nc, 1)));
  std::vector<std::int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (std::int64_t k = 0; k < K; ++k)
    for (std::int64_t t = ycol_ptr[k]; t < ycol_ptr[k + 1]; ++t) {
      const std::int64_t pos = fill[static_cast<std::size_t>(ycols[t])]++;
      occ[static_cast<std::size_t>(2 * pos)] = t;
      occ[static_cast<std::size_t>(2 * pos + 1)] = k;
    }
  d.occ_ptr.resize(cnt.size());
  d.occ.resize(occ.size());
  P2G_CUDA(cudaMemcpyAsync(d.occ_ptr.get(), cnt.data(), sizeof(std::int64_t) * cnt.size(), cudaMemcpyHostToDevice, c->stream));
  P2G_CUDA(cudaMemcpyAsync(d.occ.get(), occ.data(), sizeof(std::int64_t) * occ.size(), cudaMemcpyHostToDevice, c->stream));
  P2G_CUDA(cudaStreamSynchronize(c->stream));  // host vectors go out of scope
}

void packed_mode(p2g_ctx* c, int mode, std::int64_t K, std::int64_t J, int R, PackedDev& d, const double* dH,
                 const double* dV, const double* dW, double* dout) {
  const std::size_t RR = static_cast<std::size_t>(R) * R;
  if (mode == 1) {
    const int nb = packed_mode1_blocks(c->num_sms);
    d.part.resize(static_cast<std::size_t>(nb) * RR);
    launch_packed_mode13(1, K, J, R, d.ptr.get(), d.cols.get(), d.Y.get(), dH, dV, dW, d.part.get(), nb, c->stream);
    reduce_partials(d.part.get(), nb, static_cast<std::int64_t>(RR), dout, c->stream);
  } else if (mode == 2) {
    launch_packed_mode2(K, J, R, d.ptr.get(), d.cols.get(), d.Y.get(), dH, dW, d.occ_ptr.get(), d.occ.get(), dout,
                        c->stream);
  } else {
    const int nb = packed_mode1_blocks(c->num_sms);
    launch_packed_mode13(3, K, J, R, d.ptr.get(), d.cols.get(), d.Y.get(), dH, dV, dW, dout, nb, c->stream);
  }
}

}  // namespace

extern "C" int p2g_mttkrp_packed(p2g_ctx* c, int32_t mode, int64_t K, int64_t J, int32_t R, const int64_t* ycol_ptr,
                                 const int32_t* ycols, const double* Y, const double* H, const double* V,
                                 const double* W, double* out) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    set_device(c);
    if (mode < 1 || mode > 3) throw InvalidArgument("mttkrp: mode must be 1, 2 or 3");
    if (!H || !V || !W || !out) throw InvalidArgument("null factor");
    PackedDev d;
    upload_packed(c, K, J, R, ycol_ptr, ycols, Y, d);
    d.H.resize(static_cast<std::size_t>(R) * R);
    d.V.resize(static_cast<std::size_t>(std::max<std::int64_t>(J, 1)) * R);
    d.W.resize(static_cast<std::size_t>(std::max<std::int64_t>(K, 1)) * R);
    upload_colmajor(c, H, R, R, d.H.get());
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    upload_colmajor(c, V, J, R, d.V.get());
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    upload_colmajor(c, W, K, R, d.W.get());
    const std::int64_t rows = mode == 1 ? R : (mode == 2 ? J : K);
    d.out.resize(static_cast<std::size_t>(std::max<std::int64_t>(rows, 1)) * R);
    packed_mode(c, mode, K, J, R, d, d.H.get(), d.V.get(), d.W.get(), d.out.get());
    download_colmajor(c, d.out.get(), rows, R, out);
  });
}

extern "C" int p2g_naive_mttkrp(p2g_ctx* c, int32_t mode, int64_t K, int64_t J, int32_t R, const int64_t* ycol_ptr,
                                const int32_t* ycols, const double* Y, const double* H, const double* V,
                                const double* W, double* out) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    set_device(c);
    if (mode < 1 || mode > 3) throw InvalidArgument("mttkrp: mode must be 1, 2 or 3");
    if (!H || !V || !W || !out) throw InvalidArgument("null factor");
    PackedDev d;
    upload_packed(c, K, J, R, ycol_ptr, ycols, Y, d);
    check_finite_host(W, K * R, "khatri_rao left operand");  // kernels.hpp:37-38
    check_finite_host(mode == 3 ? V : (mode == 1 ? V : H), (mode == 2 ? R : J) * static_cast<int64_t>(R),
                      "khatri_rao right operand");
    d.H.resize(static_cast<std::size_t>(R) * R);
    d.V.resize(static_cast<std::size_t>(std::max<std::int64_t>(J, 1)) * R);
    d.W.resize(static_cast<std::size_t>(std::max<std::int64_t>(K, 1)) * R);
    upload_colmajor(c, H, R, R, d.H.get());
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    upload_colmajor(c, V, J, R, d.V.get());
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    upload_colmajor(c, W, K, R, d.W.get());
    const std::int64_t rows = mode == 1 ? R : (mode == 2 ? J : K);
    d.out.resize(static_cast<std::size_t>(std::max<std::int64_t>(rows, 1)) * R);
    NaiveScratch s;
    s.prepare(c, mode, K, J, R, d.ptr.get(), ycol_ptr[K]);
    naive_mttkrp(c, s, mode, K, J, R, d.ptr.get(), d.cols.get(), d.Y.get(), ycol_ptr[K], d.H.get(), d.V.get(),
                 d.W.get(), d.out.get());
    P2G_CUDA(cudaMemcpyAsync(out, d.out.get(), sizeof(double) * rows * R, cudaMemcpyDeviceToHost, c->stream));
    P2G_CUDA(cudaStreamSynchronize(c->stream));
  });
}

extern "C" uint64_t p2g_naive_mttkrp_bytes(int64_t K, int64_t J, int64_t R, int32_t mode) {
  try {
    return naive_bytes(K, J, R, mode);
  } catch (...) {
    return 0;
  }
}

namespace {
/// generator.hpp:36-47: Householder QR of a seeded Gaussian rows x cols
/// matrix (filled column-major from the stream), Q sign-fixed so diag(R) >= 0.
/// Output row-major into q (rows x cols).
void random_orthonormal(Rng& rng, std::int64_t rows, int cols, double* q) {
  std::vector<double> A(static_cast<std::size_t>(rows * cols));  // column-major
  for (int c = 0; c < cols; ++c)
    for (std::int64_t r = 0; r < rows; ++r) A[static_cast<std::size_t>(c * rows + r)] = rng.normal();
  std::vector<double> tau(static_cast<std::size_t>(cols)), rdiag(static_cast<std::size_t>(cols));
  for (int c = 0; c < cols; ++c) {
    double* a = A.data() + static_cast<std::size_t>(c) * rows;
    double sig = 0.0;
    for (std::int64_t r = c + 1; r < rows; ++r) sig += a[r] * a[r];
    const double alpha = a[c];
    double beta = alpha, t = 0.0;
    if (sig != 0.0) {
      beta = -std::copysign(std::sqrt(alpha * alpha + sig), alpha);
      t = (beta - alpha) / beta;
      const double inv = 1.0 / (alpha - beta);
      for (std::int64_t r = c + 1; r < rows; ++r) a[r] *= inv;  // v = (1, a[c+1..])
      for (int j = c + 1; j < cols; ++j) {
        double* b = A.data() + static_cast<std::size_t>(j) * rows;
        double dot = b[c];
        for (std::int64_t r = c + 1; r < rows; ++r) dot += a[r] * b[r];
        dot *= t;
        b[c] -= dot;
        for (std::int64_t r = c + 1; r < rows; ++r) b[r] -= dot * a[r];
      }
    }
    tau[static_cast<std::size_t>(c)] = t;
    rdiag[static_cast<std::size_t>(c)] = beta;
  }
  // Q = H_0 H_1 ... H_{cols-1} I(rows, cols), applied right to left
  std::vector<double> Q(static_cast<std::size_t>(rows * cols), 0.0);
  for (int c = 0; c < cols; ++c) Q[static_cast<std::size_t>(c) * rows + c] = 1.0;
  for (int c = cols - 1; c >= 0; --c) {
    const double* a = A.data() + static_cast<std::size_t>(c) * rows;
    const double t = tau[static_cast<std::size_t>(c)];
    if (t == 0.0) continue;
    for (int j = 0; j < cols; ++j) {
      double* qj = Q.data() + static_cast<std::size_t>(j) * rows;
      double dot = qj[c];
      for (std::int64_t r = c + 1; r < rows; ++r) dot += a[r] * qj[r];
      dot *= t;
      qj[c] -= dot;
      for (std::int64_t r = c + 1; r < rows; ++r) qj[r] -= dot * a[r];
    }
  }
  for (int c = 0; c < cols; ++c) {
    const double sg = rdiag[static_cast<std::size_t>(c)] < 0.0 ? -1.0 : 1.0;
    for (std::int64_t r = 0; r < rows; ++r)
      q[r * cols + c] = sg * Q[static_cast<std::size_t>(c) * rows + r];
  }
}

double median(std::vector<double> v) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const std::size_t n = v.size();
  return n % 2 == 1 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

double device_sum(p2g_ctx* c, const double* d, std::int64_t n) {
  std::vector<double> h(static_cast<std::size_t>(n));
  P2G_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  P2G_CUDA(cudaStreamSynchronize(c->stream));
  double s = 0.0;
  for (double x : h) s += x;
  return s;
}
}  // namespace

/// bench_mttkrp (bench.hpp:90-215) on the device over the loaded tensor.
extern "C" int p2g_bench_mttkrp(p2g_ctx* c, int32_t R, int32_t reps, uint64_t budget_bytes, uint64_t seed,
                                p2g_bench_report* rep) {
  return guarded([&] {
    require_loaded(c);
    set_device(c);
    if (!rep) throw InvalidArgument("null report");
    if (R < 1) throw InvalidArgument("bench: rank must be at least 1");
    if (R > 40) throw InvalidArgument("rank above 40 unsupported on device");
    if (reps < 1) throw InvalidArgument("bench: reps must be at least 1");
    const std::int64_t K = Ks(c), J = c->J;
    *rep = p2g_bench_report{};
    rep->K = K;
    rep->J = J;
    rep->R = R;
    rep->nnz = c->nnz;
    rep->reps = reps;
    if (budget_bytes == 0) {  // all free device memory minus a margin
      std::size_t fr = 0, tot = 0;
      P2G_CUDA(cudaMemGetInfo(&fr, &tot));
      budget_bytes = fr > (2ull << 30) ? fr - (2ull << 30) : fr / 2;
    }
    rep->budget_bytes = budget_bytes;
    // factors: one master stream, H, V, W uniform [0,1) column-major (bench.hpp:111-114)
    Rng master(seed);
    std::vector<double> H(static_cast<std::size_t>(R) * R), V(static_cast<std::size_t>(J) * R),
        W(static_cast<std::size_t>(K) * R);
    for (auto* m : {&H, &V, &W}) {
      const std::int64_t rows = static_cast<std::int64_t>(m->size()) / R;
      for (int cc = 0; cc < R; ++cc)
        for (std::int64_t r = 0; r < rows; ++r) (*m)[static_cast<std::size_t>(cc * rows + r)] = master.uniform(0.0, 1.0);
    }
    // Y_k = Q_k^T X_k with seeded random orthonormal Q_k (bench.hpp:115-129), projected on the device
    std::vector<double> Qh(static_cast<std::size_t>(c->NR) * R);
    {
      const int nt = static_cast<int>(std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
      std::vector<std::thread> th;
      std::vector<int> bad(static_cast<std::size_t>(nt), -1);
      auto work = [&](int t) {
        for (std::int64_t k = K * t / nt; k < K * (t + 1) / nt; ++k) {
          const std::int64_t I = c->srp_host[static_cast<std::size_t>(k + 1)] - c->srp_host[static_cast<std::size_t>(k)];
          if (I < R) {
            if (bad[static_cast<std::size_t>(t)] < 0) bad[static_cast<std::size_t>(t)] = static_cast<int>(k);
            continue;
          }
          Rng rk(substream_seed(seed, static_cast<std::uint64_t>(c->k_begin + k) + 1));
          random_orthonormal(rk, I, R, Qh.data() + (c->srp_host[static_cast<std::size_t>(k)] - c->srp_host[0]) * R);
        }
      };
      for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
      work(0);
      for (auto& x : th) x.join();
      for (int b : bad)
        if (b >= 0) throw DataError("rank exceeds observations for subject " + std::to_string(b));
    }
    std::vector<std::int64_t> ptr;
    std::vector<std::int32_t> cols;
    shard_cols(c, ptr, cols);
    const std::int64_t nc = ptr.back();
    PackedDev d;
    {
      // device Y + the per-column occurrence lists of the packed mode-2 kernel
      d.ptr.resize(ptr.size());
      d.cols.resize(std::max<std::size_t>(cols.size(), 1));
      d.Y.resize(std::max<std::size_t>(static_cast<std::size_t>(nc) * R, 1));
      P2G_CUDA(cudaMemcpyAsync(d.ptr.get(), ptr.data(), sizeof(std::int64_t) * ptr.size(), cudaMemcpyHostToDevice, c->stream));
      if (nc)
        P2G_CUDA(cudaMemcpyAsync(d.cols.get(), cols.data(), sizeof(std::int32_t) * nc, cudaMemcpyHostToDevice, c->stream));
      std::vector<std::int64_t> cnt(static_cast<std::size_t>(J + 1), 0);
      for (std::int64_t t = 0; t < nc; ++t) cnt[static_cast<std::size_t>(cols[static_cast<std::size_t>(t)]) + 1]++;
      for (std::int64_t j = 0; j < J; ++j) cnt[static_cast<std::size_t>(j + 1)] += cnt[static_cast<std::size_t>(j)];
      std::vector<std::int64_t> occ(static_cast<std::size_t>(2 * std::max<std::int64_t>(nc, 1)));
      std::vector<std::int64_t> fill(cnt.begin(), cnt.end() - 1);
      for (std::int64_t k = 0; k < K; ++k)
        for (std::int64_t t = ptr[static_cast<std::size_t>(k)]; t < ptr[static_cast<std::size_t>(k + 1)]; ++t) {
          const std::int64_t pos = fill[static_cast<std::size_t>(cols[static_cast<std::size_t>(t)])]++;
          occ[static_cast<std::size_t>(2 * pos)] = t;
          occ[static_cast<std::size_t>(2 * pos + 1)] = k;
        }
      d.occ_ptr.resize(cnt.size());
      d.occ.resize(occ.size());
      P2G_CUDA(cudaMemcpyAsync(d.occ_ptr.get(), cnt.data(), sizeof(std::int64_t) * cnt.size(), cudaMemcpyHostToDevice, c->stream));
      P2G_CUDA(cudaMemcpyAsync(d.occ.get(), occ.data(), sizeof(std::int64_t) * occ.size(), cudaMemcpyHostToDevice, c->stream));
      alloc_state(c, R);
      P2G_CUDA(cudaMemcpyAsync(c->Q.get(), Qh.data(), sizeof(double) * c->NR * R, cudaMemcpyHostToDevice, c->stream));
      launch_project(c, R, c->Q.get(), d.ptr.get(), d.cols.get(), d.Y.get(), c->stream);
      d.H.resize(static_cast<std::size_t>(R) * R);
      d.V.resize(static_cast<std::size_t>(std::max<std::int64_t>(J, 1)) * R);
      d.W.resize(static_cast<std::size_t>(std::max<std::int64_t>(K, 1)) * R);
      upload_colmajor(c, H.data(), R, R, d.H.get());
      P2G_CUDA(cudaStreamSynchronize(c->stream));
      upload_colmajor(c, V.data(), J, R, d.V.get());
      P2G_CUDA(cudaStreamSynchronize(c->stream));
      upload_colmajor(c, W.data(), K, R, d.W.get());
      P2G_CUDA(cudaStreamSynchronize(c->stream));
    }
    const std::int64_t rows_of[3] = {R, J, K};
    rep->specialized_device_bytes = static_cast<std::uint64_t>(
        sizeof(double) * (static_cast<std::size_t>(nc) * R + static_cast<std::size_t>(R + J + K) * R +
                          static_cast<std::size_t>(std::max<std::int64_t>(J, K)) * R) +
        sizeof(std::int64_t) * (ptr.size() + 2 * static_cast<std::size_t>(nc) + static_cast<std::size_t>(J + 1)) +
        sizeof(std::int32_t) * static_cast<std::size_t>(nc));
    cudaEvent_t e0, e1;
    P2G_CUDA(cudaEventCreate(&e0));
    P2G_CUDA(cudaEventCreate(&e1));
    auto timed = [&](auto&& fn) {
      P2G_CUDA(cudaEventRecord(e0, c->stream));
      fn();
      P2G_CUDA(cudaEventRecord(e1, c->stream));
      P2G_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      P2G_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      return static_cast<double>(ms);
    };
    DBuf<double> out;
    out.resize(static_cast<std::size_t>(std::max<std::int64_t>({R, J, K})) * R);
    // specialized sweep (one warm-up sweep first: first-launch costs are not the kernels')
    std::vector<std::vector<double>> sm(3);
    std::vector<double> sweep;
    for (int r = -1; r < reps; ++r) {
      double sw = 0.0;
      for (int mode = 1; mode <= 3; ++mode) {
        const double ms = timed([&] { packed_mode(c, mode, K, J, R, d, d.H.get(), d.V.get(), d.W.get(), out.get()); });
        if (r >= 0) {
          sm[static_cast<std::size_t>(mode - 1)].push_back(ms);
          rep->checksum_specialized += device_sum(c, out.get(), rows_of[mode - 1] * R);
        }
        sw += ms;
      }
      if (r >= 0) sweep.push_back(sw);
    }
    for (int m = 0; m < 3; ++m) rep->specialized_ms[m] = median(sm[static_cast<std::size_t>(m)]);
    rep->specialized_sweep_ms = median(sweep);
    // naive, budget-gated per mode (the materialisation bytes, mttkrp.hpp:241-253)
    bool all = true;
    std::vector<std::vector<double>> nm(3);
    for (int mode = 1; mode <= 3; ++mode) {
      rep->naive_bytes[mode - 1] = naive_bytes(K, J, R, mode);
      if (rep->naive_bytes[mode - 1] > budget_bytes) {
        rep->naive_oom[mode - 1] = 1;
        rep->naive_ms[mode - 1] = -1.0;
        all = false;
        continue;
      }
      NaiveScratch s;
      s.prepare(c, mode, K, J, R, d.ptr.get(), nc);
      for (int r = -1; r < reps; ++r) {
        const double ms = timed([&] {
          naive_mttkrp(c, s, mode, K, J, R, d.ptr.get(), d.cols.get(), d.Y.get(), nc, d.H.get(), d.V.get(), d.W.get(),
                       out.get());
        });
        if (r >= 0) {
          nm[static_cast<std::size_t>(mode - 1)].push_back(ms);
          // cuBLAS writes column-major: the same entries, so the same sum up to order
          rep->checksum_naive += device_sum(c, out.get(), rows_of[mode - 1] * R);
        }
      }
      rep->naive_ms[mode - 1] = median(nm[static_cast<std::size_t>(mode - 1)]);
    }
    if (all) {
      std::vector<double> ns;
      for (int r = 0; r < reps; ++r)
        ns.push_back(nm[0][static_cast<std::size_t>(r)] + nm[1][static_cast<std::size_t>(r)] +
                     nm[2][static_cast<std::size_t>(r)]);
      rep->naive_sweep_ms = median(ns);
      rep->speedup = rep->naive_sweep_ms / rep->specialized_sweep_ms;
    } else {
      rep->naive_sweep_oom = 1;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->state_valid = false;
  });
}

extern "C" int p2g_cp_als_iteration(p2g_ctx* c, int64_t K, int64_t J, int32_t R, const int64_t* ycol_ptr,
                                    const int32_t* ycols, const double* Y, double* H, double* V, double* W,
                                    int32_t nonneg, int32_t normalize_w, double* lambda_out, double* m3_out) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    set_device(c);
    if (!H || !V || !W) throw InvalidArgument("null factor");
    PackedDev d;
    upload_packed(c, K, J, R, ycol_ptr, ycols, Y, d);
    const std::size_t RR = static_cast<std::size_t>(R) * R;
    cudaStream_t s = c->stream;
    DBuf<double> dH, dV, dW, m1, M2, m3, gW, gV, gH, G2, G3, nH, nV, gvraw, pinv, part, gwc;
    DBuf<std::int32_t> err, work;
    dH.resize(RR);
    dV.resize(static_cast<std::size_t>(std::max<std::int64_t>(J, 1)) * R);
    dW.resize(static_cast<std::size_t>(std::max<std::int64_t>(K, 1)) * R);
    m1.resize(RR);
    M2.resize(static_cast<std::size_t>(std::max<std::int64_t>(J, 1)) * R);
    m3.resize(static_cast<std::size_t>(std::max<std::int64_t>(K, 1)) * R);
    for (DBuf<double>* b : {&gW, &gV, &gH, &G2, &G3, &gvraw, &pinv}) b->resize(RR);
    nH.resize(R);
    nV.resize(R);
    gwc.resize(RR + 1);
    part.resize(static_cast<std::size_t>(kMaxPartials) * (RR + 1));
    err.resize(1);
    P2G_CUDA(cudaMemsetAsync(err.get(), 0, sizeof(std::int32_t), s));
    check_finite_host(H, static_cast<std::int64_t>(RR), "gram operand");
    check_finite_host(V, J * R, "gram operand");
    check_finite_host(W, K * R, "gram operand");
    upload_colmajor(c, H, R, R, dH.get());
    P2G_CUDA(cudaStreamSynchronize(s));
    upload_colmajor(c, V, J, R, dV.get());
    P2G_CUDA(cudaStreamSynchronize(s));
    upload_colmajor(c, W, K, R, dW.get());
    // gram(W), gram(V) of the incoming factors
    int np = gram_partials(R, K, dW.get(), nullptr, part.get(), kMaxPartials, s);
    reduce_partials(part.get(), np, static_cast<std::int64_t>(RR + 1), gwc.get(), s);
    P2G_CUDA(cudaMemcpyAsync(gW.get(), gwc.get(), sizeof(double) * RR, cudaMemcpyDeviceToDevice, s));
    np = gram_partials(R, J, dV.get(), nullptr, part.get(), kMaxPartials, s);
    reduce_partials(part.get(), np, static_cast<std::int64_t>(RR + 1), gwc.get(), s);
    P2G_CUDA(cudaMemcpyAsync(gV.get(), gwc.get(), sizeof(double) * RR, cudaMemcpyDeviceToDevice, s));
    // H step (cp.hpp:107-112)
    packed_mode(c, 1, K, J, R, d, dH.get(), dV.get(), dW.get(), m1.get());
    launch_solve_h(R, m1.get(), gW.get(), gV.get(), dH.get(), nH.get(), gH.get(), G2.get(), s);
    // W' = W diag(nH) (cp.hpp:111)
    {
      std::vector<double> ones(static_cast<std::size_t>(R));
      DBuf<double> inv;
      inv.resize(R);
      // scale W columns by nH: reuse k_scale_cols with reciprocal norms computed on host
      std::vector<double> hnh(static_cast<std::size_t>(R));
      P2G_CUDA(cudaMemcpyAsync(hnh.data(), nH.get(), sizeof(double) * R, cudaMemcpyDeviceToHost, s));
      P2G_CUDA(cudaStreamSynchronize(s));
      for (int r = 0; r < R; ++r) ones[static_cast<std::size_t>(r)] = 1.0 / hnh[static_cast<std::size_t>(r)];
      P2G_CUDA(cudaMemcpyAsync(inv.get(), ones.data(), sizeof(double) * R, cudaMemcpyHostToDevice, s));
      launch_scale_cols(R, K, dW.get(), inv.get(), s);
      P2G_CUDA(cudaStreamSynchronize(s));
    }
    // V step (cp.hpp:115-123)
    packed_mode(c, 2, K, J, R, d, dH.get(), dV.get(), dW.get(), M2.get());
    if (nonneg) {
      work.resize(static_cast<std::size_t>(std::max<std::int64_t>(J, K)) + 1);
      launch_nnls_rows(c->nnls_ws, R, J, G2.get(), M2.get(), dV.get(), 0, err.get(), work.get(), s);
    } else {
      launch_pinv(R, G2.get(), pinv.get(), s);
      launch_rows_times(R, J, M2.get(), pinv.get(), dV.get(), s);
    }
    np = gram_partials(R, J, dV.get(), nullptr, part.get(), kMaxPartials, s);
    reduce_partials(part.get(), np, static_cast<std::int64_t>(RR + 1), gwc.get(), s);
    P2G_CUDA(cudaMemcpyAsync(gvraw.get(), gwc.get(), sizeof(double) * RR, cudaMemcpyDeviceToDevice, s));
    launch_normalize_v(R, J, dV.get(), gvraw.get(), gV.get(), nV.get(), gH.get(), G3.get(), s);
    // W step (cp.hpp:126-133)
    packed_mode(c, 3, K, J, R, d, dH.get(), dV.get(), dW.get(), m3.get());
    if (nonneg) {
      work.resize(static_cast<std::size_t>(std::max<std::int64_t>(J, K)) + 1);
      launch_nnls_rows(c->nnls_ws, R, K, G3.get(), m3.get(), dW.get(), 0, err.get(), work.get(), s);
    } else {
      launch_pinv(R, G3.get(), pinv.get(), s);
      launch_rows_times(R, K, m3.get(), pinv.get(), dW.get(), s);
    }
    std::int32_t herr = 0;
    P2G_CUDA(cudaMemcpyAsync(&herr, err.get(), sizeof(herr), cudaMemcpyDeviceToHost, s));
    P2G_CUDA(cudaStreamSynchronize(s));
    if (herr) throw NumericalError("NNLS did not converge");
    download_colmajor(c, dH.get(), R, R, H);
    download_colmajor(c, dV.get(), J, R, V);
    download_colmajor(c, dW.get(), K, R, W);
    if (m3_out) download_colmajor(c, m3.get(), K, R, m3_out);
    // lambda (cp.hpp:136-143), on host (R values)
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
      for (int64_t k = 0; k < K; ++k) acc += W[k + r * K] * W[k + r * K];
      const double nrm = std::sqrt(acc);
      if (lambda_out) lambda_out[r] = normalize_w ? nrm : 1.0;
      if (normalize_w && nrm > 0.0)
        for (int64_t k = 0; k < K; ++k) W[k + r * K] /= nrm;
    }
  });
}

extern "C" int p2g_nnls_rowwise(p2g_ctx* c, const double* G, const double* B, int64_t n, int32_t R, int32_t max_iter,
                                double* X) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    set_device(c);
    if (R < 1 || R > 40) throw InvalidArgument("nnls_rowwise: G must be square with 1 <= R <= 40");
    if (n < 0 || !G || (n > 0 && (!B || !X))) throw InvalidArgument("nnls_rowwise: bad arguments");
    check_finite_host(G, static_cast<std::int64_t>(R) * R, "nonnegative solve normal matrix");
    check_finite_host(B, n * R, "nonnegative solve right-hand side");
    if (n == 0) return;
    DBuf<double> dG, dB, dX;
    DBuf<std::int32_t> err;
    dG.resize(static_cast<std::size_t>(R) * R);
    dB.resize(static_cast<std::size_t>(n) * R);
    dX.resize(static_cast<std::size_t>(n) * R);
    err.resize(1);
    P2G_CUDA(cudaMemsetAsync(err.get(), 0, sizeof(std::int32_t), c->stream));
    upload_colmajor(c, G, R, R, dG.get());
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    upload_colmajor(c, B, n, R, dB.get());
    DBuf<std::int32_t> work;
    work.resize(static_cast<std::size_t>(n) + 1);
    launch_nnls_rows(c->nnls_ws, R, n, dG.get(), dB.get(), dX.get(), max_iter, err.get(), work.get(), c->stream);
    std::int32_t herr = 0;
    P2G_CUDA(cudaMemcpyAsync(&herr, err.get(), sizeof(herr), cudaMemcpyDeviceToHost, c->stream));
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    if (herr) throw NumericalError("NNLS did not converge");
    download_colmajor(c, dX.get(), n, R, X);
  });
}

extern "C" int p2g_pinv_small(p2g_ctx* c, const double* G, int32_t n, double* out) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    set_device(c);
    if (n < 1 || n > 40 || !G || !out) throw InvalidArgument("pinv_small: matrix must be square (1..40)");
    check_finite_host(G, static_cast<std::int64_t>(n) * n, "pseudoinverse operand");
    DBuf<double> dG, dO;
    dG.resize(static_cast<std::size_t>(n) * n);
    dO.resize(static_cast<std::size_t>(n) * n);
    upload_colmajor(c, G, n, n, dG.get());
    launch_pinv(n, dG.get(), dO.get(), c->stream);
    download_colmajor(c, dO.get(), n, n, out);
  });
}

extern "C" int p2g_economy_svd(p2g_ctx* c, const double* M, int64_t rows, int64_t cols, double* P, double* sigma,
                               double* Z) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    set_device(c);
    const std::int64_t rho = std::min(rows, cols);
    if (rows < 1 || cols < 1 || rho > svd_max_cols() || std::max(rows, cols) > (1 << 24) || !M || !P || !sigma || !Z)
      throw InvalidArgument("economy_svd: need 1 <= min(rows, cols) <= 128");
    check_finite_host(M, rows * cols, "svd operand");
    double amax = 0.0;
    for (std::int64_t e = 0; e < rows * cols; ++e) amax = std::max(amax, std::fabs(M[e]));
    if (amax == 0.0) {  // kernels.hpp:101-104
      std::fill(P, P + rows * rho, 0.0);
      std::fill(Z, Z + cols * rho, 0.0);
      std::fill(sigma, sigma + rho, 0.0);
      for (std::int64_t j = 0; j < rho; ++j) P[j * rows + j] = Z[j * cols + j] = 1.0;
      return;
    }
    // W = M (rows >= cols) or M^T (the column-major bytes of M are M^T row-major), scaled by 1 / max |entry|
    const bool tall = rows >= cols;
    const int mm = static_cast<int>(tall ? rows : cols), nn = static_cast<int>(rho);
    std::vector<double> h(static_cast<std::size_t>(rows * cols));
    for (std::int64_t e = 0; e < rows * cols; ++e) h[static_cast<std::size_t>(e)] = M[e] / amax;
    DBuf<double> dW, dV, dU, dVo, dS;
    DBuf<std::int32_t> dst;
    dW.resize(static_cast<std::size_t>(mm) * nn);
    dV.resize(static_cast<std::size_t>(nn) * nn);
    dU.resize(static_cast<std::size_t>(mm) * nn);
    dVo.resize(static_cast<std::size_t>(nn) * nn);
    dS.resize(static_cast<std::size_t>(nn));
    dst.resize(1);
    if (tall)
      upload_colmajor(c, h.data(), rows, cols, dW.get());
    else
      P2G_CUDA(cudaMemcpyAsync(dW.get(), h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, c->stream));
    launch_economy_svd(mm, nn, dW.get(), dV.get(), dU.get(), dVo.get(), dS.get(), dst.get(), c->stream);
    P2G_LAUNCHED(1);
    std::int32_t st = 0;
    P2G_CUDA(cudaMemcpyAsync(&st, dst.get(), sizeof(st), cudaMemcpyDeviceToHost, c->stream));
    P2G_CUDA(cudaMemcpyAsync(sigma, dS.get(), sizeof(double) * nn, cudaMemcpyDeviceToHost, c->stream));
    // tall: P = U (rows x rho), Z = V (cols x cols); wide: M^T = Z Sigma P^T, so Z = U (cols x rho), P = V
    download_colmajor(c, dU.get(), mm, nn, tall ? P : Z);
    download_colmajor(c, dVo.get(), nn, nn, tall ? Z : P);
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    if (st != 0) throw NumericalError("economy_svd did not converge");
    for (int j = 0; j < nn; ++j) sigma[j] *= amax;
  });
}

extern "C" int p2g_gram(p2g_ctx* c, const double* A, int64_t rows, int32_t cols, double* out) {
  return guarded([&] {
    if (!c) throw InvalidArgument("null context");
    set_device(c);
    if (cols < 1 || cols > 40 || rows < 0 || !out || (rows > 0 && !A)) throw InvalidArgument("gram: bad arguments");
    check_finite_host(A, rows * cols, "gram operand");
    const std::size_t RR = static_cast<std::size_t>(cols) * cols;
    DBuf<double> dA, part, res;
    dA.resize(static_cast<std::size_t>(std::max<std::int64_t>(rows, 1)) * cols);
    part.resize(static_cast<std::size_t>(kMaxPartials) * (RR + 1));
    res.resize(RR + 1);
    if (rows > 0) upload_colmajor(c, A, rows, cols, dA.get());
    const int np = gram_partials(cols, rows, dA.get(), nullptr, part.get(), kMaxPartials, c->stream);
    reduce_partials(part.get(), np, static_cast<std::int64_t>(RR + 1), res.get(), c->stream);
    download_colmajor(c, res.get(), cols, cols, out);
  });
}
