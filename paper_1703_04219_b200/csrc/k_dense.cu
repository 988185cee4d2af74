// Dense helpers of the CP step on the GPU: Gram partials with a fixed
// reduction tree, the batched row-wise NNLS (K4), and the replicated R x R
// updates of cp_als_iteration (cp.hpp:99-145) and the fit (solver.hpp:299-306).
#include <algorithm>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"

namespace p2g {
namespace {

constexpr int kMaxR = 40;

// ---------------------------------------------------------------------------
// gram (kernels.hpp:57-63) over n rows of a row-major n x R matrix, with the
// optional cross term sum(A o B) (solver.hpp:299).  Block b owns the static
// row range [n*b/nb, n*(b+1)/nb); partial layout: R*R entries then cross.
// ---------------------------------------------------------------------------
template <int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_gram_partial(int R, std::int64_t n, const double* __restrict__ A, const double* __restrict__ B,
                   double* __restrict__ partials) {
  __shared__ double ch[WPB][32 * kMaxR];
  __shared__ double acc_s[WPB][kMaxR * kMaxR + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int RR = R * R;
  for (int e = lane; e <= RR; e += 32) acc_s[wid][e] = 0.0;
  const std::int64_t row0 = n * blockIdx.x / gridDim.x, row1 = n * (blockIdx.x + 1) / gridDim.x;
  double cross = 0.0;
  for (std::int64_t b0 = row0 + static_cast<std::int64_t>(wid) * 32; b0 < row1; b0 += 32 * WPB) {
    const int nr = static_cast<int>(row1 - b0 < 32 ? row1 - b0 : 32);
    for (int idx = lane; idx < nr * R; idx += 32) {
      const int r = idx / R, c = idx - (idx / R) * R;
      const double a = A[(b0 + r) * R + c];
      ch[wid][r * kMaxR + c] = a;
      if (B) cross = fma(a, B[(b0 + r) * R + c], cross);
    }
    __syncwarp();
    for (int e = lane; e < RR; e += 32) {
      const int x = e / R, y = e - (e / R) * R;
      if (y > x) continue;  // lower triangle; mirrored below (exact symmetry)
      double acc = acc_s[wid][e];
      for (int r = 0; r < nr; ++r) acc = fma(ch[wid][r * kMaxR + x], ch[wid][r * kMaxR + y], acc);
      acc_s[wid][e] = acc;
    }
    __syncwarp();
  }
  cross = dev::warp_sum(cross);
  if (lane == 0) acc_s[wid][RR] = cross;
  __syncthreads();
  if (wid == 0) {
    double* out = partials + static_cast<std::int64_t>(blockIdx.x) * (RR + 1);
    for (int e = lane; e <= RR; e += 32) {
      int src = e;
      if (e < RR) {
        const int x = e / R, y = e - (e / R) * R;
        if (y > x) src = y * R + x;
      }
      double acc = 0.0;
      for (int w = 0; w < WPB; ++w) acc += acc_s[w][src];
      out[e] = acc;
    }
  }
}

__global__ void k_reduce_partials(const double* __restrict__ partials, int nparts, std::int64_t len,
                                  double* __restrict__ out) {
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < len;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    // pairwise tree over parts (parallel.hpp:115-124 style): fixed order
    double acc = 0.0;
    for (int p = 0; p < nparts; ++p) acc += partials[static_cast<std::int64_t>(p) * len + e];
    out[e] = acc;
  }
}

// ---------------------------------------------------------------------------
// K4: batched NNLS, one warp per row, faithful to nnls_single
// (kernels.hpp:115-185): same entering rule (argmax w_j > 1e-10, first index
// on ties), same step / drop rule (1e-14 * max(1, max|x|)), same cap.  The
// passive subproblem G_pp s = b_p is solved by Cholesky (equal to the
// reference's pinv_small(G_pp) b_p when G_pp is positive definite); a
// non-positive pivot falls back to the eigen pseudo-inverse.
// ---------------------------------------------------------------------------
constexpr int kNnlsFastN0 = 12;  // largest zero set the fast warm path solves

/// G^{-1} for the NNLS fast warm path: Gauss-Jordan without pivoting on the
/// SPD Gram (one warp); out[R * R] = 1 when every pivot was positive and
/// finite, else 0 (the fast path is then off for this launch).
template <int RP>
__global__ void k_ginv(int R, const double* __restrict__ G, double* __restrict__ out) {
  __shared__ double A[RP][2 * RP + 1];
  __shared__ double f[RP];
  const int lane = threadIdx.x;
  for (int e = lane; e < R * 2 * R; e += 32) {
    const int i = e / (2 * R), j = e - i * 2 * R;
    A[i][j] = j < R ? G[i * R + j] : (j - R == i ? 1.0 : 0.0);
  }
  __syncwarp();
  bool ok = true;
  for (int k = 0; k < R && ok; ++k) {
    const double piv = A[k][k];
    ok = piv > 0.0 && isfinite(piv);
    if (!ok) break;
    const double ip = 1.0 / piv;
    __syncwarp();
    for (int j = lane; j < 2 * R; j += 32) A[k][j] *= ip;
    for (int i = lane; i < R; i += 32) f[i] = i == k ? 0.0 : A[i][k];
    __syncwarp();
    for (int e = lane; e < R * 2 * R; e += 32) {
      const int i = e / (2 * R), j = e - i * 2 * R;
      if (i != k) A[i][j] = fma(-f[i], A[k][j], A[i][j]);
    }
    __syncwarp();
  }
  for (int e = lane; e < R * R; e += 32) {
    const int i = e / R, j = e - i * R;
    out[e] = 0.5 * (A[i][R + j] + A[j][R + i]);
  }
  if (lane == 0) out[R * R] = ok ? 1.0 : 0.0;
}

template <int RP>
struct NnlsSmem {
  // L (RP*RP) + b, x, w, s, sp (RP each) + cs (RP+2) ; ints: pset RP, pq RP+2.
  // The pseudo-inverse fallback's three RP*RP work matrices live in a global
  // per-warp slab (rarely touched, L1/L2): keeping them in shared memory
  // capped the kernel at 4 warps per SM at R = 40.
  static constexpr int kDoubles = RP * RP + 5 * RP + RP + 2;
  static constexpr int kInts = 2 * RP + 2;
};

template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_nnls(int R, std::int64_t n, const double* __restrict__ G, const double* __restrict__ B, double* __restrict__ X,
           int cap, std::int32_t* err, const std::int32_t* __restrict__ rowlist, const std::int32_t* __restrict__ nlist,
           unsigned long long* __restrict__ masks, int warm, double* __restrict__ pinv_slab,
           const double* __restrict__ ginv) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Gs = smem;
  double* Gi = Gs + RP * RP;  // G^{-1} (fast warm path), when ginv is valid
  double* base = Gi + RP * RP + wid * (NnlsSmem<RP>::kDoubles + (NnlsSmem<RP>::kInts + 1) / 2);
  double* L = base;
  double* PA = pinv_slab + (static_cast<std::int64_t>(blockIdx.x) * WPB + wid) * 3 * RP * RP;
  double* PE = PA + RP * RP;
  double* PO = PE + RP * RP;
  double* b = L + RP * RP;
  double* x = b + RP;
  double* w = x + RP;
  double* sv = w + RP;
  double* sp = sv + RP;
  double* cs = sp + RP;
  int* pset = reinterpret_cast<int*>(cs + RP + 2);
  int* pq = pset + RP;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gs[e] = G[e];
  const bool fast = ginv && ginv[R * R] == 1.0;
  if (fast)
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gi[e] = ginv[e];
  __syncthreads();
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  const std::int64_t nrows = rowlist ? static_cast<std::int64_t>(*nlist) : n;
  for (std::int64_t it = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; it < nrows; it += nwarps) {
    const std::int64_t row = rowlist ? static_cast<std::int64_t>(rowlist[it]) : it;
    for (int r = lane; r < R; r += 32) {
      const double v = B[row * R + r];
      b[r] = v;
      w[r] = v;
      x[r] = 0.0;
    }
    // Warm start (optional, as in k_nnls_thread): begin from the row's previous
    // passive set; an infeasible warm solve sheds its non-positive coordinates
    // and retries (x = 0 throughout), an emptied set is the reference's cold start.
    const unsigned long long full = R >= 64 ? ~0ull : ((1ull << R) - 1ull);
    unsigned long long passive = (masks && warm) ? (masks[row] & full) : 0ull;
    if (fast && !(masks && warm)) {
      // cold row: start from the support of the unconstrained solution G^{-1} b
      // (any starting passive set reaches the same unique NNLS optimum; an
      // infeasible start sheds coordinates and falls back to the cold path)
      for (int r = lane; r < R; r += 32) {
        double acc = 0.0;
        for (int c = 0; c < R; ++c) acc = fma(Gi[r * R + c], b[c], acc);
        if (acc > 0.0) passive |= 1ull << r;
      }
      for (int o = 16; o > 0; o >>= 1) passive |= __shfl_xor_sync(dev::kFull, passive, o);
    }
    bool warm_phase = passive != 0ull;
    int iters = 0;
    bool failed = false;
    __syncwarp();
    // Fast warm path: G is shared by every row, so with G^{-1} precomputed the
    // passive solve G_PP s = b_P is a Schur complement on the zero set N,
    //   s = (Gi_PP - Gi_PN Gi_NN^{-1} Gi_NP) b_P,
    // an |N| x |N| Cholesky instead of a |P| x |P| one.  Accepted only at the
    // reference's optimum (s > 0 on P, no entering coordinate w_j > 1e-10 off
    // P: nnls_single's KKT test); otherwise the row takes the general path.
    if (fast && warm_phase && masks) {
      const unsigned long long nmask = full & ~passive;
      const int n0 = __popcll(nmask);
      if (n0 <= kNnlsFastN0) {
        for (int r = lane; r < R; r += 32)
          if ((nmask >> r) & 1ull) pq[__popcll(nmask & ((1ull << r) - 1ull))] = r;
        for (int r = lane; r < R; r += 32) {  // t = Gi[:, P] b_P
          double acc = 0.0;
          for (int c = 0; c < R; ++c)
            if ((passive >> c) & 1ull) acc = fma(Gi[r * R + c], b[c], acc);
          sp[r] = acc;
        }
        __syncwarp();
        int ok = 1;
        if (n0 > 0) {
          if (lane == 0) {  // Gi_NN z = t_N by Cholesky on one lane (n0 <= kNnlsFastN0)
            for (int i = 0; i < n0 && ok; ++i)
              for (int j = 0; j <= i; ++j) {
                double acc = Gi[pq[i] * R + pq[j]];
                for (int c = 0; c < j; ++c) acc = fma(-L[i * n0 + c], L[j * n0 + c], acc);
                if (i == j) {
                  if (!(acc > 0.0) || !isfinite(acc)) {
                    ok = 0;
                    break;
                  }
                  L[i * n0 + i] = sqrt(acc);
                } else {
                  L[i * n0 + j] = acc / L[j * n0 + j];
                }
              }
            if (ok) {
              for (int i = 0; i < n0; ++i) {
                double acc = sp[pq[i]];
                for (int c = 0; c < i; ++c) acc = fma(-L[i * n0 + c], sv[c], acc);
                sv[i] = acc / L[i * n0 + i];
              }
              for (int i = n0 - 1; i >= 0; --i) {
                double acc = sv[i];
                for (int c = i + 1; c < n0; ++c) acc = fma(-L[c * n0 + i], sv[c], acc);
                sv[i] = acc / L[i * n0 + i];
              }
            }
          }
          ok = __shfl_sync(dev::kFull, ok, 0);
          __syncwarp();
        }
        if (ok) {
          for (int r = lane; r < R; r += 32) {
            double acc = 0.0;
            if ((passive >> r) & 1ull) {
              acc = sp[r];
              for (int a2 = 0; a2 < n0; ++a2) acc = fma(-Gi[r * R + pq[a2]], sv[a2], acc);
            }
            x[r] = acc;
          }
          __syncwarp();
          bool good = true;
          for (int r = lane; r < R; r += 32) {
            if ((passive >> r) & 1ull) {
              good = good && x[r] > 0.0 && isfinite(x[r]);
            } else {
              double acc = 0.0;
              for (int c = 0; c < R; ++c) acc = fma(Gs[r * R + c], x[c], acc);
              good = good && !(b[r] - acc > 1e-10);
            }
          }
          if (__all_sync(dev::kFull, good)) {
            if (lane == 0) masks[row] = passive;
            for (int r = lane; r < R; r += 32) X[row * R + r] = x[r];
            __syncwarp();
            continue;
          }
          for (int r = lane; r < R; r += 32) x[r] = 0.0;
          __syncwarp();
        }
      }
    }
    while (true) {
     if (!warm_phase) {
      // entering coordinate: argmax_{j not passive, w_j > 1e-10} w_j, first index on ties
      double best = 1e-10;
      int enter = -1;
      for (int r = lane; r < R; r += 32) {
        if (!((passive >> r) & 1ull) && w[r] > best) {
          best = w[r];
          enter = r;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(dev::kFull, best, o);
        const int oe = __shfl_xor_sync(dev::kFull, enter, o);
        if (oe >= 0 && (enter < 0 || ob > best || (ob == best && oe < enter))) {
          best = ob;
          enter = oe;
        }
      }
      if (enter < 0) break;
      passive |= 1ull << enter;
     }
      while (true) {
        if (++iters > cap) {
          failed = true;
          break;
        }
        const int np = __popcll(passive);
        for (int r = lane; r < R; r += 32)
          if ((passive >> r) & 1ull) pset[__popcll(passive & ((1ull << r) - 1ull))] = r;
        __syncwarp();
        for (int e = lane; e < np * np; e += 32) {
          const int i = e / np, j = e - (e / np) * np;
          L[e] = Gs[pset[i] * R + pset[j]];
        }
        for (int a2 = lane; a2 < np; a2 += 32) sp[a2] = b[pset[a2]];
        __syncwarp();
        // Cholesky (right-looking, lower), then two triangular solves.
        bool ok = true;
        for (int jj = 0; jj < np; ++jj) {
          const double d = L[jj * np + jj];
          ok = ok && d > 0.0 && isfinite(d);
          if (!ok) break;
          const double sd = sqrt(d);
          __syncwarp();
          for (int i = jj + 1 + lane; i < np; i += 32) L[i * np + jj] /= sd;
          if (lane == 0) L[jj * np + jj] = sd;
          __syncwarp();
          const int m = np - jj - 1;
          for (int e = lane; e < m * m; e += 32) {
            const int i = jj + 1 + e / m, c = jj + 1 + (e - (e / m) * m);
            if (c <= i) L[i * np + c] -= L[i * np + jj] * L[c * np + jj];
          }
          __syncwarp();
        }
        if (ok) {
          for (int jj = 0; jj < np; ++jj) {  // L y = b
            const double y = sp[jj] / L[jj * np + jj];
            __syncwarp();
            for (int i = jj + 1 + lane; i < np; i += 32) sp[i] -= L[i * np + jj] * y;
            if (lane == 0) sp[jj] = y;
            __syncwarp();
          }
          for (int jj = np - 1; jj >= 0; --jj) {  // L^T s = y
            const double y = sp[jj] / L[jj * np + jj];
            __syncwarp();
            for (int i = lane; i < jj; i += 32) sp[i] -= L[jj * np + i] * y;
            if (lane == 0) sp[jj] = y;
            __syncwarp();
          }
        } else {
          // pseudo-inverse route, exactly the reference's pinv_small(G_pp) b_p
          __syncwarp();
          for (int e = lane; e < np * np; e += 32) {
            const int i = e / np, j = e - (e / np) * np;
            L[e] = Gs[pset[i] * R + pset[j]];
          }
          __syncwarp();
          dev::warp_pinv_sym(L, PO, PA, PE, cs, pq, np, lane);
          double tmp[2] = {0.0, 0.0};
          for (int a2 = lane, t = 0; a2 < np && t < 2; a2 += 32, ++t) {
            double acc = 0.0;
            for (int c = 0; c < np; ++c) acc = fma(PO[a2 * np + c], b[pset[c]], acc);
            tmp[t] = acc;
          }
          __syncwarp();
          for (int a2 = lane, t = 0; a2 < np && t < 2; a2 += 32, ++t) sp[a2] = tmp[t];
          __syncwarp();
        }
        bool allpos = true;
        for (int a2 = lane; a2 < np; a2 += 32) allpos = allpos && sp[a2] > 0.0;
        allpos = __all_sync(dev::kFull, allpos);
        if (allpos) {
          for (int r = lane; r < R; r += 32) x[r] = 0.0;
          __syncwarp();
          for (int a2 = lane; a2 < np; a2 += 32) x[pset[a2]] = sp[a2];
          __syncwarp();
          break;
        }
        if (warm_phase) {  // x = 0: drop the non-positive coordinates and re-solve
          unsigned long long drop = 0ull;
          for (int a2 = lane; a2 < np; a2 += 32)
            if (!(sp[a2] > 0.0)) drop |= 1ull << pset[a2];
          for (int o = 16; o > 0; o >>= 1) drop |= __shfl_xor_sync(dev::kFull, drop, o);
          passive &= ~drop;
          __syncwarp();
          if (passive == 0ull) break;
          continue;
        }
        // step toward s until the first passive coordinate hits zero
        for (int r = lane; r < R; r += 32) sv[r] = 0.0;
        __syncwarp();
        for (int a2 = lane; a2 < np; a2 += 32) sv[pset[a2]] = sp[a2];
        __syncwarp();
        double alpha = __longlong_as_double(0x7ff0000000000000ll);  // +inf
        for (int a2 = lane; a2 < np; a2 += 32) {
          if (sp[a2] <= 0.0) {
            const int j = pset[a2];
            const double denom = x[j] - sv[j];
            const double step = denom > 0.0 ? x[j] / denom : 0.0;
            alpha = fmin(alpha, step);
          }
        }
        alpha = -dev::warp_max(-alpha);
        for (int a2 = lane; a2 < np; a2 += 32) {
          const int j = pset[a2];
          x[j] += alpha * (sv[j] - x[j]);
        }
        __syncwarp();
        double xm = 0.0;
        for (int r = lane; r < R; r += 32) xm = fmax(xm, fabs(x[r]));
        xm = dev::warp_max(xm);
        const double drop_tol = 1e-14 * fmax(1.0, xm);
        unsigned long long drop = 0ull;
        for (int a2 = lane; a2 < np; a2 += 32) {
          const int j = pset[a2];
          if (x[j] <= drop_tol) {
            x[j] = 0.0;
            drop |= 1ull << j;
          }
        }
        for (int o = 16; o > 0; o >>= 1) drop |= __shfl_xor_sync(dev::kFull, drop, o);
        passive &= ~drop;
        __syncwarp();
      }
      warm_phase = false;
      if (failed) break;
      // w = b - G x
      for (int r = lane; r < R; r += 32) {
        double acc = 0.0;
        for (int c = 0; c < R; ++c) acc = fma(Gs[r * R + c], x[c], acc);
        w[r] = b[r] - acc;
      }
      __syncwarp();
    }
    if (failed && lane == 0) atomicAdd(err, 1);
    if (masks && lane == 0) masks[row] = passive;
    for (int r = lane; r < R; r += 32) X[row * R + r] = x[r];
    __syncwarp();
  }
}

__global__ void k_rows_times(int R, std::int64_t n, const double* __restrict__ B, const double* __restrict__ P,
                             double* __restrict__ X) {
  __shared__ double Ps[kMaxR * kMaxR];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Ps[e] = P[e];
  __syncthreads();
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n * R;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = e / R;
    const int c = static_cast<int>(e - i * R);
    double acc = 0.0;
    for (int a = 0; a < R; ++a) acc = fma(B[i * R + a], Ps[a * R + c], acc);
    X[e] = acc;
  }
}

struct SmallWs {
  double A[kMaxR * kMaxR], E[kMaxR * kMaxR], T[kMaxR * kMaxR], U[kMaxR * kMaxR];
  double cs[kMaxR + 2];
  int pq[kMaxR + 2];
};

__global__ void k_pinv(int n, const double* __restrict__ G, double* __restrict__ out) {
  extern __shared__ double sm[];
  SmallWs& ws = *reinterpret_cast<SmallWs*>(sm);
  const int lane = threadIdx.x;
  for (int e = lane; e < n * n; e += 32) ws.U[e] = G[e];
  __syncwarp();
  dev::warp_pinv_sym(ws.U, ws.T, ws.A, ws.E, ws.cs, ws.pq, n, lane);
  for (int e = lane; e < n * n; e += 32) out[e] = ws.T[e];
}

/// H step of cp_als_iteration (cp.hpp:105-111) + the V-step Gram (cp.hpp:117):
/// G1 = gram(W) o gram(V); H = m1 pinv(G1); normalize columns (norms nH,
/// zero columns untouched); gramH = H^T H; G2 = (nH nH^T o gram(W)) o gramH.
__global__ void k_solve_h(int R, const double* __restrict__ m1, const double* __restrict__ gramW,
                          const double* __restrict__ gramV, double* __restrict__ H, double* __restrict__ nH,
                          double* __restrict__ gramH, double* __restrict__ G2) {
  extern __shared__ double sm[];
  SmallWs& ws = *reinterpret_cast<SmallWs*>(sm);
  const int lane = threadIdx.x;
  const int RR = R * R;
  for (int e = lane; e < RR; e += 32) ws.U[e] = gramW[e] * gramV[e];
  __syncwarp();
  dev::warp_pinv_sym(ws.U, ws.T, ws.A, ws.E, ws.cs, ws.pq, R, lane);  // T = pinv(G1)
  dev::wmm(ws.U, m1, ws.T, R, lane);                                   // U = H (unnormalized)
  // column norms
  for (int c = lane; c < R; c += 32) {
    double acc = 0.0;
    for (int i = 0; i < R; ++i) acc = fma(ws.U[i * R + c], ws.U[i * R + c], acc);
    const double nrm = sqrt(acc);
    ws.cs[c] = nrm > 0.0 ? nrm : 1.0;
    nH[c] = nrm > 0.0 ? nrm : 1.0;
  }
  __syncwarp();
  for (int e = lane; e < RR; e += 32) {
    const int c = e - (e / R) * R;
    const double h = ws.U[e] / ws.cs[c];
    ws.U[e] = h;
    H[e] = h;
  }
  __syncwarp();
  dev::wmm_tn(ws.A, ws.U, ws.U, R, lane);  // gram(H)
  for (int e = lane; e < RR; e += 32) {
    const int i = e / R, j = e - (e / R) * R;
    gramH[e] = ws.A[e];
    G2[e] = ws.cs[i] * gramW[e] * ws.cs[j] * ws.A[e];
  }
}

/// V normalization (cp.hpp:122): nV from gram(V_raw) diagonal, then gramV =
/// D^-1 gram(V_raw) D^-1 and G3 = gramV o gramH (cp.hpp:128).
__global__ void k_norm_v_small(int R, const double* __restrict__ gramV_raw, double* __restrict__ gramV,
                               double* __restrict__ nV, const double* __restrict__ gramH, double* __restrict__ G3) {
  const int lane = threadIdx.x;
  __shared__ double nv[kMaxR];
  for (int c = lane; c < R; c += 32) {
    const double nrm = sqrt(gramV_raw[c * R + c]);
    nv[c] = nrm > 0.0 ? nrm : 1.0;
    nV[c] = nv[c];
  }
  __syncwarp();
  for (int e = lane; e < R * R; e += 32) {
    const int i = e / R, j = e - (e / R) * R;
    const double g = gramV_raw[e] / (nv[i] * nv[j]);
    gramV[e] = g;
    G3[e] = g * gramH[e];
  }
}

__global__ void k_scale_cols(int R, std::int64_t n, double* __restrict__ A, const double* __restrict__ norms) {
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n * R;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e % R);
    A[e] /= norms[c];
  }
}

/// Fit (solver.hpp:299-306): cross and gram(W) come reduced in gw_cross
/// (R*R entries then cross); C = gram(H) o gram(V); model = sum(C o gram(W)).
__global__ void k_fit(int R, const double* __restrict__ gw_cross, const double* __restrict__ gramH,
                      const double* __restrict__ gramV, double norm_x, double* __restrict__ gramW,
                      double* __restrict__ scal) {
  const int lane = threadIdx.x;
  const int RR = R * R;
  double model = 0.0;
  for (int e = lane; e < RR; e += 32) {
    const double gw = gw_cross[e];
    gramW[e] = gw;
    model = fma(gramH[e] * gramV[e], gw, model);
  }
  model = dev::warp_sum(model);
  if (lane == 0) {
    const double cross = gw_cross[RR];
    const double resid = fmax(0.0, norm_x - 2.0 * cross + model);
    scal[0] = 1.0 - resid / norm_x;
    scal[1] = resid;
    scal[2] = cross;
    scal[3] = model;
  }
}

__global__ void k_transpose(const double* __restrict__ in, double* __restrict__ out, std::int64_t rows,
                            std::int64_t cols) {
  // in: column-major rows x cols ; out: row-major rows x cols
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = e / cols, j = e - (e / cols) * cols;
    out[e] = in[i + j * rows];
  }
}

__global__ void k_fill(double* A, std::int64_t n, double v) {
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    A[e] = v;
}

__global__ void k_identity(double* A, int n) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) A[e] = (e / n == e % n) ? 1.0 : 0.0;
}

__global__ void k_hadamard(const double* A, const double* B, double* C, int n) {
  for (int e = threadIdx.x; e < n; e += blockDim.x) C[e] = A[e] * B[e];
}

int elem_grid(std::int64_t n) {
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + 255) / 256, 148 * 16)));
}

constexpr std::size_t kSmallSmem = sizeof(SmallWs);

/// Opt the single-warp R x R kernels into > 48 KB of dynamic shared memory.
void small_smem_optin() {
  static bool done = false;
  if (done) return;
  P2G_CUDA(cudaFuncSetAttribute(k_pinv, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmallSmem)));
  P2G_CUDA(cudaFuncSetAttribute(k_solve_h, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmallSmem)));
  done = true;
}

template <int RP>
void nnls_launch(NnlsWork& ws, int R, std::int64_t n, const double* G, const double* B, double* X, int cap, std::int32_t* err,
                 const std::int32_t* rowlist, const std::int32_t* nlist, unsigned long long* masks, int warm,
                 cudaStream_t s) {
  constexpr int WPB = RP <= 16 ? 8 : 4;
  const std::size_t per_warp = sizeof(double) * (NnlsSmem<RP>::kDoubles + (NnlsSmem<RP>::kInts + 1) / 2);
  const std::size_t smem = sizeof(double) * 2 * RP * RP + WPB * per_warp;
  auto kern = k_nnls<RP, WPB>;
  P2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const std::int64_t want = (n + WPB - 1) / WPB;
  const int blocks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(want, 148 * 16)));
  // pinv fallback workspace and G^{-1}: the context's (grown on demand)
  ws.slab.resize(static_cast<std::size_t>(blocks) * WPB * 3 * RP * RP);
  const bool fast = !rowlist && RP > 16;
  if (fast) {
    ws.ginv.resize(static_cast<std::size_t>(RP) * RP + 1);
    k_ginv<RP><<<1, 32, 0, s>>>(R, G, ws.ginv.get());
  }
  kern<<<blocks, WPB * 32, smem, s>>>(R, n, G, B, X, cap, err, rowlist, nlist, masks, warm, ws.slab.get(),
                                      fast ? ws.ginv.get() : nullptr);
}

template <int RP>
void nnls_warp(NnlsWork& ws, int R, std::int64_t n, const double* G, const double* B, double* X, int cap,
               std::int32_t* err, const std::int32_t* rowlist, const std::int32_t* nlist, unsigned long long* masks,
               int warm, cudaStream_t s) {
  nnls_launch<RP>(ws, R, n, G, B, X, cap, err, rowlist, nlist, masks, warm, s);
}

void nnls_warp_any(NnlsWork& ws, int R, std::int64_t n, const double* G, const double* B, double* X, int cap, std::int32_t* err,
                   const std::int32_t* rowlist, const std::int32_t* nlist, cudaStream_t s,
                   unsigned long long* masks = nullptr, int warm = 0) {
  if (R <= 8)
    nnls_warp<8>(ws, R, n, G, B, X, cap, err, rowlist, nlist, masks, warm, s);
  else if (R <= 16)
    nnls_warp<16>(ws, R, n, G, B, X, cap, err, rowlist, nlist, masks, warm, s);
  else if (R <= 32)
    nnls_warp<32>(ws, R, n, G, B, X, cap, err, rowlist, nlist, masks, warm, s);
  else if (R <= 40)
    nnls_warp<40>(ws, R, n, G, B, X, cap, err, rowlist, nlist, masks, warm, s);
  else
    throw InvalidArgument("rank above 40 unsupported");
}

}  // namespace

int gram_partials(int R, std::int64_t n, const double* A, const double* B, double* partials, int max_blocks,
                  cudaStream_t s) {
  constexpr int WPB = 2;  // 2 x (32x40 + 40x40+1) doubles of static smem < 48 KB
  const int blocks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + 63) / 64, max_blocks)));
  k_gram_partial<WPB><<<blocks, WPB * 32, 0, s>>>(R, n, A, B, partials);
  P2G_LAUNCHED(1);
  return blocks;
}

void reduce_partials(const double* partials, int nparts, std::int64_t len, double* out, cudaStream_t s) {
  k_reduce_partials<<<elem_grid(len), 256, 0, s>>>(partials, nparts, len, out);
  P2G_LAUNCHED(1);
}

/// G^{-1} of an R <= 16 Gram into the context's workspace (out[R*R] =
/// validity), for the thread-per-row NNLS's cold start.
const double* launch_ginv_small(NnlsWork& ws, int R, const double* G, cudaStream_t s) {
  ws.ginv_small.resize(16 * 16 + 1);
  k_ginv<16><<<1, 32, 0, s>>>(R, G, ws.ginv_small.get());
  P2G_LAUNCHED(1);
  return ws.ginv_small.get();
}

void launch_nnls_rows(NnlsWork& ws, int R, std::int64_t n, const double* G, const double* B, double* X, int max_iter,
                      std::int32_t* err, std::int32_t* work, cudaStream_t s, unsigned* masks, int warm,
                      unsigned long long* masks64) {
  if (n == 0) return;
  const int cap = max_iter > 0 ? max_iter : 30 * R;
  if (R <= kSmallRankMax && work) {
    // thread per row; rows whose passive Cholesky meets a non-positive pivot
    // are re-solved by the warp kernel with the pseudo-inverse (work[0] = count).
    P2G_CUDA(cudaMemsetAsync(work, 0, sizeof(std::int32_t), s));
    const double* gi = (masks && !warm) ? launch_ginv_small(ws, R, G, s) : nullptr;  // cold rows: G^{-1} b support
    launch_nnls_thread(R, n, G, B, X, max_iter, err, work + 1, work, masks, warm, s, gi);
    nnls_warp_any(ws, R, n, G, B, X, cap, err, work + 1, work, s);
    P2G_LAUNCHED(1);
    return;
  }
  nnls_warp_any(ws, R, n, G, B, X, cap, err, nullptr, nullptr, s, masks64, masks64 ? warm : 0);
  P2G_LAUNCHED(1);
}

void launch_rows_times(int R, std::int64_t n, const double* B, const double* P, double* X, cudaStream_t s) {
  if (n == 0) return;
  k_rows_times<<<elem_grid(n * R), 256, 0, s>>>(R, n, B, P, X);
  P2G_LAUNCHED(1);
}

void launch_pinv(int n, const double* G, double* out, cudaStream_t s) {
  if (n > kMaxR) throw InvalidArgument("pinv: size above 40 unsupported on device");
  small_smem_optin();
  k_pinv<<<1, 32, kSmallSmem, s>>>(n, G, out);
  P2G_LAUNCHED(1);
}

void launch_solve_h(int R, const double* m1, const double* gramW, const double* gramV, double* H, double* nH,
                    double* gramH, double* G2, cudaStream_t s) {
  small_smem_optin();
  k_solve_h<<<1, 32, kSmallSmem, s>>>(R, m1, gramW, gramV, H, nH, gramH, G2);
  P2G_LAUNCHED(1);
}

void launch_normalize_v(int R, std::int64_t J, double* V, const double* gramV_raw, double* gramV, double* nV,
                        const double* gramH, double* G3, cudaStream_t s) {
  k_norm_v_small<<<1, 32, 0, s>>>(R, gramV_raw, gramV, nV, gramH, G3);
  k_scale_cols<<<elem_grid(J * R), 256, 0, s>>>(R, J, V, nV);
  P2G_LAUNCHED(2);
}

void launch_fit(int R, const double* gw_cross, const double* gramH, const double* gramV, double norm_x,
                double* gramW, double* scal, cudaStream_t s) {
  k_fit<<<1, 32, 0, s>>>(R, gw_cross, gramH, gramV, norm_x, gramW, scal);
  P2G_LAUNCHED(1);
}

void launch_scale_cols(int R, std::int64_t n, double* A, const double* norms, cudaStream_t s) {
  if (n == 0) return;
  k_scale_cols<<<elem_grid(n * R), 256, 0, s>>>(R, n, A, norms);
  P2G_LAUNCHED(1);
}

void launch_transpose(const double* in, double* out, std::int64_t rows, std::int64_t cols, cudaStream_t s) {
  if (rows * cols == 0) return;
  k_transpose<<<elem_grid(rows * cols), 256, 0, s>>>(in, out, rows, cols);
  P2G_LAUNCHED(1);
}

void launch_fill_identity(double* A, int n, cudaStream_t s) {
  k_identity<<<1, 256, 0, s>>>(A, n);
  P2G_LAUNCHED(1);
}

void launch_fill(double* A, std::int64_t n, double v, cudaStream_t s) {
  if (n == 0) return;
  k_fill<<<elem_grid(n), 256, 0, s>>>(A, n, v);
  P2G_LAUNCHED(1);
}

void launch_hadamard(const double* A, const double* B, double* C, int n, cudaStream_t s) {
  k_hadamard<<<1, 256, 0, s>>>(A, B, C, n);
  P2G_LAUNCHED(1);
}

}  // namespace p2g
