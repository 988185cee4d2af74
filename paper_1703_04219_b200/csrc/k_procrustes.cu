// Accurate Procrustes path over the flagged subjects, fused with their
// mode-1 MTTKRP partial.
//
// Replaces procrustes_update (solver.hpp:173-193) for the subjects the fast
// paths (k_polar_small for R <= 16, k_procrustes_large_w for R > 16) flag
// P2G_FLAG_ACCURATE: rank-deficient or ill-conditioned targets, non-finite
// operands, non-converged Jacobi.  k_procrustes_accurate is a one-sided
// Jacobi SVD of A = X_k V diag(W_k) H^T (backward stable like Eigen's
// JacobiSVD, kernels.hpp:105), preconditioned with the fast path's
// eigenvectors, with the canonical rank-deficiency rule D5
// (oracle/p2_oracle.hpp canonical_polar).  m1_k = Q_k^T (X_k V) diag(W_k).
#include <algorithm>

#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"

namespace p2g {
namespace {

constexpr double kNullRatio = 1e-26;  // sigma^2 <= kNullRatio * sigma_max^2 -> null direction (D5, round-off level)

struct K1Args {
  ShardArgs X;
  int R;
  const double* H;  // R x R row-major
  const double* V;  // J x R row-major
  const double* W;  // K_s x R row-major
  double* Q;        // NR x R row-major
  std::int32_t* flags;
  double* m1_partials;  // gridDim.x x R x R
  double* scratch;      // accurate path: per-warp I_max x R slabs
  std::int64_t max_rows;
  std::int32_t* counters;  // [2] = non-finite operand seen
  const double* Ebuf;      // accurate path preconditioner (K x R x R) or null
  const std::int32_t* list;   // accurate path: flagged subjects, ascending (device), or null
  const std::int32_t* nlist;  // its length (device)
  double* Shat;            // Q-free outputs (K x R x R) or null: Q = A Shat + L Chat
  double* Chat;
};


// ---------------------------------------------------------------------------
// Accurate path: one-sided Jacobi SVD of A = XV D H^T, canonical rule D5.
// One warp per flagged subject; A lives in a per-warp global scratch slab
// (L1/L2 resident: the flagged set is ~1-5% of subjects).
// ---------------------------------------------------------------------------
template <int RP>
struct AccSmem {
  // Shared memory per warp holds only what the Hestenes sweeps touch: Vj plus
  // s, sig, cs, pq, idx.  The other R x R work matrices (T, M1, B, Es, Ee, TN)
  // and the row chunks live in the warp's global slab next to A (L1/L2): with
  // all seven in shared memory (112 KB at R = 40) one warp ran per SM.
  static constexpr int kPerWarpDoubles = RP * RP + 3 * RP + 2 * (RP + 2) + RP;
  __host__ __device__ static constexpr std::size_t slab(std::int64_t max_rows, int R) {
    return 6 * static_cast<std::size_t>(RP) * RP + 64 * static_cast<std::size_t>(RP) +
           static_cast<std::size_t>(max_rows > 1 ? max_rows : 1) * R;
  }
};

template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_procrustes_accurate(K1Args a, double* m1_partials_acc) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int R = a.R;
  const int RR = R * R;
  double* Hs = smem;
  double* base = smem + RP * RP + wid * AccSmem<RP>::kPerWarpDoubles;
  const std::int64_t gw = static_cast<std::int64_t>(blockIdx.x) * WPB + wid;
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  double* slab = a.scratch + gw * AccSmem<RP>::slab(a.max_rows, R);
  double* T = slab;
  double* M1 = T + RP * RP;
  double* B = M1 + RP * RP;
  double* EA = B + RP * RP;
  double* EE = EA + RP * RP;
  double* TN = EE + RP * RP;
  double* qch = TN + RP * RP;
  double* xch = qch + 32 * RP;
  double* A = xch + 32 * RP;  // I x R row-major
  double* Vj = base;
  double* s = Vj + RP * RP;
  double* sig = s + RP;
  double* cs = sig + RP;
  int* pq = reinterpret_cast<int*>(cs + RP + 2);
  int* strong = reinterpret_cast<int*>(cs + 2 * (RP + 2));  // RP ints: 1 if strong
  (void)strong;

  for (int e = threadIdx.x; e < RR; e += blockDim.x) Hs[e] = a.H[e];
  for (int e = lane; e < RR; e += 32) M1[e] = 0.0;
  __syncthreads();


  // Flagged subjects come as a compacted, ascending list; warp gw takes the
  // contiguous share [gw L / W, (gw + 1) L / W): equal counts per warp and a
  // schedule independent of timing (the m1 partials stay deterministic).
  const std::int64_t L = a.list ? static_cast<std::int64_t>(*a.nlist) : a.X.K;
  const std::int64_t it0 = a.list ? gw * L / nwarps : gw;
  const std::int64_t it1 = a.list ? (gw + 1) * L / nwarps : a.X.K;
  const std::int64_t istep = a.list ? 1 : nwarps;
  for (std::int64_t it = it0; it < it1; it += istep) {
    const std::int64_t k = a.list ? static_cast<std::int64_t>(a.list[it]) : it;
    if (a.flags[k] != P2G_FLAG_ACCURATE) continue;
    const std::int64_t r0 = a.X.srp[k];
    const int I = static_cast<int>(a.X.srp[k + 1] - r0);
    for (int r = lane; r < R; r += 32) s[r] = a.W[k * R + r];  // R may exceed 32
    __syncwarp();
    for (int e = lane; e < RR; e += 32) {
      const int i = e / R, j = e - (e / R) * R;
      T[e] = s[i] * Hs[j * R + i];
    }
    __syncwarp();
    // Preconditioner: eigenvectors E of A^T A from the fast path (small-R
    // pipeline).  B = A E has nearly orthogonal columns, so the Hestenes
    // sweeps below converge in 1-3 sweeps; V = E V' afterwards.
    const double* Ek = a.Ebuf ? a.Ebuf + k * RR : nullptr;
    if (Ek) {
      for (int e = lane; e < RR; e += 32) {
        const int i = e / R, j = e - (e / R) * R;
        double acc = 0.0;
        for (int c = 0; c < R; ++c) acc = fma(T[i * R + c], Ek[c * R + j], acc);
        B[e] = acc;
      }
      __syncwarp();
      for (int e = lane; e < RR; e += 32) T[e] = B[e];
      __syncwarp();
    }
    // A = XV T (solver.hpp:189-190, transposed)
    double amax = 0.0;
    bool finite = true;
    for (int i = lane; i < I; i += 32) {
      double xv[RP];
      dev::csr_row_times<RP>(xv, a.X.ci, a.X.val, a.X.rp[r0 + i], a.X.rp[r0 + i + 1], a.V, R);
      for (int c = 0; c < R; ++c) {
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < RP; ++r)
          if (r < R) v = fma(xv[r], T[r * R + c], v);
        A[i * R + c] = v;
        finite &= isfinite(v);
        amax = fmax(amax, fabs(v));
      }
    }
    finite = __all_sync(dev::kFull, finite);
    amax = dev::warp_max(amax);
    __syncwarp();
    if (!finite) {  // common.hpp:50-53 on the svd operand (kernels.hpp:99)
      if (lane == 0) {
        atomicAdd(a.counters + 2, 1);
        a.flags[k] = P2G_FLAG_DEGENERATE;
      }
      __syncwarp();
      continue;
    }
    int flag = P2G_FLAG_ACCURATE;
    int rho = 0;
    if (amax == 0.0) {
      // kernels.hpp:101-104: M == 0 -> Q = I(I_k, R).
      flag = P2G_FLAG_DEFICIENT;
      for (int e = lane; e < RR; e += 32) Vj[e] = 0.0;  // no strong part
      for (int r = lane; r < R; r += 32) sig[r] = 0.0;
      __syncwarp();
      for (int e = lane; e < RR; e += 32) Vj[e] = (e / R == e % R) ? 1.0 : 0.0;
      __syncwarp();
    } else {
      const double inv = 1.0 / amax;
      for (int i = lane; i < I; i += 32)
        for (int c = 0; c < R; ++c) A[i * R + c] *= inv;
      for (int e = lane; e < RR; e += 32) Vj[e] = (e / R == e % R) ? 1.0 : 0.0;
      __syncwarp();
      // Hestenes sweeps (same rotation formulas and skip rule as the oracle's
      // one_sided_jacobi), round-robin ordering: the R/2 disjoint column pairs
      // of a round go to groups of g = 32 / (R/2) lanes (g = 1 at R = 40, 6 at
      // R = 10: the small ranks used to leave 27 of 32 lanes idle); a group
      // splits the rows, sums its (alpha, beta, gamma) partials in a fixed
      // lane order (every lane of the group gets the same bits) and rotates
      // its rows of the pair's two columns of A and V.
      {
        const int mm = (R + 1) & ~1, hh = mm / 2;
        const int g = RP > 16 ? 1 : 32 / hh;  // compile-time 1 above R = 16 (unit-stride row loops)
        const int pr = lane / g, sub = lane - pr * g;
        const bool act = pr < hh;
        const int base = act ? pr * g : 0;
        for (int sweep = 0; sweep < 80; ++sweep) {
          bool rot = false;
          for (int round = 0; round < mm - 1; ++round) {
            int p = 0, q = mm;
            if (act) {
              if (pr == 0) {
                p = round;
                q = mm - 1;
              } else {
                p = (round + pr) % (mm - 1);
                q = (round - pr + (mm - 1)) % (mm - 1);
              }
              if (p > q) {
                const int t = p;
                p = q;
                q = t;
              }
            }
            const bool valid = act && q < R;
            double al = 0.0, be = 0.0, ga = 0.0;
            if (valid)
              for (int i = sub; i < I; i += g) {
                const double x = A[i * R + p], y = A[i * R + q];
                al = fma(x, x, al);
                be = fma(y, y, be);
                ga = fma(x, y, ga);
              }
            if (g > 1) {
              double sa = 0.0, sb = 0.0, sg = 0.0;
              for (int j = 0; j < g; ++j) {
                sa += __shfl_sync(dev::kFull, al, base + j);
                sb += __shfl_sync(dev::kFull, be, base + j);
                sg += __shfl_sync(dev::kFull, ga, base + j);
              }
              al = sa;
              be = sb;
              ga = sg;
            }
            if (valid && !(ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be))) {
              rot = true;
              const double zeta = (be - al) / (2.0 * ga);
              const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
              const double c = 1.0 / sqrt(1.0 + t * t);
              const double sn = c * t;
              // R > 16: 8 rows' loads ahead of their stores (possible aliasing
              // keeps them in order otherwise); R <= 16 keeps its register budget
              constexpr int UB = RP > 16 ? 8 : 1;
              for (int i0 = sub; i0 < I; i0 += UB * g) {
                double x[UB], y[UB];
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                  const int i = i0 + u * g;
                  x[u] = i < I ? A[i * R + p] : 0.0;
                  y[u] = i < I ? A[i * R + q] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                  const int i = i0 + u * g;
                  if (i < I) {
                    A[i * R + p] = c * x[u] - sn * y[u];
                    A[i * R + q] = sn * x[u] + c * y[u];
                  }
                }
              }
              for (int r = sub; r < R; r += g) {
                const double x = Vj[r * R + p], y = Vj[r * R + q];
                Vj[r * R + p] = c * x - sn * y;
                Vj[r * R + q] = sn * x + c * y;
              }
            }
            __syncwarp();
          }
          if (!__any_sync(dev::kFull, rot)) break;
        }
      }
      if (Ek) {  // right singular vectors of A = E V'
        for (int e = lane; e < RR; e += 32) {
          const int i = e / R, j = e - (e / R) * R;
          double acc = 0.0;
          for (int c = 0; c < R; ++c) acc = fma(Ek[i * R + c], Vj[c * R + j], acc);
          B[e] = acc;
        }
        __syncwarp();
        for (int e = lane; e < RR; e += 32) Vj[e] = B[e];
        __syncwarp();
      }
      // singular values (of the scaled A), U columns in place
      for (int c = 0; c < R; ++c) {
        double acc = 0.0;
        for (int i = lane; i < I; i += 32) acc = fma(A[i * R + c], A[i * R + c], acc);
        acc = dev::warp_sum(acc);
        if (lane == 0) sig[c] = sqrt(acc);
      }
      __syncwarp();
      double smax = 0.0;
      for (int c = 0; c < R; ++c) smax = fmax(smax, sig[c]);
      for (int c = 0; c < R; ++c)
        if (sig[c] * sig[c] > kNullRatio * smax * smax) ++rho;
      for (int i = lane; i < I; i += 32)
        for (int c = 0; c < R; ++c) {
          const double sc = sig[c];
          A[i * R + c] = (sc * sc > kNullRatio * smax * smax) ? A[i * R + c] / sc : 0.0;
        }
      __syncwarp();
      flag = rho == R ? P2G_FLAG_ACCURATE : P2G_FLAG_DEFICIENT;
    }
    // Completion for rho < R (D5): Q = U Vs^T + polar(N) Vn^T,
    // N = L Vn - U (U^T L Vn), N^T N = I - B^T B, B = U^T L Vn (rho x nn).
    // Strong columns c: sig[c]^2 > thr (A col c holds U_c); null columns: A col c == 0.
    double smax2 = 0.0;
    for (int c = 0; c < R; ++c) smax2 = fmax(smax2, sig[c] * sig[c]);
    const int nn = R - rho;
    if (nn > 0) {
      // B (R x R buffer, only strong rows / null cols used): B[c][d] = sum_{i<R} U[i][c] Vn[i][d]
      for (int e = lane; e < RR; e += 32) {
        const int c = e / R, d = e - (e / R) * R;
        double acc = 0.0;
        const bool cs_ = amax != 0.0 && sig[c] * sig[c] > kNullRatio * smax2;
        const bool dn = !(amax != 0.0 && sig[d] * sig[d] > kNullRatio * smax2);
        if (cs_ && dn)
          for (int i = 0; i < R; ++i) acc = fma(A[i * R + c], Vj[i * R + d], acc);
        B[e] = acc;
      }
      __syncwarp();
      // polar(N) as the oracle computes it: N = L Vn - U (U^T L Vn) built
      // explicitly in the (zeroed) null columns of A, then one-sided Jacobi
      // over the null-column pairs (same rotations and threshold as
      // one_sided_jacobi).  TN = V_N diag(1/sigma_N) V_N^T, so polar(N) = N TN.
      // (Forming N^T N = I - B^T B instead cancels catastrophically when |N|
      // is small: relative error eps / |N|^2.)
      if (lane == 0) {
        int cnt = 0;
        for (int c = 0; c < R; ++c)
          if (!(amax != 0.0 && sig[c] * sig[c] > kNullRatio * smax2)) pq[cnt++] = c;
      }
      __syncwarp();
      for (int i = lane; i < I; i += 32)
        for (int x = 0; x < nn; ++x) {
          const int d = pq[x];
          double v = (i < R) ? Vj[i * R + d] : 0.0;
          for (int c = 0; c < R; ++c) v -= A[i * R + c] * B[c * R + d];  // B = 0 on null rows c
          A[i * R + d] = v;
        }
      for (int e = lane; e < nn * nn; e += 32) EE[e] = (e / nn == e % nn) ? 1.0 : 0.0;
      __syncwarp();
      for (int sweep = 0; sweep < 80; ++sweep) {
        int rotated = 0;
        for (int x = 0; x < nn - 1; ++x)
          for (int y = x + 1; y < nn; ++y) {
            const int p = pq[x], q = pq[y];
            double al = 0.0, be = 0.0, ga = 0.0;
            for (int i = lane; i < I; i += 32) {
              const double u = A[i * R + p], w = A[i * R + q];
              al = fma(u, u, al);
              be = fma(w, w, be);
              ga = fma(u, w, ga);
            }
            al = dev::warp_sum(al);
            be = dev::warp_sum(be);
            ga = dev::warp_sum(ga);
            if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
            rotated = 1;
            const double zeta = (be - al) / (2.0 * ga);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + t * t);
            const double sn = c * t;
            for (int i = lane; i < I; i += 32) {
              const double u = A[i * R + p], w = A[i * R + q];
              A[i * R + p] = c * u - sn * w;
              A[i * R + q] = sn * u + c * w;
            }
            for (int r = lane; r < nn; r += 32) {
              const double u = EE[r * nn + x], w = EE[r * nn + y];
              EE[r * nn + x] = c * u - sn * w;
              EE[r * nn + y] = sn * u + c * w;
            }
            __syncwarp();
          }
        if (!rotated) break;
      }
      for (int x = 0; x < nn; ++x) {
        double acc = 0.0;
        for (int i = lane; i < I; i += 32) acc = fma(A[i * R + pq[x]], A[i * R + pq[x]], acc);
        acc = dev::warp_sum(acc);
        if (lane == 0) EA[x] = sqrt(acc);  // sigma_N
      }
      __syncwarp();
      double emin = 1e308;
      for (int x = 0; x < nn; ++x) emin = fmin(emin, EA[x] * EA[x]);
      if (!(emin > 1e-8)) flag = P2G_FLAG_DEGENERATE;
      for (int e = lane; e < nn * nn; e += 32) {
        const int x = e / nn, y = e - (e / nn) * nn;
        double acc = 0.0;
        for (int m = 0; m < nn; ++m) acc += EE[x * nn + m] * EE[y * nn + m] / fmax(EA[m], 1e-300);
        TN[e] = acc;
      }
      __syncwarp();
    }
    // Q-free form for the streaming kernels: Q = A Shat + L Chat with
    //   Shat = sum_c V_c V_c^T / sigma_c - sum_c V_c / sigma_c (B TN Vn^T)_c
    //   Chat = Vn TN Vn^T
    // (strong c; sigma of the unscaled A = sig * amax).
    if (a.Shat) {
      double* Sh = a.Shat + k * RR;
      double* Ch = a.Chat + k * RR;
      for (int e = lane; e < RR; e += 32) {
        const int i = e / R, j = e - (e / R) * R;
        double sh = 0.0, chv = 0.0;
        for (int c = 0; c < R; ++c) {
          const bool strong_c = amax != 0.0 && sig[c] * sig[c] > kNullRatio * smax2;
          if (!strong_c) continue;
          double vj = Vj[j * R + c];
          if (nn > 0) {  // subtract (B TN Vn^T)(c, j)
            int x = 0;
            for (int d = 0; d < R; ++d) {
              const bool dn = !(amax != 0.0 && sig[d] * sig[d] > kNullRatio * smax2);
              if (!dn) continue;
              double btn = 0.0;  // (B TN)(c, x)
              int y = 0;
              for (int d2 = 0; d2 < R; ++d2) {
                const bool dn2 = !(amax != 0.0 && sig[d2] * sig[d2] > kNullRatio * smax2);
                if (!dn2) continue;
                btn = fma(B[c * R + d2], TN[y * nn + x], btn);
                ++y;
              }
              vj -= btn * Vj[j * R + d];
              ++x;
            }
          }
          sh = fma(Vj[i * R + c] / (sig[c] * amax), vj, sh);
        }
        if (nn > 0) {
          int x = 0;
          for (int d = 0; d < R; ++d) {
            const bool dn = !(amax != 0.0 && sig[d] * sig[d] > kNullRatio * smax2);
            if (!dn) continue;
            int y = 0;
            for (int d2 = 0; d2 < R; ++d2) {
              const bool dn2 = !(amax != 0.0 && sig[d2] * sig[d2] > kNullRatio * smax2);
              if (!dn2) continue;
              chv = fma(Vj[i * R + d] * TN[x * nn + y], Vj[j * R + d2], chv);
              ++y;
            }
            ++x;
          }
        }
        Sh[e] = sh;
        Ch[e] = chv;
      }
    }
    // Q rows (lane = row), then m1_k = Q^T XV D through 32-row chunks.
    for (int b = 0; b < I; b += 32) {
      const int i = b + lane;
      const int nr = min(32, I - b);
      double xv[RP];
      double q[RP];
#pragma unroll
      for (int r = 0; r < RP; ++r) q[r] = 0.0;
      if (i < I) {
        dev::csr_row_times<RP>(xv, a.X.ci, a.X.val, a.X.rp[r0 + i], a.X.rp[r0 + i + 1], a.V, R);
        // strong part: sum_c U[i][c] Vj[:, c]
        for (int c = 0; c < R; ++c) {
          const bool strong_c = amax != 0.0 && sig[c] * sig[c] > kNullRatio * smax2;
          if (!strong_c) continue;
          const double u = A[i * R + c];
#pragma unroll
          for (int r = 0; r < RP; ++r)
            if (r < R) q[r] = fma(u, Vj[r * R + c], q[r]);
        }
        if (nn > 0) {
          // N[i][x] = (i<R ? Vn[i][x] : 0) - sum_c U[i][c] B[c][dx]; polar row = N[i] TN
          double nrow[RP];
          int cnt = 0;
          for (int d = 0; d < R; ++d) {
            const bool isnull = !(amax != 0.0 && sig[d] * sig[d] > kNullRatio * smax2);
            if (!isnull) continue;
            double v = (i < R) ? Vj[i * R + d] : 0.0;
            for (int c = 0; c < R; ++c) v -= A[i * R + c] * B[c * R + d];
            nrow[cnt < RP ? cnt : RP - 1] = v;
            ++cnt;
          }
          int xi = 0;
          for (int d = 0; d < R; ++d) {
            const bool isnull = !(amax != 0.0 && sig[d] * sig[d] > kNullRatio * smax2);
            if (!isnull) continue;
            double pn = 0.0;
            for (int y = 0; y < nn; ++y) pn = fma(nrow[y < RP ? y : RP - 1], TN[y * nn + xi], pn);
#pragma unroll
            for (int r = 0; r < RP; ++r)
              if (r < R) q[r] = fma(pn, Vj[r * R + d], q[r]);
            ++xi;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < RP; ++r) xv[r] = 0.0;
      }
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        qch[lane * RP + r] = q[r];
        xch[lane * RP + r] = (r < R) ? xv[r] * s[r] : 0.0;
      }
      __syncwarp();
      double* qdst = a.Q + (r0 + b) * R;
      if (a.Q)
        for (int idx = lane; idx < nr * R; idx += 32) qdst[idx] = qch[(idx / R) * RP + (idx - (idx / R) * R)];
      for (int e = lane; e < RR; e += 32) {
        const int x = e / R, y = e - (e / R) * R;
        double acc = M1[e];
        for (int rr = 0; rr < nr; ++rr) acc = fma(qch[rr * RP + x], xch[rr * RP + y], acc);
        M1[e] = acc;
      }
      __syncwarp();
    }
    if (lane == 0) a.flags[k] = flag;
    __syncwarp();
  }
  __syncthreads();
  if (wid == 0) {
    for (int e = lane; e < RR; e += 32) {
      double acc = 0.0;
      for (int w = 0; w < WPB; ++w)
        acc += a.scratch[(static_cast<std::int64_t>(blockIdx.x) * WPB + w) * AccSmem<RP>::slab(a.max_rows, R) +
                         RP * RP + e];
      m1_partials_acc[static_cast<std::int64_t>(blockIdx.x) * RR + e] = acc;
    }
  }
}

__global__ void k_flag_bytes(std::int64_t K, const std::int32_t* __restrict__ flags, unsigned char* __restrict__ out) {
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < K;
       k += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    out[k] = flags[k] == P2G_FLAG_ACCURATE ? 1 : 0;
}

/// Ascending list of the subjects flagged for the accurate path (stable select).
void compact_flagged(p2g_ctx* c, const std::int32_t* flags, cudaStream_t s) {
  const std::int64_t K = c->k_end - c->k_begin;
  c->acc_list.resize(static_cast<std::size_t>(std::max<std::int64_t>(K, 1)) + 1);
  c->acc_bytes.resize(static_cast<std::size_t>(std::max<std::int64_t>(K, 1)));
  std::int32_t* nsel = c->acc_list.get() + std::max<std::int64_t>(K, 1);
  if (K == 0) {
    P2G_CUDA(cudaMemsetAsync(nsel, 0, sizeof(std::int32_t), s));
    return;
  }
  const int blocks = static_cast<int>(std::min<std::int64_t>((K + 255) / 256, 148 * 16));
  k_flag_bytes<<<blocks, 256, 0, s>>>(K, flags, c->acc_bytes.get());
  thrust::counting_iterator<std::int32_t> idx(0);
  std::size_t tbytes = 0;
  P2G_CUDA(cub::DeviceSelect::Flagged(nullptr, tbytes, idx, c->acc_bytes.get(), c->acc_list.get(), nsel,
                                      static_cast<int>(K), s));
  c->acc_temp.resize(tbytes);
  P2G_CUDA(cub::DeviceSelect::Flagged(c->acc_temp.get(), tbytes, idx, c->acc_bytes.get(), c->acc_list.get(), nsel,
                                      static_cast<int>(K), s));
}

template <int RP>
constexpr int acc_wpb() {
  return 4;
}

template <int RP>
int acc_blocks(const p2g_ctx* c) {  // 4-warp CTAs: 8 warps/SM at R > 16 (254 registers), 16 below
  return std::max(1, c->num_sms * (RP <= 16 ? 4 : 2));
}

template <int RP>
void launch_acc(p2g_ctx* c, const K1Args& a, double* m1p, cudaStream_t s) {
  constexpr int WPB = acc_wpb<RP>();
  const std::size_t smem = sizeof(double) * (RP * RP + WPB * AccSmem<RP>::kPerWarpDoubles);
  auto kern = k_procrustes_accurate<RP, WPB>;
  P2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<acc_blocks<RP>(c), WPB * 32, smem, s>>>(a, m1p);
  P2G_LAUNCHED(1);
}

}  // namespace

#define P2G_RP_DISPATCH(R, CALL)                         \
  do {                                                   \
    if ((R) <= 2) {                                      \
      constexpr int RP_ = 2;                             \
      CALL;                                              \
    } else if ((R) <= 4) {                               \
      constexpr int RP_ = 4;                             \
      CALL;                                              \
    } else if ((R) <= 5) {                               \
      constexpr int RP_ = 5;                             \
      CALL;                                              \
    } else if ((R) <= 8) {                               \
      constexpr int RP_ = 8;                             \
      CALL;                                              \
    } else if ((R) <= 10) {                              \
      constexpr int RP_ = 10;                            \
      CALL;                                              \
    } else if ((R) <= 16) {                              \
      constexpr int RP_ = 16;                            \
      CALL;                                              \
    } else if ((R) <= 24) {                              \
      constexpr int RP_ = 24;                            \
      CALL;                                              \
    } else if ((R) <= 32) {                              \
      constexpr int RP_ = 32;                            \
      CALL;                                              \
    } else if ((R) <= 40) {                              \
      constexpr int RP_ = 40;                            \
      CALL;                                              \
    } else {                                             \
      throw InvalidArgument("rank above 40 unsupported"); \
    }                                                    \
  } while (0)

int launch_procrustes_accurate(p2g_ctx* c, int R, const double* H, const double* V, const double* W, double* Q,
                               std::int32_t* flags, double* m1_partials, const double* Ebuf, double* Shat,
                               double* Chat, cudaStream_t s) {
  K1Args a{};
  a.Ebuf = Ebuf;
  a.Shat = Shat;
  a.Chat = Chat;
  a.X = ShardArgs{c->srp.get(), c->rp.get(), c->ci.get(), c->val.get(), c->k_end - c->k_begin, c->NR, c->nnz, c->J};
  a.R = R;
  a.H = H;
  a.V = V;
  a.W = W;
  a.Q = Q;
  a.flags = flags;
  a.max_rows = c->max_rows;
  a.counters = c->counters.get();
  compact_flagged(c, flags, s);
  P2G_LAUNCHED(2);
  a.list = c->acc_list.get();
  a.nlist = c->acc_list.get() + std::max<std::int64_t>(c->k_end - c->k_begin, 1);
  int blocks = 0, wpb = 1;
  P2G_RP_DISPATCH(R, (blocks = acc_blocks<RP_>(c), wpb = acc_wpb<RP_>()));
  // Per-warp global slabs: A (I_max x R) of the subject in flight and the
  // R x R work matrices (AccSmem).
  std::size_t per_warp = 0;
  P2G_RP_DISPATCH(R, per_warp = AccSmem<RP_>::slab(c->max_rows, R));
  grow_scratch(c->acc_scratch, static_cast<std::size_t>(blocks) * wpb * per_warp, "accurate Procrustes path",
               c->max_rows);
  a.scratch = c->acc_scratch.get();
  P2G_RP_DISPATCH(R, launch_acc<RP_>(c, a, m1_partials, s));
  return blocks;
}

int procrustes_accurate_blocks(p2g_ctx* c, int R) {
  int blocks = 0;
  P2G_RP_DISPATCH(R, blocks = acc_blocks<RP_>(c));
  return blocks;
}

}  // namespace p2g
