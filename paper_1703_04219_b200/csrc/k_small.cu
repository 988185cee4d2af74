// Small-rank (R <= 16) pipeline of the Procrustes step and the batched NNLS.
//
// The R x R dense work of the Procrustes step (eigendecomposition of the
// Gram matrix, the polar factor) is inherently serial per subject.  A warp
// cooperating on one 10 x 10 Jacobi spends most issue slots on index math,
// shuffles and synchronisation (profiles/: ~28.8K warp instructions per
// subject).  Here each thread owns one subject: the packed Gram matrix lives
// in registers (static indices from fully unrolled rotations), the
// eigenvectors in the thread's column of a [element][lane] shared-memory
// array (conflict-free: all lanes touch the same element index).
//
// Split of K1 (procrustes_update, solver.hpp:173-193, + mode-1 partial):
//   K1a  k_gram_c      warp per subject: C_k = (X_k V)^T (X_k V), packed lower
//   K1b  k_polar_small thread per subject: G = H D C D H^T, Jacobi eig,
//                      S = G^{-1/2}, m1_k = S H D C D, flags
//   K1c  k_qrows       warp per subject: Q_k = X_k V D H^T S (rows, coalesced)
// The accurate path (k_procrustes.cu) takes the flagged subjects.
#include <algorithm>
#include <cstdlib>
#include <utility>

#include <cub/device/device_radix_sort.cuh>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"

namespace p2g {
namespace {

constexpr int LD = 33;  // [element][lane] stride (conflict-free both ways)

__host__ __device__ constexpr int tri(int i, int j) { return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i; }

// ---------------------------------------------------------------------------
// K1a: C_k = XV^T XV (packed lower triangle) for every subject.
// ---------------------------------------------------------------------------
template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_gram_c(ShardArgs X, int R, const double* __restrict__ V, double* __restrict__ Cbuf) {
  __shared__ double chunk[WPB][32 * RP];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* ch = chunk[wid];
  constexpr int NTP = RP * (RP + 1) / 2;
  constexpr int kTri = (NTP + 31) / 32;
  const int nt = R * (R + 1) / 2;
  int ea[kTri], eb[kTri];
#pragma unroll
  for (int t = 0; t < kTri; ++t) {
    const int e = lane + 32 * t;
    int x = 0;
    while ((x + 1) * (x + 2) / 2 <= e) ++x;
    ea[t] = x;
    eb[t] = e - x * (x + 1) / 2;
  }
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < X.K; k += nwarps) {
    const std::int64_t r0 = X.srp[k];
    const int I = static_cast<int>(X.srp[k + 1] - r0);
    double cacc[kTri];
#pragma unroll
    for (int t = 0; t < kTri; ++t) cacc[t] = 0.0;
    for (int b = 0; b < I; b += 32) {
      const int i = b + lane;
      const int nr = min(32, I - b);
      double xv[RP];
      if (i < I) {
        dev::csr_row_times<RP>(xv, X.ci, X.val, X.rp[r0 + i], X.rp[r0 + i + 1], V, R);
      } else {
#pragma unroll
        for (int r = 0; r < RP; ++r) xv[r] = 0.0;
      }
#pragma unroll
      for (int r = 0; r < RP; ++r) ch[lane * RP + r] = xv[r];
      __syncwarp();
#pragma unroll
      for (int t = 0; t < kTri; ++t) {
        if (lane + 32 * t < nt) {
          double acc = cacc[t];
          for (int rr = 0; rr < nr; ++rr) acc = fma(ch[rr * RP + ea[t]], ch[rr * RP + eb[t]], acc);
          cacc[t] = acc;
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int t = 0; t < kTri; ++t)
      if (lane + 32 * t < nt) Cbuf[k * nt + lane + 32 * t] = cacc[t];
  }
}

// ---------------------------------------------------------------------------
// K1b: thread-per-subject polar factor.  Jacobi on G = H C' H^T with
// C' = D C D (rotation form of the oracle / Numerical Recipes); the fast path
// keeps the subject when lambda_min >= kFastRatio lambda_max, otherwise flags
// it for the accurate path and hands it the eigenvectors as a preconditioner.
//
// Ordering: parallel (tournament) rounds.  In every round the MP/2 rotations
// act on the fixed physical slot pairs (2i, 2i+1), so they are independent
// instruction streams (ILP) with compile-time register indices; after each
// round the register-resident G is permuted by the fixed tournament shift
// sigma, which brings the next round's pairs into the same slots.  The round
// loop itself is not unrolled, keeping the code inside the instruction cache
// (a fully unrolled sweep stalled on "no_instructions", profiles/).
// Eigenvectors stay in logical order in shared memory; their columns are
// addressed through the runtime slot -> index map L(r, s).
// ---------------------------------------------------------------------------
constexpr double kFastRatio = 1e-6;
constexpr int kMaxSweeps = 16;  // not converged -> accurate path

/// Logical index held by physical slot s in round r (M players, M even).
__host__ __device__ constexpr int rr_slot(int M, int r, int s) {
  return s == 0 ? r : (s == 1 ? M - 1 : ((s & 1) == 0 ? (r + s / 2) % (M - 1) : (r - s / 2 + (M - 1)) % (M - 1)));
}

/// Physical slot holding logical index i at the start of a sweep (round 0).
__host__ __device__ constexpr int rr_inv0(int M, int i) {
  return i == 0 ? 0 : (i == M - 1 ? 1 : (i <= M / 2 - 1 ? 2 * i : 2 * (M - 1 - i) + 1));
}

/// Physical slot that slot s moves to between consecutive rounds.
__host__ __device__ constexpr int rr_sigma(int M, int s) {
  if (s == 1) return 1;
  const int d = s == 0 ? 0 : ((s & 1) == 0 ? s / 2 : (M - 1) - s / 2);
  const int d2 = (d - 1 + (M - 1)) % (M - 1);
  return d2 == 0 ? 0 : (d2 <= M / 2 - 1 ? 2 * d2 : 2 * ((M - 1) - d2) + 1);
}

/// Cycle decomposition (compile time) of the packed-index permutation
/// e = tri(x, y) -> tri(sigma x, sigma y).  cyc lists each cycle as
/// e0, perm(e0), perm(perm(e0)), ...
template <int MP>
struct PermCycles {
  static constexpr int NT = MP * (MP + 1) / 2;
  int cyc[NT] = {};
  int start[NT] = {};
  int len[NT] = {};
  int ncycles = 0;
  constexpr PermCycles() {
    int perm[NT] = {};
    for (int x = 0; x < MP; ++x)
      for (int y = 0; y <= x; ++y) perm[tri(x, y)] = tri(rr_sigma(MP, x), rr_sigma(MP, y));
    bool seen[NT] = {};
    int pos = 0;
    for (int e0 = 0; e0 < NT; ++e0) {
      if (seen[e0]) continue;
      start[ncycles] = pos;
      int e = e0, n = 0;
      while (!seen[e]) {
        seen[e] = true;
        cyc[pos++] = e;
        ++n;
        e = perm[e];
      }
      len[ncycles++] = n;
    }
  }
};

template <int MP>
struct PermTable {
  static constexpr PermCycles<MP> value{};
  /// index of the cycle containing flattened position t
  static constexpr int cycle_of(int t) {
    int c = 0;
    while (c + 1 < value.ncycles && value.start[c + 1] <= t) ++c;
    return c;
  }
};

/// One step of the cycle walk at flattened position T.
template <int MP, int T>
__device__ __forceinline__ void perm_step(double (&g)[MP * (MP + 1) / 2], double& carry) {
  constexpr int c = PermTable<MP>::cycle_of(T);
  constexpr int s = PermTable<MP>::value.start[c];
  constexpr int n = PermTable<MP>::value.len[c];
  constexpr int e = PermTable<MP>::value.cyc[T];
  constexpr int e0 = PermTable<MP>::value.cyc[s];
  if constexpr (n == 1) {
    // fixed point
  } else if constexpr (T == s) {
    carry = g[e];
  } else {
    const double tmp = g[e];
    g[e] = carry;
    carry = tmp;
    if constexpr (T == s + n - 1) g[e0] = carry;
  }
}

template <int MP, int... Ts>
__device__ __forceinline__ void perm_steps(double (&g)[MP * (MP + 1) / 2], double& carry,
                                           std::integer_sequence<int, Ts...>) {
  (perm_step<MP, Ts>(g, carry), ...);
}

/// E lives in the thread's pair-packed column store: logical element
/// (row k, column a) at ec = a * MP + k, unit ec / 2 of 16 bytes at
/// (unit * 32 + lane): a rotation streams both columns with LDS.128/STS.128,
/// and the 32 lanes of a warp hit 32 consecutive 16-byte words.
template <int MP>
__device__ __forceinline__ void jacobi_round(double (&g)[MP * (MP + 1) / 2], double2* E2, int r) {
  constexpr int H = MP / 2;
  double cs[H], sn[H], tt[H], ap[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int p = 2 * i, q = 2 * i + 1;
    const double apq = g[tri(q, p)];
    const double app = g[tri(p, p)], aqq = g[tri(q, q)];
    cs[i] = 1.0;
    sn[i] = 0.0;
    tt[i] = 0.0;
    ap[i] = 0.0;
    const double a2 = apq * apq;
    const double d = aqq - app;
    const double rho2 = fma(d, d, 4.0 * a2);
    // (rho2 > 1e-300 keeps the approximate rsqrt in its normal range; with
    // max |G| = 1 a smaller pair is far below the convergence threshold.)
    if (a2 > 4.84e-36 * fabs(app * aqq) && rho2 > 1e-300) {
      // t = tan(phi) of the annihilating rotation (the oracle's
      // sign(theta) / (|theta| + sqrt(theta^2 + 1)), theta = d / 2apq),
      // from cos(2 phi) = |d| / rho, sin(2 phi) = 2 apq sign(d) / rho,
      // rho = sqrt(d^2 + 4 apq^2): two reciprocal square roots, no division.
      const double u = dev::rsqrt_nr(rho2);
      const double cos2 = fabs(d) * u;
      const double sin2 = (d >= 0.0 ? 2.0 : -2.0) * apq * u;
      const double x = fma(0.5, cos2, 0.5);  // cos^2(phi)
      const double rc = dev::rsqrt_nr(x);     // 1 / cos(phi)
      const double s = 0.5 * sin2 * rc;
      cs[i] = x * rc;
      sn[i] = s;
      tt[i] = s * rc;
      ap[i] = apq;
    }
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int p = 2 * i, q = 2 * i + 1;
    g[tri(p, p)] -= tt[i] * ap[i];
    g[tri(q, q)] += tt[i] * ap[i];
    if (sn[i] != 0.0) g[tri(q, p)] = 0.0;
  }
  // constant-bound loops (a dependent inner trip count is not fully
  // unrolled, and the runtime indices then demote g to local memory)
#pragma unroll
  for (int i1 = 0; i1 < H; ++i1)
#pragma unroll
    for (int i2 = 0; i2 < H; ++i2) {
      if (i2 <= i1) continue;
      const int p1 = 2 * i1, q1 = p1 + 1, p2 = 2 * i2, q2 = p2 + 1;
      const double c1 = cs[i1], s1 = sn[i1], c2 = cs[i2], s2 = sn[i2];
      const double x11 = g[tri(p1, p2)], x12 = g[tri(p1, q2)], x21 = g[tri(q1, p2)], x22 = g[tri(q1, q2)];
      const double y11 = c2 * x11 - s2 * x12, y12 = s2 * x11 + c2 * x12;
      const double y21 = c2 * x21 - s2 * x22, y22 = s2 * x21 + c2 * x22;
      g[tri(p1, p2)] = c1 * y11 - s1 * y21;
      g[tri(q1, p2)] = s1 * y11 + c1 * y21;
      g[tri(p1, q2)] = c1 * y12 - s1 * y22;
      g[tri(q1, q2)] = s1 * y12 + c1 * y22;
    }
  // eigenvectors (logical order): columns a = L(r,2i), b = L(r,2i+1)
#pragma unroll
  for (int i = 0; i < H; ++i) {
    if (sn[i] == 0.0) continue;
    const int a = rr_slot(MP, r, 2 * i), b = rr_slot(MP, r, 2 * i + 1);
    const double c = cs[i], s = sn[i];
    double2* ea = E2 + a * H * 32;
    double2* eb = E2 + b * H * 32;
    // both columns loaded before any store (the compiler cannot tell that
    // columns a and b do not overlap and would otherwise serialise each
    // load behind the previous store)
    double2 va[H], vb[H];
#pragma unroll
    for (int kk = 0; kk < H; ++kk) {
      va[kk] = ea[kk * 32];
      vb[kk] = eb[kk * 32];
    }
#pragma unroll
    for (int kk = 0; kk < H; ++kk) {
      ea[kk * 32] = make_double2(c * va[kk].x - s * vb[kk].x, c * va[kk].y - s * vb[kk].y);
      eb[kk * 32] = make_double2(s * va[kk].x + c * vb[kk].x, s * va[kk].y + c * vb[kk].y);
    }
  }
  // physical permutation g_new[tri(sigma x, sigma y)] = g_old[tri(x, y)],
  // applied along its cycles with a single carried register (all indices
  // are template constants, so g stays in registers).
  double carry = 0.0;
  perm_steps<MP>(g, carry, std::make_integer_sequence<int, MP*(MP + 1) / 2>{});
}

template <int RP>
struct PolarSmem {
  static constexpr int MP = (RP + 1) & ~1;
  static constexpr int NT = MP * (MP + 1) / 2;
  // per-lane doubles: E (MP x MP), later C' (NT) + an m1 column (MP)
  static constexpr int kLane = ((MP * MP > NT + MP ? MP * MP : NT + MP) + 1) & ~1;
  static constexpr int kPerWarp = kLane * 32;
};

template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_polar_small(std::int64_t K, int R, const double* __restrict__ H, const double* __restrict__ W,
                  const double* __restrict__ Cbuf, double* __restrict__ Sbuf, double* __restrict__ Ewarm, int /*warm*/,
                  std::int32_t* __restrict__ flags, double* __restrict__ m1_partials, int* __restrict__ dbg,
                  const std::int32_t* __restrict__ perm, std::uint8_t* __restrict__ sweeps_out) {
  extern __shared__ double smem[];
  constexpr int MP = PolarSmem<RP>::MP;
  constexpr int NT = PolarSmem<RP>::NT;
  constexpr int HP = MP / 2;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Hs = smem;                                   // R x R row-major
  double* M1w = Hs + MP * MP;                          // WPB x (R x R) warp accumulators
  double* Ew = M1w + WPB * MP * MP + wid * PolarSmem<RP>::kPerWarp;
  double2* E2 = reinterpret_cast<double2*>(Ew) + lane;
  // scalar element e of lane l's store
  auto el = [&](int l, int e) -> double& { return Ew[((e >> 1) * 32 + l) * 2 + (e & 1)]; };
  const int nt = R * (R + 1) / 2;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Hs[e] = H[e];
  for (int e = lane; e < MP * MP; e += 32) M1w[wid * MP * MP + e] = 0.0;
  __syncthreads();

  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t kb = (static_cast<std::int64_t>(blockIdx.x) * WPB + wid) * 32; kb < K; kb += nwarps * 32) {
    // subjects in the order of the previous step's sweep counts (perm), so a
    // warp's 32 subjects need similar numbers of sweeps (the warp runs until
    // its slowest lane converges)
    const bool active = kb + lane < K;
    const std::int64_t k = active ? (perm ? static_cast<std::int64_t>(perm[kb + lane]) : kb + lane) : K;
    const int nk = static_cast<int>(min(static_cast<std::int64_t>(32), K - kb));
    double s[MP];
#pragma unroll
    for (int r = 0; r < MP; ++r) s[r] = (active && r < R) ? W[k * R + r] : 0.0;
    // G = H C' H^T with C' = D C D held in registers; rows of G go to this
    // lane's store physically permuted (slot x holds logical rr_slot(MP,0,x)).
    {
      double cp[NT];
#pragma unroll
      for (int a = 0; a < MP; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) cp[tri(a, b)] = (active && a < R) ? s[a] * Cbuf[k * nt + tri(a, b)] * s[b] : 0.0;
#pragma unroll
      for (int i = 0; i < MP; ++i) {
        double z[MP];  // row i of H C'
#pragma unroll
        for (int b = 0; b < MP; ++b) z[b] = 0.0;
        if (i < R) {
#pragma unroll
          for (int a = 0; a < MP; ++a) {
            if (a >= R) continue;
            const double h = Hs[i * R + a];
#pragma unroll
            for (int b = 0; b < MP; ++b) z[b] = fma(h, cp[tri(a, b)], z[b]);
          }
        }
#pragma unroll
        for (int j = 0; j <= i; ++j) {
          double acc = 0.0;
          if (i < R) {
#pragma unroll
            for (int b = 0; b < MP; ++b)
              if (b < R) acc = fma(z[b], Hs[j * R + b], acc);
          } else {
            acc = i == j ? 1.0 : 0.0;  // padding: identity block
          }
          el(lane, tri(rr_inv0(MP, i), rr_inv0(MP, j))) = acc;
        }
      }
    }
    double g[NT];
#pragma unroll
    for (int e = 0; e < NT; ++e) g[e] = el(lane, e);
    double gmax = 0.0;
    bool finite = true;
#pragma unroll
    for (int e = 0; e < NT; ++e) {
      finite &= isfinite(g[e]);
      gmax = fmax(gmax, fabs(g[e]));
    }
    bool ok = active && finite && gmax > 0.0;
    // scale to max |G| = 1 (the rotation formulas square entries)
    const double gscale = ok ? 1.0 / gmax : 1.0;
#pragma unroll
    for (int e = 0; e < NT; ++e) g[e] *= gscale;
    // E = I
#pragma unroll
    for (int u = 0; u < MP * HP; ++u) {
      const int a = u / HP, kk = u - a * HP;
      E2[u * 32] = make_double2(2 * kk == a ? 1.0 : 0.0, 2 * kk + 1 == a ? 1.0 : 0.0);
    }
    int sweeps = 0;
    if (ok) {
      bool converged = false;
      for (int sweep = 0; sweep < kMaxSweeps; ++sweep, ++sweeps) {
        double off = 0.0, dia = 0.0;
#pragma unroll
        for (int i = 0; i < MP; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) {
            if (i == j)
              dia = fma(g[tri(i, i)], g[tri(i, i)], dia);
            else
              off = fma(g[tri(i, j)], g[tri(i, j)], off);
          }
        if (off <= 1e-32 * dia) {
          converged = true;
          break;
        }
#pragma unroll 1
        for (int r = 0; r < MP - 1; ++r) jacobi_round<MP>(g, E2, r);
      }
      ok = converged;
    }
    if (active && sweeps_out) sweeps_out[k] = static_cast<std::uint8_t>(sweeps);
    if (dbg) {  // sweep statistics: sum per subject, max, sum of per-warp max, warps
      int wmax = sweeps;
      for (int o = 16; o > 0; o >>= 1) wmax = max(wmax, __shfl_xor_sync(dev::kFull, wmax, o));
      atomicAdd(dbg + 0, sweeps);
      atomicMax(dbg + 1, sweeps);
      if (lane == 0) {
        atomicAdd(dbg + 2, wmax);
        atomicAdd(dbg + 3, 1);
      }
    }
    // eigenvalues in logical order (unscaled)
    double lam[MP];
#pragma unroll
    for (int x = 0; x < MP; ++x) lam[rr_slot(MP, 0, x)] = g[tri(x, x)] * gmax;
    if (ok) {
      double lmax = 0.0, lmin = 1e308;
#pragma unroll
      for (int i = 0; i < MP; ++i)
        if (i < R) {
          lmax = fmax(lmax, lam[i]);
          lmin = fmin(lmin, lam[i]);
        }
      ok = lmax > 0.0 && lmin >= kFastRatio * lmax;
    }
    if (active) flags[k] = ok ? P2G_FLAG_FULL_RANK : P2G_FLAG_ACCURATE;
    // Eigenvectors -> Ewarm (row-major E[i][j]) for the accurate path's
    // preconditioner, flagged subjects only.
    if (active && !ok) {
      double* ew = Ewarm + k * R * R;
#pragma unroll
      for (int j = 0; j < MP; ++j)
#pragma unroll
        for (int i = 0; i < MP; ++i)
          if (i < R && j < R) ew[i * R + j] = el(lane, j * MP + i);
    }
    // S = E diag(lambda^-1/2) E^T (logical packed, into g), column by column of E
#pragma unroll
    for (int m = 0; m < MP; ++m) lam[m] = (ok && m < R) ? rsqrt(lam[m]) : 0.0;
#pragma unroll
    for (int e = 0; e < NT; ++e) g[e] = 0.0;
#pragma unroll
    for (int m = 0; m < MP; ++m) {
      double col[MP];
#pragma unroll
      for (int kk = 0; kk < HP; ++kk) {
        const double2 v = E2[(m * HP + kk) * 32];
        col[2 * kk] = v.x;
        col[2 * kk + 1] = v.y;
      }
#pragma unroll
      for (int i = 0; i < MP; ++i) {
        const double li = lam[m] * col[i];
#pragma unroll
        for (int j = 0; j <= i; ++j) g[tri(i, j)] = fma(li, col[j], g[tri(i, j)]);
      }
    }
    // m1_k = S (H C'): C' (zero unless ok) into slots [0, NT), column j of
    // m1_k into slots [NT, NT + R); the warp sums each column over its 32
    // subjects through shared memory (fixed order) into the warp accumulator.
#pragma unroll
    for (int a = 0; a < MP; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b)
        el(lane, tri(a, b)) = (ok && a < R) ? s[a] * Cbuf[k * nt + tri(a, b)] * s[b] : 0.0;
#pragma unroll 1
    for (int j = 0; j < R; ++j) {
      double y[MP];
#pragma unroll
      for (int c = 0; c < MP; ++c) y[c] = 0.0;
#pragma unroll
      for (int a = 0; a < MP; ++a) {
        if (a >= R) continue;
        const double caj = el(lane, a >= j ? tri(a, j) : tri(j, a));
#pragma unroll
        for (int c = 0; c < MP; ++c)
          if (c < R) y[c] = fma(Hs[c * R + a], caj, y[c]);
      }
#pragma unroll
      for (int i = 0; i < MP; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < MP; ++c) acc = fma(g[i >= c ? tri(i, c) : tri(c, i)], y[c], acc);
        if (i < R) el(lane, NT + i) = acc;
      }
      __syncwarp();
      if (lane < R) {
        double acc = 0.0;
        for (int t = 0; t < 32; ++t) acc += el((lane + t) & 31, NT + lane);
        M1w[wid * MP * MP + lane * R + j] += acc;
      }
      __syncwarp();
    }
    // S out (logical packed), staged through the store for coalesced rows.
#pragma unroll
    for (int e = 0; e < NT; ++e) el(lane, e) = g[e];
    __syncwarp();
    for (int sub = 0; sub < nk; ++sub) {
      const std::int64_t ks = __shfl_sync(dev::kFull, k, sub);
      for (int e = lane; e < nt; e += 32) Sbuf[ks * nt + e] = el(sub, e);
    }
    __syncwarp();
  }
  __syncthreads();
  if (wid == 0)
    for (int e = lane; e < R * R; e += 32) {
      double acc = 0.0;
      for (int w = 0; w < WPB; ++w) acc += M1w[w * MP * MP + e];
      m1_partials[static_cast<std::int64_t>(blockIdx.x) * R * R + e] = acc;
    }
}

// ---------------------------------------------------------------------------
// Q-free forms.  With P_k = D H^T S_k (S_k = G_k^{-1/2}, packed symmetric,
// fast path) or P_k = D H^T Shat_k plus the completion term L Chat_k
// (accurate / rank-deficient subjects, full R x R in Shat/Chat), the
// Procrustes factor is Q_k = (X_k V) P_k + L Chat_k with V, H, W the factors
// the Procrustes step used.  Mode 2 and mode 3 rebuild Q rows on the fly from
// the CSR instead of reading a materialised Q (4 GB at cfg2), and mode 3 also
// emits next iteration's Gram C = (X_k V_t)^T (X_k V_t).
// ---------------------------------------------------------------------------

/// Builds P = D H^T S for subject k in shared memory (R x R row-major) and
/// returns whether the completion term applies (flagged subject).
template <int RP>
__device__ __forceinline__ bool build_p(int R, std::int64_t k, std::int32_t flag, const double* __restrict__ Sbuf,
                                        const double* __restrict__ Shat, const double* Hs, const double* __restrict__ W,
                                        double* S, double* P, int lane) {
  const int RR = R * R;
  const bool flagged = flag != P2G_FLAG_FULL_RANK;
  if (!flagged) {
    const int nt = R * (R + 1) / 2;
    for (int e = lane; e < nt; e += 32) {
      int x = 0;
      while ((x + 1) * (x + 2) / 2 <= e) ++x;
      const int y = e - x * (x + 1) / 2;
      const double v = Sbuf[k * nt + e];
      S[x * R + y] = v;
      S[y * R + x] = v;
    }
  } else {
    for (int e = lane; e < RR; e += 32) S[e] = Shat[k * RR + e];
  }
  __syncwarp();
  for (int e = lane; e < RR; e += 32) {
    const int a = e / R, b = e - (e / R) * R;
    double acc = 0.0;
    for (int c = 0; c < R; ++c) acc = fma(Hs[c * R + a], S[c * R + b], acc);
    P[e] = acc * W[k * R + a];
  }
  __syncwarp();
  return flagged;
}

/// Export: Q rows of every subject (p2g_fit Q_out, p2g_procrustes).
template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_qrows(ShardArgs X, int R, const double* __restrict__ H, const double* __restrict__ V,
            const double* __restrict__ W, const double* __restrict__ Sbuf, const double* __restrict__ Shat,
            const double* __restrict__ Chat, const std::int32_t* __restrict__ flags, double* __restrict__ Q) {
  __shared__ double Hs[RP * RP];
  __shared__ double Ps[WPB][RP * RP];
  __shared__ double Ss[WPB][RP * RP];
  __shared__ double chunk[WPB][32 * RP];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Hs[e] = H[e];
  __syncthreads();
  double* P = Ps[wid];
  double* S = Ss[wid];
  double* ch = chunk[wid];
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < X.K; k += nwarps) {
    const std::int32_t flag = flags[k];
    const bool flagged = build_p<RP>(R, k, flag, Sbuf, Shat, Hs, W, S, P, lane);
    const std::int64_t r0 = X.srp[k];
    const int I = static_cast<int>(X.srp[k + 1] - r0);
    for (int b0 = 0; b0 < I; b0 += 32) {
      const int i = b0 + lane;
      const int nr = min(32, I - b0);
      if (i < I) {
        double xv[RP];
        dev::csr_row_times<RP>(xv, X.ci, X.val, X.rp[r0 + i], X.rp[r0 + i + 1], V, R);
#pragma unroll
        for (int c = 0; c < RP; ++c) {
          if (c < R) {
            double q = (flagged && i < R) ? Chat[k * R * R + i * R + c] : 0.0;
#pragma unroll
            for (int r = 0; r < RP; ++r)
              if (r < R) q = fma(xv[r], P[r * R + c], q);
            ch[lane * RP + c] = q;
          }
        }
      }
      __syncwarp();
      double* qdst = Q + (r0 + b0) * R;
      for (int idx = lane; idx < nr * R; idx += 32) qdst[idx] = ch[(idx / R) * RP + (idx - (idx / R) * R)];
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// Thread-per-row NNLS (kernels.hpp:115-185) for R <= 16: identical control
// flow to nnls_single; passive solves by Cholesky in the thread's column of
// a [element][lane] shared array, falling back to a flag for the warp path
// when a pivot is not positive (the reference's pinv semantics).
// ---------------------------------------------------------------------------
template <int RP>
struct NnlsThreadSmem {
  static constexpr int NT = RP * (RP + 1) / 2;
  static constexpr int kPerWarp = (NT + RP) * LD;  // L, sp
};

template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_nnls_thread(int R, std::int64_t n, const double* __restrict__ G, const double* __restrict__ B,
                  double* __restrict__ X, int cap, std::int32_t* __restrict__ err, std::int32_t* __restrict__ redo,
                  std::int32_t* __restrict__ n_redo, unsigned* __restrict__ masks, int warm,
                  const double* __restrict__ ginv) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Gs = smem;
  double* Gi = Gs + RP * RP;  // G^{-1} (cold start), RP x RP
  double* Lw = Gi + RP * RP + wid * NnlsThreadSmem<RP>::kPerWarp;
  double* spw = Lw + NnlsThreadSmem<RP>::NT * LD;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gs[e] = G[e];
  const bool cold_gi = ginv && !(masks && warm) && ginv[R * R] == 1.0;
  if (cold_gi)  // k_ginv<16> wrote R x R row-major (stride R), validity at [R * R]
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gi[e] = ginv[e];
  __syncthreads();
  auto L = [&](int i, int j) -> double& { return Lw[tri(i, j) * LD + lane]; };
  auto SP = [&](int i) -> double& { return spw[i * LD + lane]; };
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t row = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; row < n; row += stride) {
    double b[RP], x[RP], w[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      b[r] = r < R ? B[row * R + r] : 0.0;
      w[r] = b[r];
      x[r] = 0.0;
    }
    // Warm start (optional): begin from the row's previous passive set.  The
    // optimum is unique (G positive definite), so only the path changes; an
    // infeasible warm solve sheds its non-positive coordinates and retries,
    // and an emptied set falls back to the reference's cold start.
    unsigned passive = (masks && warm) ? (masks[row] & ((R >= 32) ? ~0u : ((1u << R) - 1u))) : 0u;
    if (cold_gi) {  // cold row: start from the support of G^{-1} b (same unique optimum)
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        if (r >= R) continue;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < RP; ++c)
          if (c < R) acc = fma(Gi[r * R + c], b[c], acc);
        if (acc > 0.0) passive |= 1u << r;
      }
    }
    bool warm_phase = passive != 0u;
    int iters = 0;
    bool failed = false, chol_fail = false;
    while (true) {
      if (!warm_phase) {
        double best = 1e-10;
        int enter = -1;
#pragma unroll
        for (int r = 0; r < RP; ++r)
          if (r < R && !((passive >> r) & 1u) && w[r] > best) {
            best = w[r];
            enter = r;
          }
        if (enter < 0) break;
        passive |= 1u << enter;
      }
      while (true) {
        if (++iters > cap) {
          failed = true;
          break;
        }
        int pset[RP];
        int np = 0;
#pragma unroll
        for (int r = 0; r < RP; ++r)
          if ((passive >> r) & 1u) pset[np++] = r;
        // Cholesky of G_pp (lower, packed) in shared memory
        for (int i = 0; i < np; ++i) {
          for (int j = 0; j <= i; ++j) {
            double acc = Gs[pset[i] * R + pset[j]];
            for (int m = 0; m < j; ++m) acc -= L(i, m) * L(j, m);
            if (i == j) {
              if (!(acc > 0.0)) {
                chol_fail = true;
                break;
              }
              L(i, i) = sqrt(acc);
            } else {
              L(i, j) = acc / L(j, j);
            }
          }
          if (chol_fail) break;
        }
        if (chol_fail) break;
        for (int i = 0; i < np; ++i) {  // L y = b_p
          double acc = 0.0;
#pragma unroll
          for (int r = 0; r < RP; ++r)
            if (r == pset[i]) acc = b[r];
          for (int m = 0; m < i; ++m) acc -= L(i, m) * SP(m);
          SP(i) = acc / L(i, i);
        }
        for (int i = np - 1; i >= 0; --i) {  // L^T s = y
          double acc = SP(i);
          for (int m = i + 1; m < np; ++m) acc -= L(m, i) * SP(m);
          SP(i) = acc / L(i, i);
        }
        bool allpos = true;
        for (int a = 0; a < np; ++a) allpos &= SP(a) > 0.0;
        double sv[RP];
#pragma unroll
        for (int r = 0; r < RP; ++r) sv[r] = 0.0;
        for (int a = 0; a < np; ++a) {
          const double v = SP(a);
#pragma unroll
          for (int r = 0; r < RP; ++r)
            if (r == pset[a]) sv[r] = v;
        }
        if (allpos) {
#pragma unroll
          for (int r = 0; r < RP; ++r) x[r] = sv[r];
          break;
        }
        if (warm_phase) {  // x = 0 here: drop the non-positive coordinates and re-solve
#pragma unroll
          for (int r = 0; r < RP; ++r)
            if (((passive >> r) & 1u) && sv[r] <= 0.0) passive &= ~(1u << r);
          if (passive == 0u) break;
          continue;
        }
        double alpha = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
        for (int r = 0; r < RP; ++r)
          if (((passive >> r) & 1u) && sv[r] <= 0.0) {
            const double denom = x[r] - sv[r];
            alpha = fmin(alpha, denom > 0.0 ? x[r] / denom : 0.0);
          }
        double xm = 0.0;
#pragma unroll
        for (int r = 0; r < RP; ++r)
          if ((passive >> r) & 1u) x[r] += alpha * (sv[r] - x[r]);
#pragma unroll
        for (int r = 0; r < RP; ++r) xm = fmax(xm, fabs(x[r]));
        const double drop_tol = 1e-14 * fmax(1.0, xm);
#pragma unroll
        for (int r = 0; r < RP; ++r)
          if (((passive >> r) & 1u) && x[r] <= drop_tol) {
            x[r] = 0.0;
            passive &= ~(1u << r);
          }
      }
      warm_phase = false;
      if (failed || chol_fail) break;
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        if (r >= R) continue;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < RP; ++c)
          if (c < R) acc = fma(Gs[r * R + c], x[c], acc);
        w[r] = b[r] - acc;
      }
    }
    if (chol_fail) {  // this row is re-solved by the warp kernel (pinv route)
      redo[atomicAdd(n_redo, 1)] = static_cast<std::int32_t>(row);
      continue;
    }
    if (failed) atomicAdd(err, 1);
    if (masks) masks[row] = passive;
#pragma unroll
    for (int r = 0; r < RP; ++r)
      if (r < R) X[row * R + r] = x[r];
  }
}

template <int RP>
constexpr int gram_wpb() {
  int w = 8;
  while (w > 1 && w * 32 * RP * 8 > 40 * 1024) --w;
  return w;
}

__global__ void k_iota32(std::int64_t n, std::int32_t* __restrict__ out) {
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<std::int32_t>(i);
}

void fill_iota(std::int32_t* out, std::int64_t n, cudaStream_t s) {
  k_iota32<<<static_cast<int>(std::min<std::int64_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(n, out);
}

int grid_cap(std::int64_t work_warps, int wpb, int num_sms, int per_sm) {
  const std::int64_t want = (work_warps + wpb - 1) / wpb;
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(want, static_cast<std::int64_t>(num_sms) * per_sm)));
}

}  // namespace

#define P2G_SMALL_DISPATCH(R, CALL)                       \
  do {                                                    \
    if ((R) <= 2) {                                       \
      constexpr int RP_ = 2;                              \
      CALL;                                               \
    } else if ((R) <= 4) {                                \
      constexpr int RP_ = 4;                              \
      CALL;                                               \
    } else if ((R) <= 5) {                                \
      constexpr int RP_ = 5;                              \
      CALL;                                               \
    } else if ((R) <= 8) {                                \
      constexpr int RP_ = 8;                              \
      CALL;                                               \
    } else if ((R) <= 10) {                               \
      constexpr int RP_ = 10;                             \
      CALL;                                               \
    } else if ((R) <= 12) {                               \
      constexpr int RP_ = 12;                             \
      CALL;                                               \
    } else if ((R) <= 16) {                               \
      constexpr int RP_ = 16;                             \
      CALL;                                               \
    } else {                                              \
      throw InvalidArgument("small-rank path needs R <= 16"); \
    }                                                     \
  } while (0)

static ShardArgs shard_args_s(p2g_ctx* c) {
  return ShardArgs{c->srp.get(), c->rp.get(), c->ci.get(), c->val.get(), c->k_end - c->k_begin, c->NR, c->nnz, c->J};
}

void launch_gram_c(p2g_ctx* c, int R, const double* V, double* Cbuf, cudaStream_t s) {
  const ShardArgs X = shard_args_s(c);
  P2G_SMALL_DISPATCH(R, ({
                       constexpr int WPB = gram_wpb<RP_>();
                       k_gram_c<RP_, WPB><<<grid_cap(X.K, WPB, c->num_sms, 16), WPB * 32, 0, s>>>(X, R, V, Cbuf);
                     }));
  P2G_LAUNCHED(1);
}

template <int RP>
static int polar_launch(p2g_ctx* c, std::int64_t K, int R, const double* H, const double* W, const double* Cbuf,
                        double* Sbuf, double* Ewarm, int warm, std::int32_t* flags, double* m1p, int max_blocks,
                        const std::int32_t* perm, std::uint8_t* sweeps_out, cudaStream_t s) {
  constexpr int WPB = RP <= 10 ? 4 : 2;
  constexpr int MP = PolarSmem<RP>::MP;
  const std::size_t smem = sizeof(double) * (MP * MP + WPB * MP * MP + WPB * PolarSmem<RP>::kPerWarp);
  auto kern = k_polar_small<RP, WPB>;
  P2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  P2G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPB * 32, smem));
  const int blocks = grid_cap((K + 31) / 32, WPB, c->num_sms, std::max(per_sm, 1));
  const int nb = std::min(blocks, max_blocks);
  kern<<<nb, WPB * 32, smem, s>>>(K, R, H, W, Cbuf, Sbuf, Ewarm, warm, flags, m1p,
                                  c->opt.debug ? c->counters.get() + 4 : nullptr, perm, sweeps_out);
  return nb;
}

int launch_polar_small(p2g_ctx* c, int R, const double* H, const double* W, const double* Cbuf, double* Sbuf,
                       double* Ewarm, int warm, std::int32_t* flags, double* m1_partials, int max_blocks,
                       cudaStream_t s) {
  const std::int64_t K = c->k_end - c->k_begin;
  // order subjects by the previous step's sweep counts (stable, 5-bit keys)
  c->polar_sweeps.resize(static_cast<std::size_t>(std::max<std::int64_t>(K, 1)));
  const std::int32_t* perm = nullptr;
  if (c->polar_sweeps_valid && K > 0 && c->opt.polar_sort) {
    c->polar_perm.resize(static_cast<std::size_t>(2 * K));
    c->polar_keys.resize(static_cast<std::size_t>(K));
    std::int32_t* iota = c->polar_perm.get() + K;
    fill_iota(iota, K, s);
    std::size_t tbytes = 0;
    P2G_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tbytes, c->polar_sweeps.get(), c->polar_keys.get(), iota,
                                             c->polar_perm.get(), static_cast<int>(K), 0, 5, s));
    c->polar_temp.resize(tbytes);
    P2G_CUDA(cub::DeviceRadixSort::SortPairs(c->polar_temp.get(), tbytes, c->polar_sweeps.get(), c->polar_keys.get(),
                                             iota, c->polar_perm.get(), static_cast<int>(K), 0, 5, s));
    P2G_LAUNCHED(2);
    perm = c->polar_perm.get();
  }
  int nb = 0;
  P2G_SMALL_DISPATCH(R, nb = polar_launch<RP_>(c, K, R, H, W, Cbuf, Sbuf, Ewarm, warm, flags, m1_partials, max_blocks,
                                               perm, c->polar_sweeps.get(), s));
  c->polar_sweeps_valid = true;
  P2G_LAUNCHED(1);
  return nb;
}

void launch_qrows(p2g_ctx* c, int R, const double* H, const double* V, const double* W, const double* Sbuf,
                  const double* Shat, const double* Chat, const std::int32_t* flags, double* Q, cudaStream_t s) {
  const ShardArgs X = shard_args_s(c);
  P2G_SMALL_DISPATCH(R, ({
                       constexpr int WPB = RP_ <= 10 ? 8 : 4;
                       k_qrows<RP_, WPB><<<grid_cap(X.K, WPB, c->num_sms, 16), WPB * 32, 0, s>>>(
                           X, R, H, V, W, Sbuf, Shat, Chat, flags, Q);
                     }));
  P2G_LAUNCHED(1);
}

template <int RP>
static void nnls_thread_launch(int R, std::int64_t n, const double* G, const double* B, double* X, int cap,
                               std::int32_t* err, std::int32_t* redo, std::int32_t* n_redo, unsigned* masks, int warm,
                               cudaStream_t s, const double* ginv) {
  constexpr int WPB = 4;
  const std::size_t smem = sizeof(double) * (2 * RP * RP + WPB * NnlsThreadSmem<RP>::kPerWarp);
  auto kern = k_nnls_thread<RP, WPB>;
  P2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int blocks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + 127) / 128, 148 * 16)));
  kern<<<blocks, WPB * 32, smem, s>>>(R, n, G, B, X, cap, err, redo, n_redo, masks, warm, ginv);
}

void launch_nnls_thread(int R, std::int64_t n, const double* G, const double* B, double* X, int max_iter,
                        std::int32_t* err, std::int32_t* redo, std::int32_t* n_redo, unsigned* masks, int warm,
                        cudaStream_t s, const double* ginv) {
  if (n == 0) return;
  const int cap = max_iter > 0 ? max_iter : 30 * R;
  P2G_SMALL_DISPATCH(R, nnls_thread_launch<RP_>(R, n, G, B, X, cap, err, redo, n_redo, masks, warm, s, ginv));
  P2G_LAUNCHED(1);
}

}  // namespace p2g
