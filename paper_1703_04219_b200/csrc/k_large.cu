// Large-rank (R > 16) Procrustes step fused with the mode-1 partial.
//
// Replaces procrustes_update (solver.hpp:173-193) over all subjects for
// R > 16.  The oracle takes the polar factor from a one-sided Jacobi SVD of
// A_k = X_k V diag(W_k) H^T (I_k x R).  At R = 40 a sweep is R(R-1)/2 = 780
// column pairs of length I_k, and unpreconditioned A needs ~10 sweeps: far
// too slow, and the Gram route (eig of A^T A) squares the condition number.
//
// B200 design: one warp per subject, persistent (k_procrustes_large_w below).
//   E    = right singular vectors of A from the previous Procrustes step
//          (Ewarm, K x R x R in HBM; identity on the first step)
//   X~   = X_k V D (lane per row),  B = A E = X~ (H^T E)      (DMMA)
//   M    = B^T B,  F = B^T X~                                   (DMMA)
//   two-sided Jacobi on M with the oracle's rotation: in exact arithmetic
//   the one-sided Jacobi of B.  With E from the previous step the columns of
//   B are nearly orthogonal, the case in which two-sided Jacobi on M has the
//   relative accuracy of one-sided Jacobi on B (Demmel-Veselic); when they
//   are not (first step, or factors moved), E is refreshed from this solve
//   and the subject is redone once if it is also ill-conditioned
//   (sigma_min^2 < 1e-6 sigma_max^2; otherwise the Gram route's eps kappa^2
//   error is below 1e-10, as in the small-R fast path).  The sweeps stop at a
//   scaled off-diagonal of 1e-4 and M'^{-1/2} gets a second-order correction
//   (below).  V_A = E V',  Q = B V' S' V_A^T = B Z,  m1_k = Q^T X~ = Z^T F.
// Rank-deficient (canonical rule D5), non-finite or non-converged subjects
// are flagged P2G_FLAG_ACCURATE and finished by k_procrustes_accurate, which
// takes V_A (stored in Ewarm) as its preconditioner.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"

namespace p2g {
namespace {

#include "jacobi_plan40.inc"

constexpr int kLgMaxSweeps = 40;
constexpr double kTinyL = 1e-24;  // M_pp below this x max diag: near-null column (covers D5's 1e-26)

struct LgArgs {
  ShardArgs X;
  int R;
  const double* H;  // R x R row-major
  const double* V;  // J x R row-major
  const double* W;  // K_s x R row-major
  double* Q;        // NR x R row-major
  std::int32_t* flags;
  double* m1_partials;  // gridDim.x x R x R
  double* Ewarm;        // K_s x R x R row-major: E in, V_A out
  int ew_valid;
  double* slab;  // per CTA: 2 x max_rows x R (B rows, X~ rows)
  std::int64_t max_rows;
  int* dbg;  // optional: [0] sweeps, [1] max sweeps, [2] redone subjects, [3] subjects
  const double* XV;  // optional: X V rows (NR x R) from the previous mode-3 pass
};

// ---------------------------------------------------------------------------
// One warp owns a subject: M and V' live in the warp's shared memory (V'
// rows 0..31 in registers during the sweeps), every R x R (and I x R)
// product runs on the fp64
// tensor cores (DMMA m8n8k4) over per-warp slabs in global memory (L1/L2
// resident), and the sweeps stop early:
//
//   Jacobi stops once the scaled off-diagonal max |M'_pq| / sqrt(M'_pp M'_qq)
//   is at most kTauL = 1e-4 (instead of ~1e-12, one to two sweeps fewer), and
//   S' = M'^{-1/2} comes from the second-order Daleckii-Krein expansion of
//   f(x) = x^{-1/2} about Lambda = diag(M'), with N = M' - Lambda:
//     S' = f(Lambda) + sum_pq f[l_p, l_q] N_pq + sum_pqr f[l_p, l_r, l_q] N_pr N_rq
//   f's divided differences have closed forms in s = sqrt(l), u = 1/s,
//   P_pq = 1/(s_p + s_q) and A = P o N:
//     S'_pq = delta_pq u_p + u_p u_q (C1 - A + P o C2)_pq,
//     C1 = A diag(u) A,  C2 = A A
//   (no eigenvalue gaps appear, so clustered eigenvalues are harmless).  The
//   truncation error in Q is O(R tau^3): measured 2.4e-12 at tau = 1e-4 (8e-11 at 3e-4) with every
//   scaled off-diagonal at tau).  Then G^{-1/2} = E' S' E'^T with E' = E V',
//   Z = V' S' E'^T, Q = B Z and m1_k = Z^T F as before.
// ---------------------------------------------------------------------------
// During the sweeps M is kept in its upper triangle only (M[min * LDM + max]):
// half the shared-memory stores of a full symmetric update.
constexpr double kTauL = 1e-4;   // Jacobi stop: max scaled off-diagonal (truncation error <= 3e-12 measured)
constexpr double kSkipL = 1e-5;  // rotations below this scaled size are skipped (threshold Jacobi; the second-order correction covers them)

template <int RP, bool EXACT = false>
struct LgWarp {
  // exact R = 40 runs the physical-order Jacobi round (jacobi_plan40.inc)
  static constexpr bool kPhys = RP == 40 && EXACT;
  static constexpr int LDM = RP + 1;  // M: odd leading dimension (column walks conflict free)
  static constexpr int LDV = RP + 2;  // V'^T: even, 16-byte rows for the paired updates
  static constexpr int LDP = RP + 1;  // kPhys: rotated rows of the physical-order M (odd stride)
  static constexpr int kMat = kPhys ? RP * LDP : RP * LDM;  // M (kPhys: Jacobi buffer 0)
  static constexpr int kVt = kPhys ? RP * LDP : RP * LDV;   // V'^T (kPhys: Jacobi buffer 1)
  static constexpr int NBLK = (RP / 2) * (RP / 2 - 1) / 2;  // off-diagonal 2 x 2 blocks (slot i1 < i2)
  // CTA tables, in doubles (even): uint16 block and round-robin tables; kPhys: the per-lane
  // plan (uint4 [6][32] and uint [6][32] per block, uint4 [32] diagonal blocks), the element
  // addresses (uint16 [820], by triangular index) and the elements in address order (uint [820])
  static constexpr int kTri = RP * (RP + 1) / 2;
  static constexpr int kTabD =
      kPhys ? ((16 * 7 * 32 + 4 * 6 * 32 + 6 * kTri + 15) / 16) * 2 : ((NBLK + (RP - 1) * (RP / 2) + 7) / 8) * 2;
  // M, V'^T, w, u (1/sqrt diag), then per pair slot and double-buffered: (c, s), t M_pq, int4 offsets
  // (kPhys: (c, s) only)
  static constexpr int kWarpD = kMat + kVt + 2 * RP + (kPhys ? 2 * RP + 2 : 2 * (RP + RP / 2 + RP));  // kPhys: + 2 mbarriers
  static constexpr int kWarpDE = (kWarpD + 1) & ~1;
  static constexpr int pick_wpb() {
    int w = 16;
    while (w > 1 && (kTabD + w * kWarpDE) * 8 > 227 * 1024) --w;
    return w;
  }
  static constexpr int WPB = pick_wpb();
  static constexpr std::size_t kSmem = sizeof(double) * (kTabD + WPB * kWarpDE);
  static constexpr int NB = RP / 8;  // 8-wide tensor tiles (RP multiple of 8)
  // per-warp global slab: B, X~ (max_rows x R each), T, F, E, N, M1 (R x R), s (R)
  __host__ __device__ static std::size_t slab_doubles(std::int64_t max_rows, int R) {
    if (kPhys) return static_cast<std::size_t>(R) * R + RP;  // the m1 partial and sqrt(diag M') (rows streamed, E in place)
    return 2 * static_cast<std::size_t>(max_rows > 1 ? max_rows : 1) * R +
           5 * static_cast<std::size_t>(R) * R + RP;
  }
};

/// Logical index held by physical position x (pair slot x / 2, p side for even
/// x, q side for odd x) in round 0 of the round-robin of sched below; after a
/// round every position moves along one fixed cycle (see the V' rows below).
__host__ __device__ constexpr int rr_l0(int m, int x) {
  return (x & 1) ? ((x >> 1) == 0 ? m - 1 : m - 1 - (x >> 1)) : (x >> 1);
}

/// dst[e] = src[e], e < n, by a warp: 8 loads in flight per lane ahead of
/// the stores (global to global: the compiler cannot reorder them itself).
__device__ __forceinline__ void warp_copy(double* dst, const double* src, int n, int lane) {
  for (int e0 = 0; e0 < n; e0 += 256) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + lane + 32 * u;
      t[u] = e < n ? src[e] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + lane + 32 * u;
      if (e < n) dst[e] = t[u];
    }
  }
}

/// out(i, j) for i < rows, j < R of the product sum_c a(i, c) b(c, j), c < R,
/// on DMMA m8n8k4 (row.col): lane (fm, fk) feeds A[fm][fk] and B[fk][fm] and
/// holds C[fm][2 fk + h].  8-row tiles of the output in turn, all RP/8
/// column tiles at once.
template <int RP, bool EXACT, class FA, class FB, class Epi>
__device__ __forceinline__ void warp_mm(int rows, int R, FA fa, FB fb, Epi epi) {
  constexpr int NB = RP / 8;
  const int lane = threadIdx.x & 31, fm = lane >> 2, fk = lane & 3;
  // two 8-row tiles per pass: every B fragment (a shared-memory or global load per lane) feeds two
  // DMMAs; the accumulation order per output element is that of one tile at a time
#pragma unroll 1
  for (int i0 = 0; i0 < rows; i0 += 16) {
    const int ia = i0 + fm, ib = i0 + 8 + fm;
    const bool va = ia < rows, vb = ib < rows;
    double acc[2][NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[0][b][0] = acc[0][b][1] = acc[1][b][0] = acc[1][b][1] = 0.0;
#pragma unroll 2
    for (int k4 = 0; k4 < RP; k4 += 4) {
      const int c = k4 + fk;
      const bool cv = EXACT || c < R;
      const double xa = (va && cv) ? fa(ia, c) : 0.0;
      const double xb = (vb && cv) ? fa(ib, c) : 0.0;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int j = 8 * b + fm;
        const double y = (cv && (EXACT || j < R)) ? fb(c, j) : 0.0;
        dev::dmma884(acc[0][b], xa, y);
        dev::dmma884(acc[1][b], xb, y);
      }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int i = t ? ib : ia;
      if (i < rows) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 8 * b + 2 * fk + h;
            if (EXACT || j < R) epi(i, j, acc[t][b][h]);
          }
      }
    }
  }
}

template <int RP, bool EXACT>
__global__ void __launch_bounds__(LgWarp<RP>::WPB * 32, 1) k_procrustes_large_w(LgArgs a) {
  using L = LgWarp<RP, EXACT>;
  constexpr int LDM = L::LDM, LDV = L::LDV, NB = L::NB, WPB = L::WPB;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int R = EXACT ? RP : a.R;
  const int RR = R * R;
  const int m = (R + 1) & ~1, half = m / 2, nblk = half * (half - 1) / 2;
  // exact R = 40: the physical-order Jacobi round (jacobi_plan40.inc)
  constexpr bool kPhys = L::kPhys;
  constexpr int LDVx = kPhys ? LDM : LDV;  // V'^T leading dimension after the sweeps
  std::uint16_t* blk = reinterpret_cast<std::uint16_t*>(smem);  // 2 x 2 block (slot i1, slot i2) of M
  std::uint16_t* sched = blk + L::NBLK;                         // round-robin (p, q) per (round, slot)
  uint4* pplan = reinterpret_cast<uint4*>(smem);                // kPhys: [6][32] blocks, [32] diagonal
  unsigned* pplan5 = reinterpret_cast<unsigned*>(pplan + 7 * 32);  // kPhys: [6][32] 5th word of a block
  unsigned* pelem = pplan5 + 6 * 32;  // kPhys: M's elements in address order (addr | x << 16 | y << 24)
  std::uint16_t* paddr = reinterpret_cast<std::uint16_t*>(pelem + L::kTri);  // kPhys: address of (x <= y)
  double* M = smem + L::kTabD + wid * L::kWarpDE;
  double* Vt = M + L::kMat;  // V'^T: Vt[p * LDV + k] = V'(k, p)
  double* w = Vt + L::kVt;
  double* u = w + RP;
  // per slot, double-buffered by round parity: (c, s), t M_pq, and the offsets
  // (p LDM, q LDM, p, q; q < 0: no pair)
  double2* rotb = reinterpret_cast<double2*>(u + RP);
  double* rtb = reinterpret_cast<double*>(rotb + RP);
  int4* ofsb = reinterpret_cast<int4*>(rtb + RP);
  if constexpr (kPhys) {
    // the plan as byte offsets: rot(i1) | rot(i2) << 16 (16 B per slot), the rest 8 B per element
    for (int e = threadIdx.x; e < L::kTri; e += blockDim.x) {
      pelem[e] = c_plan_elem[e];
      paddr[e] = c_plan_addr[e];
    }
    for (int e = threadIdx.x; e < 6 * 32; e += blockDim.x) {  // block j of lane l: [j][l] (4 words) + [j][l]
      const int j = e >> 5, l = e & 31;
      pplan[32 * j + l] = make_uint4(c_plan_blk[l][j][0] * 16u, c_plan_blk[l][j][1] * 8u, c_plan_blk[l][j][2] * 8u,
                                     c_plan_blk[l][j][3] * 8u);
      pplan5[32 * j + l] = c_plan_blk[l][j][4] * 8u;
    }
    for (int l = threadIdx.x; l < 32; l += blockDim.x)
      pplan[6 * 32 + l] = l < 20 ? make_uint4(c_plan_diag[l][0] * 8u, c_plan_diag[l][1] * 8u, c_plan_diag[l][2] * 8u, 0u)
                                 : make_uint4(0u, 0u, 0u, 0u);
  } else
  for (int it = threadIdx.x; it < nblk; it += blockDim.x) {  // (the slots' own 2 x 2 blocks: param_store)
    int i1 = 0, r = it;
    while (r >= half - 1 - i1) {
      r -= half - 1 - i1;
      ++i1;
    }
    blk[it] = static_cast<std::uint16_t>((i1 << 8) | (i1 + 1 + r));
  }
  if constexpr (!kPhys)
  for (int it = threadIdx.x; it < (m - 1) * half; it += blockDim.x) {
    const int round = it / half, l = it - round * half;
    int p, q;
    if (l == 0) {
      p = round;
      q = m - 1;
    } else {
      p = (round + l) % (m - 1);
      q = (round - l + (m - 1)) % (m - 1);
    }
    // no p < q swap: slots l of a round then touch the consecutive indices
    // round + l and round - l, so the lanes of a block row hit consecutive
    // shared-memory words (conflict-free); the rotation is symmetric in p, q
    sched[it] = static_cast<std::uint16_t>(p | ((q < R ? q : 0xff) << 8));
  }
  __syncthreads();
  // this lane's share of every round: 2 x 2 blocks (slot i1 | i2 << 8) of M
  // and (slot | column offset << 8) items of V'^T, fixed for the whole kernel
  constexpr int kLaneBlk = (L::NBLK + 31) / 32;
  // V' rows 0..31 of an exact-R subject live in registers (one row per lane,
  // below); only rows 32..R-1 (R = 40) stay as shared-memory items
  constexpr int kRegRows = EXACT ? (RP < 32 ? RP : 32) : 0;
  constexpr int kSmemKp = RP / 2 - kRegRows / 2;  // column pairs of V'^T still in shared memory
  constexpr int kLaneVit = kSmemKp > 0 ? (kSmemKp * (RP / 2) + 31) / 32 : 1;
  int lblk[kLaneBlk], lvit[kLaneVit];
#pragma unroll
  for (int j = 0; j < kLaneBlk; ++j) {
    const int it = lane + 32 * j;
    lblk[j] = it < nblk ? ((blk[it] >> 8) | ((blk[it] & 0xff) << 8)) : -1;
  }
  {
    const int kp0 = kRegRows / 2;
    const int nkp = ((R + 1) >> 1) - kp0;
#pragma unroll
    for (int j = 0; j < kLaneVit; ++j) {
      const int it = lane + 32 * j;
      const int sl = nkp > 0 ? it / nkp : 0, kp = kp0 + (nkp > 0 ? it - sl * nkp : 0);  // consecutive lanes: consecutive 16-byte units
      lvit[j] = (nkp > 0 && it < nkp * half) ? (sl | ((2 * kp) << 8)) : -1;
    }
  }
  const std::int64_t gw = static_cast<std::int64_t>(blockIdx.x) * WPB + wid;
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  double* slab = a.slab + gw * L::slab_doubles(a.max_rows, R);
  if constexpr (kPhys) {
    // Exact R = 40.  X~ = X_k V D is streamed in 8-row tiles from the X V rows
    // of the last mode-3 pass (a.XV, always given): B = X~ T' (T' = H^T E) is
    // formed tile by tile and only its Gram M = B^T B is kept; after the
    // sweeps Q = X~ W with W = T' Z, Z = V' S' E'^T, and m1 += Q^T X~
    // (= Z^T B^T X~ of the generic path), again tile by tile.  E is updated in
    // place in Ewarm (a row tile of E' = E V' depends only on the same rows of
    // E).  The product order is the generic path's: W = H^T (E' S' E'^T)
    // measured 30x further from the oracle on cfg5's ill-conditioned subjects.
    // After the sweeps every R x R operand lives in the warp's two shared buffers
    // (the ~24 KB of L1 left beside 229 KB of shared memory cannot hold per-warp
    // global scratch, whose reads were L2 round trips): W is formed as
    // ((H^T E') S') E'^T, each product in place over its left operand's row tiles.
    // Per-warp global scratch: the m1 partial and sqrt(diag M').
    constexpr int LDS = LDM;
    double* const M1 = slab;       // this warp's m1 partial
    double* const sv = M1 + RR;    // sqrt(M'_pp)
    double* const Ms0 = M;         // shared buffer 0 (the M region)
    double* const Ms1 = M + L::kMat;  // shared buffer 1 (the V'^T region)
    for (int e = lane; e < RR; e += 32) M1[e] = 0.0;
    const int fm = lane >> 2, fk = lane & 3, fn = 2 * (lane & 3);
    // X V row tiles (8 rows x 320 B, contiguous in HBM) arrive by TMA bulk copies into two
    // staging slots behind the B tile of buffer 0, one mbarrier per slot, two tiles in flight
    const unsigned mbar0 = dev::smem_uniform(rotb + RP), mbar1 = mbar0 + 8u;
    const unsigned st0 = dev::smem_uniform(Ms0 + 8 * LDS), st1 = st0 + 8u * 8 * RP;
    unsigned ph0 = 0, ph1 = 0;
    if (lane == 0) {
      dev::mbar_init(mbar0, 1);
      dev::mbar_init(mbar1, 1);
      dev::fence_mbar_init();
    }
    __syncwarp();
    for (std::int64_t k = gw; k < a.X.K; k += nwarps) {
      const std::int64_t r0 = a.X.srp[k];
      const int I = static_cast<int>(a.X.srp[k + 1] - r0);
      for (int r = lane; r < RP; r += 32) w[r] = a.W[k * RP + r];
      double* Ek = a.Ewarm + k * RR;  // E: read and updated in place
      if (!a.ew_valid)
        for (int e = lane; e < RR; e += 32) Ek[e] = (e / RP == e % RP) ? 1.0 : 0.0;
      const double* xvk = a.XV + r0 * RP;
      // the next subject's E and X V rows on their way into L2 while this one's sweeps run
      if (lane == 0 && k + nwarps < a.X.K) {
        const std::int64_t kn = k + nwarps, rn = a.X.srp[kn];
        if (a.ew_valid) dev::prefetch_l2_bulk(a.Ewarm + kn * RR, RR * 8u);
        dev::prefetch_l2_bulk(a.XV + rn * RP, static_cast<unsigned>(a.X.srp[kn + 1] - rn) * (RP * 8u));
      }
      int flag = P2G_FLAG_FULL_RANK;
      for (int pass = 0; pass < 2; ++pass) {
        __syncwarp();
        // T' = H^T E into the slab and shared buffer 1
        warp_mm<RP, true>(
            RP, RP, [&](int i, int c) { return __ldg(a.H + c * RP + i); }, [&](int c, int j) { return Ek[c * RP + j]; },
            [&](int i, int j, double v) { Ms1[i * LDS + j] = v; });
        __syncwarp();
        // M = B^T B over 8-row tiles of B = X~ T' (tiles staged in buffer 0)
        bool finite = true;
        {
          double accM[NB * (NB + 1) / 2][2];
#pragma unroll
          for (int t = 0; t < NB * (NB + 1) / 2; ++t) accM[t][0] = accM[t][1] = 0.0;
          auto tile_in = [&](int t, unsigned st, unsigned mbar) {  // rows 8 t .. of X V into a staging slot
            const int rows = I - 8 * t < 8 ? I - 8 * t : 8;
            if (lane == 0) dev::bulk_g2s(st, xvk + static_cast<std::int64_t>(8 * t) * RP, rows * (RP * 8u), mbar);
          };
          const int ntiles = (I + 7) >> 3;
          dev::fence_proxy_async();  // the slots were last written by this warp's own stores
          __syncwarp();
          if (ntiles > 0) tile_in(0, st0, mbar0);
          if (ntiles > 1) tile_in(1, st1, mbar1);
          for (int t = 0; t < ntiles; ++t) {
            const int i = 8 * t + fm;
            const bool iv = i < I;
            const bool odd = t & 1;
            const unsigned st = odd ? st1 : st0;
            dev::mbar_wait(odd ? mbar1 : mbar0, odd ? ph1 : ph0);
            if (odd)
              ph1 ^= 1u;
            else
              ph0 ^= 1u;
            double accB[NB][2];
#pragma unroll
            for (int b = 0; b < NB; ++b) accB[b][0] = accB[b][1] = 0.0;
#pragma unroll
            for (int k4 = 0; k4 < RP; k4 += 4) {
              const double x = iv ? dev::lds64<0>(st + 8u * (fm * RP + k4 + fk)) * w[k4 + fk] : 0.0;
#pragma unroll
              for (int b = 0; b < NB; ++b) dev::dmma884(accB[b], x, Ms1[(k4 + fk) * LDS + 8 * b + fm]);
            }
            __syncwarp();  // every lane has read the slot: refill it with tile t + 2
            if (t + 2 < ntiles) tile_in(t + 2, st, odd ? mbar1 : mbar0);
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              Ms0[fm * LDS + 8 * b + fn] = accB[b][0];
              Ms0[fm * LDS + 8 * b + fn + 1] = accB[b][1];
            }
            __syncwarp();
#pragma unroll
            for (int kk = 0; kk < 8; kk += 4) {
              double f[NB];
#pragma unroll
              for (int b = 0; b < NB; ++b) f[b] = Ms0[(kk + fk) * LDS + 8 * b + fm];
              int t2 = 0;
#pragma unroll
              for (int bi = 0; bi < NB; ++bi)
#pragma unroll
                for (int bj = 0; bj <= bi; ++bj) dev::dmma884(accM[t2++], f[bi], f[bj]);
            }
          }
          __syncwarp();
          // the upper triangle in physical (round-0) order into buffer 0:
          // logical l sits at position 2l (l < 20), 2 (39 - l) + 1 (l >= 20; 39 -> 1)
          int t = 0;
#pragma unroll
          for (int bi = 0; bi < NB; ++bi)
#pragma unroll
            for (int bj = 0; bj <= bi; ++bj, ++t) {
              const int i = 8 * bi + fm;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int j = 8 * bj + fn + h;
                if (bi > bj || i <= j) {
                  const int xi = i == 39 ? 1 : (i < 20 ? 2 * i : 2 * (39 - i) + 1);
                  const int xj = j == 39 ? 1 : (j < 20 ? 2 * j : 2 * (39 - j) + 1);
                  const int x = min(xi, xj), y = max(xi, xj);
                  M[paddr[x * (2 * RP + 1 - x) / 2 + y - x]] = accM[t][h];
                }
                finite &= isfinite(accM[t][h]);
              }
            }
        }
        finite = __all_sync(dev::kFull, finite);
        __syncwarp();
        if (!finite) {  // the accurate path re-checks the operand; no preconditioner from here
          for (int e = lane; e < RR; e += 32) Ek[e] = (e / RP == e % RP) ? 1.0 : 0.0;
          __syncwarp();
          flag = P2G_FLAG_ACCURATE;
          break;
        }
        bool converged = false;
        int sweeps = 0;
        double off = 0.0;  // scaled off-diagonal mass at the start of the pass
        double* Mx = M;    // after the sweeps: M' (logical order, full)
        double* Vx = Vt;   // and V'^T (Vx[p * LDVx + k] = V'(k, p))
        {
        // Physical-order round (jacobi_plan40.inc): slot i's
        // pair sits at positions (2i, 2i + 1) of M, V' rows and V' row chunks;
        // after each round every position's content moves one step along the
        // fixed cycle sigma, so all addresses are static.  M ping-pongs between
        // the M region (buffer 0) and the V'^T region (buffer 1).
        constexpr int kBuf = L::kMat * 8;  // bytes from buffer 0 to buffer 1
        const unsigned mb = dev::smem_uniform(M);
        const unsigned rb = dev::smem_uniform(rotb);  // (c, s) per slot, 2 x 20 double2
        // V' in registers as 32 tiles of 5 rows x 10 positions (5 slots): lane (rg, ch) holds rows
        // 5 rg .. 5 rg + 4 at positions 10 ch .. 10 ch + 9, so a lane needs 5 of the round's 20 rotation
        // pairs (5 loads instead of the 25 of a row-per-lane layout; the sigma step crosses chunks
        // with two shuffles per row)
        const int ch = lane & 3, rg = lane >> 2;
        double vt[5][10];
#pragma unroll
        for (int r = 0; r < 5; ++r)
#pragma unroll
          for (int k = 0; k < 10; ++k) vt[r][k] = rr_l0(RP, 10 * ch + k) == 5 * rg + r ? 1.0 : 0.0;
        double tiny = 0.0;
        // Scaled ("fast") rotations: M = D M~ D off the diagonal and V' = V~ D with a scale d_x per
        // position (both columns of a rotation shrink by the same cosine), so a rotation is
        // col_p += na col_q, col_q += nb col_p with na = -t d_q / d_p, nb = t d_p / d_q: two FMAs per
        // element pair instead of four operations, and a dependency depth of one.  The diagonal
        // entries stay unscaled (only the slot lanes touch them).  (d_x, 1 / d_x) follow the positions
        // along sigma in the tail of each Jacobi buffer.
        constexpr unsigned kDs = kPlanDoubles * 8u;
        static_assert(kPlanDoubles + 2 * RP <= L::kMat, "scales behind the elements");
        const unsigned dsp = kDs + 16u * (lane == 0 ? 3 : 2 * lane - 2);                    // sigma(2 lane)
        const unsigned dsq = kDs + 16u * (lane == 0 ? 1 : (lane == 19 ? 38 : 2 * lane + 3));  // sigma(2 lane + 1)
        struct Dg {
          double al, be, gs;  // M_pp, M_qq (true), M~_pq (scaled)
        };
        // slot `lane` (< 20): its diagonal block from the buffer at `rd` ...
        // this lane's static share of every round (pplan, byte offsets): blocks
        // {rot(i1) | rot(i2) << 16, r_pp | r_pq, r_qp | r_qq, w_pp | w_pq} + {w_qp | w_qq}
        // and (lanes < 20) its slot's diagonal block {r_pp | r_qq, r_pq | w_pp, w_qq | w_pq}
        const unsigned pb = dev::smem_uniform(pplan) + 16u * lane;
        const unsigned p5 = dev::smem_uniform(pplan5) + 4u * lane;
        auto par_load = [&](unsigned rd) {
          Dg d{0.0, 0.0, 0.0};
          if (lane < 20) {
            const uint4 g = dev::lds128u(pb + 16u * 6 * 32);
            const unsigned dg[3] = {g.x, g.y, g.z};
            d.al = dev::lds64<0>(rd + (dg[0] & 0xffffu));
            d.be = dev::lds64<0>(rd + (dg[0] >> 16));
            d.gs = dev::lds64<0>(rd + (dg[1] & 0xffffu));
          }
          return d;
        };
        // ... its rotation (c, s) into the rot buffer at `ro`, the rotated
        // block's sigma-images into the buffer at `wr` (rotation as in the
        // generic path)
        auto par_store = [&](const Dg& d, unsigned rd, unsigned wr, unsigned ro) {
          // (d, 1 / d) of positions 2 lane, 2 lane + 1
          const double2 sp = lane < 20 ? dev::lds128<0>(rd + kDs + 32u * lane) : make_double2(1.0, 1.0);
          const double2 sq = lane < 20 ? dev::lds128<0>(rd + kDs + 32u * lane + 16u) : make_double2(1.0, 1.0);
          const double ga = d.gs * (sp.x * sq.x);
          const bool on = d.al > tiny && d.be > tiny && ga * ga > (kSkipL * kSkipL) * (d.al * d.be);
          const double dd = d.be - d.al, g2 = 2.0 * ga;
          const double h = on ? fma(dd, dd, g2 * g2) : 1.0;
          const double rh = h * dev::rsqrt_nr(h);
          const double tt = on ? (dd >= 0.0 ? g2 : -g2) * dev::rcp_nr(fabs(dd) + rh) : 0.0;
          const double dt = __dmul_rn(tt, ga);
          if (lane < 20) {
            const uint4 g = dev::lds128u(pb + 16u * 6 * 32);
            const unsigned dg[3] = {g.x, g.y, g.z};
            dev::sts128<0>(ro + 16u * lane, -tt * (sq.x * sp.y), tt * (sp.x * sq.y));
            dev::sts64<0>(wr + (dg[1] >> 16), on ? d.al - dt : d.al);
            dev::sts64<0>(wr + (dg[2] & 0xffffu), on ? d.be + dt : d.be);
            dev::sts64<0>(wr + (dg[2] >> 16), on ? 0.0 : d.gs);
            // the positions' scales shrink by c = (1 + t^2)^{-1/2} and move along sigma
            const double t2 = fma(tt, tt, 1.0);
            const double c = on ? dev::rsqrt_nr(t2) : 1.0, ic = on ? t2 * c : 1.0;
            dev::sts128<0>(wr + dsp, c * sp.x, ic * sp.y);
            dev::sts128<0>(wr + dsq, c * sq.x, ic * sq.y);
          }
        };
        // M <- J^T M J over this lane's six 2 x 2 blocks, two at a time (their
        // loads ahead of their stores), written to their sigma-images
        auto blocks = [&](unsigned rd, unsigned wr, unsigned ro) {
#pragma unroll
          for (int j0 = 0; j0 < 6; j0 += 2) {
            double2 r1[2], r2[2];
            double x[2][4];
            unsigned q4[2];
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const uint4 q = dev::lds128u(pb + 16u * 32 * (j0 + v));
              q4[v] = q.w;
              r1[v] = dev::lds128<0>(ro + (q.x & 0xffffu));
              r2[v] = dev::lds128<0>(ro + (q.x >> 16));
              x[v][0] = dev::lds64<0>(rd + (q.y & 0xffffu));  // pp
              x[v][1] = dev::lds64<0>(rd + (q.y >> 16));      // pq
              x[v][2] = dev::lds64<0>(rd + (q.z & 0xffffu));  // qp
              x[v][3] = dev::lds64<0>(rd + (q.z >> 16));      // qq
            }
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const unsigned w5 = dev::lds32u(p5 + 4u * 32 * (j0 + v));
              const double a1 = r1[v].x, b1 = r1[v].y, a2 = r2[v].x, b2 = r2[v].y;
              const double x11 = x[v][0], x12 = x[v][1], x21 = x[v][2], x22 = x[v][3];
              const double y11 = fma(a2, x12, x11), y12 = fma(b2, x11, x12);
              const double y21 = fma(a2, x22, x21), y22 = fma(b2, x21, x22);
              dev::sts64<0>(wr + (q4[v] & 0xffffu), fma(a1, y21, y11));
              dev::sts64<0>(wr + (q4[v] >> 16), fma(a1, y22, y12));
              dev::sts64<0>(wr + (w5 & 0xffffu), fma(b1, y11, y21));
              dev::sts64<0>(wr + (w5 >> 16), fma(b1, y12, y22));
            }
          }
        };
        // V' <- V' J on the register tile, then one step along sigma
        auto vupd = [&](unsigned ro) {
          const unsigned cb = ro + 80u * ch;
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const double2 r = dev::lds128<0>(cb + 16u * k);
#pragma unroll
            for (int q = 0; q < 5; ++q) {
              const double x0 = vt[q][2 * k], y0 = vt[q][2 * k + 1];
              vt[q][2 * k] = fma(r.x, y0, x0);
              vt[q][2 * k + 1] = fma(r.y, x0, y0);
            }
          }
          // positions 10 ch + 8 <- 10 ch + 10 (next chunk) and 10 ch + 1 <- 10 ch - 1
          // (previous chunk); chunk 0 holds the cycle's ends 3 <- 0 and 1 (fixed)
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            double* v = vt[q];
            const double dn = __shfl_down_sync(dev::kFull, v[0], 1);
            const double up = __shfl_up_sync(dev::kFull, v[9], 1);
            const double o0 = v[0], o1 = v[1], o9 = v[9];
            v[0] = v[2];
            v[2] = v[4];
            v[4] = v[6];
            v[6] = v[8];
            v[8] = ch == 3 ? o9 : dn;
            v[9] = v[7];
            v[7] = v[5];
            v[5] = v[3];
            v[3] = ch == 0 ? o0 : o1;
            v[1] = ch == 0 ? o1 : up;
          }
        };
        // one sweep (m - 1 = 39 rounds) from buffer A to buffer B: rounds in
        // pairs (A -> B with rot buffer 0, B -> A with rot buffer 1), then the last
        auto run_sweep = [&](unsigned A, unsigned B) {
          par_store(par_load(A), A, B, rb);
          __syncwarp();
          // one round per iteration (the two buffers and the two rotation buffers swap roles):
          // the loop body stays small for the instruction caches
#pragma unroll 1
          for (int rr = 0; rr < RP - 2; ++rr) {
            // roles by round parity, computed from the (uniform) round counter so that the
            // addresses stay in uniform registers (one wavefront per same-address load)
            const unsigned par = static_cast<unsigned>(rr) & 1u;
            const unsigned ra = par ? B : A, wb = par ? A : B;
            const unsigned ro = rb + 320u * par, ro2 = rb + 320u * (par ^ 1u);
            blocks(ra, wb, ro);
            __syncwarp();
            {
              const Dg d = par_load(wb);
              vupd(ro);
              par_store(d, wb, ra, ro2);
            }
            __syncwarp();
          }
          const unsigned ra = A, wb = B, ro = rb;  // 38 rounds done: round 39 as round 1
          blocks(ra, wb, ro);
          __syncwarp();
          vupd(ro);
          __syncwarp();
        };
        int cur = 0;  // the buffer holding M at sweep boundaries (round-0 arrangement)
        for (int x = lane; x < RP; x += 32) M[kPlanDoubles + 2 * x] = M[kPlanDoubles + 2 * x + 1] = 1.0;
        auto at = [&](const double* Mc, int x, int y) {  // element (x <= y)
          return Mc[paddr[x * (2 * RP + 1 - x) / 2 + y - x]];
        };
        for (int sweep = 0; sweep < kLgMaxSweeps; ++sweep, ++sweeps) {
          double* Mc = M + cur * L::kMat;
          const double d0 = at(Mc, lane, lane), d1 = lane < 8 ? at(Mc, 32 + lane, 32 + lane) : 0.0;
          const double dmax = dev::warp_max(fmax(d0, d1));
          tiny = kTinyL * dmax;
          // u_x = d_x / sqrt(M_xx): M~_xy u_x u_y is the scaled off-diagonal; 1 / d_x refreshed (no drift)
          {
            double* ds = Mc + kPlanDoubles;
            const double s0 = ds[2 * lane];
            u[lane] = d0 > tiny ? s0 / sqrt(d0) : 0.0;
            ds[2 * lane + 1] = 1.0 / s0;
            if (lane < 8) {
              const double s1 = ds[2 * (32 + lane)];
              u[32 + lane] = d1 > tiny ? s1 / sqrt(d1) : 0.0;
              ds[2 * (32 + lane) + 1] = 1.0 / s1;
            }
          }
          __syncwarp();
          // scaled off-diagonal over the elements in address order (the diagonal adds 1 each)
          double omax = 0.0, osum = 0.0;
#pragma unroll 2
          for (int e0 = 0; e0 < L::kTri; e0 += 64) {
            const int ea = e0 + lane, eb = e0 + 32 + lane;
            const unsigned pa = pelem[ea < L::kTri ? ea : 0], pb2 = pelem[eb < L::kTri ? eb : 0];
            const double va = Mc[pa & 0xffffu] * u[(pa >> 16) & 0xffu] * u[pa >> 24];
            const double vb = Mc[pb2 & 0xffffu] * u[(pb2 >> 16) & 0xffu] * u[pb2 >> 24];
            const bool oa = ea < L::kTri && ((pa >> 16) & 0xffu) != (pa >> 24);
            const bool ob = eb < L::kTri && ((pb2 >> 16) & 0xffu) != (pb2 >> 24);
            if (oa) {
              omax = fmax(omax, fabs(va));
              osum = fma(va, va, osum);
            }
            if (ob) {
              omax = fmax(omax, fabs(vb));
              osum = fma(vb, vb, osum);
            }
          }
          omax = dev::warp_max(omax);
          if (sweep == 0) {
            off = 2.0 * dev::warp_sum(osum);  // both triangles, as in the generic path
            if (a.dbg && lane == 0) {
              const int b = omax <= 0.0 ? 0 : min(9, max(0, static_cast<int>(floor(log10(omax))) + 9));
              atomicAdd(a.dbg + 4 + b, 1);
            }
          }
          if (omax <= kTauL) {
            converged = true;
            break;
          }
          run_sweep(mb + static_cast<unsigned>(cur * kBuf), mb + static_cast<unsigned>((cur ^ 1) * kBuf));
          cur ^= 1;
        }
        // M' in logical order (full) into the other buffer, V'^T into this one
        {
          const double* Mc = M + cur * L::kMat;
          double* Ml = M + (cur ^ 1) * L::kMat;
          __syncwarp();
          for (int x = lane; x < RP; x += 32) u[x] = Mc[kPlanDoubles + 2 * x];  // the positions' scales
          __syncwarp();
          for (int e = lane; e < RP * RP; e += 32) {
            const int p = e / RP, q = e - p * RP;
            const int xp = p == RP - 1 ? 1 : (p < RP / 2 ? 2 * p : 2 * (RP - 1 - p) + 1);
            const int xq = q == RP - 1 ? 1 : (q < RP / 2 ? 2 * q : 2 * (RP - 1 - q) + 1);
            const double v = at(Mc, min(xp, xq), max(xp, xq));
            Ml[p * LDM + q] = p == q ? v : v * (u[xp] * u[xq]);
          }
          __syncwarp();
          double* V2 = M + cur * L::kMat;
#pragma unroll
          for (int q = 0; q < 5; ++q)
#pragma unroll
            for (int k = 0; k < 10; ++k) V2[rr_l0(RP, 10 * ch + k) * LDM + 5 * rg + q] = vt[q][k] * u[10 * ch + k];
          __syncwarp();
          Mx = Ml;
          Vx = V2;
        }
        }
        if (a.dbg && lane == 0) {
          atomicAdd(a.dbg + 16 + min(sweeps, 9), 1);
          atomicAdd(a.dbg + 0, sweeps);
          atomicMax(a.dbg + 1, sweeps);
          if (pass == 0) atomicAdd(a.dbg + 3, 1);
          if (pass == 1) atomicAdd(a.dbg + 2, 1);
        }
        // E <- E V', in place (row tile i of E' reads only row tile i of E)
        warp_mm<RP, true>(
            RP, RP, [&](int i, int c) { return Ek[i * RP + c]; }, [&](int c, int j) { return Vx[j * LDVx + c]; },
            [&](int i, int j, double v) { Ek[i * RP + j] = v; });
        __syncwarp();
        if (!converged) {
          flag = P2G_FLAG_ACCURATE;
          break;
        }
        double smax2 = 0.0, smin2 = 1e308;
        for (int j = 0; j < RP; ++j) {
          smax2 = fmax(smax2, Mx[j * LDM + j]);
          smin2 = fmin(smin2, Mx[j * LDM + j]);
        }
        if (!(smax2 > 0.0) || !(smin2 > kTinyL * smax2)) {
          flag = P2G_FLAG_ACCURATE;
          break;
        }
        if (pass == 0 && off > 0.25 && smin2 < 1e-6 * smax2) continue;
        // S' = M'^{-1/2} (second order about the diagonal): A = P o N in place over M'
        // (P_pq = 1 / (s_p + s_q)), S' into V''s buffer (V' is dead: E' = E V' is stored)
        for (int p = lane; p < RP; p += 32) {
          const double sq = sqrt(Mx[p * LDM + p]);
          sv[p] = sq;
          u[p] = 1.0 / sq;
        }
        __syncwarp();
        for (int e = lane; e < RR; e += 32) {
          const int p = e / RP, q = e - p * RP;
          Mx[p * LDM + q] = p == q ? 0.0 : dev::rcp_nr(sv[p] + sv[q]) * Mx[p * LDM + q];
        }
        __syncwarp();
        double* const Sx = Vx;
        {
#pragma unroll 1
          for (int bi = 0; bi < NB; ++bi) {
            const int i = 8 * bi + fm;
            double c1[NB][2], c2[NB][2];
#pragma unroll
            for (int b = 0; b < NB; ++b) c1[b][0] = c1[b][1] = c2[b][0] = c2[b][1] = 0.0;
#pragma unroll 2
            for (int k4 = 0; k4 < RP; k4 += 4) {
              const int c = k4 + fk;
              const double x = Mx[i * LDM + c];
              const double xu = x * u[c];
#pragma unroll
              for (int b = 0; b < NB; ++b) {
                const double y = Mx[c * LDM + 8 * b + fm];
                dev::dmma884(c1[b], xu, y);
                dev::dmma884(c2[b], x, y);
              }
            }
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int j = 8 * b + fn + h;
                const double corr = c1[b][h] - Mx[i * LDM + j] + dev::rcp_nr(sv[i] + sv[j]) * c2[b][h];
                Sx[i * LDM + j] = (i == j ? u[i] : 0.0) + u[i] * u[j] * corr;
              }
          }
        }
        __syncwarp();
        // T'' = H^T E' over A, then ((T'' S') E'^T) in place: the DMMA of a row tile is warp-wide,
        // so every lane has read the tile's left operand before any lane's epilogue overwrites it
        double* const Wsm = Mx;
        warp_mm<RP, true>(
            RP, RP, [&](int i, int c) { return __ldg(a.H + c * RP + i); }, [&](int c, int j) { return Ek[c * RP + j]; },
            [&](int i, int j, double v) { Wsm[i * LDS + j] = v; });
        __syncwarp();
        warp_mm<RP, true>(
            RP, RP, [&](int i, int c) { return Wsm[i * LDS + c]; }, [&](int c, int j) { return Sx[c * LDM + j]; },
            [&](int i, int j, double v) { Wsm[i * LDS + j] = v; });
        __syncwarp();
        warp_mm<RP, true>(
            RP, RP, [&](int i, int c) { return Wsm[i * LDS + c]; }, [&](int c, int j) { return Ek[j * RP + c]; },
            [&](int i, int j, double v) { Wsm[i * LDS + j] = v; });
        __syncwarp();
        double* const Xst = Sx;  // then: 8 x 41 X~ tile and 8 x 41 Q tile (S' is dead)
        double* const Qst = Sx + 8 * LDS;
        // Q = X~ W and m1 += Q^T X~, tile by tile
        {
          double m1a[NB][NB][2];
#pragma unroll
          for (int p = 0; p < NB; ++p)
#pragma unroll
            for (int b = 0; b < NB; ++b) m1a[p][b][0] = m1a[p][b][1] = 0.0;
          double* Qk = a.Q + r0 * RP;
          for (int i0 = 0; i0 < I; i0 += 8) {
            // the tile's X~ rows (a contiguous 8 x 40 block of X V, coalesced) into Xst
#pragma unroll
            for (int v = 0; v < 10; ++v) {
              const int e = lane + 32 * v, row = e / RP, col = e - row * RP;
              Xst[row * LDS + col] = i0 + row < I ? __ldg(xvk + static_cast<std::int64_t>(i0) * RP + e) * w[col] : 0.0;
            }
            __syncwarp();
            double accQ[NB][2];
#pragma unroll
            for (int b = 0; b < NB; ++b) accQ[b][0] = accQ[b][1] = 0.0;
#pragma unroll
            for (int k4 = 0; k4 < RP; k4 += 4) {
              const double x = Xst[fm * LDS + k4 + fk];
#pragma unroll
              for (int b = 0; b < NB; ++b) dev::dmma884(accQ[b], x, Wsm[(k4 + fk) * LDS + 8 * b + fm]);
            }
            if (i0 + fm < I) {
#pragma unroll
              for (int b = 0; b < NB; ++b)
                *reinterpret_cast<double2*>(Qk + static_cast<std::int64_t>(i0 + fm) * RP + 8 * b + fn) =
                    make_double2(accQ[b][0], accQ[b][1]);
            }
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              Qst[fm * LDS + 8 * b + fn] = accQ[b][0];
              Qst[fm * LDS + 8 * b + fn + 1] = accQ[b][1];
            }
            __syncwarp();
#pragma unroll
            for (int kk = 0; kk < 8; kk += 4) {
              double fq[NB], fx[NB];
#pragma unroll
              for (int b = 0; b < NB; ++b) {
                fq[b] = Qst[(kk + fk) * LDS + 8 * b + fm];
                fx[b] = Xst[(kk + fk) * LDS + 8 * b + fm];
              }
#pragma unroll
              for (int p = 0; p < NB; ++p)
#pragma unroll
                for (int b = 0; b < NB; ++b) dev::dmma884(m1a[p][b], fq[p], fx[b]);
            }
            __syncwarp();
          }
#pragma unroll
          for (int p = 0; p < NB; ++p)
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
              for (int h = 0; h < 2; ++h) M1[(8 * p + fm) * RP + 8 * b + fn + h] += m1a[p][b][h];
        }
        __syncwarp();
        break;
      }
      if (lane == 0) a.flags[k] = flag;
      __syncwarp();
    }
    for (int e = lane; e < RR; e += 32) a.m1_partials[gw * RR + e] = M1[e];
    return;
  }

  double* Bs = slab;                  // I x R rows of B = X~ H^T E
  double* Xs = Bs + a.max_rows * R;   // I x R rows of X~ = X V D
  double* Ts = Xs + a.max_rows * R;   // H^T E; later A = P o N; later Z
  double* Fs = Ts + RR;               // F = B^T X~
  double* Es = Fs + RR;               // E (R x R)
  double* Ns = Es + RR;               // scratch: E V', P, V' S'
  double* M1 = Ns + RR;               // this warp's m1 partial
  double* sv = M1 + RR;               // sqrt(M'_pp)
  for (int e = lane; e < RR; e += 32) M1[e] = 0.0;
  for (std::int64_t k = gw; k < a.X.K; k += nwarps) {
    const std::int64_t r0 = a.X.srp[k];
    const int I = static_cast<int>(a.X.srp[k + 1] - r0);
    for (int r = lane; r < R; r += 32) w[r] = a.W[k * R + r];
    double* Ek = a.Ewarm + k * RR;
    if (a.ew_valid)
      warp_copy(Es, Ek, RR, lane);
    else
      for (int e = lane; e < RR; e += 32) Es[e] = (e / R == e % R) ? 1.0 : 0.0;
    __syncwarp();
    // rows of X~ = X_k V D: from the previous mode-3 pass's X V rows when
    // available (a coalesced copy), else gathered (lane per row)
    if (a.XV) {  // 8 loads in flight per lane before the stores (they would alias)
      const double* xs = a.XV + r0 * R;
      const int n = I * R;
      for (int e0 = 0; e0 < n; e0 += 256) {
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + lane + 32 * u;
          t[u] = e < n ? __ldg(xs + e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + lane + 32 * u;
          if (e < n) Xs[e] = t[u] * w[e % R];
        }
      }
    } else
    for (int i = lane; i < I; i += 32) {
      double xv[RP];
      dev::csr_row_times<RP>(xv, a.X.ci, a.X.val, a.X.rp[r0 + i], a.X.rp[r0 + i + 1], a.V, R);
      double* xrow = Xs + static_cast<std::int64_t>(i) * R;
#pragma unroll
      for (int c = 0; c < RP; ++c)
        if (c < R) xrow[c] = xv[c] * w[c];
    }
    int flag = P2G_FLAG_FULL_RANK;
    for (int pass = 0; pass < 2; ++pass) {
      __syncwarp();
      // T' = H^T E, then B = X~ T' (= X_k V D H^T E)
      warp_mm<RP, EXACT>(
          R, R, [&](int i, int c) { return __ldg(a.H + c * R + i); }, [&](int c, int j) { return Es[c * R + j]; },
          [&](int i, int j, double v) { Ts[i * R + j] = v; });
      __syncwarp();
      warp_mm<RP, EXACT>(
          I, R, [&](int i, int c) { return Xs[i * R + c]; }, [&](int c, int j) { return Ts[c * R + j]; },
          [&](int i, int j, double v) { Bs[i * R + j] = v; });
      __syncwarp();
      // M = B^T B (lower tiles) into shared memory, F = B^T X~ into the slab
      bool finite = true;
      {
        const int fm = lane >> 2, fk = lane & 3, fn = 2 * (lane & 3);
        double acc[NB * (NB + 1) / 2][2];
#pragma unroll
        for (int t = 0; t < NB * (NB + 1) / 2; ++t) acc[t][0] = acc[t][1] = 0.0;
        for (int k4 = 0; k4 < I; k4 += 4) {
          const int r = k4 + fk;
          double f[NB];
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const int col = 8 * b + fm;
            f[b] = (r < I && (EXACT || col < R)) ? Bs[static_cast<std::int64_t>(r) * R + col] : 0.0;
          }
          int t = 0;
#pragma unroll
          for (int bi = 0; bi < NB; ++bi)
#pragma unroll
            for (int bj = 0; bj <= bi; ++bj) dev::dmma884(acc[t++], f[bi], f[bj]);
        }
        int t = 0;
#pragma unroll
        for (int bi = 0; bi < NB; ++bi)
#pragma unroll
          for (int bj = 0; bj <= bi; ++bj, ++t) {
            const int i = 8 * bi + fm;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j = 8 * bj + fn + h;
              if (EXACT || (i < R && j < R)) {
                M[i * LDM + j] = acc[t][h];
                M[j * LDM + i] = acc[t][h];
                finite &= isfinite(acc[t][h]);
              }
            }
          }
      }
      {
        const int fm = lane >> 2, fk = lane & 3, fn = 2 * (lane & 3);
#pragma unroll 1
        for (int bi = 0; bi < NB; ++bi) {
          double acc[NB][2];
#pragma unroll
          for (int bj = 0; bj < NB; ++bj) acc[bj][0] = acc[bj][1] = 0.0;
          for (int k4 = 0; k4 < I; k4 += 4) {
            const int r = k4 + fk;
            const int ci = 8 * bi + fm;
            const double fa = (r < I && (EXACT || ci < R)) ? Bs[static_cast<std::int64_t>(r) * R + ci] : 0.0;
#pragma unroll
            for (int bj = 0; bj < NB; ++bj) {
              const int cj = 8 * bj + fm;
              const double fb = (r < I && (EXACT || cj < R)) ? Xs[static_cast<std::int64_t>(r) * R + cj] : 0.0;
              dev::dmma884(acc[bj], fa, fb);
            }
          }
#pragma unroll
          for (int bj = 0; bj < NB; ++bj) {
            const int i = 8 * bi + fm;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j = 8 * bj + fn + h;
              if (EXACT || (i < R && j < R)) {
                Fs[i * R + j] = acc[bj][h];
                finite &= isfinite(acc[bj][h]);
              }
            }
          }
        }
      }
      finite = __all_sync(dev::kFull, finite);
      __syncwarp();
      if (!finite) {  // the accurate path re-checks the operand; no preconditioner from here
        for (int e = lane; e < RR; e += 32) Es[e] = (e / R == e % R) ? 1.0 : 0.0;
        __syncwarp();
        flag = P2G_FLAG_ACCURATE;
        break;
      }
      bool converged = false;
      int sweeps = 0;
      double off = 0.0;  // scaled off-diagonal mass at the start of the pass
      double* Mx = M;    // after the sweeps: M' (logical order, full)
      double* Vx = Vt;   // and V'^T (Vx[p * LDVx + k] = V'(k, p))
    // V' = I; row `lane` of V' also in registers, in round-0 physical order
      for (int e = lane; e < R * LDV; e += 32) {
        const int p = e / LDV, kk = e - p * LDV;
        Vt[e] = p == kk ? 1.0 : 0.0;
      }
      double vreg[kRegRows > 0 ? RP : 1];
#pragma unroll
      for (int x = 0; x < (kRegRows > 0 ? RP : 1); ++x) vreg[x] = rr_l0(RP, x) == lane ? 1.0 : 0.0;
      for (int sweep = 0; sweep < kLgMaxSweeps; ++sweep, ++sweeps) {
        double dmax = 0.0;
        for (int j = 0; j < R; ++j) dmax = fmax(dmax, M[j * LDM + j]);
        const double tiny = kTinyL * dmax;
        for (int p = lane; p < R; p += 32) {
          const double d = M[p * LDM + p];
          u[p] = d > tiny ? 1.0 / sqrt(d) : 0.0;
        }
        __syncwarp();
        double omax = 0.0, osum = 0.0;
        for (int e = lane; e < RR; e += 32) {
          const int p = e / R, q = e - p * R;
          const double x = M[p < q ? p * LDM + q : q * LDM + p] * u[p] * u[q];
          if (p != q) {
            omax = fmax(omax, fabs(x));
            osum = fma(x, x, osum);
          }
        }
        omax = dev::warp_max(omax);
        if (sweep == 0) {
          off = dev::warp_sum(osum);
          if (a.dbg && lane == 0) {
            const int b = omax <= 0.0 ? 0 : min(9, max(0, static_cast<int>(floor(log10(omax))) + 9));
            atomicAdd(a.dbg + 4 + b, 1);
          }
        }
        if (omax <= kTauL) {
          converged = true;
          break;
        }
        // Rotation parameters of one round's slot (lanes < half store them).
        // Split into the shared-memory loads and a pure-ALU tail, so that the
        // tail of round r + 1 can be scheduled among round r's V' updates.
        struct PIn {
          double al, be, ga;
          int p, q;
        };
        auto param_load = [&](int round) {
          PIn in;
          const int pq = sched[round * half + (lane < half ? lane : 0)];
          in.p = pq & 0xff;
          in.q = pq >> 8;
          const int qq = in.q != 0xff ? in.q : in.p;
          in.al = M[in.p * LDM + in.p];
          in.be = M[qq * LDM + qq];
          in.ga = in.q != 0xff ? M[in.p < qq ? in.p * LDM + qq : qq * LDM + in.p] : 0.0;
          return in;
        };
        auto param_store = [&](const PIn& in, int buf, bool diag) {
          const bool on = in.q != 0xff && in.al > tiny && in.be > tiny &&
                          in.ga * in.ga > (kSkipL * kSkipL) * (in.al * in.be);
          // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al) / (2 ga),
          // without divisions: t = sign(d) 2ga / (|d| + sqrt(d^2 + 4ga^2))
          const double d = in.be - in.al, g2 = 2.0 * in.ga;
          const double h = on ? fma(d, d, g2 * g2) : 1.0;
          const double rh = h * dev::rsqrt_nr(h);
          const double tt = on ? (d >= 0.0 ? g2 : -g2) * dev::rcp_nr(fabs(d) + rh) : 0.0;
          const double c = on ? dev::rsqrt_nr(fma(tt, tt, 1.0)) : 1.0;
          if (lane < half) {
            // the slot's own 2 x 2 block (M_pp, M_qq, M_pq) is updated here, by
            // the lane that holds its old values: no other block of the round
            // touches these entries, and the next parameter load follows the
            // round's block updates
            if (on && diag) {  // (not for the wrapped-around load of the sweep's last round)
              const double dt = __dmul_rn(tt, in.ga);
              M[in.p * LDM + in.p] = in.al - dt;
              M[in.q * LDM + in.q] = in.be + dt;
              M[in.p < in.q ? in.p * LDM + in.q : in.q * LDM + in.p] = 0.0;
            }
            rotb[buf * (RP / 2) + lane] = make_double2(c, c * tt);
            rtb[buf * (RP / 2) + lane] = tt * in.ga;
            ofsb[buf * (RP / 2) + lane] = in.q != 0xff ? make_int4(in.p * LDM, in.q * LDM, in.p, in.q)
                                                      : make_int4(in.p * LDM, -1, in.p, -1);
          }
        };
        param_store(param_load(0), 0, true);
        __syncwarp();
        for (int round = 0; round < m - 1; ++round) {
          const int buf = round & 1;
          const double2* rot = rotb + buf * (RP / 2);
          const int4* ofs = ofsb + buf * (RP / 2);
          // M <- J^T M J over this lane's 2 x 2 blocks of slot pairs
#pragma unroll
          for (int j = 0; j < kLaneBlk; ++j) {
            const int b = lblk[j];
            if (b < 0) continue;
            const int i1 = b & 0xff, i2 = b >> 8;
            const double2 r1 = rot[i1], r2 = rot[i2];
            if (r1.y == 0.0 && r2.y == 0.0) continue;
            const int4 o1 = ofs[i1], o2 = ofs[i2];
            if (!EXACT && (o1.w < 0 || o2.w < 0)) {  // odd R: 1 x 2 block against the dummy slot's index
              const bool d1 = o1.w < 0;
              const int ar = d1 ? o1.x : o2.x, ac = d1 ? o1.z : o2.z;  // the single index (row / column offsets)
              const int ur = d1 ? o2.x : o1.x, uc = d1 ? o2.z : o1.z;
              const int vr = d1 ? o2.y : o1.y, vc = d1 ? o2.w : o1.w;
              const double cc = d1 ? r2.x : r1.x, ss = d1 ? r2.y : r1.y;
              const int au = ac < uc ? ar + uc : ur + ac, av = ac < vc ? ar + vc : vr + ac;
              const double xu = M[au], xv = M[av];
              M[au] = cc * xu - ss * xv;
              M[av] = ss * xu + cc * xv;
              continue;
            }
            const double c1 = r1.x, s1 = r1.y, c2 = r2.x, s2 = r2.y;
            // upper-triangle (canonical) addresses: row index < column index
            const int e11 = o1.z < o2.z ? o1.x + o2.z : o2.x + o1.z;
            const int e12 = o1.z < o2.w ? o1.x + o2.w : o2.y + o1.z;
            const int e21 = o1.w < o2.z ? o1.y + o2.z : o2.x + o1.w;
            const int e22 = o1.w < o2.w ? o1.y + o2.w : o2.y + o1.w;
            const double x11 = M[e11], x12 = M[e12], x21 = M[e21], x22 = M[e22];
            const double y11 = c2 * x11 - s2 * x12, y12 = s2 * x11 + c2 * x12;
            const double y21 = c2 * x21 - s2 * x22, y22 = s2 * x21 + c2 * x22;
            const double z11 = c1 * y11 - s1 * y21, z21 = s1 * y11 + c1 * y21;
            const double z12 = c1 * y12 - s1 * y22, z22 = s1 * y12 + c1 * y22;
            M[e11] = z11;
            M[e12] = z12;
            M[e21] = z21;
            M[e22] = z22;
          }
          __syncwarp();
          // next round's parameter loads (M is final for this round) ...
          const PIn nxt = param_load(round + 1 < m - 1 ? round + 1 : 0);
          // ... V' <- V' J.  Register rows: slot i's pair sits at positions
          // (2i, 2i+1); afterwards every position moves one step along the
          // fixed cycle 0 <- 2 <- ... <- RP-2 <- RP-1 <- RP-3 <- ... <- 3 <- 0
          // (position 1, index RP-1, stays), which is how the round-robin's
          // pairs advance, so the next round's pairs are again (2i, 2i+1) ...
          if constexpr (kRegRows > 0) {
#pragma unroll
            for (int i = 0; i < RP / 2; ++i) {
              const double2 r = rot[i];
              const double x0 = vreg[2 * i], y0 = vreg[2 * i + 1];
              vreg[2 * i] = r.x * x0 - r.y * y0;
              vreg[2 * i + 1] = r.y * x0 + r.x * y0;
            }
            const double t0 = vreg[0];
#pragma unroll
            for (int l = 0; l < RP / 2 - 1; ++l) vreg[2 * l] = vreg[2 * l + 2];
            vreg[RP - 2] = vreg[RP - 1];
#pragma unroll
            for (int l = RP / 2 - 1; l >= 2; --l) vreg[2 * l + 1] = vreg[2 * l - 1];
            vreg[3] = t0;
          }
          // ... shared-memory rows: p, q of V'^T (offset p LDV = p LDM + p) over
          // this lane's column pairs, branch-free so the parameter tail interleaves ...
#pragma unroll
          for (int j = 0; j < (kSmemKp > 0 ? kLaneVit : 0); ++j) {
            const int v = lvit[j];
            const int sl = v & 0xff, kc = (v >> 8) & 0xff;
            const double2 r = rot[v < 0 ? 0 : sl];
            const int4 o = ofs[v < 0 ? 0 : sl];
            const bool on = v >= 0 && r.y != 0.0;
            double2* vp = reinterpret_cast<double2*>(Vt + (on ? o.x + o.z + kc : 0));
            double2* vq = reinterpret_cast<double2*>(Vt + (on ? o.y + o.w + kc : 0));
            const double2 x = *vp, y = *vq;
            if (on) {
              *vp = make_double2(r.x * x.x - r.y * y.x, r.x * x.y - r.y * y.y);
              *vq = make_double2(r.y * x.x + r.x * y.x, r.y * x.y + r.x * y.y);
            }
          }
          // ... and the parameters into the other buffer
          param_store(nxt, buf ^ 1, round + 1 < m - 1);
          __syncwarp();
        }
      }
      // register rows back (whole sweeps bring positions back to round-0 order)
      if constexpr (kRegRows > 0) {
        if (lane < R) {
#pragma unroll
          for (int x = 0; x < RP; ++x) Vt[rr_l0(RP, x) * LDV + lane] = vreg[x];
        }
        __syncwarp();
      }
          if (a.dbg && lane == 0) {
        atomicAdd(a.dbg + 16 + min(sweeps, 9), 1);
        atomicAdd(a.dbg + 0, sweeps);
        atomicMax(a.dbg + 1, sweeps);
        if (pass == 0) atomicAdd(a.dbg + 3, 1);
        if (pass == 1) atomicAdd(a.dbg + 2, 1);
      }
      // E <- E V'
      warp_mm<RP, EXACT>(
          R, R, [&](int i, int c) { return Es[i * R + c]; }, [&](int c, int j) { return Vx[j * LDVx + c]; },
          [&](int i, int j, double v) { Ns[i * R + j] = v; });
      __syncwarp();
      warp_copy(Es, Ns, RR, lane);
      __syncwarp();
      if (!converged) {
        flag = P2G_FLAG_ACCURATE;
        break;
      }
      double smax2 = 0.0, smin2 = 1e308;
      for (int j = 0; j < R; ++j) {
        smax2 = fmax(smax2, Mx[j * LDM + j]);
        smin2 = fmin(smin2, Mx[j * LDM + j]);
      }
      if (!(smax2 > 0.0) || !(smin2 > kTinyL * smax2)) {
        flag = P2G_FLAG_ACCURATE;
        break;
      }
      if (pass == 0 && off > 0.25 && smin2 < 1e-6 * smax2) continue;
      // S' = M'^{-1/2} (second order about the diagonal) into M
      for (int p = lane; p < R; p += 32) {
        const double s = sqrt(Mx[p * LDM + p]);
        sv[p] = s;
        u[p] = 1.0 / s;
      }
      __syncwarp();
      for (int e = lane; e < RR; e += 32) {
        const int p = e / R, q = e - p * R;
        const double P = 1.0 / (sv[p] + sv[q]);
        Ns[e] = P;
        Ts[e] = p == q ? 0.0 : P * Mx[p < q ? p * LDM + q : q * LDM + p];
      }
      __syncwarp();
      {
        const int fm = lane >> 2, fk = lane & 3;
#pragma unroll 1
        for (int bi = 0; bi < NB; ++bi) {
          const int i = 8 * bi + fm;
          double c1[NB][2], c2[NB][2];
#pragma unroll
          for (int b = 0; b < NB; ++b) c1[b][0] = c1[b][1] = c2[b][0] = c2[b][1] = 0.0;
#pragma unroll 2
          for (int k4 = 0; k4 < RP; k4 += 4) {
            const int c = k4 + fk;
            const bool ok = EXACT || (i < R && c < R);
            const double x = ok ? Ts[i * R + c] : 0.0;
            const double xu = ok ? x * u[c] : 0.0;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              const int j = 8 * b + fm;
              const double y = (EXACT || (c < R && j < R)) ? Ts[c * R + j] : 0.0;
              dev::dmma884(c1[b], xu, y);
              dev::dmma884(c2[b], x, y);
            }
          }
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j = 8 * b + 2 * fk + h;
              if (EXACT || (i < R && j < R)) {
                const double corr = c1[b][h] - Ts[i * R + j] + Ns[i * R + j] * c2[b][h];
                Mx[i * LDM + j] = (i == j ? u[i] : 0.0) + u[i] * u[j] * corr;
              }
            }
        }
      }
      __syncwarp();
      // Y = V' S' into Ns, Z = Y E'^T into Ts
      warp_mm<RP, EXACT>(
          R, R, [&](int i, int c) { return Vx[c * LDVx + i]; }, [&](int c, int j) { return Mx[c * LDM + j]; },
          [&](int i, int j, double v) { Ns[i * R + j] = v; });
      __syncwarp();
      warp_mm<RP, EXACT>(
          R, R, [&](int i, int c) { return Ns[i * R + c]; }, [&](int c, int j) { return Es[j * R + c]; },
          [&](int i, int j, double v) { Ts[i * R + j] = v; });
      __syncwarp();
      // m1 += Z^T F;  Q = B Z
      warp_mm<RP, EXACT>(
          R, R, [&](int i, int c) { return Ts[c * R + i]; }, [&](int c, int j) { return Fs[c * R + j]; },
          [&](int i, int j, double v) { M1[i * R + j] += v; });
      double* Qk = a.Q + r0 * R;
      warp_mm<RP, EXACT>(
          I, R, [&](int i, int c) { return Bs[i * R + c]; }, [&](int c, int j) { return Ts[c * R + j]; },
          [&](int i, int j, double v) { Qk[static_cast<std::int64_t>(i) * R + j] = v; });
      __syncwarp();
      break;
    }
    warp_copy(Ek, Es, RR, lane);
    if (lane == 0) a.flags[k] = flag;
    __syncwarp();
  }
  for (int e = lane; e < RR; e += 32) a.m1_partials[gw * RR + e] = M1[e];
}

template <int RP, bool EXACT>
int launch_large_w(p2g_ctx* c, LgArgs a, int max_partials, cudaStream_t s) {
  using L = LgWarp<RP, EXACT>;
  auto kern = k_procrustes_large_w<RP, EXACT>;
  P2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(L::kSmem)));
  const std::int64_t K = a.X.K;
  const int blocks = static_cast<int>(std::max<std::int64_t>(
      1, std::min<std::int64_t>({(K + L::WPB - 1) / L::WPB, static_cast<std::int64_t>(c->num_sms),
                                 static_cast<std::int64_t>(max_partials / L::WPB)})));
  grow_scratch(c->acc_scratch, static_cast<std::size_t>(blocks) * L::WPB * L::slab_doubles(a.max_rows, a.R),
               "large-rank Procrustes path", a.max_rows);
  a.slab = c->acc_scratch.get();
  kern<<<blocks, L::WPB * 32, L::kSmem, s>>>(a);
  return blocks * L::WPB;  // one m1 partial per warp
}

}  // namespace

int launch_procrustes_large(p2g_ctx* c, int R, const double* H, const double* V, const double* W, double* Q,
                            std::int32_t* flags, double* m1_partials, double* Ewarm, int ew_valid, int max_blocks,
                            cudaStream_t s, const double* XV_in) {
  LgArgs a{};
  a.XV = XV_in;
  a.X = ShardArgs{c->srp.get(), c->rp.get(), c->ci.get(), c->val.get(), c->k_end - c->k_begin, c->NR, c->nnz, c->J};
  a.R = R;
  a.H = H;
  a.V = V;
  a.W = W;
  a.Q = Q;
  a.flags = flags;
  a.m1_partials = m1_partials;
  a.Ewarm = Ewarm;
  a.ew_valid = ew_valid;
  a.max_rows = c->max_rows;
  a.dbg = c->opt.debug ? c->counters.get() + 4 : nullptr;
  if (a.X.K == 0) return 0;
  if (R == 40 && !a.XV) {  // the R = 40 kernel streams X V rows: form them (first step of a fit)
    launch_xv_rows(c, R, V, c->Ubuf.get(), s);
    a.XV = c->Ubuf.get();
  }
  int blocks = 0;
  if (R == 24)
    blocks = launch_large_w<24, true>(c, a, max_blocks, s);
  else if (R == 32)
    blocks = launch_large_w<32, true>(c, a, max_blocks, s);
  else if (R == 40)
    blocks = launch_large_w<40, true>(c, a, max_blocks, s);
  else if (R <= 24)
    blocks = launch_large_w<24, false>(c, a, max_blocks, s);
  else if (R <= 32)
    blocks = launch_large_w<32, false>(c, a, max_blocks, s);
  else if (R <= 40)
    blocks = launch_large_w<40, false>(c, a, max_blocks, s);
  else
    throw InvalidArgument("rank above 40 unsupported");
  P2G_LAUNCHED(1);
  return blocks;
}

}  // namespace p2g
