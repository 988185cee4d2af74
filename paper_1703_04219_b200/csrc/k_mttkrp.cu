// K3 — SPARTan slice-wise MTTKRP on the GPU, plus K2 (projection) and the
// packed-Y boundary kernels.
//
// Fused-loop (Q-based) forms, SURVEY.md §3.2 / north_star:
//   mode 2 (mttkrp.hpp:111-138):  M2 = sum_k X_k^T (Q_k H diag(W_k))   J x R
//   mode 3 (mttkrp.hpp:143-166):  M3(k,:) = colwise-dot(Q_k H, X_k V)  K x R
//   mode 1 (mttkrp.hpp:81-106):   M1 = sum_k Q_k^T (X_k V) diag(W_k)  R x R
// They equal the reference's Y-based kernels on Y_k = Q_k^T X_k
// (project_slice, solver.hpp:197-208) without materialising Y (F5).
#include <algorithm>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"

namespace p2g {
namespace {

/// Leading dimension of staged rows: odd, so 32 lanes reading their own rows
/// hit distinct banks (an even stride such as 40 is a 16-way conflict).
template <int RP>
constexpr int CLD = RP | 1;

template <int RP>
__device__ __forceinline__ void stage_rows(double* chunk, const double* __restrict__ src, int nr, int R, int lane) {
  // rows at the odd stride CLD<RP> (conflict-free when lanes walk their own row)
  for (int row = 0; row < nr; ++row)
    for (int c = lane; c < R; c += 32) chunk[row * CLD<RP> + c] = __ldg(src + row * R + c);
  __syncwarp();
}

// ---------------------------------------------------------------------------
// mode 2: one warp per subject; U' = Q_k (H diag(W_k o nH)) row by row, then
// scattered into M2 with fp64 reductions in L2 (RED.ADD.F64).
// ---------------------------------------------------------------------------
template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_mode2(ShardArgs X, int R, const double* __restrict__ Q, const double* __restrict__ H,
            const double* __restrict__ W, const double* __restrict__ nH, double* __restrict__ M2) {
  __shared__ double HWs[WPB][RP * RP];
  __shared__ double chunk[WPB][32 * CLD<RP>];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* HW = HWs[wid];
  double* ch = chunk[wid];
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < X.K; k += nwarps) {
    const std::int64_t r0 = X.srp[k];
    const int I = static_cast<int>(X.srp[k + 1] - r0);
    for (int e = lane; e < R * R; e += 32) {
      const int b = e - (e / R) * R;
      const double w = W[k * R + b] * (nH ? nH[b] : 1.0);
      HW[e] = H[e] * w;
    }
    __syncwarp();
    for (int b0 = 0; b0 < I; b0 += 32) {
      const int nr = min(32, I - b0);
      stage_rows<RP>(ch, Q + (r0 + b0) * R, nr, R, lane);
      if (lane < nr) {
        double u[RP];
#pragma unroll
        for (int c = 0; c < RP; ++c) {
          double acc = 0.0;
          if (c < R) {
#pragma unroll
            for (int a = 0; a < RP; ++a)
              if (a < R) acc = fma(ch[lane * CLD<RP> + a], HW[a * R + c], acc);
          }
          u[c] = acc;
        }
        const std::int64_t p0 = X.rp[r0 + b0 + lane], p1 = X.rp[r0 + b0 + lane + 1];
        for (std::int64_t p = p0; p < p1; ++p) {
          const int j = __ldg(X.ci + p);
          const double v = __ldg(X.val + p);
          double* dst = M2 + static_cast<std::int64_t>(j) * R;
#pragma unroll
          for (int c = 0; c < RP; ++c)
            if (c < R) atomicAdd(dst + c, v * u[c]);
        }
      }
      __syncwarp();
    }
  }
}


// ---------------------------------------------------------------------------
// mode 3: one warp per subject; M3(k,c) = sum_i (Q_k H)(i,c) (X_k V)(i,c).
// ---------------------------------------------------------------------------
template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_mode3(ShardArgs X, int R, const double* __restrict__ Q, const double* __restrict__ H,
            const double* __restrict__ V, double* __restrict__ M3) {
  __shared__ double Hs[RP * RP];
  __shared__ double chunk[WPB][32 * CLD<RP>];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Hs[e] = H[e];
  __syncthreads();
  double* ch = chunk[wid];
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < X.K; k += nwarps) {
    const std::int64_t r0 = X.srp[k];
    const int I = static_cast<int>(X.srp[k + 1] - r0);
    double part[RP];
#pragma unroll
    for (int c = 0; c < RP; ++c) part[c] = 0.0;
    for (int b0 = 0; b0 < I; b0 += 32) {
      const int nr = min(32, I - b0);
      stage_rows<RP>(ch, Q + (r0 + b0) * R, nr, R, lane);
      if (lane < nr) {
        double xv[RP];
        dev::csr_row_times<RP>(xv, X.ci, X.val, X.rp[r0 + b0 + lane], X.rp[r0 + b0 + lane + 1], V, R);
#pragma unroll
        for (int c = 0; c < RP; ++c) {
          if (c < R) {
            double qh = 0.0;
#pragma unroll
            for (int a = 0; a < RP; ++a)
              if (a < R) qh = fma(ch[lane * CLD<RP> + a], Hs[a * R + c], qh);
            part[c] = fma(qh, xv[c], part[c]);
          }
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int c = 0; c < RP; ++c) {
      if (c < R) {
        const double t = dev::warp_sum(part[c]);
        if (lane == 0) M3[k * R + c] = t;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// mode 3 for R > 16 on the fp64 tensor cores: per subject, 8-row tiles of
// P = Q_k H (DMMA m8n8k4: Q fragments straight from HBM, H from shared
// memory) meet the matching fragment of X_k V, which each lane gathers for
// its own row (lane (fm, fk) holds row fm, columns 8b + 2fk + {0, 1} in the
// C layout); the column sums over rows are a 3-step shuffle over fm.
// Per subject: Q read once (coalesced 32-byte sectors), CSR streamed once,
// V rows from L2.  The tile's CSR entries (a contiguous range: its 8 rows)
// are first staged in shared memory with coalesced loads, so a lane's
// gather chain is a shared-memory read followed by the V-row load, and kU
// entries of its row are in flight at once (the kernel is bound by the
// latency of this chain, not by L2 throughput).
// ---------------------------------------------------------------------------
constexpr int kM3Stage = 256;  // staged entries per warp (a tile holds ~70 at cfg4)

template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_mode3_mma(ShardArgs X, int R, const double* __restrict__ Q, const double* __restrict__ H,
                const double* __restrict__ V, double* __restrict__ M3, double* __restrict__ XV) {
  constexpr int NB = RP / 8;
  constexpr int kU = 4;  // entries of a row in flight per lane
  __shared__ double Hs[RP * RP];  // H zero-padded to RP x RP, row-major
  __shared__ double vst[WPB][kM3Stage];
  __shared__ std::int32_t cst[WPB][kM3Stage];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, fm = lane >> 2, fk = lane & 3;
  for (int e = threadIdx.x; e < RP * RP; e += blockDim.x) {
    const int a = e / RP, c = e - a * RP;
    Hs[e] = (a < R && c < R) ? H[a * R + c] : 0.0;
  }
  __syncthreads();
  const bool even = (R & 1) == 0;
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < X.K; k += nwarps) {
    const std::int64_t r0 = X.srp[k];
    const int I = static_cast<int>(X.srp[k + 1] - r0);
    double m3p[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) m3p[b][0] = m3p[b][1] = 0.0;
    for (int i0 = 0; i0 < I; i0 += 8) {
      const int i = i0 + fm;
      const bool iv = i < I;
      const double* qrow = Q + (r0 + i) * R;
      double acc[NB][2];
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[b][0] = acc[b][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < RP; k4 += 4) {
        const int c = k4 + fk;
        const double x = (iv && c < R) ? __ldg(qrow + c) : 0.0;
#pragma unroll
        for (int b = 0; b < NB; ++b) dev::dmma884(acc[b], x, Hs[c * RP + 8 * b + fm]);
      }
      double xv[NB][2];
#pragma unroll
      for (int b = 0; b < NB; ++b) xv[b][0] = xv[b][1] = 0.0;
      const std::int64_t pa = X.rp[r0 + i0], pb = X.rp[r0 + min(i0 + 8, I)];
      const std::int64_t p0 = iv ? X.rp[r0 + i] : pa, p1 = iv ? X.rp[r0 + i + 1] : pa;
      for (std::int64_t cb = pa; cb < pb; cb += kM3Stage) {
        const int nc = static_cast<int>(pb - cb < kM3Stage ? pb - cb : kM3Stage);
        __syncwarp();
        for (int t = lane; t < nc; t += 32) {
          cst[wid][t] = __ldg(X.ci + cb + t);
          vst[wid][t] = __ldg(X.val + cb + t);
        }
        __syncwarp();
        const int q0 = static_cast<int>((p0 > cb ? p0 : cb) - cb), q1 = static_cast<int>((p1 < cb + nc ? p1 : cb + nc) - cb);
        // kU entries at a time (the same per-row accumulation order as the
        // other paths: entries ascending)
        for (int q = q0; q < q1; q += kU) {
          double v[kU];
          const double* vr[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const bool on = q + u < q1;
            v[u] = on ? vst[wid][q + u] : 0.0;
            vr[u] = V + static_cast<std::int64_t>(on ? cst[wid][q + u] : 0) * R;
          }
          double2 y[kU][NB];
#pragma unroll
          for (int u = 0; u < kU; ++u)
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              const int c = 8 * b + 2 * fk;
              if (even) {
                y[u][b] = (c < R && q + u < q1) ? __ldg(reinterpret_cast<const double2*>(vr[u] + c))
                                                : make_double2(0.0, 0.0);
              } else {
                y[u][b].x = (c < R && q + u < q1) ? __ldg(vr[u] + c) : 0.0;
                y[u][b].y = (c + 1 < R && q + u < q1) ? __ldg(vr[u] + c + 1) : 0.0;
              }
            }
#pragma unroll
          for (int u = 0; u < kU; ++u)
            if (q + u < q1) {
#pragma unroll
              for (int b = 0; b < NB; ++b) {
                xv[b][0] = fma(v[u], y[u][b].x, xv[b][0]);
                xv[b][1] = fma(v[u], y[u][b].y, xv[b][1]);
              }
            }
        }
      }
      if (XV && iv) {  // X_k V rows for the next Procrustes step (it would re-gather them)
        double* xr = XV + (r0 + i) * R;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int c = 8 * b + 2 * fk;
          if (even) {
            if (c < R) *reinterpret_cast<double2*>(xr + c) = make_double2(xv[b][0], xv[b][1]);
          } else {
            if (c < R) xr[c] = xv[b][0];
            if (c + 1 < R) xr[c + 1] = xv[b][1];
          }
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        m3p[b][0] = fma(acc[b][0], xv[b][0], m3p[b][0]);
        m3p[b][1] = fma(acc[b][1], xv[b][1], m3p[b][1]);
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double t = m3p[b][h];
        t += __shfl_xor_sync(dev::kFull, t, 4);
        t += __shfl_xor_sync(dev::kFull, t, 8);
        t += __shfl_xor_sync(dev::kFull, t, 16);
        const int c = 8 * b + 2 * fk + h;
        if (fm == 0 && c < R) M3[k * R + c] = t;
      }
  }
}

// ---------------------------------------------------------------------------
// mode 3 for exact R in {24, 32, 40} (the fused loop's R > 16 path): warp per
// subject in two phases.
//  A. X_k V rows: kG = 32 / (R / 4) lane groups take kG rows at a time; a
//     group reads a V row with R / 4 lanes of 32-byte loads (one row per
//     group per instruction, 4 entries in flight).  The rows' CSR entries are
//     staged 32 at a time in registers (coalesced) and broadcast by shuffles.
//     Each row is written to XV (the next Procrustes step reads it) with
//     32-byte stores.  Per-row accumulation order: entries ascending, as in
//     the other paths.
//  B. 8-row tiles of P = Q_k H (DMMA; Q fragments from HBM, H from shared
//     memory) meet the matching fragment of the X_k V rows just written
//     (L2-resident), and m3 = column sums of P o X_k V (3-step shuffle over
//     the tile's rows), in the same order as k_mode3_mma.
// ---------------------------------------------------------------------------
template <int RP, int WPB, bool M3OUT = true>
__global__ void __launch_bounds__(WPB * 32)
    k_mode3_rows(ShardArgs X, const double* __restrict__ Q, const double* __restrict__ H,
                 const double* __restrict__ V, double* __restrict__ M3, double* __restrict__ XV) {
  constexpr int NB = RP / 8;
  constexpr int kL = RP / 4, kG = 32 / kL;
  static_assert(RP % 8 == 0, "exact R, multiple of 8");
  __shared__ double Hs[RP * RP];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, fm = lane >> 2, fk = lane & 3;
  const int g = lane / kL, sub = lane - g * kL;
  const bool act = g < kG;
  if constexpr (M3OUT) {
    for (int e = threadIdx.x; e < RP * RP; e += blockDim.x) Hs[e] = H[e];
    __syncthreads();
  }
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < X.K; k += nwarps) {
    const std::int64_t r0 = X.srp[k];
    const int I = static_cast<int>(X.srp[k + 1] - r0);
    // A: X_k V rows
    for (int i0 = 0; i0 < I; i0 += kG) {
      const int i = i0 + g;
      const bool iv = act && i < I;
      const std::int64_t pa = X.rp[r0 + i0], pb = X.rp[r0 + (i0 + kG < I ? i0 + kG : I)];
      const std::int64_t p0 = iv ? X.rp[r0 + i] : pa, p1 = iv ? X.rp[r0 + i + 1] : pa;
      double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
      for (std::int64_t cb = pa; cb < pb; cb += 32) {
        const int m = static_cast<int>(pb - cb < 32 ? pb - cb : 32);
        const std::int32_t cc = lane < m ? __ldg(X.ci + cb + lane) : 0;
        const double vv = lane < m ? __ldg(X.val + cb + lane) : 0.0;
        const int t0 = static_cast<int>((p0 > cb ? p0 : cb) - cb);
        const int n = static_cast<int>((p1 < cb + m ? p1 : cb + m) - cb) - t0;
        const int nmax = __reduce_max_sync(dev::kFull, n > 0 ? n : 0);
        for (int u = 0; u < nmax; u += 4) {
          double w[4];
          double4 y[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t = t0 + u + j;
            const int col = __shfl_sync(dev::kFull, cc, t & 31);
            const double vj = __shfl_sync(dev::kFull, vv, t & 31);
            const bool on = u + j < n;
            w[j] = on ? vj : 0.0;
            y[j] = on ? dev::ldg256(V + static_cast<std::size_t>(col) * RP + 4 * sub)
                      : make_double4(0.0, 0.0, 0.0, 0.0);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (u + j < n) {
              acc.x = fma(w[j], y[j].x, acc.x);
              acc.y = fma(w[j], y[j].y, acc.y);
              acc.z = fma(w[j], y[j].z, acc.z);
              acc.w = fma(w[j], y[j].w, acc.w);
            }
        }
      }
      if (iv) dev::stg256(XV + (r0 + i) * RP + 4 * sub, acc);
    }
    if constexpr (!M3OUT) continue;
    __syncwarp();
    // B: m3 from P = Q_k H and the X_k V rows
    double m3p[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) m3p[b][0] = m3p[b][1] = 0.0;
    for (int i0 = 0; i0 < I; i0 += 8) {
      const int i = i0 + fm;
      const bool iv = i < I;
      const double* qrow = Q + (r0 + i) * RP;
      double acc[NB][2];
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[b][0] = acc[b][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < RP; k4 += 4) {
        const double x = iv ? __ldg(qrow + k4 + fk) : 0.0;
#pragma unroll
        for (int b = 0; b < NB; ++b) dev::dmma884(acc[b], x, Hs[(k4 + fk) * RP + 8 * b + fm]);
      }
      const double* xr = XV + (r0 + i) * RP;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const double2 xv = iv ? *reinterpret_cast<const double2*>(xr + 8 * b + 2 * fk) : make_double2(0.0, 0.0);
        m3p[b][0] = fma(acc[b][0], xv.x, m3p[b][0]);
        m3p[b][1] = fma(acc[b][1], xv.y, m3p[b][1]);
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double t = m3p[b][h];
        t += __shfl_xor_sync(dev::kFull, t, 4);
        t += __shfl_xor_sync(dev::kFull, t, 8);
        t += __shfl_xor_sync(dev::kFull, t, 16);
        if (fm == 0) M3[k * RP + 8 * b + 2 * fk + h] = t;
      }
  }
}

// ---------------------------------------------------------------------------
// mode 1 from a given Q (the p2g_mttkrp_q hook; the fused loop gets M1 from
// K1): m1 += Q_k^T (XV o W_k) through 32-row chunks.
// ---------------------------------------------------------------------------
template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_mode1_q(ShardArgs X, int R, const double* __restrict__ Q, const double* __restrict__ V,
              const double* __restrict__ W, double* __restrict__ partials) {
  __shared__ double qch[WPB][32 * CLD<RP>];
  __shared__ double xch[WPB][32 * CLD<RP>];
  __shared__ double acc_s[WPB][RP * RP];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int RR = R * R;
  for (int e = lane; e < RR; e += 32) acc_s[wid][e] = 0.0;
  __syncwarp();
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < X.K; k += nwarps) {
    const std::int64_t r0 = X.srp[k];
    const int I = static_cast<int>(X.srp[k + 1] - r0);
    for (int b0 = 0; b0 < I; b0 += 32) {
      const int nr = min(32, I - b0);
      stage_rows<RP>(qch[wid], Q + (r0 + b0) * R, nr, R, lane);
      double xv[RP];
      if (lane < nr) {
        dev::csr_row_times<RP>(xv, X.ci, X.val, X.rp[r0 + b0 + lane], X.rp[r0 + b0 + lane + 1], V, R);
#pragma unroll
        for (int c = 0; c < RP; ++c)
          if (c < R) xch[wid][lane * CLD<RP> + c] = xv[c] * W[k * R + c];
      }
      __syncwarp();
      for (int e = lane; e < RR; e += 32) {
        const int x = e / R, y = e - (e / R) * R;
        double acc = acc_s[wid][e];
        for (int rr = 0; rr < nr; ++rr) acc = fma(qch[wid][rr * CLD<RP> + x], xch[wid][rr * CLD<RP> + y], acc);
        acc_s[wid][e] = acc;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (wid == 0)
    for (int e = lane; e < RR; e += 32) {
      double acc = 0.0;
      for (int w = 0; w < WPB; ++w) acc += acc_s[w][e];
      partials[static_cast<std::int64_t>(blockIdx.x) * RR + e] = acc;
    }
}

// ---------------------------------------------------------------------------
// K2 projection (solver.hpp:197-208): packed Y_k(:, c) = sum over entries of
// column cols_k[c] of v * Q_k(row, :).  One warp per subject, lane per
// distinct column, rows visited in ascending order (deterministic).
// ---------------------------------------------------------------------------
template <int RP>
__global__ void k_project(ShardArgs X, int R, const double* __restrict__ Q, const std::int64_t* __restrict__ ycol_ptr,
                          const std::int32_t* __restrict__ ycols, double* __restrict__ Y) {
  const int lane = threadIdx.x & 31;
  const std::int64_t gw = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (std::int64_t k = gw; k < X.K; k += nwarps) {
    const std::int64_t r0 = X.srp[k];
    const int I = static_cast<int>(X.srp[k + 1] - r0);
    const std::int64_t c0 = ycol_ptr[k], c1 = ycol_ptr[k + 1];
    for (std::int64_t cc = c0 + lane; cc < c1; cc += 32) {
      const int col = ycols[cc];
      double acc[RP];
#pragma unroll
      for (int r = 0; r < RP; ++r) acc[r] = 0.0;
      for (int i = 0; i < I; ++i) {
        std::int64_t lo = X.rp[r0 + i], hi = X.rp[r0 + i + 1];
        while (lo < hi) {  // lower_bound
          const std::int64_t mid = (lo + hi) >> 1;
          if (X.ci[mid] < col)
            lo = mid + 1;
          else
            hi = mid;
        }
        if (lo < X.rp[r0 + i + 1] && X.ci[lo] == col) {
          const double v = X.val[lo];
#pragma unroll
          for (int r = 0; r < RP; ++r)
            if (r < R) acc[r] = fma(v, Q[(r0 + i) * R + r], acc[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < RP; ++r)
        if (r < R) Y[cc * R + r] = acc[r];
    }
  }
}

// ---------------------------------------------------------------------------
// Packed-Y MTTKRP (the reference's own kernels, mttkrp.hpp:81-166), used by
// the boundary entry points p2g_mttkrp_packed / p2g_cp_als_iteration.
// Y: per slice an R x c_k column-major block at Y + ycol_ptr[k]*R.
// ---------------------------------------------------------------------------
struct PackedArgs {
  std::int64_t K, J;
  int R;
  const std::int64_t* ycol_ptr;
  const std::int32_t* ycols;
  const double* Y;
  const double* H;
  const double* V;
  const double* W;
};

template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_packed_mode13(PackedArgs a, int mode, double* __restrict__ out) {
  // mode 1: per-block R x R partials into out[blockIdx]; mode 3: rows of out.
  __shared__ double prod_s[WPB][RP * RP];
  __shared__ double acc_s[WPB][RP * RP];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int R = a.R, RR = R * R;
  for (int e = lane; e < RR; e += 32) acc_s[wid][e] = 0.0;
  __syncwarp();
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < a.K; k += nwarps) {
    const std::int64_t c0 = a.ycol_ptr[k], c1 = a.ycol_ptr[k + 1];
    if (c1 == c0) continue;  // mttkrp.hpp:98,159 skip empty slices
    // prod = Y_k V(cols_k, :)   (R x R)
    for (int e = lane; e < RR; e += 32) {
      const int x = e / R, y = e - (e / R) * R;
      double acc = 0.0;
      for (std::int64_t c = c0; c < c1; ++c) acc = fma(a.Y[c * R + x], a.V[static_cast<std::int64_t>(a.ycols[c]) * R + y], acc);
      prod_s[wid][e] = acc;
    }
    __syncwarp();
    if (mode == 1) {
      for (int e = lane; e < RR; e += 32) {
        const int y = e - (e / R) * R;
        acc_s[wid][e] = fma(prod_s[wid][e], a.W[k * R + y], acc_s[wid][e]);
      }
    } else {
      for (int y = lane; y < R; y += 32) {
        double acc = 0.0;
        for (int x = 0; x < R; ++x) acc = fma(a.H[x * R + y], prod_s[wid][x * R + y], acc);
        out[k * R + y] = acc;
      }
    }
    __syncwarp();
  }
  if (mode == 1) {
    __syncthreads();
    if (wid == 0)
      for (int e = lane; e < RR; e += 32) {
        double acc = 0.0;
        for (int w = 0; w < WPB; ++w) acc += acc_s[w][e];
        out[static_cast<std::int64_t>(blockIdx.x) * RR + e] = acc;
      }
  }
}

/// mode 2 on packed Y, deterministic: one warp per output row j walks the
/// (slice, column) occurrences of j in slice order (col_occ built on host).
__global__ void k_packed_mode2(PackedArgs a, const std::int64_t* __restrict__ occ_ptr,
                               const std::int64_t* __restrict__ occ, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const std::int64_t gw = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int R = a.R;
  for (std::int64_t j = gw; j < a.J; j += nwarps) {
    for (int y = lane; y < R; y += 32) {
      double acc = 0.0;
      for (std::int64_t t = occ_ptr[j]; t < occ_ptr[j + 1]; ++t) {
        const std::int64_t c = occ[2 * t], k = occ[2 * t + 1];
        double tv = 0.0;  // (Y_k^T H)(c, y)
        for (int x = 0; x < R; ++x) tv = fma(a.Y[c * R + x], a.H[x * R + y], tv);
        acc = fma(tv, a.W[k * R + y], acc);
      }
      out[j * R + y] = acc;
    }
  }
}

/// Warps per block so that static shared memory stays within 48 KB.
constexpr int fit_wpb(int per_warp_doubles, int fixed_doubles) {
  int w = 8;
  while (w > 1 && (w * per_warp_doubles + fixed_doubles) * 8 > 48 * 1024) --w;
  return w;
}

int grid_for(std::int64_t warps, int wpb, int num_sms, int per_sm = 8) {
  const std::int64_t want = (warps + wpb - 1) / wpb;
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(want, static_cast<std::int64_t>(num_sms) * per_sm)));
}

}  // namespace

#define P2G_RP_DISPATCH2(R, CALL)                           \
  do {                                                      \
    if ((R) <= 2) {                                         \
      constexpr int RP_ = 2;                                \
      CALL;                                                 \
    } else if ((R) <= 4) {                                  \
      constexpr int RP_ = 4;                                \
      CALL;                                                 \
    } else if ((R) <= 5) {                                  \
      constexpr int RP_ = 5;                                \
      CALL;                                                 \
    } else if ((R) <= 8) {                                  \
      constexpr int RP_ = 8;                                \
      CALL;                                                 \
    } else if ((R) <= 10) {                                 \
      constexpr int RP_ = 10;                               \
      CALL;                                                 \
    } else if ((R) <= 16) {                                 \
      constexpr int RP_ = 16;                               \
      CALL;                                                 \
    } else if ((R) <= 24) {                                 \
      constexpr int RP_ = 24;                               \
      CALL;                                                 \
    } else if ((R) <= 32) {                                 \
      constexpr int RP_ = 32;                               \
      CALL;                                                 \
    } else if ((R) <= 40) {                                 \
      constexpr int RP_ = 40;                               \
      CALL;                                                 \
    } else {                                                \
      throw InvalidArgument("rank above 40 unsupported");   \
    }                                                       \
  } while (0)

// R <= 16 only (row-per-lane kernels that spill at larger R; their callers
// take the R > 16 branch first, so no larger instantiation is emitted).
#define P2G_RP_DISPATCH_SMALL(R, CALL)                        \
  do {                                                        \
    if ((R) <= 2) {                                           \
      constexpr int RP_ = 2;                                  \
      CALL;                                                   \
    } else if ((R) <= 4) {                                    \
      constexpr int RP_ = 4;                                  \
      CALL;                                                   \
    } else if ((R) <= 5) {                                    \
      constexpr int RP_ = 5;                                  \
      CALL;                                                   \
    } else if ((R) <= 8) {                                    \
      constexpr int RP_ = 8;                                  \
      CALL;                                                   \
    } else if ((R) <= 10) {                                   \
      constexpr int RP_ = 10;                                 \
      CALL;                                                   \
    } else if ((R) <= 16) {                                   \
      constexpr int RP_ = 16;                                 \
      CALL;                                                   \
    } else {                                                  \
      throw InvalidArgument("rank above 16 on a small-R path"); \
    }                                                         \
  } while (0)

static ShardArgs shard_args(p2g_ctx* c) {
  return ShardArgs{c->srp.get(), c->rp.get(), c->ci.get(), c->val.get(), c->k_end - c->k_begin, c->NR, c->nnz, c->J};
}

void launch_mode2(p2g_ctx* c, int R, const double* Q, const double* H, const double* W, const double* nH, double* M2,
                  cudaStream_t s) {
  const ShardArgs X = shard_args(c);
  // L2 fp64 reductions (the packed/hook path; the fused loop uses the
  // atomics-free CSC form).  On-chip accumulation was measured and dropped:
  // shared-memory fp64 atomicAdd lowers to an ATOMS.CAST.SPIN CAS loop on
  // sm_100a (14.3 ms vs 5.4 ms at cfg2).
  P2G_CUDA(cudaMemsetAsync(M2, 0, sizeof(double) * c->J * R, s));
  P2G_RP_DISPATCH2(R, ({
                     constexpr int WPB = fit_wpb(RP_ * RP_ + 32 * CLD<RP_>, 0);
                     k_mode2<RP_, WPB><<<grid_for(X.K, WPB, c->num_sms), WPB * 32, 0, s>>>(X, R, Q, H, W, nH, M2);
                   }));
  P2G_LAUNCHED(1);
}

void launch_mode3(p2g_ctx* c, int R, const double* Q, const double* H, const double* V, double* m3,
                  cudaStream_t s, double* XV_out) {
  const ShardArgs X = shard_args(c);
  if (R > 16 || XV_out) {  // the row-per-lane form spills above R = 16; the large-R loop wants X V rows
    constexpr int WPB = 8;
    if (XV_out && (R == 24 || R == 32 || R == 40)) {  // the fused loop: X V rows kept for Procrustes
      // resident blocks only (the subjects are split statically over the grid)
      auto run = [&](auto kern) {
        int per_sm = 0;
        P2G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPB * 32, 0));
        kern<<<grid_for(X.K, WPB, c->num_sms, std::max(per_sm, 1)), WPB * 32, 0, s>>>(X, Q, H, V, m3, XV_out);
      };
      if (R == 24)
        run(k_mode3_rows<24, WPB>);
      else if (R == 32)
        run(k_mode3_rows<32, WPB>);
      else
        run(k_mode3_rows<40, WPB>);
      P2G_LAUNCHED(1);
      return;
    }
    if (R <= 24)
      k_mode3_mma<24, WPB><<<grid_for(X.K, WPB, c->num_sms, 4), WPB * 32, 0, s>>>(X, R, Q, H, V, m3, XV_out);
    else if (R <= 32)
      k_mode3_mma<32, WPB><<<grid_for(X.K, WPB, c->num_sms, 4), WPB * 32, 0, s>>>(X, R, Q, H, V, m3, XV_out);
    else if (R <= 40)
      k_mode3_mma<40, WPB><<<grid_for(X.K, WPB, c->num_sms, 4), WPB * 32, 0, s>>>(X, R, Q, H, V, m3, XV_out);
    else
      throw InvalidArgument("rank above 40 unsupported");
    P2G_LAUNCHED(1);
    return;
  }
  P2G_RP_DISPATCH_SMALL(R, ({
                         constexpr int WPB = fit_wpb(32 * CLD<RP_>, RP_ * RP_);
                         k_mode3<RP_, WPB><<<grid_for(X.K, WPB, c->num_sms), WPB * 32, 0, s>>>(X, R, Q, H, V, m3);
                       }));
  P2G_LAUNCHED(1);
}

void launch_xv_rows(p2g_ctx* c, int R, const double* V, double* XV, cudaStream_t s) {
  const ShardArgs X = shard_args(c);
  constexpr int WPB = 8;
  auto run = [&](auto kern) {
    int per_sm = 0;
    P2G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPB * 32, 0));
    kern<<<grid_for(X.K, WPB, c->num_sms, std::max(per_sm, 1)), WPB * 32, 0, s>>>(X, nullptr, nullptr, V, nullptr, XV);
  };
  if (R == 24)
    run(k_mode3_rows<24, WPB, false>);
  else if (R == 32)
    run(k_mode3_rows<32, WPB, false>);
  else if (R == 40)
    run(k_mode3_rows<40, WPB, false>);
  else
    throw InvalidArgument("X V rows: exact R in {24, 32, 40}");
  P2G_LAUNCHED(1);
}

void launch_mode1_q(p2g_ctx* c, int R, const double* Q, const double* V, const double* W, double* partials,
                    int nblocks, cudaStream_t s) {
  const ShardArgs X = shard_args(c);
  P2G_RP_DISPATCH2(R, ({
                     constexpr int WPB = fit_wpb(64 * CLD<RP_> + RP_ * RP_, 0);
                     k_mode1_q<RP_, WPB><<<nblocks, WPB * 32, 0, s>>>(X, R, Q, V, W, partials);
                   }));
  P2G_LAUNCHED(1);
}

void launch_project(p2g_ctx* c, int R, const double* Q, const std::int64_t* ycol_ptr, const std::int32_t* ycols,
                    double* Y, cudaStream_t s) {
  const ShardArgs X = shard_args(c);
  P2G_RP_DISPATCH2(R, (k_project<RP_><<<grid_for(X.K, 4, c->num_sms), 128, 0, s>>>(X, R, Q, ycol_ptr, ycols, Y)));
  P2G_LAUNCHED(1);
}

int packed_mode1_blocks(int num_sms) { return num_sms * 2; }

void launch_packed_mode13(int mode, std::int64_t K, std::int64_t J, int R, const std::int64_t* ycol_ptr,
                          const std::int32_t* ycols, const double* Y, const double* H, const double* V,
                          const double* W, double* out, int nblocks, cudaStream_t s) {
  PackedArgs a{K, J, R, ycol_ptr, ycols, Y, H, V, W};
  P2G_RP_DISPATCH2(R, ({
                     constexpr int WPB = fit_wpb(2 * RP_ * RP_, 0);
                     k_packed_mode13<RP_, WPB><<<nblocks, WPB * 32, 0, s>>>(a, mode, out);
                   }));
  P2G_LAUNCHED(1);
}

void launch_packed_mode2(std::int64_t K, std::int64_t J, int R, const std::int64_t* ycol_ptr,
                         const std::int32_t* ycols, const double* Y, const double* H, const double* W,
                         const std::int64_t* occ_ptr, const std::int64_t* occ, double* out, cudaStream_t s) {
  PackedArgs a{K, J, R, ycol_ptr, ycols, Y, H, nullptr, W};
  const int blocks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((J + 3) / 4, 4096)));
  k_packed_mode2<<<blocks, 128, 0, s>>>(a, occ_ptr, occ, out);
  P2G_LAUNCHED(1);
}

}  // namespace p2g
