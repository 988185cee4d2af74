// Small-rank (R <= 16) streaming passes of the Q-free iteration: mode 2 and
// mode 3 (+ next iteration's Gram C), restated from mttkrp.hpp:111-166 with
// Q_k = X_k V P_k (+ L Chat_k) rebuilt on the fly (see k_small.cu).
//
// Layout (B200-first):
//  * one warp owns a batch of SB consecutive subjects.  Setup builds the
//    batch's R x R row operators T_s in shared memory, [element][subject]
//    (stride SB+1: lanes of different subjects hit different banks):
//        mode 3:  T3_s = diag(w_s) Hprev^T S_s H_t          (q_i = xv_i T3)
//        mode 2:  T2_s = T3_s diag(w_s o nH)                (u_i = xv_i T2)
//    with S_s the packed fast-path factor or the accurate path's full Shat.
//    Each lane computes R/LPS rows of one subject's T (LPS = 32/SB lanes
//    per subject), all indices compile-time (exact-R template).
//  * the batch's rows (contiguous in the CSR) stream in chunks of 32, one
//    row per lane, across subject boundaries (full lanes regardless of I_k);
//    each lane finds its subject in the batch row offsets.
//  * mode 2 writes the row factors u_i (coalesced); M2 = X^T U is read out
//    from the CSC copy without atomics (k_csc.cu).
//  * mode 3 stages the xn and q rows in shared memory and accumulates the
//    next iteration's Gram C = Xn^T Xn and m3 = diag(Q^T Xn) on the fp64
//    tensor cores (DMMA m8n8k4, 4-row k-steps per subject segment, rows of
//    other subjects masked to zero), flushing at subject boundaries
//    (warp-uniform control, fixed order: deterministic).
#include <algorithm>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"

namespace p2g {
namespace {

template <int R>
struct StreamCfg {
  // subjects per batch: the largest power of two keeping a lane's share of
  // the setup (NRL rows of B, R doubles each) within ~32 registers' doubles
  static constexpr int pick_sb() {
    int sb = 32;
    while (sb > 4 && ((R + 32 / sb - 1) / (32 / sb)) * R > 32) sb /= 2;
    return sb;
  }
  static constexpr int SB = pick_sb();
  static constexpr int SBP = SB + 1;                          // [element][subject] stride
  static constexpr int LPS = 32 / SB;                         // lanes per subject in setup
  static constexpr int NRL = (R + LPS - 1) / LPS;             // T rows per lane
  static constexpr int RR = R * R;
  static constexpr int NT = R * (R + 1) / 2;
  static constexpr int WPB = 4;
  static constexpr int kWarpT = RR * SBP;                     // doubles
  static constexpr int UM2 = 4;                               // rows per lane in flight (mode 2)
  static constexpr int UM3 = 1;                               // rows per lane in flight (mode 3)
  static constexpr int NB = (R + 7) / 8;                      // 8 x 8 tensor tiles per side (mode 3)
  static constexpr int XS = NB == 1 ? 12 : 20;                // staged row stride: conflict-free fragments
  static constexpr int kWarpCh = 2 * 32 * UM3 * XS;           // doubles (mode 3: xn and q rows)
};

__host__ __device__ constexpr int tri_idx(int i, int j) { return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i; }

/// Builds T_s for the warp's batch [k0, k0 + nb) into Tw ([e][s], stride SBP).
/// MODE 2 additionally scales column c by w_s[c] * nH[c].
template <int R, int MODE>
__device__ __forceinline__ void build_batch_ops(std::int64_t k0, int nb, const double* Hs, const double* Hts,
                                                const double* __restrict__ nH, const double* __restrict__ Wprev,
                                                const double* __restrict__ Sbuf, const double* __restrict__ Shat,
                                                const std::int32_t* fl, double* Tw, int lane) {
  using C = StreamCfg<R>;
  // 1. stage S_s (full, row-major [c][b]) into the T area: every load of
  //    the batch issued before any store (one dependent load at a time left
  //    the setup latency-bound)
  if constexpr (MODE == 2) {  // (mode 2: the batched form below costs a CTA per SM in registers)
#pragma unroll 4
    for (int idx = lane; idx < nb * C::RR; idx += 32) {
      const int s = idx / C::RR, e = idx - s * C::RR;
      const int c = e / R, b = e - c * R;
      const std::int64_t k = k0 + s;
      Tw[e * C::SBP + s] =
          fl[s] != P2G_FLAG_FULL_RANK ? __ldg(Shat + k * C::RR + e) : __ldg(Sbuf + k * C::NT + tri_idx(c, b));
    }
  } else {
  constexpr int NIT = (C::SB * C::RR + 31) / 32;
  double vv[NIT];
#pragma unroll
  for (int j = 0; j < NIT; ++j) {
    const int idx = lane + 32 * j;
    const int s = idx / C::RR, e = idx - s * C::RR;
    const int c = e / R, b = e - c * R;
    const std::int64_t k = k0 + s;
    vv[j] = idx < nb * C::RR
                ? (fl[s] != P2G_FLAG_FULL_RANK ? Shat[k * C::RR + e] : Sbuf[k * C::NT + tri_idx(c, b)])
                : 0.0;
  }
#pragma unroll
  for (int j = 0; j < NIT; ++j) {
    const int idx = lane + 32 * j;
    const int s = idx / C::RR, e = idx - s * C::RR;
    if (idx < nb * C::RR) Tw[e * C::SBP + s] = vv[j];
  }
  }
  __syncwarp();
  // 2. B rows a = q + LPS m of subject s: B[a][b] = sum_c H[c][a] S[c][b]
  const int s = lane % C::SB, q = lane / C::SB;
  const bool act = s < nb;
  double Bm[C::NRL][R];
#pragma unroll
  for (int m = 0; m < C::NRL; ++m) {
    const int a = q + C::LPS * m;
#pragma unroll
    for (int b = 0; b < R; ++b) Bm[m][b] = 0.0;
    if (act && a < R) {
#pragma unroll
      for (int c = 0; c < R; ++c) {
        const double h = Hs[c * R + a];
#pragma unroll
        for (int b = 0; b < R; ++b) Bm[m][b] = fma(h, Tw[(c * R + b) * C::SBP + s], Bm[m][b]);
      }
    }
  }
  __syncwarp();
  // 3. T rows: T[a][c'] = w_a sum_b B[a][b] Ht[b][c'] (x w_c' nH_c' in mode 2)
  const double* wk = Wprev + (k0 + s) * R;
  double cs[R];
#pragma unroll
  for (int c = 0; c < R; ++c) cs[c] = (MODE == 2 && act) ? wk[c] * nH[c] : 1.0;
#pragma unroll
  for (int m = 0; m < C::NRL; ++m) {
    const int a = q + C::LPS * m;
    if (!act || a >= R) continue;
    const double wa = wk[a];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < R; ++b) acc = fma(Bm[m][b], Hts[b * R + c], acc);
      Tw[(a * R + c) * C::SBP + s] = acc * wa * cs[c];
    }
  }
  __syncwarp();
}

/// Mode 2 row factors: u_i = xv_i T2_s (+ Chat_i H_t diag(w o nH)) -> U (NR x R);
/// M2 = X^T U follows from the CSC pass (k_csc.cu).
template <int R>
__global__ void __launch_bounds__(StreamCfg<R>::WPB * 32)
    k_mode2_sb(ShardArgs X, const double* __restrict__ Hprev, const double* __restrict__ Vprev,
               const double* __restrict__ Wprev, const double* __restrict__ Ht, const double* __restrict__ nH,
               const double* __restrict__ Sbuf, const double* __restrict__ Shat, const double* __restrict__ Chat,
               const std::int32_t* __restrict__ flags, double* __restrict__ U, const double* __restrict__ XV) {
  using C = StreamCfg<R>;
  extern __shared__ double smem[];
  __shared__ std::int32_t rowoff_s[C::WPB][C::SB + 1];
  __shared__ std::int32_t fl_s[C::WPB][C::SB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Hs = smem;
  double* Hts = Hs + C::RR;
  double* Tw = Hts + C::RR + wid * C::kWarpT;
  std::int32_t* rowoff = rowoff_s[wid];
  std::int32_t* fl = fl_s[wid];
  for (int e = threadIdx.x; e < C::RR; e += blockDim.x) {
    Hs[e] = Hprev[e];
    Hts[e] = Ht[e];
  }
  __syncthreads();
  const std::int64_t nbatch = (X.K + C::SB - 1) / C::SB;
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * C::WPB;
  for (std::int64_t bt = static_cast<std::int64_t>(blockIdx.x) * C::WPB + wid; bt < nbatch; bt += nwarps) {
    const std::int64_t k0 = bt * C::SB;
    const int nb = static_cast<int>(min(static_cast<std::int64_t>(C::SB), X.K - k0));
    const std::int64_t row0 = X.srp[k0];
    const int nrows = static_cast<int>(X.srp[k0 + nb] - row0);
    for (int s = lane; s <= C::SB; s += 32) rowoff[s] = s <= nb ? static_cast<int>(X.srp[k0 + s] - row0) : nrows;
    if (lane < C::SB) fl[lane] = lane < nb ? flags[k0 + lane] : P2G_FLAG_FULL_RANK;
    __syncwarp();
    build_batch_ops<R, 2>(k0, nb, Hs, Hts, nH, Wprev, Sbuf, Shat, fl, Tw, lane);
    int sl = 0;
    constexpr int UR = C::UM2;
    for (int cb = 0; cb < nrows; cb += 32 * UR) {
      std::int64_t p0[UR], p1[UR];
      int su[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const int r = cb + lane + 32 * u;
        p0[u] = p1[u] = 0;
        su[u] = -1;
        if (r < nrows) {
          while (rowoff[sl + 1] <= r) ++sl;
          su[u] = sl;
          if (!XV) {  // the row extents are only needed to gather
            p0[u] = __ldg(X.rp + row0 + r);
            p1[u] = __ldg(X.rp + row0 + r + 1);
          }
        }
      }
      double xv[UR][R];
      if (XV) {  // X V_prev rows left by the previous mode-3 pass (a streaming read, no V gathers)
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const double* xr = XV + (row0 + cb + lane + 32 * u) * R;
#pragma unroll
          for (int a = 0; a < R; ++a) xv[u][a] = su[u] >= 0 ? __ldg(xr + a) : 0.0;
        }
      } else {
        dev::csr_rows_times<R, UR, 1>(xv, xv, X.ci, X.val, p0, p1, Vprev, Vprev);
      }
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const int s_ = su[u];
        if (s_ < 0) continue;
        double uv[R];
#pragma unroll
        for (int c = 0; c < R; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < R; ++a) acc = fma(xv[u][a], Tw[(a * R + c) * C::SBP + s_], acc);
          uv[c] = acc;
        }
        const int i = cb + lane + 32 * u - rowoff[s_];
        if (fl[s_] != P2G_FLAG_FULL_RANK && i < R) {  // completion term L Chat (rows < R)
          const std::int64_t k = k0 + s_;
          const double* chr = Chat + k * C::RR + i * R;
#pragma unroll
          for (int c = 0; c < R; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int b = 0; b < R; ++b) acc = fma(chr[b], Hts[b * R + c], acc);
            uv[c] = fma(acc, Wprev[k * R + c] * nH[c], uv[c]);
          }
        }
        double* urow = U + (row0 + cb + lane + 32 * u) * R;  // consecutive lanes, consecutive rows
#pragma unroll
        for (int c = 0; c < R; ++c) urow[c] = uv[c];
      }
    }
    __syncwarp();
  }
}

/// Mode 3 fused with next iteration's Gram:
///   m3(k,c) = sum_i (xv_prev,i T3_s + Chat_i H_t)_c (xv_new,i)_c,
///   C_k     = sum_i xv_new,i^T xv_new,i (packed lower).
template <int R>
__global__ void __launch_bounds__(StreamCfg<R>::WPB * 32)
    k_mode3_sb(ShardArgs X, const double* __restrict__ Hprev, const double* __restrict__ Vprev,
               const double* __restrict__ Wprev, const double* __restrict__ Ht, const double* __restrict__ Vt,
               const double* __restrict__ Sbuf, const double* __restrict__ Shat, const double* __restrict__ Chat,
               const std::int32_t* __restrict__ flags, double* __restrict__ M3, double* __restrict__ Cnext,
               double* __restrict__ XV, int xv_in) {
  using C = StreamCfg<R>;
  extern __shared__ double smem[];
  __shared__ std::int32_t rowoff_s[C::WPB][C::SB + 1];
  __shared__ std::int32_t fl_s[C::WPB][C::SB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Hs = smem;
  double* Hts = Hs + C::RR;
  double* Tw = Hts + C::RR + wid * (C::kWarpT + C::kWarpCh);
  double* ch = Tw + C::kWarpT;
  std::int32_t* rowoff = rowoff_s[wid];
  std::int32_t* fl = fl_s[wid];
  for (int e = threadIdx.x; e < C::RR; e += blockDim.x) {
    Hs[e] = Hprev[e];
    Hts[e] = Ht[e];
  }
  __syncthreads();
  const std::int64_t nbatch = (X.K + C::SB - 1) / C::SB;
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * C::WPB;
  for (std::int64_t bt = static_cast<std::int64_t>(blockIdx.x) * C::WPB + wid; bt < nbatch; bt += nwarps) {
    const std::int64_t k0 = bt * C::SB;
    const int nb = static_cast<int>(min(static_cast<std::int64_t>(C::SB), X.K - k0));
    const std::int64_t row0 = X.srp[k0];
    const int nrows = static_cast<int>(X.srp[k0 + nb] - row0);
    for (int s = lane; s <= C::SB; s += 32) rowoff[s] = s <= nb ? static_cast<int>(X.srp[k0 + s] - row0) : nrows;
    if (lane < C::SB) fl[lane] = lane < nb ? flags[k0 + lane] : P2G_FLAG_FULL_RANK;
    __syncwarp();
    build_batch_ops<R, 3>(k0, nb, Hs, Hts, nullptr, Wprev, Sbuf, Shat, fl, Tw, lane);
    // fp64 tensor-core accumulators (DMMA m8n8k4, fragment: c0 = C[lane/4][2(lane%4)],
    // c1 = C[lane/4][2(lane%4)+1]): Gram tiles (0,0), (1,0), (1,1) of Xn^T Xn and the
    // diagonal tiles of Q^T Xn (m3 = its diagonal)
    double g00[2] = {0.0, 0.0}, g10[2] = {0.0, 0.0}, g11[2] = {0.0, 0.0};
    double d00[2] = {0.0, 0.0}, d11[2] = {0.0, 0.0};
    int cur = 0;  // subject being accumulated (warp-uniform)
    const int fm = lane >> 2, fn = 2 * (lane & 3);
    auto flush = [&](int s) {
      const std::int64_t k = k0 + s;
      double* cn = Cnext + k * C::NT;
      auto put = [&](int a, int b, double v) {
        if (a < R && b <= a) cn[a * (a + 1) / 2 + b] = v;
      };
      put(fm, fn, g00[0]);
      put(fm, fn + 1, g00[1]);
      if (fm == fn && fm < R) M3[k * R + fm] = d00[0];
      if (fm == fn + 1 && fm < R) M3[k * R + fm] = d00[1];
      if constexpr (C::NB == 2) {
        put(8 + fm, fn, g10[0]);
        put(8 + fm, fn + 1, g10[1]);
        put(8 + fm, 8 + fn, g11[0]);
        put(8 + fm, 8 + fn + 1, g11[1]);
        if (fm == fn && 8 + fm < R) M3[k * R + 8 + fm] = d11[0];
        if (fm == fn + 1 && 8 + fm < R) M3[k * R + 8 + fm] = d11[1];
      }
      g00[0] = g00[1] = g10[0] = g10[1] = g11[0] = g11[1] = 0.0;
      d00[0] = d00[1] = d11[0] = d11[1] = 0.0;
    };
    int sl = 0;
    constexpr int UR = C::UM3;
    for (int cb = 0; cb < nrows; cb += 32 * UR) {
      const int nr = min(32 * UR, nrows - cb);
      std::int64_t p0[UR], p1[UR];
      int su[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const int r = cb + lane + 32 * u;
        p0[u] = p1[u] = 0;
        su[u] = -1;
        if (r < nrows) {
          while (rowoff[sl + 1] <= r) ++sl;
          su[u] = sl;
          p0[u] = __ldg(X.rp + row0 + r);
          p1[u] = __ldg(X.rp + row0 + r + 1);
        }
      }
      double xp[UR][R], xn[UR][R];  // both gathers share the entry stream
      if (xv_in) {  // X V_prev rows from the previous pass; only V_t is gathered
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const double* xr = XV + (row0 + cb + lane + 32 * u) * R;
#pragma unroll
          for (int a = 0; a < R; ++a) xp[u][a] = su[u] >= 0 ? xr[a] : 0.0;
        }
        dev::csr_rows_times<R, UR, 1>(xn, xn, X.ci, X.val, p0, p1, Vt, Vt);
      } else {
        dev::csr_rows_times<R, UR, 2>(xp, xn, X.ci, X.val, p0, p1, Vprev, Vt);
      }
      if (XV) {  // X V_t rows for the next iteration (each lane rewrites its own rows)
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          if (su[u] < 0) continue;
          double* xr = XV + (row0 + cb + lane + 32 * u) * R;
#pragma unroll
          for (int a = 0; a < R; ++a) xr[a] = xn[u][a];
        }
      }
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const int s_ = su[u];
        if (s_ < 0) continue;
        double qv[R];
#pragma unroll
        for (int c = 0; c < R; ++c) {
          double a0 = 0.0;
#pragma unroll
          for (int a = 0; a < R; ++a) a0 = fma(xp[u][a], Tw[(a * R + c) * C::SBP + s_], a0);
          qv[c] = a0;
        }
        const int i = cb + lane + 32 * u - rowoff[s_];
        if (fl[s_] != P2G_FLAG_FULL_RANK && i < R) {  // completion term L Chat (rows < R)
          const double* chr = Chat + (k0 + s_) * C::RR + i * R;
#pragma unroll
          for (int c = 0; c < R; ++c) {
            double a0 = 0.0;
#pragma unroll
            for (int b = 0; b < R; ++b) a0 = fma(chr[b], Hts[b * R + c], a0);
            qv[c] += a0;
          }
        }
        double* xs = ch + (lane + 32 * u) * C::XS;
        double* qs = xs + 32 * UR * C::XS;
#pragma unroll
        for (int a = 0; a < 8 * C::NB; ++a) {
          xs[a] = a < R ? xn[u][a] : 0.0;
          qs[a] = a < R ? qv[a] : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < UR; ++u)
        if (su[u] < 0) {  // past the batch: zero rows accumulate nothing
          double* xs = ch + (lane + 32 * u) * C::XS;
          double* qs = xs + 32 * UR * C::XS;
#pragma unroll
          for (int a = 0; a < 8 * C::NB; ++a) xs[a] = qs[a] = 0.0;
        }
      __syncwarp();
      // per subject segment [ss, se) of the chunk: 4-row k-steps on the tensor
      // cores, rows outside the segment enter as zeros (warp-uniform control)
      int ss = 0;
      while (ss < nr) {
        const int end = rowoff[cur + 1] - cb;
        if (end <= ss) {  // subject closed at or before this point
          flush(cur++);
          continue;
        }
        const int se = min(end, nr);
        for (int k4 = ss & ~3; k4 < se; k4 += 4) {
          const int r = k4 + (lane & 3);
          const bool in = r >= ss && r < se;
          const double* xr = ch + r * C::XS;
          const double* qr = xr + 32 * UR * C::XS;
          const double x0 = in ? xr[fm] : 0.0, q0 = in ? qr[fm] : 0.0;
          dev::dmma884(g00, x0, x0);
          dev::dmma884(d00, q0, x0);
          if constexpr (C::NB == 2) {
            const double x1 = in ? xr[8 + fm] : 0.0, q1 = in ? qr[8 + fm] : 0.0;
            dev::dmma884(g10, x1, x0);
            dev::dmma884(g11, x1, x1);
            dev::dmma884(d11, q1, x1);
          }
        }
        if (end <= nr) flush(cur++);
        ss = se;
      }
      __syncwarp();
    }
    for (; cur < nb; ++cur) flush(cur);
  }
}

template <int R>
int stream_blocks(p2g_ctx* c, const void* kern, std::size_t smem) {
  using C = StreamCfg<R>;
  int per_sm = 0;
  P2G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPB * 32, smem));
  const std::int64_t nbatch = (c->k_end - c->k_begin + C::SB - 1) / C::SB;
  const std::int64_t want = (nbatch + C::WPB - 1) / C::WPB;
  return static_cast<int>(std::max<std::int64_t>(
      1, std::min<std::int64_t>(want, static_cast<std::int64_t>(c->num_sms) * std::max(per_sm, 1))));
}

ShardArgs shard_args_st(p2g_ctx* c) {
  return ShardArgs{c->srp.get(), c->rp.get(), c->ci.get(), c->val.get(), c->k_end - c->k_begin, c->NR, c->nnz, c->J};
}

template <int R>
void mode2_sb(p2g_ctx* c, const double* Hprev, const double* Vprev, const double* Wprev, const double* Ht,
              const double* nH, const double* Sbuf, const double* Shat, const double* Chat, const std::int32_t* flags,
              double* U, cudaStream_t s, const double* XV) {
  using C = StreamCfg<R>;
  const std::size_t smem = sizeof(double) * (2 * C::RR + C::WPB * C::kWarpT);
  auto kern = k_mode2_sb<R>;
  P2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int nb = stream_blocks<R>(c, reinterpret_cast<const void*>(kern), smem);
  kern<<<nb, C::WPB * 32, smem, s>>>(shard_args_st(c), Hprev, Vprev, Wprev, Ht, nH, Sbuf, Shat, Chat, flags, U, XV);
}

template <int R>
void mode3_sb(p2g_ctx* c, const double* Hprev, const double* Vprev, const double* Wprev, const double* Ht,
              const double* Vt, const double* Sbuf, const double* Shat, const double* Chat, const std::int32_t* flags,
              double* M3, double* Cnext, cudaStream_t s, double* XV, int xv_in) {
  using C = StreamCfg<R>;
  const std::size_t smem = sizeof(double) * (2 * C::RR + C::WPB * (C::kWarpT + C::kWarpCh));
  auto kern = k_mode3_sb<R>;
  P2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int nb = stream_blocks<R>(c, reinterpret_cast<const void*>(kern), smem);
  kern<<<nb, C::WPB * 32, smem, s>>>(shard_args_st(c), Hprev, Vprev, Wprev, Ht, Vt, Sbuf, Shat, Chat, flags, M3,
                                     Cnext, XV, xv_in);
}

}  // namespace

#define P2G_EXACT_R_DISPATCH(R, CALL)                                   \
  switch (R) {                                                          \
    case 1: { constexpr int R_ = 1; CALL; } break;                      \
    case 2: { constexpr int R_ = 2; CALL; } break;                      \
    case 3: { constexpr int R_ = 3; CALL; } break;                      \
    case 4: { constexpr int R_ = 4; CALL; } break;                      \
    case 5: { constexpr int R_ = 5; CALL; } break;                      \
    case 6: { constexpr int R_ = 6; CALL; } break;                      \
    case 7: { constexpr int R_ = 7; CALL; } break;                      \
    case 8: { constexpr int R_ = 8; CALL; } break;                      \
    case 9: { constexpr int R_ = 9; CALL; } break;                      \
    case 10: { constexpr int R_ = 10; CALL; } break;                    \
    case 11: { constexpr int R_ = 11; CALL; } break;                    \
    case 12: { constexpr int R_ = 12; CALL; } break;                    \
    case 13: { constexpr int R_ = 13; CALL; } break;                    \
    case 14: { constexpr int R_ = 14; CALL; } break;                    \
    case 15: { constexpr int R_ = 15; CALL; } break;                    \
    case 16: { constexpr int R_ = 16; CALL; } break;                    \
    default: throw InvalidArgument("small-rank streaming path needs R <= 16"); \
  }

void launch_mode2_qf(p2g_ctx* c, int R, const double* Hprev, const double* Vprev, const double* Wprev,
                     const double* Ht, const double* nH, const double* Sbuf, const double* Shat, const double* Chat,
                     const std::int32_t* flags, double* U, cudaStream_t s, const double* XV) {
  if (c->k_end > c->k_begin) {
    P2G_EXACT_R_DISPATCH(R, (mode2_sb<R_>(c, Hprev, Vprev, Wprev, Ht, nH, Sbuf, Shat, Chat, flags, U, s, XV)));
    P2G_LAUNCHED(1);
  }
}

void launch_mode3_qf(p2g_ctx* c, int R, const double* Hprev, const double* Vprev, const double* Wprev,
                     const double* Ht, const double* Vt, const double* Sbuf, const double* Shat, const double* Chat,
                     const std::int32_t* flags, double* M3, double* Cnext, cudaStream_t s, double* XV,
                     int xv_in) {
  if (c->k_end > c->k_begin) {
    P2G_EXACT_R_DISPATCH(R, (mode3_sb<R_>(c, Hprev, Vprev, Wprev, Ht, Vt, Sbuf, Shat, Chat, flags, M3, Cnext, s, XV,
                                          xv_in)));
    P2G_LAUNCHED(1);
  }
}

}  // namespace p2g
