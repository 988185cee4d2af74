// Atomics-free mode-2 MTTKRP: M2 = X^T U over a column-major copy of the shard.
//
// mttkrp_mode2 (mttkrp.hpp:111-138) is M2 = sum_k X_k^T U_k with row factors
// U_k = Q_k H diag(W_k o nH).  Scattering v * u_i into M2 with L2 fp64
// reductions costs one L2 request per (entry, column) pair: 630M requests per
// iteration at cfg2, where ncu shows L1/L2 at 77%/64% of their request
// throughput (profiles/).  Instead, each row's u_i is written once (the
// streaming kernels produce it coalesced), and M2 is read out from a
// column-major copy of the shard built at load time:
//   M2[j, :] = sum_{(i, v) in column j} v * U[i, :]
// The copy is ordered by (row block, column), row blocks of 2^17 rows: the
// segments in flight share one or two row blocks of U (10 MB at R = 10,
// 42 MB at R = 40), so the random U-row gathers hit L2 instead of DRAM.
// A segment is a run of one (row block, column) cut at kSeg entries (Zipf
// columns of cfg5 stay balanced); one thread sums a segment, and a second
// pass adds each column's segment partials in row-block order:
// deterministic, no atomics.
#include <algorithm>
#include <cstring>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"

namespace p2g {
namespace {

constexpr std::int64_t kSeg = 256;  // entries per segment (one thread)
constexpr int kRowBlockBits = 16;   // row blocks of 2^16 rows (U block 21 MB at R = 40)

__global__ void k_row_expand(std::int64_t NR, const std::int64_t* __restrict__ rp, std::int32_t* __restrict__ row_of) {
  for (std::int64_t r = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < NR;
       r += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    for (std::int64_t p = rp[r]; p < rp[r + 1]; ++p) row_of[p] = static_cast<std::int32_t>(r);
}

__global__ void k_iota(std::int64_t n, std::int32_t* __restrict__ out) {
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<std::int32_t>(i);
}

__global__ void k_csc_gather(std::int64_t n, const std::int32_t* __restrict__ perm, const std::int32_t* __restrict__ row_of,
                             const double* __restrict__ val, std::int32_t* __restrict__ crow, double* __restrict__ cval) {
  for (std::int64_t q = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int32_t p = perm[q];
    crow[q] = row_of[p];
    cval[q] = val[p];
  }
}

__global__ void k_block_keys(std::int64_t n, std::int64_t J, const std::int32_t* __restrict__ row_of,
                             const std::int32_t* __restrict__ ci, std::uint64_t* __restrict__ keys) {
  for (std::int64_t p = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    keys[p] = static_cast<std::uint64_t>(row_of[p] >> kRowBlockBits) * static_cast<std::uint64_t>(J) +
              static_cast<std::uint64_t>(ci[p]);
}

/// run_start[q] candidates: q where the (block, column) key changes, else 0 (max-scanned).
__global__ void k_run_marks(std::int64_t n, const std::uint64_t* __restrict__ keys, std::int64_t* __restrict__ mark) {
  for (std::int64_t q = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    mark[q] = (q == 0 || keys[q] != keys[q - 1]) ? q : 0;
}

/// Segment heads: a new run, or every kSeg entries inside a run.
__global__ void k_seg_heads(std::int64_t n, const std::int64_t* __restrict__ run_start, unsigned char* __restrict__ head) {
  for (std::int64_t q = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    head[q] = ((q - run_start[q]) % kSeg) == 0 ? 1 : 0;
}

/// Per segment: column-major key col * nblk + block (for the per-column lists).
__global__ void k_seg_colkeys(std::int64_t nseg, std::int64_t J, std::int64_t nblk, const std::int64_t* __restrict__ seg_beg,
                              const std::uint64_t* __restrict__ keys, std::uint64_t* __restrict__ ckey,
                              std::int32_t* __restrict__ ids) {
  for (std::int64_t s = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < nseg;
       s += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::uint64_t k = keys[seg_beg[s]];
    const std::uint64_t blk = k / static_cast<std::uint64_t>(J), col = k - blk * static_cast<std::uint64_t>(J);
    ckey[s] = col * static_cast<std::uint64_t>(nblk) + blk;
    ids[s] = static_cast<std::int32_t>(s);
  }
}

/// ptr[j] = first position whose key / nblk >= j (binary search over sorted keys).
__global__ void k_key_ptr(std::int64_t J, std::int64_t n, std::int64_t div, const std::uint64_t* __restrict__ keys,
                          std::int64_t* __restrict__ ptr) {
  for (std::int64_t j = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j <= J;
       j += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    std::int64_t lo = 0, hi = n;
    while (lo < hi) {
      const std::int64_t mid = (lo + hi) >> 1;
      if (static_cast<std::int64_t>(keys[mid] / static_cast<std::uint64_t>(div)) < j)
        lo = mid + 1;
      else
        hi = mid;
    }
    ptr[j] = lo;
  }
}

int grid_for(std::int64_t n, int threads) {
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + threads - 1) / threads, 148 * 32)));
}

/// Thread per segment: partial[s, :] = sum over the segment's entries of v * U[row, :].
/// Consecutive threads hold consecutive segments of the same row block.
template <int RP>
__global__ void __launch_bounds__(128) k_seg_spmm(int R, std::int64_t nseg, std::int64_t n,
                                                  const std::int64_t* __restrict__ seg_beg,
                                                  const std::int32_t* __restrict__ crow,
                                                  const double* __restrict__ cval, const double* __restrict__ U,
                                                  double* __restrict__ partial) {
  for (std::int64_t s = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < nseg;
       s += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    double acc[RP];
#pragma unroll
    for (int c = 0; c < RP; ++c) acc[c] = 0.0;
    const std::int64_t q1 = s + 1 < nseg ? seg_beg[s + 1] : n;
    for (std::int64_t q = seg_beg[s]; q < q1; ++q) {
      const double v = cval[q];
      const double* u = U + static_cast<std::int64_t>(crow[q]) * R;
      if constexpr (RP % 2 == 0) {
        if ((R & 1) == 0) {
#pragma unroll
          for (int c = 0; c < RP; c += 2)
            if (c < R) {
              const double2 x = __ldg(reinterpret_cast<const double2*>(u + c));
              acc[c] = fma(v, x.x, acc[c]);
              acc[c + 1] = fma(v, x.y, acc[c + 1]);
            }
          continue;
        }
      }
#pragma unroll
      for (int c = 0; c < RP; ++c)
        if (c < R) acc[c] = fma(v, __ldg(u + c), acc[c]);
    }
    double* out = partial + s * R;
#pragma unroll
    for (int c = 0; c < RP; ++c)
      if (c < R) out[c] = acc[c];
  }
}

/// R > 16 (exact R, R % 4 == 0): warp per segment.  A U row (8 R bytes) is
/// read by R / 4 lanes with 32-byte loads, so three lane groups take three
/// entries per warp instruction (entries t = g mod 3 to group g, 4 in flight
/// per group); the segment's entries are staged 32 at a time in registers and
/// broadcast by shuffles, and the three group sums are added in a fixed order
/// at the end of the segment (deterministic).  Warps claim segments one at a
/// time from a counter, so the warps in flight always work near one frontier
/// -- one row block of U (21 MB at R = 40), which stays in L2.  (A static
/// grid-stride drifts: warps that drew short segments run ahead, and the
/// window spread over ~20 row blocks, re-reading U from DRAM 3x; claiming
/// chunks of 16 segments widened it the same way.)
template <int RP>
__global__ void __launch_bounds__(256) k_seg_spmm_w(std::int64_t nseg, std::int64_t n,
                                                    const std::int64_t* __restrict__ seg_beg,
                                                    const std::int32_t* __restrict__ crow,
                                                    const double* __restrict__ cval, const double* __restrict__ U,
                                                    double* __restrict__ partial, unsigned long long* next) {
  constexpr int kL = RP / 4;     // lanes per U row
  constexpr int kG = 32 / kL;    // entries per warp instruction
  static_assert(RP % 4 == 0 && kL <= 32 && kG >= 1, "exact R, multiple of 4");
  const int lane = threadIdx.x & 31;
  const int g = lane / kL, sub = lane - g * kL;
  const bool act = g < kG;
  const int c = 4 * sub;
  while (true) {
    unsigned long long s0 = 0;
    if (lane == 0) s0 = atomicAdd(next, 1ull);
    s0 = __shfl_sync(dev::kFull, s0, 0);
    if (s0 >= static_cast<unsigned long long>(nseg)) break;
    const std::int64_t s = static_cast<std::int64_t>(s0);
    const std::int64_t q0 = seg_beg[s], q1 = s + 1 < nseg ? seg_beg[s + 1] : n;
    double4 a = make_double4(0.0, 0.0, 0.0, 0.0);
    for (std::int64_t qb = q0; qb < q1; qb += 32) {
      const int m = static_cast<int>(q1 - qb < 32 ? q1 - qb : 32);
      const std::int32_t rr = lane < m ? __ldg(crow + qb + lane) : 0;
      const double vv = lane < m ? __ldg(cval + qb + lane) : 0.0;
      for (int t0 = 0; t0 < m; t0 += 4 * kG) {
        double v[4];
        double4 y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + kG * u + g;  // this group's entry
          const int r = __shfl_sync(dev::kFull, rr, t & 31);
          const double w = __shfl_sync(dev::kFull, vv, t & 31);
          const bool on = act && t < m;
          v[u] = on ? w : 0.0;
          y[u] = on ? dev::ldg256(U + static_cast<std::size_t>(r) * RP + c) : make_double4(0.0, 0.0, 0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a.x = fma(v[u], y[u].x, a.x);
          a.y = fma(v[u], y[u].y, a.y);
          a.z = fma(v[u], y[u].z, a.z);
          a.w = fma(v[u], y[u].w, a.w);
        }
      }
    }
    // group sums in a fixed order: group 0 + group 1 + ... (lanes sub + kL g)
#pragma unroll
    for (int h = 1; h < kG; ++h) {
      const int src = sub + kL * h;
      const double bx = __shfl_sync(dev::kFull, a.x, src), by = __shfl_sync(dev::kFull, a.y, src);
      const double bz = __shfl_sync(dev::kFull, a.z, src), bw = __shfl_sync(dev::kFull, a.w, src);
      if (g == 0) {
        a.x += bx;
        a.y += by;
        a.z += bz;
        a.w += bw;
      }
    }
    if (g == 0) {
      double* o = partial + s * RP + c;
      *reinterpret_cast<double2*>(o) = make_double2(a.x, a.y);
      *reinterpret_cast<double2*>(o + 2) = make_double2(a.z, a.w);
    }
  }
}

/// M2[j, c] = sum of column j's segment partials, in row-block order.
__global__ void k_seg_reduce(int R, std::int64_t J, const std::int64_t* __restrict__ seg_ptr,
                             const std::int32_t* __restrict__ seg_ids, const double* __restrict__ partial,
                             double* __restrict__ M2) {
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < J * R;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t j = e / R;
    const int c = static_cast<int>(e - j * R);
    double t = 0.0;
    for (std::int64_t q = seg_ptr[j]; q < seg_ptr[j + 1]; ++q) t += partial[static_cast<std::int64_t>(seg_ids[q]) * R + c];
    M2[e] = t;
  }
}

/// U = Q_k H diag(W_k o nH) row factors for R > 16 on the fp64 tensor cores:
/// warp per subject.  H (zero-padded to RP x RP) is shared by every subject, so
/// one copy per CTA sits in shared memory (row stride RP + 4: the B fragments of
/// a half-warp, 4 rows x 4 columns, fall on 16 different bank pairs) and the
/// per-subject column scale w_k o nH is applied to the C fragments instead of
/// being folded into a per-warp copy of H (round 1: 12.8 KB per warp rebuilt per
/// subject, 16 warps per SM).  8-row tiles of Q_k are DMMA A fragments straight
/// from HBM (one tile's ten loads in flight per lane, 24+ warps per SM); U rows
/// stored as 16-byte pairs.
template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32, 3)
    k_urows(ShardArgs X, int R, const double* __restrict__ Q, const double* __restrict__ H,
            const double* __restrict__ W, const double* __restrict__ nH, double* __restrict__ U) {
  constexpr int NB = RP / 8, LDH = RP + 4;
  __shared__ double Hs[RP * LDH];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, fm = lane >> 2, fk = lane & 3;
  for (int e = threadIdx.x; e < RP * RP; e += blockDim.x) {
    const int a = e / RP, c = e - a * RP;
    Hs[a * LDH + c] = (a < R && c < R) ? H[a * R + c] : 0.0;
  }
  __syncthreads();
  const bool even = (R & 1) == 0;
  const unsigned hb = static_cast<unsigned>(__cvta_generic_to_shared(Hs)) + 8u * static_cast<unsigned>(fk * LDH + fm);
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < X.K; k += nwarps) {
    const std::int64_t r0 = X.srp[k];
    const int I = static_cast<int>(X.srp[k + 1] - r0);
    double sc[NB][2];  // this lane's columns of w_k o nH
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 8 * b + 2 * fk + h;
        sc[b][h] = c < R ? __ldg(W + k * R + c) * __ldg(nH + c) : 0.0;
      }
    for (int i0 = 0; i0 < I; i0 += 8) {
      const int i = i0 + fm;
      const double* qrow = Q + (r0 + i) * R;
      double x[RP / 4];
#pragma unroll
      for (int k4 = 0; k4 < RP; k4 += 4) {
        const int c = k4 + fk;
        x[k4 / 4] = (i < I && c < R) ? __ldg(qrow + c) : 0.0;
      }
      double acc[NB][2];
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[b][0] = acc[b][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < RP; k4 += 4)
#pragma unroll
        for (int b = 0; b < NB; ++b)  // (asm loads: kept in the loop, not hoisted into 100 registers)
          dev::dmma884(acc[b], x[k4 / 4], dev::lds64<0>(hb + 8u * static_cast<unsigned>(k4 * LDH + 8 * b)));
      if (i < I) {
        double* urow = U + (r0 + i) * R;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int c = 8 * b + 2 * fk;
          const double u0 = acc[b][0] * sc[b][0], u1 = acc[b][1] * sc[b][1];
          if (even) {
            if (c < R) *reinterpret_cast<double2*>(urow + c) = make_double2(u0, u1);
          } else {
            if (c < R) urow[c] = u0;
            if (c + 1 < R) urow[c + 1] = u1;
          }
        }
      }
    }
  }
}

}  // namespace

void build_csc(p2g_ctx* c) {
  sync_csc(c);
  const std::int64_t n = c->nnz, J = c->J;
  if (n > static_cast<std::int64_t>(0x7fffffff) || c->NR > static_cast<std::int64_t>(0x7fffffff))
    throw InvalidArgument("shard too large for 32-bit CSC indices");
  if (!c->side) {
    P2G_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    P2G_CUDA(cudaEventCreateWithFlags(&c->ev_upload, cudaEventDisableTiming));
    P2G_CUDA(cudaEventCreateWithFlags(&c->ev_csc, cudaEventDisableTiming));
  }
  // phase A on the side stream, behind everything the load queued so far
  P2G_CUDA(cudaEventRecord(c->ev_upload, c->stream));
  P2G_CUDA(cudaStreamWaitEvent(c->side, c->ev_upload, 0));
  cudaStream_t s = c->side;
  const std::int64_t nblk = (c->NR >> kRowBlockBits) + 1;
  c->csc_row.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  c->csc_val.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  c->seg_ptr.resize(static_cast<std::size_t>(J + 1));
  c->nseg = 0;
  if (n == 0) {
    P2G_CUDA(cudaMemsetAsync(c->seg_ptr.get(), 0, sizeof(std::int64_t) * (J + 1), c->stream));
    P2G_CUDA(cudaStreamSynchronize(c->stream));
    return;
  }
  c->csc_rowof.resize(static_cast<std::size_t>(n));
  c->csc_iota.resize(static_cast<std::size_t>(n));
  c->csc_perm.resize(static_cast<std::size_t>(n));
  c->csc_keys.resize(static_cast<std::size_t>(n));
  c->csc_skeys.resize(static_cast<std::size_t>(n));
  std::int32_t* row_of = c->csc_rowof.get();
  std::int32_t* iota = c->csc_iota.get();
  std::int32_t* perm = c->csc_perm.get();
  std::uint64_t* keys = c->csc_keys.get();
  std::uint64_t* skeys = c->csc_skeys.get();
  k_row_expand<<<grid_for(c->NR, 256), 256, 0, s>>>(c->NR, c->rp.get(), row_of);
  k_iota<<<grid_for(n, 256), 256, 0, s>>>(n, iota);
  k_block_keys<<<grid_for(n, 256), 256, 0, s>>>(n, J, row_of, c->ci.get(), keys);
  int bits = 1;
  while ((std::uint64_t{1} << bits) < static_cast<std::uint64_t>(nblk * J)) ++bits;
  std::size_t tbytes = 0, tb2 = 0, tb3 = 0;
  P2G_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tbytes, keys, skeys, iota, perm, static_cast<int>(n), 0, bits, s));
  c->csc_mark.resize(static_cast<std::size_t>(n));
  c->csc_runstart.resize(static_cast<std::size_t>(n));
  P2G_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb2, c->csc_mark.get(), c->csc_runstart.get(), cub::Max(),
                                          static_cast<int>(n), s));
  c->csc_head.resize(static_cast<std::size_t>(n));
  c->seg_beg.resize(static_cast<std::size_t>(n));
  c->csc_nsel.resize(1);
  thrust::counting_iterator<std::int64_t> idx(0);
  P2G_CUDA(cub::DeviceSelect::Flagged(nullptr, tb3, idx, c->csc_head.get(), c->seg_beg.get(), c->csc_nsel.get(),
                                      static_cast<int>(n), s));
  // one temp allocation for the three passes (no frees, which would sync the device)
  c->csc_temp.resize(std::max({tbytes, tb2, tb3}));
  tbytes = c->csc_temp.n;
  // LSD radix sort: stable, so a (row block, column) run keeps CSR (row-ascending) order
  P2G_CUDA(cub::DeviceRadixSort::SortPairs(c->csc_temp.get(), tbytes, keys, skeys, iota, perm, static_cast<int>(n), 0,
                                           bits, s));
  k_csc_gather<<<grid_for(n, 256), 256, 0, s>>>(n, perm, row_of, c->val.get(), c->csc_row.get(), c->csc_val.get());
  // segment heads: run starts (max-scan of change positions), split every kSeg
  k_run_marks<<<grid_for(n, 256), 256, 0, s>>>(n, skeys, c->csc_mark.get());
  tb2 = c->csc_temp.n;
  P2G_CUDA(cub::DeviceScan::InclusiveScan(c->csc_temp.get(), tb2, c->csc_mark.get(), c->csc_runstart.get(),
                                          cub::Max(), static_cast<int>(n), s));
  k_seg_heads<<<grid_for(n, 256), 256, 0, s>>>(n, c->csc_runstart.get(), c->csc_head.get());
  tb3 = c->csc_temp.n;
  P2G_CUDA(cub::DeviceSelect::Flagged(c->csc_temp.get(), tb3, idx, c->csc_head.get(), c->seg_beg.get(),
                                      c->csc_nsel.get(), static_cast<int>(n), s));
  P2G_CUDA(cudaMemcpyAsync(c->pinned + 60, c->csc_nsel.get(), sizeof(std::int64_t), cudaMemcpyDeviceToHost, s));
  c->csc_pending = true;
}

/// Phase B of the CSC build (per-column segment lists in row-block order:
/// segment ids sorted by col * nblk + block), then the main stream waits for it.
void ensure_csc(p2g_ctx* c) {
  if (!c->csc_pending) return;
  cudaStream_t s = c->side;
  P2G_CUDA(cudaStreamSynchronize(s));  // phase A done: the segment count is on the host
  std::int64_t nseg = 0;
  std::memcpy(&nseg, c->pinned + 60, sizeof(nseg));
  c->nseg = nseg;
  const std::int64_t J = c->J;
  const std::int64_t nblk = (c->NR >> kRowBlockBits) + 1;
  c->csc_ck.resize(static_cast<std::size_t>(nseg));
  c->csc_sck.resize(static_cast<std::size_t>(nseg));
  c->csc_ids.resize(static_cast<std::size_t>(nseg));
  c->seg_ids.resize(static_cast<std::size_t>(nseg));
  k_seg_colkeys<<<grid_for(nseg, 256), 256, 0, s>>>(nseg, J, nblk, c->seg_beg.get(), c->csc_skeys.get(),
                                                    c->csc_ck.get(), c->csc_ids.get());
  int cbits = 1;
  while ((std::uint64_t{1} << cbits) < static_cast<std::uint64_t>(nblk * J)) ++cbits;
  std::size_t tbytes = 0;
  P2G_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tbytes, c->csc_ck.get(), c->csc_sck.get(), c->csc_ids.get(),
                                           c->seg_ids.get(), static_cast<int>(nseg), 0, cbits, s));
  c->csc_temp.resize(tbytes);
  tbytes = c->csc_temp.n;
  P2G_CUDA(cub::DeviceRadixSort::SortPairs(c->csc_temp.get(), tbytes, c->csc_ck.get(), c->csc_sck.get(),
                                           c->csc_ids.get(), c->seg_ids.get(), static_cast<int>(nseg), 0, cbits, s));
  k_key_ptr<<<grid_for(J + 1, 256), 256, 0, s>>>(J, nseg, nblk, c->csc_sck.get(), c->seg_ptr.get());
  P2G_CUDA(cudaEventRecord(c->ev_csc, s));
  P2G_CUDA(cudaStreamWaitEvent(c->stream, c->ev_csc, 0));
  c->csc_pending = false;
}

/// Completes any pending build and waits for the side stream (before the
/// shard buffers it reads are replaced, and at teardown).
void sync_csc(p2g_ctx* c) {
  ensure_csc(c);
  if (c->side) P2G_CUDA(cudaStreamSynchronize(c->side));
}

template <int RP>
static void seg_spmm(p2g_ctx* c, int R, const double* U, cudaStream_t s) {
  if constexpr (RP > 16) {
    if (R == RP) {  // exact R: constant strides, 32-byte row loads (R = 24, 32, 40)
      c->seg_next.resize(1);
      P2G_CUDA(cudaMemsetAsync(c->seg_next.get(), 0, sizeof(unsigned long long), s));
      int per_sm = 0;
      P2G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_seg_spmm_w<RP>, 256, 0));
      const int blocks = static_cast<int>(std::max<std::int64_t>(
          1, std::min<std::int64_t>((c->nseg + 7) / 8, static_cast<std::int64_t>(c->num_sms) * std::max(per_sm, 1))));
      k_seg_spmm_w<RP><<<blocks, 256, 0, s>>>(c->nseg, c->nnz, c->seg_beg.get(), c->csc_row.get(), c->csc_val.get(),
                                               U, c->seg_part.get(), c->seg_next.get());
      return;
    }
  }
  k_seg_spmm<RP><<<grid_for(c->nseg, 128), 128, 0, s>>>(R, c->nseg, c->nnz, c->seg_beg.get(), c->csc_row.get(),
                                                        c->csc_val.get(), U, c->seg_part.get());
}

void launch_csc_mode2(p2g_ctx* c, int R, const double* U, double* M2, cudaStream_t s) {
  ensure_csc(c);
  c->seg_part.resize(static_cast<std::size_t>(std::max<std::int64_t>(c->nseg, 1)) * R);
  if (c->nseg > 0) {
    if (R <= 2)
      seg_spmm<2>(c, R, U, s);
    else if (R <= 4)
      seg_spmm<4>(c, R, U, s);
    else if (R <= 6)
      seg_spmm<6>(c, R, U, s);
    else if (R <= 8)
      seg_spmm<8>(c, R, U, s);
    else if (R <= 10)
      seg_spmm<10>(c, R, U, s);
    else if (R <= 12)
      seg_spmm<12>(c, R, U, s);
    else if (R <= 16)
      seg_spmm<16>(c, R, U, s);
    else if (R <= 24)
      seg_spmm<24>(c, R, U, s);
    else if (R <= 32)
      seg_spmm<32>(c, R, U, s);
    else if (R <= 40)
      seg_spmm<40>(c, R, U, s);
    else
      throw InvalidArgument("rank above 40 unsupported");
    P2G_LAUNCHED(1);
  }
  k_seg_reduce<<<grid_for(c->J * R, 256), 256, 0, s>>>(R, c->J, c->seg_ptr.get(), c->seg_ids.get(), c->seg_part.get(), M2);
  P2G_LAUNCHED(1);
}

template <int RP>
static void urows(p2g_ctx* c, int R, const double* Q, const double* H, const double* W, const double* nH, double* U,
                  cudaStream_t s) {
  constexpr int WPB = 8;
  auto kern = k_urows<RP, WPB>;
  const ShardArgs X{c->srp.get(), c->rp.get(), c->ci.get(), c->val.get(), c->k_end - c->k_begin, c->NR, c->nnz, c->J};
  const int blocks =
      static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((X.K + WPB - 1) / WPB, c->num_sms * 8)));
  kern<<<blocks, WPB * 32, 0, s>>>(X, R, Q, H, W, nH, U);
}

void launch_urows_large(p2g_ctx* c, int R, const double* Q, const double* H, const double* W, const double* nH,
                        double* U, cudaStream_t s) {
  if (c->k_end <= c->k_begin) return;
  if (R <= 24)
    urows<24>(c, R, Q, H, W, nH, U, s);
  else if (R <= 32)
    urows<32>(c, R, Q, H, W, nH, U, s);
  else if (R <= 40)
    urows<40>(c, R, Q, H, W, nH, U, s);
  else
    throw InvalidArgument("rank above 40 unsupported");
  P2G_LAUNCHED(1);
}

}  // namespace p2g
