// Atomics-free mode-2 MTTKRP: M2 = X^T U over a column-major copy of the shard.
//
// mttkrp_mode2 (mttkrp.hpp:111-138) is M2 = sum_k X_k^T U_k with row factors
// U_k = Q_k H diag(W_k o nH).  Scattering v * u_i into M2 with L2 fp64
// reductions costs one L2 request per (entry, column) pair: 630M requests per
// iteration at cfg2, where ncu shows L1/L2 at 77%/64% of their request
// throughput (profiles/).  Instead, each row's u_i is written once (the
// streaming kernels produce it coalesced), and M2 is read out column by
// column from a CSC copy of the shard built at load time:
//   M2[j, :] = sum_{(i, v) in column j} v * U[i, :]
// Columns are cut into segments of at most kSeg entries (hot Zipf columns of
// cfg5 stay balanced); one CTA sums a segment, and a second pass adds a
// column's segment partials in order: deterministic, no atomics.
#include <algorithm>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"

namespace p2g {
namespace {

constexpr std::int64_t kSeg = 4096;
constexpr int kSpThreads = 128;

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

/// col_ptr[j] = first position of key >= j in the sorted keys (binary search).
__global__ void k_col_ptr(std::int64_t J, std::int64_t n, const std::int32_t* __restrict__ keys,
                          std::int64_t* __restrict__ col_ptr) {
  for (std::int64_t j = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j <= J;
       j += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    std::int64_t lo = 0, hi = n;
    while (lo < hi) {
      const std::int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < j)
        lo = mid + 1;
      else
        hi = mid;
    }
    col_ptr[j] = lo;
  }
}

int grid_for(std::int64_t n, int threads) {
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + threads - 1) / threads, 148 * 32)));
}

/// One CTA per segment: partial[s, :] = sum over the segment's entries of v * U[row, :].
template <int RP>
__global__ void __launch_bounds__(kSpThreads) k_seg_spmm(int R, std::int64_t nseg, const std::int64_t* __restrict__ seg_beg,
                                                         const std::int64_t* __restrict__ seg_end,
                                                         const std::int32_t* __restrict__ crow,
                                                         const double* __restrict__ cval, const double* __restrict__ U,
                                                         double* __restrict__ partial) {
  extern __shared__ double red[];  // kSpThreads x (RP + 1)
  const int tid = threadIdx.x;
  for (std::int64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    double acc[RP];
#pragma unroll
    for (int c = 0; c < RP; ++c) acc[c] = 0.0;
    const std::int64_t q1 = seg_end[s];
    for (std::int64_t q = seg_beg[s] + tid; q < q1; q += kSpThreads) {
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
#pragma unroll
    for (int c = 0; c < RP; ++c) red[tid * (RP + 1) + c] = acc[c];
    __syncthreads();
    for (int c = tid; c < R; c += kSpThreads) {
      double t = 0.0;
      for (int i = 0; i < kSpThreads; ++i) t += red[i * (RP + 1) + c];
      partial[s * R + c] = t;
    }
    __syncthreads();
  }
}

/// M2[j, c] = sum of column j's segment partials, in segment order.
__global__ void k_seg_reduce(int R, std::int64_t J, const std::int64_t* __restrict__ seg_ptr,
                             const double* __restrict__ partial, double* __restrict__ M2) {
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < J * R;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t j = e / R;
    const int c = static_cast<int>(e - j * R);
    double t = 0.0;
    for (std::int64_t s = seg_ptr[j]; s < seg_ptr[j + 1]; ++s) t += partial[s * R + c];
    M2[e] = t;
  }
}

/// U rows of the large-R path: u_i = q_i H diag(w_k o nH), warp per subject.
template <int RP, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_urows(ShardArgs X, int R, const double* __restrict__ Q, const double* __restrict__ H,
            const double* __restrict__ W, const double* __restrict__ nH, double* __restrict__ U) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* HW = sm + wid * RP * (RP + 1);  // R x R, ld RP + 1
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * WPB;
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * WPB + wid; k < X.K; k += nwarps) {
    for (int a = 0; a < R; ++a)
      for (int c = lane; c < R; c += 32) HW[a * (RP + 1) + c] = H[a * R + c] * W[k * R + c] * nH[c];
    __syncwarp();
    const std::int64_t r0 = X.srp[k], r1 = X.srp[k + 1];
    for (std::int64_t i = r0 + lane; i < r1; i += 32) {
      double q[RP];
#pragma unroll
      for (int a = 0; a < RP; ++a) q[a] = a < R ? Q[i * R + a] : 0.0;
      for (int c = 0; c < R; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < RP; ++a)
          if (a < R) acc = fma(q[a], HW[a * (RP + 1) + c], acc);
        U[i * R + c] = acc;
      }
    }
    __syncwarp();
  }
}

}  // namespace

void build_csc(p2g_ctx* c) {
  cudaStream_t s = c->stream;
  const std::int64_t n = c->nnz, J = c->J;
  c->col_ptr.resize(static_cast<std::size_t>(J + 1));
  c->csc_row.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  c->csc_val.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  if (n > static_cast<std::int64_t>(0x7fffffff) || c->NR > static_cast<std::int64_t>(0x7fffffff))
    throw InvalidArgument("shard too large for 32-bit CSC indices");
  std::vector<std::int64_t> cp(static_cast<std::size_t>(J + 1), 0);
  if (n > 0) {
    DBuf<std::int32_t> row_of, keys, iota, perm;
    row_of.resize(static_cast<std::size_t>(n));
    keys.resize(static_cast<std::size_t>(n));
    iota.resize(static_cast<std::size_t>(n));
    perm.resize(static_cast<std::size_t>(n));
    k_row_expand<<<grid_for(c->NR, 256), 256, 0, s>>>(c->NR, c->rp.get(), row_of.get());
    k_iota<<<grid_for(n, 256), 256, 0, s>>>(n, iota.get());
    int bits = 1;
    while ((std::int64_t{1} << bits) < J) ++bits;
    std::size_t tbytes = 0;
    P2G_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tbytes, c->ci.get(), keys.get(), iota.get(), perm.get(),
                                             static_cast<int>(n), 0, bits, s));
    DBuf<unsigned char> temp;
    temp.resize(tbytes);
    // LSD radix sort: stable, so entries of a column keep CSR (row-ascending) order
    P2G_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tbytes, c->ci.get(), keys.get(), iota.get(), perm.get(),
                                             static_cast<int>(n), 0, bits, s));
    k_csc_gather<<<grid_for(n, 256), 256, 0, s>>>(n, perm.get(), row_of.get(), c->val.get(), c->csc_row.get(),
                                                  c->csc_val.get());
    k_col_ptr<<<grid_for(J + 1, 256), 256, 0, s>>>(J, n, keys.get(), c->col_ptr.get());
    P2G_CUDA(cudaMemcpyAsync(cp.data(), c->col_ptr.get(), sizeof(std::int64_t) * (J + 1), cudaMemcpyDeviceToHost, s));
    P2G_CUDA(cudaStreamSynchronize(s));
  }
  // segment table (host; J entries)
  std::vector<std::int64_t> sp(static_cast<std::size_t>(J + 1), 0), sb, se;
  for (std::int64_t j = 0; j < J; ++j) {
    const std::int64_t a = cp[static_cast<std::size_t>(j)], b = cp[static_cast<std::size_t>(j + 1)];
    for (std::int64_t q = a; q < b; q += kSeg) {
      sb.push_back(q);
      se.push_back(std::min(b, q + kSeg));
    }
    sp[static_cast<std::size_t>(j + 1)] = static_cast<std::int64_t>(sb.size());
  }
  c->nseg = static_cast<std::int64_t>(sb.size());
  c->seg_ptr.resize(sp.size());
  c->seg_beg.resize(std::max<std::size_t>(sb.size(), 1));
  c->seg_end.resize(std::max<std::size_t>(se.size(), 1));
  P2G_CUDA(cudaMemcpyAsync(c->seg_ptr.get(), sp.data(), sizeof(std::int64_t) * sp.size(), cudaMemcpyHostToDevice, s));
  if (!sb.empty()) {
    P2G_CUDA(cudaMemcpyAsync(c->seg_beg.get(), sb.data(), sizeof(std::int64_t) * sb.size(), cudaMemcpyHostToDevice, s));
    P2G_CUDA(cudaMemcpyAsync(c->seg_end.get(), se.data(), sizeof(std::int64_t) * se.size(), cudaMemcpyHostToDevice, s));
  }
  P2G_CUDA(cudaStreamSynchronize(s));
}

template <int RP>
static void seg_spmm(p2g_ctx* c, int R, const double* U, cudaStream_t s) {
  const std::size_t smem = sizeof(double) * kSpThreads * (RP + 1);
  auto kern = k_seg_spmm<RP>;
  P2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int blocks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(c->nseg, 148 * 16)));
  kern<<<blocks, kSpThreads, smem, s>>>(R, c->nseg, c->seg_beg.get(), c->seg_end.get(), c->csc_row.get(),
                                        c->csc_val.get(), U, c->seg_part.get());
}

void launch_csc_mode2(p2g_ctx* c, int R, const double* U, double* M2, cudaStream_t s) {
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
  k_seg_reduce<<<grid_for(c->J * R, 256), 256, 0, s>>>(R, c->J, c->seg_ptr.get(), c->seg_part.get(), M2);
  P2G_LAUNCHED(1);
}

template <int RP>
static void urows(p2g_ctx* c, int R, const double* Q, const double* H, const double* W, const double* nH, double* U,
                  cudaStream_t s) {
  constexpr int WPB = 4;
  const std::size_t smem = sizeof(double) * WPB * RP * (RP + 1);
  auto kern = k_urows<RP, WPB>;
  P2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const ShardArgs X{c->srp.get(), c->rp.get(), c->ci.get(), c->val.get(), c->k_end - c->k_begin, c->NR, c->nnz, c->J};
  const int blocks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((X.K + WPB - 1) / WPB, 148 * 8)));
  kern<<<blocks, WPB * 32, smem, s>>>(X, R, Q, H, W, nH, U);
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
