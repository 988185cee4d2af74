// Eye initialisation: V = |leading R eigenvectors|
// of the column Gram matrix C = sum_k X_k^T X_k (solver.hpp:133-164).
//
// C is J x J and is built from non-zero column pairs only, as the reference
// does: C(a, b) = sum over rows r holding both a and b of x_ra x_rb (rows of
// different subjects never meet, so the sum over slices is the sum over the
// stacked rows).  Device layout: a column-major copy of the CSR by a stable
// radix sort of the column ids (rows stay ascending inside a column), then
// one warp per column b walks b's rows and scatters x_rb * x_r. into its own
// accumulator (shared memory when J fits, else its own row of C in global
// memory).  The lanes of a warp hold distinct columns of one row, and each
// warp owns its column, so there are no atomics and the order is fixed:
// C(a, b) and C(b, a) are the same products in the same row order (C is
// exactly symmetric).  With several ranks the shard Grams are allreduced.
// The eigenvectors come from cuSOLVER syevdx (only the top R), a plain
// library eigensolver as SURVEY.md 8(f) plans.
#include <algorithm>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"
#include "p2g_libs.hpp"

namespace p2g {
namespace {

__global__ void k_init_rows(std::int64_t NR, const std::int64_t* __restrict__ rp, std::int32_t* __restrict__ row_of) {
  for (std::int64_t r = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < NR;
       r += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    for (std::int64_t p = rp[r]; p < rp[r + 1]; ++p) row_of[p] = static_cast<std::int32_t>(r);
}

__global__ void k_init_iota(std::int64_t n, std::int64_t* __restrict__ out) {
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    out[i] = i;
}

/// ptr[j] = first sorted position with column >= j.
__global__ void k_init_colptr(std::int64_t J, std::int64_t n, const std::int32_t* __restrict__ cols,
                              std::int64_t* __restrict__ ptr) {
  for (std::int64_t j = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j <= J;
       j += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    std::int64_t lo = 0, hi = n;
    while (lo < hi) {
      const std::int64_t mid = (lo + hi) >> 1;
      if (cols[mid] < j)
        lo = mid + 1;
      else
        hi = mid;
    }
    ptr[j] = lo;
  }
}

/// One warp per column b: C[b, :] = sum over b's rows r (ascending) of
/// x_rb * X[r, :].  SMEM: the accumulator lives in shared memory (J doubles
/// per warp), else directly in C's row b (owned by this warp).
template <bool SMEM>
__global__ void __launch_bounds__(128) k_col_gram(std::int64_t J, const std::int64_t* __restrict__ colptr,
                                                  const std::int64_t* __restrict__ perm,
                                                  const std::int32_t* __restrict__ row_of,
                                                  const std::int64_t* __restrict__ rp,
                                                  const std::int32_t* __restrict__ ci,
                                                  const double* __restrict__ val, double* __restrict__ C) {
  extern __shared__ double acc_s[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  for (std::int64_t b = static_cast<std::int64_t>(blockIdx.x) * wpb + wid; b < J;
       b += static_cast<std::int64_t>(gridDim.x) * wpb) {
    double* acc = SMEM ? acc_s + static_cast<std::int64_t>(wid) * J : C + b * J;
    for (std::int64_t a = lane; a < J; a += 32) acc[a] = 0.0;
    __syncwarp();
    for (std::int64_t q = colptr[b]; q < colptr[b + 1]; ++q) {
      const std::int64_t p_b = perm[q];
      const double x = val[p_b];
      const std::int32_t r = row_of[p_b];
      const std::int64_t p0 = rp[r], p1 = rp[r + 1];
      for (std::int64_t p = p0 + lane; p < p1; p += 32) acc[ci[p]] = fma(x, val[p], acc[ci[p]]);
      __syncwarp();
    }
    if (SMEM) {
      for (std::int64_t a = lane; a < J; a += 32) C[b * J + a] = acc[a];
      __syncwarp();
    }
  }
}

__global__ void k_eye_v(std::int64_t J, int R, int m, const double* __restrict__ Z, double* __restrict__ V) {
  // V row-major J x R: V[j, r] = |Z(j, m - 1 - r)| (syevdx: ascending, column-major)
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < J * R;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t j = e / R;
    const int r = static_cast<int>(e - j * R);
    V[e] = fabs(Z[static_cast<std::int64_t>(m - 1 - r) * J + j]);
  }
}

int grid(std::int64_t n, int t) {
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + t - 1) / t, 148 * 32)));
}

}  // namespace

void build_column_gram(p2g_ctx* c, double* C) {
  const std::int64_t J = c->J, n = c->nnz, NR = c->NR;
  cudaStream_t s = c->stream;
  DBuf<std::int32_t> row_of, cols_sorted;
  DBuf<std::int64_t> idx, perm, colptr;
  row_of.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  cols_sorted.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  idx.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  perm.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  colptr.resize(static_cast<std::size_t>(J + 1));
  k_init_rows<<<grid(NR, 256), 256, 0, s>>>(NR, c->rp.get(), row_of.get());
  k_init_iota<<<grid(n, 256), 256, 0, s>>>(n, idx.get());
  P2G_LAUNCHED(2);
  // stable sort of the entry indices by column: rows stay ascending per column
  int bits = 1;
  while ((1ll << bits) < J) ++bits;
  std::size_t tmp = 0;
  P2G_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, c->ci.get(), cols_sorted.get(), idx.get(), perm.get(), n, 0,
                                           bits, s));
  DBuf<unsigned char> tbuf;
  tbuf.resize(std::max<std::size_t>(tmp, 1));
  P2G_CUDA(cub::DeviceRadixSort::SortPairs(tbuf.get(), tmp, c->ci.get(), cols_sorted.get(), idx.get(), perm.get(), n,
                                           0, bits, s));
  k_init_colptr<<<grid(J + 1, 256), 256, 0, s>>>(J, n, cols_sorted.get(), colptr.get());
  P2G_LAUNCHED(3);  // (incl. the radix sort's passes, counted once)
  constexpr int kWpb = 4;
  const std::size_t smem = sizeof(double) * kWpb * static_cast<std::size_t>(J);
  const int blocks = grid(J, kWpb);
  if (smem <= 200 * 1024) {
    P2G_CUDA(cudaFuncSetAttribute(k_col_gram<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_col_gram<true><<<blocks, 32 * kWpb, smem, s>>>(J, colptr.get(), perm.get(), row_of.get(), c->rp.get(),
                                                      c->ci.get(), c->val.get(), C);
  } else {
    k_col_gram<false><<<blocks, 32 * kWpb, 0, s>>>(J, colptr.get(), perm.get(), row_of.get(), c->rp.get(),
                                                    c->ci.get(), c->val.get(), C);
  }
  P2G_LAUNCHED(1);
  P2G_CUDA(cudaStreamSynchronize(s));
}

/// V (row-major J x R) = |top-R eigenvectors of C| (C J x J, overwritten).
void eye_vectors(p2g_ctx* c, double* C, int R, double* V) {
  const std::int64_t J = c->J;
  if (J > 2147483647ll / std::max<std::int64_t>(J, 1)) throw InvalidArgument("eye init: J too large for a dense J x J eigenproblem");
  SolverLib& L = solver_lib();
  cusolverDnHandle_t h = nullptr;
  if (L.Create(&h) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnCreate failed");
  struct Guard {
    SolverLib& L;
    cusolverDnHandle_t h;
    ~Guard() { L.Destroy(h); }
  } g{L, h};
  L.SetStream(h, c->stream);
  const int n = static_cast<int>(J);
  DBuf<double> w;
  w.resize(static_cast<std::size_t>(n));
  int m = 0, lwork = 0;
  if (L.DsyevdxBuf(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, C, n, 0.0, 0.0,
                   n - R + 1, n, &m, w.get(), &lwork) != CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDnDsyevdx_bufferSize failed");
  DBuf<double> work;
  work.resize(static_cast<std::size_t>(std::max(lwork, 1)));
  DBuf<int> info;
  info.resize(1);
  if (L.Dsyevdx(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, C, n, 0.0, 0.0,
                n - R + 1, n, &m, w.get(), work.get(), lwork, info.get()) != CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDnDsyevdx failed");
  int hinfo = 0;
  P2G_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  P2G_CUDA(cudaStreamSynchronize(c->stream));
  if (hinfo != 0) throw NumericalError("eye init: eigensolver did not converge (info " + std::to_string(hinfo) + ")");
  if (m < R) throw NumericalError("eye init: eigensolver returned fewer than R vectors");
  k_eye_v<<<grid(J * R, 256), 256, 0, c->stream>>>(J, R, m, C, V);
  P2G_LAUNCHED(1);
}

}  // namespace p2g
