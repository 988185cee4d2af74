// Naive MTTKRP on the device: the baseline the
// paper's slice-wise reformulation beats (mttkrp.hpp:198-235).  It
// materialises the dense mode-n unfolding of the R x J x K tensor {Y_k} and
// the full Khatri-Rao product, then multiplies them -- a plain GEMM, so the
// multiply is cuBLAS DGEMM.  Layouts (column-major, as the reference):
//   mode 1: A (R x J K),  column j + J k  = Y_k(:, j);  KRP = khatri_rao(W, V) (K J x R)
//   mode 2: A (J x R K),  column i + R k  = Y_k(i, :)^T; KRP = khatri_rao(W, H) (K R x R)
//   mode 3: A (K x R J),  column i + R j  = Y_k(i, j);  KRP = khatri_rao(V, H) (J R x R)
// khatri_rao(A, B) row a * rows(B) + b = B(b, :) o A(a, :) (kernels.hpp:34-44).
// Factors arrive row-major (the library's device layout).
#include <algorithm>

#include "dev_common.cuh"
#include "p2g_ctx.hpp"
#include "p2g_libs.hpp"

namespace p2g {
namespace {

int grid(std::int64_t n, int t) {
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + t - 1) / t, 148 * 32)));
}

/// Scatter the packed columns of every Y_k into the zeroed unfolding.
__global__ void k_unfold(int mode, std::int64_t K, std::int64_t J, int R, const std::int64_t* __restrict__ ptr,
                         const std::int32_t* __restrict__ cols, const std::int64_t* __restrict__ subj_of,
                         const double* __restrict__ Y, double* __restrict__ A, std::int64_t nc) {
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nc * R;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t t = e / R;
    const int i = static_cast<int>(e - t * R);
    const std::int64_t k = subj_of[t], j = cols[t];
    const double y = Y[e];
    std::int64_t idx;
    if (mode == 1)
      idx = (j + J * k) * R + i;                    // (i, j + J k), ld R
    else if (mode == 2)
      idx = (static_cast<std::int64_t>(i) + R * k) * J + j;  // (j, i + R k), ld J
    else
      idx = (static_cast<std::int64_t>(i) + static_cast<std::int64_t>(R) * j) * K + k;  // (k, i + R j), ld K
    A[idx] = y;
  }
}

/// KRP (na * nb x R, column-major) = khatri_rao(A (na x R), B (nb x R)), both row-major.
__global__ void k_khatri_rao(std::int64_t na, std::int64_t nb, int R, const double* __restrict__ A,
                             const double* __restrict__ B, double* __restrict__ out) {
  const std::int64_t rows = na * nb;
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * R;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t c = e / rows, row = e - c * rows;
    const std::int64_t a = row / nb, b = row - a * nb;
    out[e] = B[b * R + c] * A[a * R + c];
  }
}

__global__ void k_subj_of(std::int64_t K, const std::int64_t* __restrict__ ptr, std::int64_t* __restrict__ subj_of) {
  for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < K;
       k += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    for (std::int64_t t = ptr[k]; t < ptr[k + 1]; ++t) subj_of[t] = k;
}

struct BlasHandle {
  cublasHandle_t h = nullptr;
  ~BlasHandle() {
    if (h) blas_lib().Destroy(h);
  }
};

}  // namespace

std::uint64_t naive_bytes(std::int64_t K, std::int64_t J, std::int64_t R, int mode) {
  const auto k = static_cast<std::uint64_t>(K), j = static_cast<std::uint64_t>(J), r = static_cast<std::uint64_t>(R);
  std::uint64_t unfolded = 0, krp = 0, result = 0;
  switch (mode) {  // mttkrp.hpp:241-253
    case 1: unfolded = r * j * k; krp = k * j * r; result = r * r; break;
    case 2: unfolded = j * r * k; krp = k * r * r; result = j * r; break;
    case 3: unfolded = k * r * j; krp = j * r * r; result = k * r; break;
    default: throw InvalidArgument("mttkrp: mode must be 1, 2 or 3");
  }
  return 8 * (unfolded + krp + result);
}

void NaiveScratch::prepare(p2g_ctx* c, int mode, std::int64_t K, std::int64_t J, int R, const std::int64_t* ptr,
                           std::int64_t nc) {
  const std::int64_t R64 = R;
  const std::int64_t ncols = mode == 1 ? J * K : (mode == 2 ? R64 * K : R64 * J);
  const std::int64_t lda = mode == 1 ? R64 : (mode == 2 ? J : K);
  const std::int64_t kr = mode == 1 ? K * J : (mode == 2 ? K * R64 : J * R64);
  if (ncols > 2147483647ll || lda > 2147483647ll || kr > 2147483647ll)
    throw InvalidArgument("naive mttkrp: unfolding exceeds the 32-bit GEMM dimensions");
  A.resize(static_cast<std::size_t>(std::max<std::int64_t>(lda * ncols, 1)));
  KRP.resize(static_cast<std::size_t>(std::max<std::int64_t>(kr * R64, 1)));
  subj_of.resize(static_cast<std::size_t>(std::max<std::int64_t>(nc, 1)));
  k_subj_of<<<grid(K, 256), 256, 0, c->stream>>>(K, ptr, subj_of.get());
  P2G_LAUNCHED(1);
}

/// out (column-major rows x R) = naive MTTKRP of packed Y on the device.
void naive_mttkrp(p2g_ctx* c, NaiveScratch& s, int mode, std::int64_t K, std::int64_t J, int R,
                  const std::int64_t* ptr, const std::int32_t* cols, const double* Y, std::int64_t nc, const double* H,
                  const double* V, const double* W, double* out) {
  const std::int64_t R64 = R;
  const std::int64_t ncols = mode == 1 ? J * K : (mode == 2 ? R64 * K : R64 * J);
  const std::int64_t lda = mode == 1 ? R64 : (mode == 2 ? J : K);
  const std::int64_t kr = mode == 1 ? K * J : (mode == 2 ? K * R64 : J * R64);
  cudaStream_t st = c->stream;
  // materialise: the dense unfolding (zeros, then the stored columns) and the Khatri-Rao product
  P2G_CUDA(cudaMemsetAsync(s.A.get(), 0, sizeof(double) * static_cast<std::size_t>(lda * ncols), st));
  k_unfold<<<grid(nc * R64, 256), 256, 0, st>>>(mode, K, J, R, ptr, cols, s.subj_of.get(), Y, s.A.get(), nc);
  if (mode == 1)
    k_khatri_rao<<<grid(kr * R64, 256), 256, 0, st>>>(K, J, R, W, V, s.KRP.get());
  else if (mode == 2)
    k_khatri_rao<<<grid(kr * R64, 256), 256, 0, st>>>(K, R64, R, W, H, s.KRP.get());
  else
    k_khatri_rao<<<grid(kr * R64, 256), 256, 0, st>>>(J, R64, R, V, H, s.KRP.get());
  P2G_LAUNCHED(2);
  if (!s.blas) {
    BlasLib& L = blas_lib();
    if (L.Create(&s.blas) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasCreate failed");
    L.SetMathMode(s.blas, CUBLAS_DEFAULT_MATH);  // true fp64 (no emulation)
  }
  BlasLib& L = blas_lib();
  L.SetStream(s.blas, st);
  const double one = 1.0, zero = 0.0;
  const int m = static_cast<int>(lda), n = R, k = static_cast<int>(ncols);
  if (L.Dgemm(s.blas, CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &one, s.A.get(), m, s.KRP.get(), k, &zero, out, m) !=
      CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDgemm failed");
}

NaiveScratch::~NaiveScratch() {
  if (blas) blas_lib().Destroy(blas);
}

}  // namespace p2g
