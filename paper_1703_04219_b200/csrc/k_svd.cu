// economy_svd (kernels.hpp:92-107) on the device: thin SVD M = P diag(sigma) Z^T,
// rho = min(m, n), singular values non-increasing.
//
// Not on the fused loop (the Procrustes kernels take their polar factors from
// eigen-solves); this is the boundary function of the drop-in
// headers.  One warp runs the one-sided (Hestenes) Jacobi the oracle restates
// for Eigen's JacobiSVD: W (mm x nn, mm >= nn: M or M^T) is rotated in place
// column pair by column pair until every pair is orthogonal to 1e-15, V
// accumulates the rotations, sigma_j = |w_j|, columns sorted by sigma.  Columns
// with sigma = 0 (relative to sigma_max) get an orthonormal completion from
// unit vectors (two Gram-Schmidt passes), as in the oracle.
#include "dev_common.cuh"
#include "p2g_ctx.hpp"

namespace p2g {
namespace {

constexpr int kSvdMaxCols = 128;

/// W: mm x nn row-major (scaled by 1 / max |entry| by the caller), V: nn x nn row-major.
/// Out: Uo (mm x nn row-major, sorted, normalised), Vo (nn x nn row-major, sorted), sig (nn).
__global__ void __launch_bounds__(32) k_economy_svd(int mm, int nn, double* __restrict__ W, double* __restrict__ V,
                                                    double* __restrict__ Uo, double* __restrict__ Vo,
                                                    double* __restrict__ sig, int* __restrict__ status) {
  __shared__ double s_sig[kSvdMaxCols];
  __shared__ int s_ord[kSvdMaxCols];
  const int lane = threadIdx.x;
  for (int e = lane; e < nn * nn; e += 32) V[e] = (e / nn == e % nn) ? 1.0 : 0.0;
  __syncwarp();
  const double tol = 1e-15;
  bool converged = false;
  for (int sweep = 0; sweep < 80 && !converged; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < nn - 1; ++p)
      for (int q = p + 1; q < nn; ++q) {
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < mm; i += 32) {
          const double x = W[static_cast<std::size_t>(i) * nn + p], y = W[static_cast<std::size_t>(i) * nn + q];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = dev::warp_sum(al);
        be = dev::warp_sum(be);
        ga = dev::warp_sum(ga);
        if (ga == 0.0 || fabs(ga) <= tol * sqrt(al * be)) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = lane; i < mm; i += 32) {
          double* r = W + static_cast<std::size_t>(i) * nn;
          const double x = r[p], y = r[q];
          r[p] = c * x - s * y;
          r[q] = s * x + c * y;
        }
        for (int i = lane; i < nn; i += 32) {
          double* r = V + static_cast<std::size_t>(i) * nn;
          const double x = r[p], y = r[q];
          r[p] = c * x - s * y;
          r[q] = s * x + c * y;
        }
        __syncwarp();
      }
    converged = !rotated;
  }
  if (lane == 0) *status = converged ? 0 : 1;
  for (int j = 0; j < nn; ++j) {
    double a = 0.0;
    for (int i = lane; i < mm; i += 32) {
      const double x = W[static_cast<std::size_t>(i) * nn + j];
      a = fma(x, x, a);
    }
    a = dev::warp_sum(a);
    if (lane == 0) s_sig[j] = sqrt(a);
  }
  __syncwarp();
  if (lane == 0) {  // stable order by sigma, non-increasing
    for (int j = 0; j < nn; ++j) s_ord[j] = j;
    for (int a = 1; a < nn; ++a) {
      const int o = s_ord[a];
      int b = a - 1;
      while (b >= 0 && s_sig[s_ord[b]] < s_sig[o]) {
        s_ord[b + 1] = s_ord[b];
        --b;
      }
      s_ord[b + 1] = o;
    }
  }
  __syncwarp();
  const double smax = s_sig[s_ord[0]];
  const double zero = smax * 2.3e-16 * (mm > nn ? mm : nn);  // sigma at rounding level of sigma_max: null column
  int nz = 0;
  for (int c = 0; c < nn; ++c) {
    const int src = s_ord[c];
    const double s = s_sig[src];
    const bool keep = s > zero;
    if (keep) nz = c + 1;  // (sorted: the kept columns come first)
    if (lane == 0) sig[c] = keep ? s : (s > 0.0 ? s : 0.0);
    for (int i = lane; i < mm; i += 32)
      Uo[static_cast<std::size_t>(i) * nn + c] = keep ? W[static_cast<std::size_t>(i) * nn + src] / s : 0.0;
    for (int i = lane; i < nn; i += 32) Vo[static_cast<std::size_t>(i) * nn + c] = V[static_cast<std::size_t>(i) * nn + src];
  }
  __syncwarp();
  // orthonormal completion of the null columns of U from unit vectors; W's first column is the scratch vector
  int cand = 0;
  for (int c = nz; c < nn; ++c) {
    while (cand < mm) {
      for (int i = lane; i < mm; i += 32) W[static_cast<std::size_t>(i) * nn] = i == cand ? 1.0 : 0.0;
      ++cand;
      __syncwarp();
      for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j < c; ++j) {
          double d = 0.0;
          for (int i = lane; i < mm; i += 32) d = fma(Uo[static_cast<std::size_t>(i) * nn + j], W[static_cast<std::size_t>(i) * nn], d);
          d = dev::warp_sum(d);
          for (int i = lane; i < mm; i += 32) W[static_cast<std::size_t>(i) * nn] -= d * Uo[static_cast<std::size_t>(i) * nn + j];
          __syncwarp();
        }
      double n2 = 0.0;
      for (int i = lane; i < mm; i += 32) {
        const double x = W[static_cast<std::size_t>(i) * nn];
        n2 = fma(x, x, n2);
      }
      n2 = sqrt(dev::warp_sum(n2));
      if (n2 > 0.5) {
        for (int i = lane; i < mm; i += 32) Uo[static_cast<std::size_t>(i) * nn + c] = W[static_cast<std::size_t>(i) * nn] / n2;
        __syncwarp();
        break;
      }
    }
  }
}

}  // namespace

int svd_max_cols() { return kSvdMaxCols; }

void launch_economy_svd(int mm, int nn, double* W, double* V, double* Uo, double* Vo, double* sig, int* status,
                        cudaStream_t s) {
  k_economy_svd<<<1, 32, 0, s>>>(mm, nn, W, V, Uo, Vo, sig, status);
}

}  // namespace p2g
