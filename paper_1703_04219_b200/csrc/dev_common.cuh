// Device-side building blocks shared by the libp2g kernels (sm_100a, fp64).
//
// All numerics are IEEE binary64 on CUDA cores (DFMA): tcgen05 has no f64
// kind on sm_100a, so the small dense R x R work runs as
// warp-cooperative code over shared memory.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace p2g {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

__device__ __forceinline__ int warp_or(int v) { return __any_sync(kFull, v); }

/// Row-major R-vector gather of V row j (V is J x R row-major).
/// 1/sqrt(x) for normal x > 0 without the library slow path (whose
/// out-of-line call forces spills in register-resident loops): the MUFU
/// approximation refined by two Newton steps, y <- y (3/2 - x/2 y^2).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

/// 1/x for normal x without the IEEE division sequence: the MUFU
/// approximation refined by two Newton steps, y <- y (2 - x y).
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

/// Bulk (TMA) prefetch of `bytes` (a multiple of 16) at the 16-byte aligned global address p
/// into L2: one instruction by one lane, no destination buffer.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

/// TMA bulk copy global -> shared with mbarrier completion (one lane issues; every lane waits).
/// Sizes are multiples of 16 bytes, both addresses 16-byte aligned.
__device__ __forceinline__ void mbar_init(unsigned mbar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
/// Orders this thread's earlier generic-proxy accesses to shared memory before later async-proxy (TMA) ones.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned mbar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

/// Shared-memory accesses at a 32-bit shared address plus a compile-time
/// byte offset (ptxas folds a warp-uniform base into [R + UR + imm]).  The
/// asm statements keep their source order, so a batch of loads written ahead
/// of a batch of stores is issued that way.
template <int IMM>
__device__ __forceinline__ double lds64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(IMM) : "memory");
  return v;
}
template <int IMM>
__device__ __forceinline__ double2 lds128(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(v.x), "=d"(v.y) : "r"(a), "n"(IMM) : "memory");
  return v;
}
template <int IMM>
__device__ __forceinline__ void sts64(unsigned a, double v) {
  asm volatile("st.shared.f64 [%0+%1], %2;" ::"r"(a), "n"(IMM), "d"(v) : "memory");
}
template <int IMM>
__device__ __forceinline__ void sts128(unsigned a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0+%1], {%2, %3};" ::"r"(a), "n"(IMM), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ uint4 lds128u(unsigned a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned lds32u(unsigned a) {
  unsigned v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
/// 32-byte read-only global load (sm_100: LDG.E.256).
__device__ __forceinline__ double4 ldg256(const double* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
/// 32-byte global store (sm_100: STG.E.256).
__device__ __forceinline__ void stg256(double* p, double4 v) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}
/// The shared address of p, made warp-uniform (a uniform register).
__device__ __forceinline__ unsigned smem_uniform(const void* p) {
  return __shfl_sync(kFull, static_cast<unsigned>(__cvta_generic_to_shared(p)), 0);
}

template <int RP>
__device__ __forceinline__ void axpy_row(double (&acc)[RP], const double* __restrict__ vrow, double a, int R) {
#pragma unroll
  for (int r = 0; r < RP; ++r)
    if (r < R) acc[r] = fma(a, __ldg(vrow + r), acc[r]);
}

/// acc = X_row . V for one CSR row (entries [p0,p1)): the X_k V product of
/// solver.hpp:182-188 restated row-wise (same per-row accumulation order:
/// columns ascending).
template <int RP>
__device__ __forceinline__ void csr_row_times(double (&acc)[RP], const int32_t* __restrict__ ci,
                                              const double* __restrict__ val, int64_t p0, int64_t p1,
                                              const double* __restrict__ V, int R) {
#pragma unroll
  for (int r = 0; r < RP; ++r) acc[r] = 0.0;
  for (int64_t p = p0; p < p1; ++p) {
    const int j = __ldg(ci + p);
    const double v = __ldg(val + p);
    axpy_row<RP>(acc, V + static_cast<int64_t>(j) * R, v, R);
  }
}

/// D += A B on the fp64 tensor cores (DMMA m8n8k4, row.col): the warp holds
/// A[lane/4][lane%4], B[lane%4][lane/4] and D[lane/4][2(lane%4) + {0,1}].
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

/// acc[u] += X_row(u) . V for U rows at once, V1 only (NV = 1) or also
/// acc2[u] += X_row(u) . V2 (NV = 2): the t-th entry of every row is loaded
/// together, so a lane keeps U independent ci -> V dependency chains in
/// flight (the streaming kernels are bound by this gather latency).  V rows
/// are read as 16-byte vectors when R is even.  Same per-row accumulation
/// order as csr_row_times (entries ascending).
template <int R, int U, int NV>
__device__ __forceinline__ void csr_rows_times(double (&acc)[U][R], double (&acc2)[U][R],
                                               const int32_t* __restrict__ ci, const double* __restrict__ val,
                                               const int64_t (&p0)[U], const int64_t (&p1)[U],
                                               const double* __restrict__ V1, const double* __restrict__ V2) {
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int a = 0; a < R; ++a) {
      acc[u][a] = 0.0;
      if (NV == 2) acc2[u][a] = 0.0;
    }
  int64_t p[U];
#pragma unroll
  for (int u = 0; u < U; ++u) p[u] = p0[u];
  while (true) {
    bool act[U], any = false;
    int j[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      act[u] = p[u] < p1[u];
      any |= act[u];
      j[u] = act[u] ? __ldg(ci + p[u]) : 0;
      v[u] = act[u] ? __ldg(val + p[u]) : 0.0;
    }
    if (!any) break;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!act[u]) continue;
      const double* r1 = V1 + static_cast<int64_t>(j[u]) * R;
      const double* r2 = V2 + static_cast<int64_t>(j[u]) * R;
      if constexpr (R % 2 == 0) {
#pragma unroll
        for (int a = 0; a < R; a += 2) {
          const double2 x = __ldg(reinterpret_cast<const double2*>(r1 + a));
          acc[u][a] = fma(v[u], x.x, acc[u][a]);
          acc[u][a + 1] = fma(v[u], x.y, acc[u][a + 1]);
          if (NV == 2) {
            const double2 y = __ldg(reinterpret_cast<const double2*>(r2 + a));
            acc2[u][a] = fma(v[u], y.x, acc2[u][a]);
            acc2[u][a + 1] = fma(v[u], y.y, acc2[u][a + 1]);
          }
        }
      } else {
#pragma unroll
        for (int a = 0; a < R; ++a) {
          acc[u][a] = fma(v[u], __ldg(r1 + a), acc[u][a]);
          if (NV == 2) acc2[u][a] = fma(v[u], __ldg(r2 + a), acc2[u][a]);
        }
      }
      ++p[u];
    }
  }
}

// ---------------------------------------------------------------------------
// Warp-cooperative small dense algebra on shared memory (row-major, ld = n).
// ---------------------------------------------------------------------------

/// C = A * B (n x n), all row-major in smem; C must not alias A or B.
__device__ __forceinline__ void wmm(double* C, const double* A, const double* B, int n, int lane) {
  for (int e = lane; e < n * n; e += kWarp) {
    const int i = e / n, j = e - (e / n) * n;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = fma(A[i * n + k], B[k * n + j], acc);
    C[e] = acc;
  }
  __syncwarp();
}

/// C = A^T * B (n x n).
__device__ __forceinline__ void wmm_tn(double* C, const double* A, const double* B, int n, int lane) {
  for (int e = lane; e < n * n; e += kWarp) {
    const int i = e / n, j = e - (e / n) * n;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = fma(A[k * n + i], B[k * n + j], acc);
    C[e] = acc;
  }
  __syncwarp();
}

/// C = A * B^T (n x n).
__device__ __forceinline__ void wmm_nt(double* C, const double* A, const double* B, int n, int lane) {
  for (int e = lane; e < n * n; e += kWarp) {
    const int i = e / n, j = e - (e / n) * n;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = fma(A[i * n + k], B[j * n + k], acc);
    C[e] = acc;
  }
  __syncwarp();
}

/// Cyclic Jacobi eigendecomposition of the symmetric n x n matrix A (smem,
/// row-major, overwritten: eigenvalues end on the diagonal), eigenvectors
/// accumulated into the columns of E.  Rotations of one round are disjoint
/// (round-robin ordering), so the warp applies them simultaneously.
/// Work arrays: cs[2*ceil(n/2)] doubles, pq[2*ceil(n/2)] ints.
/// Returns the number of sweeps used.
__device__ inline int warp_jacobi_eig(double* A, double* E, int n, double* cs, int* pq, int lane,
                                      int max_sweeps = 40) {
  for (int e = lane; e < n * n; e += kWarp) E[e] = (e / n == e % n) ? 1.0 : 0.0;
  __syncwarp();
  if (n <= 1) return 0;
  const int m = (n + 1) & ~1;  // players incl. one dummy for odd n
  const int half = m / 2;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    // Convergence: off-diagonal mass relative to the diagonal.
    double off = 0.0, dia = 0.0;
    for (int e = lane; e < n * n; e += kWarp) {
      const int i = e / n, j = e - i * n;
      const double a = A[e];
      if (i == j)
        dia = fma(a, a, dia);
      else
        off = fma(a, a, off);
    }
    off = warp_sum(off);
    dia = warp_sum(dia);
    if (off == 0.0 || off <= 1e-32 * dia) break;
    for (int round = 0; round < m - 1; ++round) {
      if (lane < half) {
        int p, q;
        if (lane == 0) {
          p = round;
          q = m - 1;
        } else {
          p = (round + lane) % (m - 1);
          q = (round - lane + (m - 1)) % (m - 1);
        }
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = A[p * n + q];
          const double app = A[p * n + p], aqq = A[q * n + q];
          if (apq != 0.0 && fabs(apq) > 1e-300 && fabs(apq) > 2.2e-16 * 0.01 * sqrt(fabs(app * aqq))) {
            const double theta = (aqq - app) / (2.0 * apq);
            const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
            c = rsqrt(fma(t, t, 1.0));
            s = t * c;
          }
        } else {
          q = -1;  // dummy pair
        }
        cs[2 * lane] = c;
        cs[2 * lane + 1] = s;
        pq[2 * lane] = p;
        pq[2 * lane + 1] = q;
      }
      __syncwarp();
      // Columns: A <- A J ; E <- E J.
      for (int it = lane; it < half * n; it += kWarp) {
        const int pr = it / n, k = it - pr * n;
        const int p = pq[2 * pr], q = pq[2 * pr + 1];
        if (q < 0) continue;
        const double c = cs[2 * pr], s = cs[2 * pr + 1];
        if (s == 0.0) continue;
        const double akp = A[k * n + p], akq = A[k * n + q];
        A[k * n + p] = c * akp - s * akq;
        A[k * n + q] = s * akp + c * akq;
        const double ekp = E[k * n + p], ekq = E[k * n + q];
        E[k * n + p] = c * ekp - s * ekq;
        E[k * n + q] = s * ekp + c * ekq;
      }
      __syncwarp();
      // Rows: A <- J^T A.
      for (int it = lane; it < half * n; it += kWarp) {
        const int pr = it / n, k = it - pr * n;
        const int p = pq[2 * pr], q = pq[2 * pr + 1];
        if (q < 0) continue;
        const double c = cs[2 * pr], s = cs[2 * pr + 1];
        if (s == 0.0) continue;
        const double apk = A[p * n + k], aqk = A[q * n + k];
        A[p * n + k] = c * apk - s * aqk;
        A[q * n + k] = s * apk + c * aqk;
      }
      __syncwarp();
      if (lane < half) {
        const int p = pq[2 * lane], q = pq[2 * lane + 1];
        if (q >= 0 && cs[2 * lane + 1] != 0.0) {
          A[p * n + q] = 0.0;
          A[q * n + p] = 0.0;
        }
      }
      __syncwarp();
    }
  }
  return sweep;
}

/// Moore-Penrose pseudo-inverse of a symmetric PSD n x n matrix (kernels.hpp:
/// 68-87): symmetrize, eig, keep eigenvalues > 1e-12 * max|lambda| and > 0.
/// G is read, out written (row-major smem); A, E, T scratch n*n each.
__device__ inline void warp_pinv_sym(const double* G, double* out, double* A, double* E, double* cs, int* pq, int n,
                                     int lane) {
  for (int e = lane; e < n * n; e += kWarp) {
    const int i = e / n, j = e - i * n;
    A[e] = 0.5 * (G[i * n + j] + G[j * n + i]);
  }
  __syncwarp();
  warp_jacobi_eig(A, E, n, cs, pq, lane);
  double amax = 0.0;
  for (int i = lane; i < n; i += kWarp) amax = fmax(amax, fabs(A[i * n + i]));
  amax = warp_max(amax);
  const double cutoff = 1e-12 * amax;
  for (int e = lane; e < n * n; e += kWarp) {
    const int i = e / n, j = e - i * n;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) {
      const double ev = A[k * n + k];
      if (ev > cutoff && ev > 0.0) acc += E[i * n + k] * E[j * n + k] / ev;
    }
    out[e] = acc;
  }
  __syncwarp();
  // exact symmetry (kernels.hpp:85)
  for (int e = lane; e < n * n; e += kWarp) {
    const int i = e / n, j = e - i * n;
    if (j > i) out[e] = out[j * n + i];
  }
  __syncwarp();
}

}  // namespace dev
}  // namespace p2g
