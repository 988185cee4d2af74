// Lazily dlopen'ed CUDA libraries for the two once-per-call dense steps that
// are plain library work: cuSOLVER syevdx (the J x J eigenproblem of the eye
// initialisation, solver.hpp:133-164) and cuBLAS DGEMM (the naive MTTKRP,
// mttkrp.hpp:208-235, which is by definition a materialised GEMM).  Loading
// them on first use keeps the hot loop's process free of both.
#pragma once

#include <cublas_v2.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <string>

#include "p2g_ctx.hpp"

namespace p2g {

struct SolverLib {
  cusolverStatus_t (*Create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*Destroy)(cusolverDnHandle_t) = nullptr;
  cusolverStatus_t (*SetStream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*DsyevdxBuf)(cusolverDnHandle_t, cusolverEigMode_t, cusolverEigRange_t, cublasFillMode_t, int,
                                 const double*, int, double, double, int, int, int*, const double*, int*) = nullptr;
  cusolverStatus_t (*Dsyevdx)(cusolverDnHandle_t, cusolverEigMode_t, cusolverEigRange_t, cublasFillMode_t, int,
                              double*, int, double, double, int, int, int*, double*, double*, int, int*) = nullptr;
};

struct BlasLib {
  cublasStatus_t (*Create)(cublasHandle_t*) = nullptr;
  cublasStatus_t (*Destroy)(cublasHandle_t) = nullptr;
  cublasStatus_t (*SetStream)(cublasHandle_t, cudaStream_t) = nullptr;
  cublasStatus_t (*Dgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const double*,
                          const double*, int, const double*, int, const double*, double*, int) = nullptr;
  cublasStatus_t (*SetMathMode)(cublasHandle_t, cublasMath_t) = nullptr;
};

template <typename F>
inline void dl_sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  if (!f) throw CudaError(std::string("missing symbol ") + name);
}

inline SolverLib& solver_lib() {
  static SolverLib L;
  static void* h = nullptr;
  if (!h) {
    void* x = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_LOCAL);
    if (!x) throw CudaError("cuSOLVER unavailable: cannot dlopen libcusolver.so.11");
    dl_sym(x, "cusolverDnCreate", L.Create);
    dl_sym(x, "cusolverDnDestroy", L.Destroy);
    dl_sym(x, "cusolverDnSetStream", L.SetStream);
    dl_sym(x, "cusolverDnDsyevdx_bufferSize", L.DsyevdxBuf);
    dl_sym(x, "cusolverDnDsyevdx", L.Dsyevdx);
    h = x;
  }
  return L;
}

inline BlasLib& blas_lib() {
  static BlasLib L;
  static void* h = nullptr;
  if (!h) {
    void* x = dlopen("libcublas.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!x) throw CudaError("cuBLAS unavailable: cannot dlopen libcublas.so.12");
    dl_sym(x, "cublasCreate_v2", L.Create);
    dl_sym(x, "cublasDestroy_v2", L.Destroy);
    dl_sym(x, "cublasSetStream_v2", L.SetStream);
    dl_sym(x, "cublasDgemm_v2", L.Dgemm);
    dl_sym(x, "cublasSetMathMode", L.SetMathMode);
    h = x;
  }
  return L;
}

}  // namespace p2g
