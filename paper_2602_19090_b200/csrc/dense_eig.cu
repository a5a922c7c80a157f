// dense_eig.cu — the Rayleigh–Ritz sub-solve of LARGE unresolved groups (R13) with a dense
// symmetric eigensolver instead of the cyclic Jacobi of cluster.cu. Same mathematics, same conventions
// (cluster.cu header): K = C·(M+Mᵀ)/2·C with C = I + R_JJ/2, K = YΘYᵀ (Θ ascending, y_kk ≥ 0, the
// largest-|·| entry of the column when y_kk = 0), Z = C·Y, λ̂_J = μ + Θ.
//
// The Jacobi core is O(m³) per sweep with one grid-wide synchronisation per rotation round (m − 1 rounds
// per sweep), which makes a 6628-column group (BASELINE c4: cnd 1e14 from an FP32 eigensolver) a
// minutes-long solve. Here the two C products, Z = C·Y and the apply T·Z are FP64-accurate products on the
// INT8 slice GEMM (ozr_api.cu oz_dgemm; the host orchestrates) and the eigen-decomposition of K is LAPACK's
// divide-and-conquer syevd from cuSOLVER
// (a library routine in the role cuBLAS plays for a plain GEMM; loaded with dlopen on first use so the
// library has no link-time dependency and binds the libcusolver.so.11 torch has already loaded, if any).
// Backward-stable like Jacobi: the eigenvectors of K are accurate to u‖K‖/gap_K, the same accuracy the
// parity tests allow the Jacobi path against the oracle's __float128 one.
#include <dlfcn.h>

#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "kernels.h"

namespace ozr {

namespace {

// ---------------------------------------------------------------- cuSOLVER (dlopen)
typedef int (*fn_create)(void**);
typedef int (*fn_destroy)(void*);
typedef int (*fn_setstream)(void*, cudaStream_t);
typedef int (*fn_syevd_bs)(void*, int, int, int, const double*, int, const double*, int*);
typedef int (*fn_syevd)(void*, int, int, int, double*, int, double*, double*, int, int*);

struct SolverApi {
  bool tried = false, ok = false;
  std::string err;
  fn_create create = nullptr;
  fn_destroy destroy = nullptr;
  fn_setstream setstream = nullptr;
  fn_syevd_bs syevd_bs = nullptr;
  fn_syevd syevd = nullptr;
};

SolverApi& api() {
  static SolverApi a;
  if (a.tried) return a;
  a.tried = true;
  void* h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, when loaded
  if (!h) h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("/usr/local/cuda/lib64/libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    a.err = std::string("dlopen libcusolver.so.11: ") + dlerror();
    return a;
  }
  a.create = reinterpret_cast<fn_create>(dlsym(h, "cusolverDnCreate"));
  a.destroy = reinterpret_cast<fn_destroy>(dlsym(h, "cusolverDnDestroy"));
  a.setstream = reinterpret_cast<fn_setstream>(dlsym(h, "cusolverDnSetStream"));
  a.syevd_bs = reinterpret_cast<fn_syevd_bs>(dlsym(h, "cusolverDnDsyevd_bufferSize"));
  a.syevd = reinterpret_cast<fn_syevd>(dlsym(h, "cusolverDnDsyevd"));
  a.ok = a.create && a.destroy && a.setstream && a.syevd_bs && a.syevd;
  if (!a.ok) a.err = "libcusolver.so.11 lacks the syevd entry points";
  return a;
}

constexpr int kEigModeVector = 1;  // CUSOLVER_EIG_MODE_VECTOR
constexpr int kFillLower = 0;      // CUBLAS_FILL_MODE_LOWER

// ---------------------------------------------------------------- kernels (m x m, column-major, ld = m)
// out = (X + Xᵀ)/2
__global__ void k_dsym(int m, const double* __restrict__ X, double* __restrict__ out) {
  const long long m2 = static_cast<long long>(m) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < m2;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int a = static_cast<int>(e % m), b = static_cast<int>(e / m);
    out[e] = 0.5 * (X[e] + X[static_cast<long long>(a) * m + b]);
  }
}

// column k of Y: sign so that y_kk ≥ 0 (the largest-|·| entry, lowest index on ties, when y_kk = 0);
// λ̂_{J_k} = μ + θ_k. One CTA per column.
__global__ void __launch_bounds__(256)
    k_dense_sign(int m, double* __restrict__ Y, const double* __restrict__ th, double mu, const int* __restrict__ J,
                 double* __restrict__ lam, const int* __restrict__ info, int* __restrict__ err) {
  __shared__ double sb[256];
  __shared__ int si[256];
  const int k = blockIdx.x;
  double* y = Y + static_cast<long long>(k) * m;
  double piv = y[k];
  if (piv == 0.0) {
    double best = -1.0;
    int bi = m;
    for (int l = threadIdx.x; l < m; l += 256) {
      const double v = fabs(y[l]);
      if (v > best) {
        best = v;
        bi = l;
      }
    }
    sb[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int t = 1; t < 256; ++t)
        if (sb[t] > sb[0] || (sb[t] == sb[0] && si[t] < si[0])) {
          sb[0] = sb[t];
          si[0] = si[t];
        }
    }
    __syncthreads();
    piv = si[0] < m ? y[si[0]] : 1.0;
  }
  const double sg = piv < 0 ? -1.0 : 1.0;
  __syncthreads();
  for (int l = threadIdx.x; l < m; l += 256) y[l] *= sg;
  if (threadIdx.x == 0) {
    lam[J[k]] = mu + th[k];
    if (k == 0 && info && *info != 0) atomicOr(err, ERR_SOLVER);
  }
}

// out = X + alpha·P (cnt elements)
__global__ void k_daxpy(long long cnt, const double* __restrict__ X, double alpha, const double* __restrict__ P,
                        double* __restrict__ out) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < cnt;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    out[e] = fma(alpha, P[e], X[e]);
}

// Ẽ'[:, J_k] (owned columns) ← (T·Z)[:, k] on the rows outside the group, (Z − I)_{a,k}·2^{g_i} on its rows
// (row i = J_a): the dense groups' part of k_cluster_apply, with T·Z from the INT8 slice GEMM.
__global__ void k_dense_scatter(const double* __restrict__ TZ, int rows, int m, const int* __restrict__ J, int grp,
                                const int* __restrict__ grp_of, const int* __restrict__ pos_of,
                                const double* __restrict__ Z, const int32_t* __restrict__ gexp, double* __restrict__ Ep,
                                long long lde, int col0, int ncols) {
  const int k = blockIdx.y;
  const int jl = J[k] - col0;
  if (jl < 0 || jl >= ncols) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    double v = TZ[static_cast<long long>(k) * rows + i];
    if (grp_of[i] == grp) {
      const int a = pos_of[i];
      v = ldexp(Z[static_cast<long long>(k) * m + a] - (a == k ? 1.0 : 0.0), gexp[i]);
    }
    Ep[static_cast<long long>(jl) * lde + i] = v;
  }
}

}  // namespace

DenseEig::~DenseEig() {
  if (handle) api().destroy(handle);
}

bool dense_eig_available(std::string* why) {
  SolverApi& a = api();
  if (!a.ok && why) *why = a.err;
  return a.ok;
}

// Workspace (doubles) syevd needs for an m x m problem; -1 when cuSOLVER is unavailable.
long long dense_eig_lwork(DenseEig& de, int m, cudaStream_t s) {
  SolverApi& a = api();
  if (!a.ok) return -1;
  if (!de.handle && a.create(&de.handle) != 0) return -1;
  if (a.setstream(de.handle, s) != 0) return -1;
  int lw = 0;
  if (a.syevd_bs(de.handle, kEigModeVector, kFillLower, m, nullptr, m, nullptr, &lw) != 0) return -1;
  return lw;
}

void launch_dense_sym(int m, const double* X, double* out, cudaStream_t s) {
  const long long m2 = static_cast<long long>(m) * m;
  const int gb = static_cast<int>(std::min<long long>((m2 + 255) / 256, 148 * 16));
  k_dsym<<<gb, 256, 0, s>>>(m, X, out);
}
void launch_dense_axpy(long long cnt, const double* X, double alpha, const double* P, double* out, cudaStream_t s) {
  const int gb = static_cast<int>(std::min<long long>((cnt + 255) / 256, 148 * 16));
  k_daxpy<<<gb, 256, 0, s>>>(cnt, X, alpha, P, out);
}
cudaError_t dense_syevd(DenseEig& de, int m, double* K, double* th, cudaStream_t s) {
  SolverApi& a = api();
  if (!a.ok || !de.handle || a.setstream(de.handle, s) != 0) return cudaErrorNotSupported;
  if (a.syevd(de.handle, kEigModeVector, kFillLower, m, K, m, th, de.work, de.lwork, de.info) != 0)
    return cudaErrorUnknown;
  return cudaGetLastError();
}
void launch_dense_sign(int m, double* Y, const double* th, double mu, const int* J, double* lam, const int* info,
                       int* err, cudaStream_t s) {
  k_dense_sign<<<m, 256, 0, s>>>(m, Y, th, mu, J, lam, info, err);
}
void launch_dense_scatter(const double* TZ, int rows, int m, const int* J, int grp, const int* grp_of, const int* pos_of,
                          const double* Z, const int32_t* gexp, double* Ep, long long lde, int col0, int ncols,
                          cudaStream_t s) {
  k_dense_scatter<<<dim3((rows + 255) / 256 < 16 ? (rows + 255) / 256 : 16, m), 256, 0, s>>>(
      TZ, rows, m, J, grp, grp_of, pos_of, Z, gexp, Ep, lde, col0, ncols);
}

}  // namespace ozr
