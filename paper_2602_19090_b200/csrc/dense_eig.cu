// dense_eig.cu — the Rayleigh–Ritz sub-solve of LARGE unresolved groups (R13) with a dense
// symmetric eigensolver instead of the cyclic Jacobi of cluster.cu. Same mathematics, same conventions
// (cluster.cu header): K = C·(M+Mᵀ)/2·C with C = I + R_JJ/2, K = YΘYᵀ (Θ ascending, y_kk ≥ 0, the
// largest-|·| entry of the column when y_kk = 0), Z = C·Y, λ̂_J = μ + Θ.
//
// The Jacobi core is O(m³) per sweep with one grid-wide synchronisation per rotation round (m − 1 rounds
// per sweep), which makes a 6628-column group (BASELINE c4: cnd 1e14 from an FP32 eigensolver) a
// minutes-long solve. Here the two C products and Z = C·Y are FP64 SIMT GEMMs (fixed summation order:
// deterministic) and the eigen-decomposition of K is LAPACK's divide-and-conquer syevd from cuSOLVER
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
// out = Cin + alpha · P·Q, 64 x 64 output tile per CTA, 4 x 4 per thread, k-slabs of 16 in shared
// memory; every output is one fma chain over l ascending (deterministic).
constexpr int GT = 64, GK = 16;
__global__ void __launch_bounds__(256)
    k_dgemm_acc(int m, const double* __restrict__ P, const double* __restrict__ Q, const double* __restrict__ Cin,
                double alpha, double* __restrict__ out) {
  __shared__ double ps[GK][GT + 1];  // ps[l][a] = P(a0 + a, l0 + l)
  __shared__ double qs[GK][GT + 1];  // qs[l][b] = Q(l0 + l, b0 + b)
  const int a0 = blockIdx.x * GT, b0 = blockIdx.y * GT;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  for (int l0 = 0; l0 < m; l0 += GK) {
    for (int e = threadIdx.x; e < GT * GK; e += 256) {
      const int a = e % GT, l = e / GT;  // consecutive threads: consecutive rows of P's column
      ps[l][a] = (a0 + a < m && l0 + l < m) ? P[static_cast<long long>(l0 + l) * m + a0 + a] : 0.0;
      const int lq = e % GK, b = e / GK;
      qs[lq][b] = (l0 + lq < m && b0 + b < m) ? Q[static_cast<long long>(b0 + b) * m + l0 + lq] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int l = 0; l < GK; ++l) {
      double pa[4], qb[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) pa[r] = ps[l][tx + 16 * r];
#pragma unroll
      for (int c = 0; c < 4; ++c) qb[c] = qs[l][ty + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(pa[r], qb[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int a = a0 + tx + 16 * r, b = b0 + ty + 16 * c;
      if (a < m && b < m) {
        const long long o = static_cast<long long>(b) * m + a;
        out[o] = fma(alpha, acc[r][c], Cin[o]);
      }
    }
}

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
    if (k == 0 && *info != 0) atomicOr(err, ERR_SOLVER);
  }
}

void dgemm_acc(int m, const double* P, const double* Q, const double* Cin, double alpha, double* out, cudaStream_t s) {
  dim3 grid((m + GT - 1) / GT, (m + GT - 1) / GT);
  k_dgemm_acc<<<grid, 256, 0, s>>>(m, P, Q, Cin, alpha, out);
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

cudaError_t launch_cluster_dense(const ClusterLaunch& L, DenseEig& de, int m, long long o, double mu, const int* J,
                                 cudaStream_t s) {
  SolverApi& a = api();
  if (!a.ok || !de.handle || a.setstream(de.handle, s) != 0) return cudaErrorNotSupported;
  const double* M = L.Mbuf + o;
  const double* R = L.Rbuf + o;
  double* K = L.Kbuf + o;
  double* V = L.Vbuf + o;
  double* Z = L.Zbuf + o;
  double* th = L.coop_scratch;  // m eigenvalues
  const long long m2 = static_cast<long long>(m) * m;
  const int gb = static_cast<int>(std::min<long long>((m2 + 255) / 256, 148 * 16));
  k_dsym<<<gb, 256, 0, s>>>(m, M, V);           // V = K0 = (M + Mᵀ)/2
  dgemm_acc(m, R, V, V, 0.5, K, s);             // K = K0 + ½R·K0 = C·K0
  dgemm_acc(m, K, R, K, 0.5, V, s);             // V = K + ½K·R = C·K0·C
  k_dsym<<<gb, 256, 0, s>>>(m, V, K);           // K = sym(V)
  if (a.syevd(de.handle, kEigModeVector, kFillLower, m, K, m, th, de.work, de.lwork, de.info) != 0)
    return cudaErrorUnknown;
  k_dense_sign<<<m, 256, 0, s>>>(m, K, th, mu, J, L.lam, de.info, L.err);  // K = Y (signed), λ̂_J
  dgemm_acc(m, R, K, K, 0.5, Z, s);             // Z = Y + ½R·Y = C·Y
  return cudaGetLastError();
}

}  // namespace ozr
