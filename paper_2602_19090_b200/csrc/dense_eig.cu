// dense_eig.cu — elementwise pieces of the Rayleigh–Ritz sub-solve of LARGE unresolved groups (R13),
// orchestrated in ozr_api.cu: K = C·(M+Mᵀ)/2·C with C = I + R_JJ/2 and Z = C·Y as FP64-accurate INT8 slice products
// (oz_dgemm), K = YΘYᵀ by the hand-written eigensolver (syev.cu), Y's signs (y_kk ≥ 0, the largest-|·| entry of the
// column when y_kk = 0), λ̂_J = μ + Θ, and the scatter of Ẽ'[:, J]·Z — the same mathematics and conventions as the
// per-CTA Jacobi of cluster.cu, whose O(m³·sweeps) cost with m − 1 grid-wide synchronisations per sweep rules it out
// for groups of thousands of columns (BASELINE c4's FP32 start opens with 6628).
#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "kernels.h"

namespace ozr {

namespace {

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

void launch_dense_sym(int m, const double* X, double* out, cudaStream_t s) {
  const long long m2 = static_cast<long long>(m) * m;
  const int gb = static_cast<int>(std::min<long long>((m2 + 255) / 256, 148 * 16));
  k_dsym<<<gb, 256, 0, s>>>(m, X, out);
}
void launch_dense_axpy(long long cnt, const double* X, double alpha, const double* P, double* out, cudaStream_t s) {
  const int gb = static_cast<int>(std::min<long long>((cnt + 255) / 256, 148 * 16));
  k_daxpy<<<gb, 256, 0, s>>>(cnt, X, alpha, P, out);
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
