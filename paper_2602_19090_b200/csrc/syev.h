// syev.h — the hand-written dense symmetric eigensolver (syev.cu) of the large-group Rayleigh–Ritz sub-solve
// (R13). Internal.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <functional>
#include <string>
#include <utility>
#include <vector>

namespace ozr {

// Grow-only device buffers of the eigensolver (owned by the context).
struct SyevWorkspace {
  std::vector<std::pair<void*, size_t>> bufs;
  void* get(int slot, size_t bytes);
  ~SyevWorkspace();
};

// C = op(A)·B (column-major, fp64 result): A is M x K (lda), or stored K x M when a_t (op(A) = Aᵀ); B is K x N.
// Returns 0 on success. Used for the large products (D&C merges, back-transformation).
using SyevGemm = std::function<int(int M, int N, int K, const double* A, int lda, bool a_t, const double* B, int ldb,
                                   double* C, int ldc)>;

// K (m x m, ld = m, lower triangle read, destroyed) = YΘYᵀ: θ ascending (device, m), Y (device, m x m, ld = m).
// Products with a dimension ≥ big_gemm_min go to `gemm` (when set). Returns 0, or 6 (CUDA error / no
// convergence) / 8 (out of memory) with *err set.
// Stage checks (tests): d_out set — stop after the tridiagonalisation (d, e, τ out; K holds the reflectors below
// its sub-diagonal); d_in set — the divide and conquer alone on the tridiagonal (d_in, e_in): θ, Y = its eigenvectors.
struct SyevDebug {
  double* d_out = nullptr;
  double* e_out = nullptr;
  double* tau_out = nullptr;
  const double* d_in = nullptr;
  const double* e_in = nullptr;
};
int dense_syev(SyevWorkspace& w, int m, double* K, double* theta, double* Y, const SyevGemm& gemm, int big_gemm_min,
               cudaStream_t s, std::string* err, const SyevDebug* dbg = nullptr);

// pieces (tests / measurement)
int syev_trd_grid(int m);
size_t syev_trd_partials(int m, int G);
cudaError_t syev_tridiag(double* A, int m, double* d, double* e, double* tau, double* V, double* W, double* part,
                         int G, cudaStream_t s);
void syev_dgemm(int M, int N, int K, double alpha, const double* A, int lda, bool ta, const double* B, int ldb,
                double beta, double* C, int ldc, cudaStream_t s);

}  // namespace ozr
