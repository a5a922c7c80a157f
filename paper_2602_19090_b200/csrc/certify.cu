// certify.cu — the a-posteriori forward-error certificate of one sweep (reading R12).
//
// The paper stops after a fixed number of iterations and models the error only on average over
// the columns (eq. assume2 / gamma). The sweep returns X̂_new = X̂^(1)(I + Ẽ) while the exact
// eigenvectors are X = X̂^(1)(I + E), so ‖X − X̂_new‖₂ ≈ ‖E − Ẽ‖₂, Ẽ's second-order defect.
// From X̂^(1) = X(I + F), F ≈ −Ẽ, and Alg. 1's R, S, for i ≠ j
//     (Ẽ − E)_ij ≈ Q_ij / (λ̂_j − λ̂_i),   Q = ẼᵀC,   c_kj = (λ̂_k − λ̂_j)·ẽ_kj,
// up to terms bounded by ‖Ẽ‖² (added as 1.5‖Ẽ‖_F² by the host). Q only has to be accurate to a few per cent, so
// it is ONE bf16 tensor-core GEMM (the slice-GEMM kernel with kind::f16, f32 accumulator): Ẽ and C are stored
// column-scaled by powers of two (exact) in bf16, which keeps every entry's relative precision (2^-8) whatever
// its magnitude inside the column; the host measured ‖·‖₂ of D = Q∘H to 0.3 % of the exact-Q value on every
// BASELINE recipe (scratch study, R12).
//
//   k_cert_prep   Ẽ = diag(2^−g)·Ẽ' (the stored Ẽ' = diag(2^g)Ẽ is exact), its column maxima, bf16 Ẽ and C
//   (GEMM)        Q = ẼᵀC  (launch_gemm_i8 kind 1)
//   k_cert_delta  D = 2^{sE_i + sC_j}·Q_ij / (λ̂_j − λ̂_i) (fp32, i ≠ j), Σ_i D_ij² per column
//   k_pi_*        power iteration for ‖D‖₂ (D column-partitioned on P ranks: D·z all-reduced)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "certify.h"

namespace ozr {

namespace {

constexpr int CB = 256;
constexpr int PI_CHUNKS = 32;

__device__ __forceinline__ double cb_sum(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < CB / 32) ? sh[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (threadIdx.x == 0) sh[0] = v;
  __syncthreads();
  v = sh[0];
  __syncthreads();
  return v;
}
__device__ __forceinline__ double cb_max(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < CB / 32) ? sh[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (threadIdx.x == 0) sh[0] = v;
  __syncthreads();
  v = sh[0];
  __syncthreads();
  return v;
}
// ⌈log2 v⌉ for v > 0 from the exponent field (0 for v = 0)
__device__ __forceinline__ int ceil_log2_dev(double v) {
  if (v == 0.0) return 0;
  int e;
  const double m = frexp(v, &e);
  return (m == 0.5) ? e - 1 : e;
}

// one CTA per local column j (global gj = col0 + j)
__global__ void __launch_bounds__(CB)
    k_cert_prep(const double* __restrict__ Ep, long long lde, int rows, const int32_t* __restrict__ g,
                const double* __restrict__ lam, int col0, __nv_bfloat16* __restrict__ Eb, __nv_bfloat16* __restrict__ Cb,
                long long ldb, int32_t* __restrict__ sE, int32_t* __restrict__ sC, double* __restrict__ esq) {
  __shared__ double sh[CB / 32];
  const int j = blockIdx.x, gj = col0 + j;
  const double* col = Ep + static_cast<long long>(j) * lde;
  const double lj = lam[gj];
  double me = 0.0, mc = 0.0, ss = 0.0;
  for (int i = threadIdx.x; i < rows; i += CB) {
    const double e = ldexp(col[i], -g[i]);  // ẽ_ij = 2^{−g_i} ẽ'_ij, exact
    me = fmax(me, fabs(e));
    mc = fmax(mc, fabs((lam[i] - lj) * e));
    ss = fma(e, e, ss);
  }
  me = cb_max(me, sh);
  mc = cb_max(mc, sh);
  ss = cb_sum(ss, sh);
  const int se = ceil_log2_dev(me), sc = ceil_log2_dev(mc);
  __nv_bfloat16* eb = Eb + static_cast<long long>(gj) * ldb;  // Ẽ: all columns (the GEMM's A operand)
  __nv_bfloat16* cb = Cb + static_cast<long long>(j) * ldb;   // C: this rank's columns
  for (int i = threadIdx.x; i < rows; i += CB) {
    const double e = ldexp(col[i], -g[i]);
    eb[i] = __float2bfloat16_rn(static_cast<float>(ldexp(e, -se)));
    cb[i] = __float2bfloat16_rn(static_cast<float>(ldexp((lam[i] - lj) * e, -sc)));
  }
  if (threadIdx.x == 0) {
    sE[gj] = se;
    sC[j] = sc;
    esq[j] = ss;
  }
}

// one CTA per local column j: D_ij = 2^{sE_i + sC_j} Q_ij / (λ̂_j − λ̂_i), D_jj = 0; dsq[j] = Σ_i D_ij²
__global__ void __launch_bounds__(CB)
    k_cert_delta(const float* __restrict__ Q, long long ldq, int rows, const int32_t* __restrict__ sE,
                 const int32_t* __restrict__ sC, const double* __restrict__ lam, int col0, float* __restrict__ D,
                 double* __restrict__ dsq, int* __restrict__ flag) {
  __shared__ double sh[CB / 32];
  const int j = blockIdx.x, gj = col0 + j;
  const double lj = lam[gj];
  const int cj = sC[j];
  const float* q = Q + static_cast<long long>(j) * ldq;
  float* d = D + static_cast<long long>(j) * rows;
  double ss = 0.0;
  bool bad = false;
  for (int i = threadIdx.x; i < rows; i += CB) {
    double v = 0.0;
    if (i != gj) {
      const double dl = lj - lam[i];
      if (dl == 0.0) {
        bad = true;
      } else {
        v = ldexp(static_cast<double>(q[i]), sE[i] + cj) / dl;
      }
    }
    d[i] = static_cast<float>(v);
    ss = fma(v, v, ss);
  }
  ss = cb_sum(ss, sh);
  if (threadIdx.x == 0) dsq[j] = ss;
  if (bad) atomicOr(flag, 1);
}

// power iteration: y = D·z (rows), chunked over columns; then Dᵀy per column
__global__ void __launch_bounds__(CB)
    k_pi_dz(const float* __restrict__ D, int rows, int cols, const double* __restrict__ z, double* __restrict__ part) {
  const int i = blockIdx.x * CB + threadIdx.x;
  if (i >= rows) return;
  const int per = (cols + PI_CHUNKS - 1) / PI_CHUNKS;
  const int j0 = blockIdx.y * per, j1 = min(cols, j0 + per);
  double acc = 0.0;
  for (int j = j0; j < j1; ++j) acc = fma(static_cast<double>(D[static_cast<long long>(j) * rows + i]), z[j], acc);
  part[static_cast<long long>(blockIdx.y) * rows + i] = acc;
}
__global__ void k_pi_sum(const double* __restrict__ part, int rows, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double acc = 0.0;
  for (int q = 0; q < PI_CHUNKS; ++q) acc += part[static_cast<long long>(q) * rows + i];
  y[i] = acc;
}
__global__ void __launch_bounds__(CB)
    k_pi_dty(const float* __restrict__ D, int rows, const double* __restrict__ y, double* __restrict__ v) {
  __shared__ double sh[CB / 32];
  const float* c = D + static_cast<long long>(blockIdx.x) * rows;
  double acc = 0.0;
  for (int i = threadIdx.x; i < rows; i += CB) acc = fma(static_cast<double>(c[i]), y[i], acc);
  acc = cb_sum(acc, sh);
  if (threadIdx.x == 0) v[blockIdx.x] = acc;
}

}  // namespace

void launch_cert_prep(const double* Ep, long long lde, int rows, int cols, const int32_t* g, const double* lam, int col0,
                      void* Eb, void* Cb, long long ldb, int32_t* sE, int32_t* sC, double* esq, cudaStream_t s) {
  k_cert_prep<<<cols, CB, 0, s>>>(Ep, lde, rows, g, lam, col0, static_cast<__nv_bfloat16*>(Eb),
                                  static_cast<__nv_bfloat16*>(Cb), ldb, sE, sC, esq);
}
void launch_cert_delta(const float* Q, long long ldq, int rows, int cols, const int32_t* sE, const int32_t* sC,
                       const double* lam, int col0, float* D, double* dsq, int* flag, cudaStream_t s) {
  k_cert_delta<<<cols, CB, 0, s>>>(Q, ldq, rows, sE, sC, lam, col0, D, dsq, flag);
}
void launch_pi_dz(const float* D, int rows, int cols, const double* z, double* part, double* y, cudaStream_t s) {
  k_pi_dz<<<dim3((rows + CB - 1) / CB, PI_CHUNKS), CB, 0, s>>>(D, rows, cols, z, part);
  k_pi_sum<<<(rows + 255) / 256, 256, 0, s>>>(part, rows, y);
}
void launch_pi_dty(const float* D, int rows, int cols, const double* y, double* v, cudaStream_t s) {
  k_pi_dty<<<cols, CB, 0, s>>>(D, rows, y, v);
}
int cert_pi_chunks() { return PI_CHUNKS; }

}  // namespace ozr
