// certify.h — launchers of the a-posteriori forward-error certificate (certify.cu, R12). Internal.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace ozr {

// Ẽ = diag(2^−g)·Ẽ' from the stored Ẽ' (rows x cols, local columns [col0, col0 + cols)); per column j:
// sE[col0 + j] = ⌈log2 max_i |ẽ_ij|⌉, sC[j] = ⌈log2 max_i |(λ̂_i − λ̂_j) ẽ_ij|⌉, esq[j] = Σ_i ẽ_ij²,
// rsq[j] = Σ_{i≠j} (λ̂_i ẽ_ij/(λ̂_j − λ̂_i))² (the eigenvalue-rounding term of the certificate);
// Eb (bf16, column col0 + j at Eb + (col0 + j)·ldb) = ẽ·2^−sE, Cb (bf16, local column j) = (λ̂_i − λ̂_j)ẽ_ij·2^−sC.
void launch_cert_prep(const double* Ep, long long lde, int rows, int cols, const int32_t* g, const double* lam, int col0,
                      void* Eb, void* Cb, long long ldb, int32_t* sE, int32_t* sC, double* esq, double* rsq,
                      cudaStream_t s);
// Ẽ's rows as a GEMM A operand: rE[i] = row exponent of the all-gathered Eb (rows x cols, column k scaled by
// 2^−sE_k), EbT[i·ldb + k] = ẽ_ik·2^−rE_i in bf16.
void launch_cert_rowT(const void* Eb, long long ldb, int rows, int cols, const int32_t* sE, int32_t* rE, void* EbT,
                      cudaStream_t s);
// D = −(E − Ẽ) to second order (fp32, rows x cols, ld = rows): D_ij = 2^{sE_i + sC_j}·Q_ij/(λ̂_j − λ̂_i)
// − 2^{rE_i + sE_j}·P_ij, D_jj = −2^{rE_j + sE_j}·P_jj − ½esq_j (Q = ẼᵀC, P = Ẽ·Ẽ_{:,J}, ld = ldq);
// dsq[j] = Σ_i D_ij²; *flag |= 1 when two estimates are equal (no certificate).
void launch_cert_delta(const float* Q, const float* P, long long ldq, int rows, int cols, const int32_t* sE,
                       const int32_t* sC, const int32_t* rE, const double* esq, const double* lam, int col0, __nv_bfloat16* D,
                       double* dsq, int* flag, cudaStream_t s);
// y = D·z (part: cert_pi_chunks()·rows doubles of scratch); v = Dᵀ·y
void launch_pi_dz(const __nv_bfloat16* D, int rows, int cols, const double* z, double* part, double* y, cudaStream_t s);
void launch_pi_dty(const __nv_bfloat16* D, int rows, int cols, const double* y, double* v, cudaStream_t s);
int cert_pi_chunks();
// x = y − sqrt(c2[0])·x
void launch_lz_axpy(double* x, const double* y, int n, const double* c2, cudaStream_t s);

}  // namespace ozr
