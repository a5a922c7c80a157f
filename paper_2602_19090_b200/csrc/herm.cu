// herm.cu — the element-wise kernels of the Hermitian sweep (ozr_refine_step_herm; "the proposed
// method can be extended in a straightforward manner to Hermitian matrices", reading R18).
//
// A complex n x n matrix Z is carried as its real-stacked 2n x n form Ẑ = [Re Z; Im Z]; the complex product A·X̂
// is then the real product M_A·X̂s with the real symmetric embedding M_A = [[Ar, −Ai], [Ai, Ar]], X̂ᴴR is
// X̂sᵀ·[R̂, JR̂] (JR̂ = [Im R; −Re R]) and X̂Ẽ is Q·[diag(2^g)Er; −diag(2^g)Ei | diag(2^g)Ei; diag(2^g)Er] with the
// integer digits Q = [X̂r, X̂i]·diag(2^−g, 2^−g) — every product an INT8 slice product of the real kernels.
//
//   k_herm_embed     M_A from Ar, Ai
//   k_herm_lam_res   λ̂_j = Re(x̂_jᴴv_j)/(x̂_jᴴx̂_j) from the double-double V̂ (Alg. 1 line 3) and the columns of
//                    [R̂, JR̂], R = V − X̂D̂ (line 4's right operand), plus their column maxima
//   k_herm_E         Ẽ (line 5: ẽ_ij = w_ij/(λ̂_j − λ̂_i), ẽ_jj = r_j/2 + 0i) as the B operand of X̂Ẽ, ‖ẽ_j‖²
//   k_herm_Q         Q (the A operand of X̂Ẽ): the integer digits of X̂^(1) by rows, real then imaginary parts
//   k_herm_final     X̂ ← RN(X̂^(1) + U) on both parts (line 6, accsum), ν_j² = ‖x̂_j,new − x̂_j‖²
#include <cuda_runtime.h>

#include "ddmath.cuh"
#include "kernels.h"

namespace ozr {

namespace {

constexpr int HB = 256;

__device__ __forceinline__ double hsum(double v, double* sh) {  // fixed-order block sum
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < HB / 32) ? sh[threadIdx.x] : 0.0;
  if (threadIdx.x < 32)
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // valid in thread 0
}
__device__ __forceinline__ dd hsum_dd(dd v, dd* sh) {  // fixed-order block sum in double-double
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int o = 16; o; o >>= 1) {
    dd u{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
    v = dd_add(v, u);
  }
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    v = sh[0];
    for (int k = 1; k < HB / 32; ++k) v = dd_add(v, sh[k]);
  }
  return v;  // valid in thread 0
}
__device__ __forceinline__ double hmax(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < HB / 32) ? sh[threadIdx.x] : 0.0;
  if (threadIdx.x < 32)
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;  // valid in thread 0
}

__global__ void __launch_bounds__(HB) k_herm_embed(const double* __restrict__ Ar, const double* __restrict__ Ai,
                                                   long long lda, int n, double* __restrict__ M, long long ldm) {
  const int j = blockIdx.x;  // column of M (0 .. 2n)
  const int jj = j < n ? j : j - n;
  const double* cr = Ar + jj * lda;
  const double* ci = Ai + jj * lda;
  double* mc = M + j * ldm;
  for (int i = threadIdx.x; i < n; i += HB) {
    const double r = cr[i], im = ci[i];
    if (j < n) {  // [Ar; Ai]
      mc[i] = r;
      mc[n + i] = im;
    } else {      // [−Ai; Ar]
      mc[i] = -im;
      mc[n + i] = r;
    }
  }
}

// One CTA per column j (0 .. n): t = Σ_i x̂s_ij·v̂_ij over the 2n stacked rows (double-double), λ̂_j = t/s_j;
// R̂ = V̂ − X̂s·λ̂_j (double-double, RN to fp64 — its rounding, 2^-53·|R|, is far below the W budget) into column j of
// R2 and JR̂ into column n + j; rmax[j] = max_i |R̂_ij|.
__global__ void __launch_bounds__(HB) k_herm_lam_res(const double* __restrict__ Vh, const double* __restrict__ Vl,
                                                     long long ldv, const double* __restrict__ X1, long long ldx1,
                                                     const double* __restrict__ s_hi, const double* __restrict__ s_lo,
                                                     int n, double* __restrict__ lam, double* __restrict__ R2,
                                                     long long ldr, double* __restrict__ rmax) {
  __shared__ dd shd[HB / 32];
  __shared__ double shm[HB / 32];
  __shared__ double lam_s;
  const int j = blockIdx.x;
  const int n2 = 2 * n;
  const double* vh = Vh + j * ldv;
  const double* vl = Vl + j * ldv;
  const double* x1 = X1 + j * ldx1;
  dd t{0.0, 0.0};
  for (int i = threadIdx.x; i < n2; i += HB) t = dd_add(t, dd_mul_d(dd{vh[i], vl[i]}, x1[i]));
  t = hsum_dd(t, shd);
  if (threadIdx.x == 0) {
    const dd l = dd_div(t, dd{s_hi[j], s_lo[j]});
    lam_s = l.hi;
    lam[j] = l.hi;
  }
  __syncthreads();
  const double l = lam_s;
  double* r = R2 + j * ldr;
  double* jr = R2 + (static_cast<long long>(n) + j) * ldr;
  double m = 0.0;
  for (int i = threadIdx.x; i < n2; i += HB) {
    double ph, pl;
    two_prod(x1[i], l, ph, pl);
    const dd res = dd_add(dd{vh[i], vl[i]}, dd{-ph, -pl});
    const double v = res.hi;
    r[i] = v;
    if (i < n) jr[n + i] = -v;  // JR̂ = [Im R; −Re R]
    else jr[i - n] = v;
    m = fmax(m, fabs(v));
  }
  m = hmax(m, shm);
  if (threadIdx.x == 0) rmax[j] = m;
}

// Column j of Ẽ (Alg. 1 line 5) from W (n x 2n: [Wr, Wi], fp64): the B operand of U = Q·B, B (2n x 2n) =
// [E1, E2], E1 = [D Er; −D Ei], E2 = [D Ei; D Er], D = diag(2^g) (exact scalings); nrm2[j] = ‖ẽ_j‖²,
// emax[j] = max |entries of column j of E1| (= of E2).
__global__ void __launch_bounds__(HB) k_herm_E(const double* __restrict__ W, long long ldw, const double* __restrict__ lam,
                                               const double* __restrict__ r_hi, const int32_t* __restrict__ g, int n,
                                               double* __restrict__ B, long long ldb, double* __restrict__ nrm2,
                                               double* __restrict__ emax, int* __restrict__ err) {
  __shared__ double sh[HB / 32];
  const int j = blockIdx.x;
  const double lj = lam[j];
  const double* wr = W + j * ldw;
  const double* wi = W + (static_cast<long long>(n) + j) * ldw;
  double* e1 = B + j * ldb;
  double* e2 = B + (static_cast<long long>(n) + j) * ldb;
  double s2 = 0.0, m = 0.0;
  bool bad = false;
  for (int i = threadIdx.x; i < n; i += HB) {
    double er, ei;
    if (i == j) {
      er = r_hi[j] * 0.5;  // ẽ_jj = r_j/2
      ei = 0.0;
    } else {
      const double dl = __dsub_rn(lj, lam[i]);  // λ̂_j − λ̂_i
      if (dl == 0.0) bad = true;
      er = __ddiv_rn(wr[i], dl);
      ei = __ddiv_rn(wi[i], dl);
    }
    s2 = __fma_rn(er, er, __fma_rn(ei, ei, s2));
    const double sr = ldexp_fast(er, g[i]), si = ldexp_fast(ei, g[i]);
    e1[i] = sr;
    e1[n + i] = -si;
    e2[i] = si;
    e2[n + i] = sr;
    m = fmax(m, fmax(fabs(sr), fabs(si)));
  }
  if (bad) atomicOr(err, ERR_DEGENERATE);
  s2 = hsum(s2, sh);
  if (threadIdx.x == 0) nrm2[j] = s2;
  m = hmax(m, sh);
  if (threadIdx.x == 0) emax[j] = m;
}

// Q (n x 2n, column-major): Q[i, k] = x̂^(1)r_ik·2^{−g_k}, Q[i, n + k] = x̂^(1)i_ik·2^{−g_k} — exact integers
// (|q| ≤ 2^{53−β}).
__global__ void __launch_bounds__(HB) k_herm_Q(const double* __restrict__ X1, long long ldx1,
                                               const int32_t* __restrict__ g, int n, double* __restrict__ Q,
                                               long long ldq) {
  const int c = blockIdx.x;  // column of Q (0 .. 2n)
  const int k = c < n ? c : c - n;
  const double* src = X1 + k * ldx1 + (c < n ? 0 : n);
  double* dst = Q + c * ldq;
  const int e = -g[k];
  for (int i = threadIdx.x; i < n; i += HB) dst[i] = ldexp_fast(src[i], e);
}

// X̂ ← RN(X̂^(1) + U) (accsum) on both parts; U = [Ur, Ui] (n x 2n, double-double); ν_j² = ‖x̂_j,new − x̂_j‖².
__global__ void __launch_bounds__(HB) k_herm_final(const double* __restrict__ Uh, const double* __restrict__ Ul,
                                                   long long ldu, const double* __restrict__ X1, long long ldx1,
                                                   double* __restrict__ Xr, double* __restrict__ Xi, long long ldx,
                                                   int n, double* __restrict__ nu2) {
  __shared__ double sh[HB / 32];
  const int j = blockIdx.x;
  double s2 = 0.0;
  for (int part = 0; part < 2; ++part) {
    const double* uh = Uh + (static_cast<long long>(part) * n + j) * ldu;
    const double* ul = Ul + (static_cast<long long>(part) * n + j) * ldu;
    const double* x1 = X1 + j * ldx1 + part * n;
    double* x = (part ? Xi : Xr) + j * ldx;
    for (int i = threadIdx.x; i < n; i += HB) {
      double s, e;
      two_sum(x1[i], uh[i], s, e);
      const double xn = __dadd_rn(s, __dadd_rn(e, ul[i]));
      const double d = __dsub_rn(xn, x[i]);
      s2 = __fma_rn(d, d, s2);
      x[i] = xn;
    }
  }
  s2 = hsum(s2, sh);
  if (threadIdx.x == 0) nu2[j] = s2;
}

}  // namespace

void launch_herm_embed(const double* Ar, const double* Ai, long long lda, int n, double* M, long long ldm,
                       cudaStream_t s) {
  k_herm_embed<<<2 * n, HB, 0, s>>>(Ar, Ai, lda, n, M, ldm);
}
void launch_herm_lam_res(const double* Vh, const double* Vl, long long ldv, const double* X1, long long ldx1,
                         const double* s_hi, const double* s_lo, int n, double* lam, double* R2, long long ldr,
                         double* rmax, cudaStream_t s) {
  k_herm_lam_res<<<n, HB, 0, s>>>(Vh, Vl, ldv, X1, ldx1, s_hi, s_lo, n, lam, R2, ldr, rmax);
}
void launch_herm_E(const double* W, long long ldw, const double* lam, const double* r_hi, const int32_t* g, int n,
                   double* B, long long ldb, double* nrm2, double* emax, int* err, cudaStream_t s) {
  k_herm_E<<<n, HB, 0, s>>>(W, ldw, lam, r_hi, g, n, B, ldb, nrm2, emax, err);
}
void launch_herm_Q(const double* X1, long long ldx1, const int32_t* g, int n, double* Q, long long ldq,
                   cudaStream_t s) {
  k_herm_Q<<<2 * n, HB, 0, s>>>(X1, ldx1, g, n, Q, ldq);
}
void launch_herm_final(const double* Uh, const double* Ul, long long ldu, const double* X1, long long ldx1, double* Xr,
                       double* Xi, long long ldx, int n, double* nu2, cudaStream_t s) {
  k_herm_final<<<n, HB, 0, s>>>(Uh, Ul, ldu, X1, ldx1, Xr, Xi, ldx, n, nu2);
}

}  // namespace ozr
