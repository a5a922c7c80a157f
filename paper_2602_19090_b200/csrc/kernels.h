// kernels.h — launchers of the HBM-bound ozr kernels (kernels.cu). Internal, not ABI.
#pragma once
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

namespace ozr {

enum { ERR_NONFINITE = 1, ERR_RANGE = 2, ERR_DEGENERATE = 4, ERR_SOLVER = 8 };

constexpr int kMaxChunks = 8;
constexpr int kPlanGroups = 96;

// How the int32 group planes of one product are recombined:
// value = Σ_c T_c · 2^{8(L − d_last(c)) + ℓA_i + ℓB_j + scale8}, T_c = Σ_{g∈c} 256^{d_last(c) − d_g} C_g (int128).
struct RecombPlan {
  int ngroups;
  int L;
  int consecutive;  // 1: group g is the whole diagonal diag[0] + g, ngroups <= 12 — the 64-bit limb path
  int nchunks;
  int chunk_first[kMaxChunks + 1];
  int diag[kPlanGroups];
  // per-N-tile budgets (matches PairTable::tileL): column j only sums groups with diag <= tileL[j / 256]
  int tile_budgets;
  unsigned char tileL[256];
};

void launch_colmax(const double* X, long long ldx, int rows, int cols, double* w, int* err, cudaStream_t s);
void launch_x1_split(const double* X, long long ldx, int rows, int cols, int beta, int kx, const double* w, double* X1,
                     long long ldx1, int8_t* dig, long long ldd, long long pstride, int32_t* g, double* s_hi,
                     double* s_lo, double* r_hi, double* r_lo, int* err, cudaStream_t s);
void launch_split_fixed(const double* M, const double* Mlo, long long ldm, int rows, int cols, int k, int8_t* dig,
                        long long ldd, long long pstride, int32_t* ell, int* err, cudaStream_t s);
// Digits of Res = V − X̂^(1)D̂ formed on the fly from V (dd), X̂^(1) and λ̂ (local column j uses lam[j]),
// exponent per column from eR (k_recombine_V); same digits as k_split_fixed on the stored Res.
void launch_split_res(const double* Vh, const double* Vl, long long ldv, const double* X1, long long ldx1,
                      const double* lam, int rows, int cols, int k, const int32_t* eR, int8_t* dig, long long ldd,
                      long long pstride, int32_t* ell, cudaStream_t s);
void launch_transpose_i8(const int8_t* src, long long lds, long long sps, int8_t* dst, long long ldt, long long tps,
                         int rows, int cols, int planes, cudaStream_t s);
void launch_transpose_f64(const double* src, long long lds, double* dst, long long ldt, int rows, int cols,
                          cudaStream_t s);
void launch_recombine_V(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp,
                        const int32_t* ellA, const int32_t* ellB, int scale8, const double* X1, long long ldx1,
                        const double* s_hi, const double* s_lo, double* Vh, double* Vl, long long ldv,
                        double* lam_out, int32_t* eR, int* eR_max, cudaStream_t s, int allow_tma = 1,
                        const double* lam0 = nullptr);
// Unresolved pairs of k_recombine_E (cluster branch, R13): every pair (i, j), i ≠ j, with
// λ̂_i = λ̂_j or |ẽ_ij| > κ is united in the device union-find `parent` (O(n) memory, any number of
// pairs; the resulting partition is independent of the order of the unions), and *any is set.
struct EdgeOut {
  int mode;      // 0: the paper's Alg. 1 (equal λ̂ → ERR_DEGENERATE); 1: union unresolved pairs
  double kappa;
  int* parent;   // n entries, parent[i] = i on entry (launch_iota)
  int* any;
};
void launch_iota(int* p, int n, cudaStream_t s);
// dst/src: device-accessible (device or mapped pinned host memory); 8-byte units when all are 8-aligned
void launch_copy_bytes(void* dst, const void* src, size_t bytes, cudaStream_t s);
void launch_uf_flatten(int* parent, int n, cudaStream_t s);  // parent[i] ← root of i
void launch_recombine_E(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp,
                        const int32_t* ellA, const int32_t* ellB, int scale8, const double* r_hi, const double* lam,
                        const int32_t* gX, int col0, double* Ep, long long lde, double* nrm2, int* eE_max,
                        int32_t* eE_col, int* err, const EdgeOut& eo, double* nW2 /* nullable: ‖w_j‖² */,
                        cudaStream_t s, int allow_tma = 1);
// form_R: R = I − X̂^(1)ᵀX̂^(1) (local columns) from the G slice-product planes, ‖r_j‖² in nR2[j]
void launch_form_R(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp, const int32_t* g,
                   int scale8, int col0, const double* r_hi, const double* r_lo, double* R, long long ldr, double* nR2,
                   cudaStream_t s);

// Hermitian sweep (herm.cu; ozr_refine_step_herm, R18): complex n x n matrices in the real-stacked
// 2n x n form [Re; Im].
void launch_herm_embed(const double* Ar, const double* Ai, long long lda, int n, double* M, long long ldm,
                       cudaStream_t s);
void launch_herm_lam_res(const double* Vh, const double* Vl, long long ldv, const double* X1, long long ldx1,
                         const double* s_hi, const double* s_lo, int n, double* lam, double* R2, long long ldr,
                         double* rmax, cudaStream_t s);
void launch_herm_E(const double* W, long long ldw, const double* lam, const double* r_hi, const int32_t* g, int n,
                   double* B, long long ldb, double* nrm2, double* emax, int* err, cudaStream_t s);
void launch_herm_Q(const double* X1, long long ldx1, const int32_t* g, int n, double* Q, long long ldq,
                   cudaStream_t s);
void launch_herm_final(const double* Uh, const double* Ul, long long ldu, const double* X1, long long ldx1, double* Xr,
                       double* Xi, long long ldx, int n, double* nu2, cudaStream_t s);

// Cluster sub-solve (cluster.cu). Groups g = 0..ngroups-1 with members mem[goff[g] .. goff[g]+gm[g]) (global
// column indices, ascending (λ̂, index)); per-group m x m workspaces at offset gsq[g] (Σ m²) in M/R/K/V/Z.
struct ClusterLaunch {
  int ngroups, nmembers, mmax, ntiles, rows;
  int col0, ncols;    // this rank's columns [col0, col0 + ncols) (block-column partition)
  const int4* tiles;  // (group, a0, b0, m) 16 x 16 tiles of k_cluster_build
  const int *goff, *gsq, *gm, *mem, *grp_of, *pos_of;
  const double* mu;
  const int8_t* xdig;  // X̂^(1) digit planes (column-major, kx planes)
  long long ldd, pstride;
  int kx;
  const int32_t* gexp;  // g_j (LSB exponent of column j of X̂^(1))
  const double *r_hi, *r_lo;
  const int32_t* wplanes;  // W = X̂ᵀRes slice-product planes
  long long wpstride;
  const RecombPlan* rpW;
  const int32_t* ellR;
  int scale8;
  double* lam;  // in: λ̂ (Rayleigh quotients), out: λ̂_J = μ + Θ
  double *Mbuf, *Rbuf, *Kbuf, *Vbuf, *Zbuf, *T;
  int* sweeps;
  double* Ep;
  long long lde;
  double* nrm2;     // n entries, global column index
  int32_t* eE_col;  // ncols entries, local column index
  int* eE_max;
  int nsplit;                 // row splits of the exact Gram partial sums (cluster_dot_splits)
  unsigned long long* part;   // ntiles·nsplit·256·2 u64
  const int* hgm;          // host copy of gm (which groups take the cooperative whole-GPU Jacobi)
  double* coop_scratch;    // >= 5·mmax + 8 doubles
  int* coop_flags;         // >= 128 ints
  int ntiles_dot;          // the first ntiles_dot tiles (small groups) sum their Gram block from the digits
                           // (k_cluster_dot); the rest read it from Gbuf (tensor-core Gram, ozr_api.cu)
  const double* Gbuf;      // G_JJ = X̂_JᵀX̂_J rounded to fp64, at offset gsq[g] for those groups
  int dense_min;           // groups of at least this many columns take the dense solver (dense_eig.cu)
  int* err;                // error flags (ERR_SOLVER when the dense solver reports failure)
};
// Pieces of the dense sub-solve of a large group (dense_eig.cu; ozr_api.cu orchestrates with oz_dgemm):
// out = (X + Xᵀ)/2 (m x m); out = X + alpha·P (cnt elements); K ← its eigenvectors Y (ascending θ);
// Y's columns signed (y_kk ≥ 0) and λ̂_J = μ + θ; the dense group's part of the apply.
void launch_dense_sym(int m, const double* X, double* out, cudaStream_t s);
void launch_dense_axpy(long long cnt, const double* X, double alpha, const double* P, double* out, cudaStream_t s);
void launch_dense_sign(int m, double* Y, const double* th, double mu, const int* J, double* lam, const int* info,
                       int* err, cudaStream_t s);
void launch_dense_scatter(const double* TZ, int rows, int m, const int* J, int grp, const int* grp_of, const int* pos_of,
                          const double* Z, const int32_t* gexp, double* Ep, long long lde, int col0, int ncols,
                          cudaStream_t s);
size_t cluster_jacobi_smem(int mmax);
int cluster_dot_splits(int ntiles, int rows);
// build: R_JJ (all), M_JJ and T = Ẽ'[:, J] on this rank's columns (zero elsewhere; all-reduced between);
// solve: Jacobi of every group (replicated on every rank); apply: Ẽ'[:, J] and column statistics of the
// owned columns.
cudaError_t launch_cluster_build(const ClusterLaunch& L, cudaStream_t s);
// digit columns J of the k planes of `dig` (ld bytes per column) → contiguous columns of `out`; g[J] → gJ
void launch_gather_digit_cols(const int8_t* dig, long long ld, long long pstride, int k, const int* J, int m,
                              int8_t* out, long long opstride, const int32_t* g, int32_t* gJ, cudaStream_t s);
cudaError_t launch_cluster_solve(const ClusterLaunch& L, cudaStream_t s);
// apply: the groups below dense_min (the dense ones: launch_dense_scatter); colstats: every member column
cudaError_t launch_cluster_apply(const ClusterLaunch& L, cudaStream_t s);
cudaError_t launch_cluster_colstats(const ClusterLaunch& L, cudaStream_t s);
void launch_final(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp,
                  const int32_t* ellB, int scale8, const double* X1, long long ldx1, double* X, long long ldx,
                  double* nu2, double* wnext, cudaStream_t s, int allow_tma = 1, double* D = nullptr);
// power-iteration helpers (certify.cu): out[0] = Σx², v = z/√nrm2[0] (z == nullptr: a deterministic start vector)
void launch_sumsq(const double* x, int n, double* out, cudaStream_t s);
void launch_normalize(double* v, const double* z, int n, const double* nrm2, int col0, cudaStream_t s);
void launch_recombine_dd(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp,
                         const int32_t* ellA, const int32_t* ellB, int scale8, double* Ch, double* Cl, long long ldc,
                         cudaStream_t s);

}  // namespace ozr
